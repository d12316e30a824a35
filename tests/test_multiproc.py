"""N>1 path on CPU: world_size-2 `gloo` process group.  Each rank asks libpmg for its row band (pipeline-wide
cumulative halo, host-only geometry), evaluates its input band and keeps its output rows; the bands are
gathered (all_gather, the only collective — used only to assemble the image) and must reproduce the full
image bit for bit.  On a GPU box the same geometry drives pmg_run_band (bench.py --gpus N)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1909_07190_b200 as pmg
import pmg_inputs as PI
from oracle import evaluate


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, W, H, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        wl = PI.small(name, W, H)
        pipe = pmg.Pipeline(wl.text)
        o_r0, o_r1, i_r0, i_r1 = pipe.band_rows(wl.params, rank, world, opts=pmg.sched_opts(probe=False))
        inp = wl.inputs()
        band_in = {k: (v[..., i_r0:i_r1, :] if v.ndim >= 2 else v) for k, v in inp.items()}
        band = evaluate(wl.text, {"W": W, "H": i_r1 - i_r0}, band_in)
        (key, out), = band.items()
        mine = np.ascontiguousarray(out[..., o_r0 - i_r0:o_r1 - i_r0, :])
        rows = torch.tensor([o_r0, o_r1])
        all_rows = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(all_rows, rows)
        mx = max(int(r[1] - r[0]) for r in all_rows)
        pad = np.zeros(mine.shape[:-2] + (mx, mine.shape[-1]), mine.dtype)
        pad[..., :mine.shape[-2], :] = mine
        t = torch.from_numpy(pad)
        parts = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        if rank == 0:
            full = evaluate(wl.text, wl.params, inp)[key]
            stitched = np.concatenate([p.numpy()[..., :int(r[1] - r[0]), :] for p, r in zip(parts, all_rows)], axis=-2)
            q.put(("ok", bool(np.array_equal(stitched.view(np.uint8), full.view(np.uint8))),
                   [tuple(int(x) for x in r) for r in all_rows]))
    except Exception as e:  # pragma: no cover
        q.put(("err", repr(e), None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,W,H", [("harris", 40, 37), ("unsharp", 33, 29), ("blur", 16, 23)])
def test_band_sharding_world2_gloo(name, W, H):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, W, H, q)) for r in range(2)]
    for p in procs:
        p.start()
    status, same, rows = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert status == "ok", same
    assert rows == [(0, H // 2), (H // 2, H)]
    assert same, "stitched bands differ from the full-image result"


def _worker_helpers(rank, world, port, q):
    """paper_1909_07190_b200.dist on gloo: frame split + gather_frames, band rows + gather_bands (padded
    all_gather_into_tensor with unequal counts)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1909_07190_b200.dist import frame_range, gather_bands, gather_frames
        # frames: C1 blur, 7 frames over `world` ranks, each rank evaluates its own frames
        wl = PI.WORKLOADS["blur"]
        frames = PI.blur_frames(7)[:, :16, :20]
        f0, f1 = frame_range(rank, world, 7)
        small = PI.small("blur", 20, 16)
        mine = np.stack([evaluate(small.text, small.params, {"img": frames[f]})["blury"] for f in range(f0, f1)])
        allf = gather_frames(torch.from_numpy(mine), 7).numpy()
        exp = np.stack([evaluate(small.text, small.params, {"img": frames[f]})["blury"] for f in range(7)])
        ok_frames = bool(np.array_equal(allf.view(np.uint32), exp.view(np.uint32)))
        # bands: unsharp 3 planes, odd height -> unequal band rows
        wu = PI.small("unsharp", 24, 19)
        pipe = pmg.Pipeline(wu.text)
        rows = [pipe.band_rows(wu.params, b, world, opts=pmg.sched_opts(probe=False)) for b in range(world)]
        o_r0, o_r1, i_r0, i_r1 = rows[rank]
        inp = wu.inputs()
        band = evaluate(wu.text, {"W": 24, "H": i_r1 - i_r0}, {"img": inp["img"][..., i_r0:i_r1, :]})["masked"]
        full = gather_bands(torch.from_numpy(np.ascontiguousarray(band[..., o_r0 - i_r0:o_r1 - i_r0, :])),
                            [(r[0], r[1]) for r in rows]).numpy()
        ok_bands = bool(np.array_equal(full.view(np.uint32), evaluate(wu.text, wu.params, inp)["masked"].view(np.uint32)))
        if rank == 0:
            q.put(("ok", ok_frames, ok_bands, [frame_range(r, world, 7) for r in range(world)]))
    except Exception as e:  # pragma: no cover
        q.put(("err", repr(e), None, None))
    finally:
        dist.destroy_process_group()


def test_frame_split_and_gathers_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_helpers, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    status, ok_frames, ok_bands, ranges = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert status == "ok", ok_frames
    assert ranges == [(0, 4), (4, 7)]
    assert ok_frames, "gathered frames differ from the per-frame oracle"
    assert ok_bands, "gathered bands differ from the full-image oracle"
