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
