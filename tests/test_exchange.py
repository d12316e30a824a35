"""Halo-exchange bands on CPU: world_size-2 and -3 `gloo` process groups.

Every rank derives its exchange geometry from libpmg on the host (pmg_band_exchange_host: own rows per group,
workspace slots, sends / receives) and runs the transport of paper_1909_07190_b200/dist.py (batch_isend_irecv)
on a CPU "workspace" in which it wrote, for each stage, a value identifying (stage, row) into the rows it owns.
After the exchange every received row must hold exactly the owner's (stage, row) pattern, every row a band's
later groups read must be either its own or received, and the sends / receives of all ranks must pair up.
The GPU side (the kernels in this mode, stitched bands == oracle) is tests/test_gpu_exchange.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1909_07190_b200 as pmg
from paper_1909_07190_b200.dist import exchange_after, exchange_groups, rows_view

LL = "pipelines/local_laplacian_J4K4.pmg"


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _geom(band, n, W, H):
    text = open(os.path.join(os.path.dirname(__file__), "..", LL)).read()
    return pmg.Pipeline(text).band_exchange({"W": W, "H": H}, band, n, opts=pmg.sched_opts(probe=False, bands=n))


def _pattern(k, rows, row_pitch):
    # byte pattern of (stage k, row r): low byte of r, stage, high byte of r, then zeros
    r = np.arange(rows[0], rows[1])
    v = np.zeros((rows[1] - rows[0], row_pitch), np.uint8)
    v[:, 0] = r & 0xFF
    v[:, 1] = k
    v[:, 2] = (r >> 8) & 0xFF
    return torch.from_numpy(v)


def _worker(rank, world, port, W, H, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = _geom(rank, world, W, H)
        ws = torch.full((g["workspace_bytes"],), 0xEE, dtype=torch.uint8)
        for k, st in enumerate(g["stages"]):
            if st["own"][1] > st["own"][0]:
                rows_view(ws, st, st["own"]).copy_(_pattern(k, st["own"], st["row_pitch"]).expand(st["planes"], -1, -1))
        moved = 0
        for g0, g1 in exchange_groups_all(world, W, H):
            moved += exchange_after(g, ws, g1 - 1)
        bad = []
        for t in g["recv"]:
            st = g["stages"][t["stage"]]
            got = rows_view(ws, st, t["rows"])
            exp = _pattern(t["stage"], t["rows"], st["row_pitch"]).expand(st["planes"], -1, -1)
            if not torch.equal(got, exp):
                bad.append((st["name"], t["rows"]))
        # every row a later group reads is own or received
        uncovered = []
        for k, st in enumerate(g["stages"]):
            nd, own = st["need"], st["own"]
            have = set(range(*own))
            for t in g["recv"]:
                if t["stage"] == k:
                    have |= set(range(*t["rows"]))
            if not set(range(*nd)) <= have:
                uncovered.append(st["name"])
        q.put(("ok", rank, bad, uncovered, moved, len(g["send"]), len(g["recv"])))
    except Exception as e:  # pragma: no cover
        import traceback
        q.put(("err", rank, traceback.format_exc(), None, 0, 0, 0))
    finally:
        dist.destroy_process_group()


def exchange_groups_all(world, W, H):
    """The (run, exchange) steps every rank takes: the union of all bands' exchange points."""
    after = set()
    ng = 0
    for b in range(world):
        g = _geom(b, world, W, H)
        ng = len(g["groups"])
        after |= {t["after_group"] for t in g["send"]} | {t["after_group"] for t in g["recv"]}
    return exchange_groups({"groups": [None] * ng, "send": [{"after_group": a} for a in after], "recv": []})


@pytest.mark.parametrize("world,W,H", [(2, 96, 64), (3, 160, 96)])
def test_halo_exchange_gloo(world, W, H):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, W, H, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert r[0] == "ok", r[2]
        assert r[2] == [], f"rank {r[1]}: wrong rows received {r[2]}"
        assert r[3] == [], f"rank {r[1]}: rows read but neither owned nor received: {r[3]}"
    assert sum(r[5] for r in res) == sum(r[6] for r in res) > 0      # sends and receives pair up
    assert all(r[4] > 0 for r in res)


def test_exchange_geometry_partitions_rows():
    """Own rows of every group partition its row extent across the bands; image rows needed by a band are a
    fraction of what the cumulative-halo recompute needs (4-level local Laplacian, 4 bands)."""
    n, W, H = 4, 160, 96
    gs = [_geom(b, n, W, H) for b in range(n)]
    for gi in range(len(gs[0]["groups"])):
        spans = [tuple(g["groups"][gi]) for g in gs]
        assert spans[0][0] == 0 and all(spans[b][1] == spans[b + 1][0] for b in range(n - 1))
    text = open(os.path.join(os.path.dirname(__file__), "..", LL)).read()
    pipe = pmg.Pipeline(text)
    mid = 1
    _, _, i0, i1 = pipe.band_rows({"W": W, "H": H}, mid, n, opts=pmg.sched_opts(probe=False, bands=n))
    xin = gs[mid]["in"]
    assert xin[1] - xin[0] < i1 - i0
