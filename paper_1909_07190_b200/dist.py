"""Multi-GPU plumbing over torch.distributed (north_star: "a batch of frames is split per GPU;
NCCL is used only to gather bands or frames where the caller asks").  No collective is on the compute path:
each rank runs its own row band (pmg_run_band, pipeline-wide halo recomputed locally) or its own frames
(pmg_run_batch).  These helpers only split the work and, on request, assemble the result with one
all_gather_into_tensor (NCCL over NVLink on a GPU box; gloo in the CPU tests)."""
from __future__ import annotations


def frame_range(rank: int, world: int, nframes: int) -> tuple[int, int]:
    """Contiguous frames [f0, f1) of rank `rank` (the first nframes % world ranks take one more)."""
    base, extra = divmod(nframes, world)
    f0 = rank * base + min(rank, extra)
    return f0, f0 + base + (1 if rank < extra else 0)


def _gather_padded(local, counts, dim, group=None):
    """all_gather_into_tensor of `local` padded along `dim` to max(counts); returns the concatenation of every
    rank's first counts[r] entries along `dim` (on every rank)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    mx = max(counts)
    shape = list(local.shape)
    shape[dim] = mx
    pad = torch.zeros(shape, dtype=local.dtype, device=local.device)
    pad.narrow(dim, 0, local.shape[dim]).copy_(local)
    # all_gather_into_tensor concatenates along dim 0: move `dim` to the front
    pad = pad.movedim(dim, 0).contiguous()
    flat = torch.empty((world * mx, *pad.shape[1:]), dtype=pad.dtype, device=pad.device)
    dist.all_gather_into_tensor(flat, pad, group=group)
    parts = [flat[r * mx:r * mx + counts[r]] for r in range(world)]
    return torch.cat(parts, 0).movedim(0, dim)


def gather_bands(local_rows, band_rows, group=None):
    """Assemble the full image from every rank's output rows.  local_rows: this rank's liveout rows
    [out_r0, out_r1) ([..., rows, W], any device); band_rows: [(out_r0, out_r1)] of every rank in rank order."""
    counts = [r1 - r0 for r0, r1 in band_rows]
    return _gather_padded(local_rows.contiguous(), counts, local_rows.dim() - 2, group)


def gather_frames(local_frames, nframes: int, group=None):
    """Assemble a frame-major batch [nframes, ...] from every rank's contiguous frames (frame_range)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    counts = [frame_range(r, world, nframes)[1] - frame_range(r, world, nframes)[0] for r in range(world)]
    return _gather_padded(local_frames.contiguous(), counts, 0, group)


# ------------------------------------------------------------------ halo-exchange bands
# pmg_band_exchange gives every rank the same geometry: band b computes its own rows of each group and, after
# the group that produces a workspace stage, receives the rows its later groups read from the bands that own
# them.  The transport is the caller's: NCCL point-to-point here (torch.distributed batch_isend_irecv; gloo on
# CPU in the tests), or device copies when all bands live in one process (tests, bench --simulate-bands).

def rows_view(ws, st: dict, rows):
    """uint8 view [planes, hi-lo, row_pitch] of rows [lo, hi) of workspace stage `st` (its slot holds st["buf"])."""
    lo, hi = rows
    b0 = st["buf"][0]
    slot = ws.narrow(0, st["offset"], st["planes"] * st["plane_pitch"]).view(st["planes"], st["rows"], st["row_pitch"])
    return slot[:, lo - b0:hi - b0, :]


def exchange_after(geom: dict, ws, g: int, group=None):
    """The sends / receives of band geom["band"] after group g, over torch.distributed point-to-point."""
    import torch.distributed as dist
    ops, landing = [], []
    for t in geom["send"]:
        if t["after_group"] == g:
            ops.append(dist.P2POp(dist.isend, rows_view(ws, geom["stages"][t["stage"]], t["rows"]).contiguous(),
                                  t["peer"], group))
    for t in geom["recv"]:
        if t["after_group"] == g:
            dst = rows_view(ws, geom["stages"][t["stage"]], t["rows"])
            tmp = dst.new_empty(dst.shape).contiguous()
            ops.append(dist.P2POp(dist.irecv, tmp, t["peer"], group))
            landing.append((dst, tmp))
    if not ops:
        return 0
    for r in dist.batch_isend_irecv(ops):
        r.wait()
    for dst, tmp in landing:
        dst.copy_(tmp)
    return sum(t.numel() for _, t in landing)


def exchange_groups(geom: dict):
    """Runs of consecutive groups with no exchange in between: [(g0, g1)], each followed by its exchange."""
    after = {t["after_group"] for t in geom["send"]} | {t["after_group"] for t in geom["recv"]}
    runs, g0 = [], 0
    for g in range(len(geom["groups"])):
        if g in after:
            runs.append((g0, g + 1))
            g0 = g + 1
    if g0 < len(geom["groups"]):
        runs.append((g0, len(geom["groups"])))
    return runs


def exchange_points(geoms) -> set:
    """Groups after which some band exchanges rows (every rank must take the same (run, exchange) steps)."""
    pts = set()
    for gm in geoms:
        pts |= {t["after_group"] for t in gm["send"]} | {t["after_group"] for t in gm["recv"]}
    return pts


def run_band_exchange(plan, band: int, nbands: int, inputs, outputs, workspace, stream=None, group=None,
                      points=None):
    """One rank's band in halo-exchange mode: consecutive groups without an exchange run as one
    pmg_run_band_groups call; after a producing group only the halo rows move (NCCL send/recv).  inputs hold
    image rows geom["in"], outputs rows geom["out"].  Returns the bytes received."""
    import torch
    geom = plan.band_exchange(band, nbands)
    if points is None:
        points = exchange_points([plan.band_exchange(b, nbands) for b in range(nbands)])
    moved = 0
    for g0, g1 in exchange_groups({"groups": geom["groups"], "send": [{"after_group": a} for a in points], "recv": []}):
        plan.run_band_groups(band, nbands, g0, g1, inputs, outputs, workspace, stream)
        if g1 - 1 in points:
            # NCCL point-to-point is ordered after the current stream's work; the landing copies run on it too
            cur = torch.cuda.current_stream() if workspace.is_cuda else None
            if cur is not None and stream is not None and stream != cur:
                cur.wait_stream(stream)
            moved += exchange_after(geom, workspace, g1 - 1, group)
            if cur is not None and stream is not None and stream != cur:
                stream.wait_stream(cur)
    return moved


def run_bands_exchange_local(plan, nbands: int, inputs, outputs, workspaces, stream=None):
    """Every band of one image in this process (one device): group by group, all bands, then device copies of
    the halo rows between the bands' workspaces.  inputs[b] / outputs[b] / workspaces[b]: band b's buffers."""
    geoms = [plan.band_exchange(b, nbands) for b in range(nbands)]
    ng = len(geoms[0]["groups"])
    after = set()
    for gm in geoms:
        after |= {t["after_group"] for t in gm["recv"]}
    g0 = 0
    for g in range(ng):
        if g in after or g == ng - 1:
            for b in range(nbands):
                plan.run_band_groups(b, nbands, g0, g + 1, inputs[b], outputs[b], workspaces[b], stream)
            g0 = g + 1
            for b, gm in enumerate(geoms):
                for t in gm["recv"]:
                    if t["after_group"] != g:
                        continue
                    st = gm["stages"][t["stage"]]
                    src = rows_view(workspaces[t["peer"]], geoms[t["peer"]]["stages"][t["stage"]], t["rows"])
                    rows_view(workspaces[b], st, t["rows"]).copy_(src)
    return geoms
