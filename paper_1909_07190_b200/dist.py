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
