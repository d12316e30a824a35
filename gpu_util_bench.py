"""Device-input helpers shared by bench.py and __graft_entry__.smoke() (no method arithmetic)."""
import numpy as np

_SAME = {np.dtype(np.float32): np.float32, np.dtype(np.int32): np.int32, np.dtype(np.int16): np.int16,
         np.dtype(np.uint16): np.int16, np.dtype(np.uint8): np.uint8}


def device_inputs(plan, inputs_np: dict, device: int, rows=None):
    """Copy numpy inputs to 16-byte-pitched device tensors in the plan's input order; rows=(r0, r1) keeps
    only that row band of every image (band runs)."""
    import torch

    import paper_1909_07190_b200 as pmg
    out = []
    for io in plan.inputs:
        arr = inputs_np[io.name]
        if rows is not None and not io.is_table:
            arr = arr[..., rows[0]:rows[1], :]
        src = torch.from_numpy(np.ascontiguousarray(arr).view(_SAME[arr.dtype]))
        if io.is_table:
            t = torch.empty(arr.shape, dtype=pmg.pipeline._torch_dtype(io.dtype), device=f"cuda:{device}")
        else:
            t = pmg.empty_pitched(arr.shape, io.dtype, f"cuda:{device}")
        t.view(src.dtype).copy_(src.to(f"cuda:{device}"))
        out.append(t)
    return out
