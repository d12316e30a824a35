"""Helpers for the GPU parity tests: run a pipeline through the C ABI (libpmg.so) on torch tensors."""
import numpy as np

import paper_1909_07190_b200 as pmg

_SAME = {np.dtype(np.float32): np.float32, np.dtype(np.int32): np.int32, np.dtype(np.int16): np.int16,
         np.dtype(np.uint16): np.int16, np.dtype(np.uint8): np.uint8}


def to_device(arr: np.ndarray, dtype: str, device="cuda:0", pitched=True):
    """numpy -> device tensor of the pipeline dtype; images get a 16-byte-aligned row pitch."""
    import torch
    src = torch.from_numpy(np.ascontiguousarray(arr).view(_SAME[arr.dtype]))
    target = pmg.pipeline._torch_dtype(dtype)
    if not pitched or arr.ndim == 1:
        out = torch.empty(arr.shape, dtype=target, device=device)
    else:
        out = pmg.empty_pitched(arr.shape, dtype, device)
    out.view(src.dtype).copy_(src.to(device))
    return out


def to_numpy(t) -> np.ndarray:
    import torch
    if t.dtype == torch.uint16:
        return t.view(torch.int16).cpu().numpy().view(np.uint16)
    return t.cpu().numpy()


def run_gpu(text: str, params: dict, inputs: dict, opts=None, spec=None, plan=None):
    """Returns ({liveout: ndarray}, plan)."""
    import torch
    pipe = pmg.Pipeline(text) if plan is None else plan.pipeline
    if plan is None:
        plan = pmg.Plan(pipe, params, device=0, spec=spec, opts=opts)
    ins = [to_device(inputs[io.name], io.dtype, pitched=not io.is_table) for io in plan.inputs]
    outs = plan.run(ins)
    torch.cuda.synchronize()
    return {io.name: to_numpy(t) for io, t in zip(plan.outputs, outs)}, plan


def compare(got: np.ndarray, exp: np.ndarray, float_tol=1e-4, rel_range=None):
    """Bit-exact for integer outputs; for float the BJ tolerance (1e-4 abs on [0,1] images, or range-relative
    for accumulation-derived outputs).  Returns (n_not_bit_identical, max_abs_diff)."""
    assert got.shape == exp.shape, (got.shape, exp.shape)
    if exp.dtype.kind in "iu":
        np.testing.assert_array_equal(got, exp)
        return 0, 0.0
    neq = int(np.count_nonzero(got.view(np.uint32) != exp.view(np.uint32)))
    d = float(np.max(np.abs(got.astype(np.float64) - exp.astype(np.float64)))) if got.size else 0.0
    tol = float_tol if rel_range is None else rel_range * float(np.max(np.abs(exp)))
    assert d <= tol, f"max |gpu - oracle| = {d} > {tol} ({neq} elements not bit-identical)"
    return neq, d
