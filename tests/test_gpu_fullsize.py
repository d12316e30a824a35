"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py times (automatic schedule,
whole image, one pipeline run on the caller's stream), checked on sampled outputs that the demand-driven
oracle (oracle/points.py) computes one by one: random interior points plus every corner and the middle of
every edge (the border-tile kernel's territory).  Bar: bit-exact for integer outputs, and for float outputs
too by construction (reading R3); the BASELINE tolerance is asserted as the ceiling."""
import numpy as np
import pytest

import pmg_inputs as PI
from gpu_util import compare, to_device, to_numpy
from oracle import evaluate_points

pytestmark = pytest.mark.gpu

import paper_1909_07190_b200 as pmg  # noqa: E402

TOL = {"blur": dict(float_tol=1e-4), "unsharp": dict(float_tol=1e-4), "harris": dict(rel_range=1e-5),
       "local_laplacian": dict(float_tol=1e-4), "camera": {}, "pyramid_blend": dict(float_tol=1e-4)}


def sample_points(shape, n, seed):
    """n random points, plus the corners, edge midpoints and next-to-corner points of every plane."""
    rng = np.random.default_rng(seed)
    H, W = shape[-2], shape[-1]
    ys = np.array([0, 0, H - 1, H - 1, 0, H - 1, H // 2, H // 2, 1, H - 2])
    xs = np.array([0, W - 1, 0, W - 1, W // 2, W // 2, 0, W - 1, 1, W - 2])
    planes = shape[0] if len(shape) == 3 else 1
    cols = [rng.integers(0, s, size=n) for s in shape]
    cols[-2] = np.concatenate([cols[-2], np.tile(ys, planes)])
    cols[-1] = np.concatenate([cols[-1], np.tile(xs, planes)])
    if len(shape) == 3:
        cols[0] = np.concatenate([cols[0], np.repeat(np.arange(planes), len(ys))])
    return tuple(c.astype(np.int64) for c in cols)


@pytest.mark.parametrize("name", ["harris", "unsharp", "camera", "blur", "local_laplacian", "pyramid_blend"])
def test_fullsize_sampled_parity(name):
    import torch
    wl = PI.WORKLOADS[name]
    inp = wl.inputs("structured") if name in ("local_laplacian", "pyramid_blend") else wl.inputs()
    plan = pmg.Plan(pmg.Pipeline(wl.text), wl.params)              # automatic schedule, as bench.py
    ins = [to_device(inp[io.name], io.dtype, pitched=not io.is_table) for io in plan.inputs]
    outs = plan.run(ins)
    torch.cuda.synchronize()
    (io, out), = zip(plan.outputs, outs)
    got = to_numpy(out)
    pts = sample_points(got.shape, 24 if name in ("local_laplacian", "pyramid_blend") else 96, seed=11)
    exp = evaluate_points(wl.text, wl.params, inp, io.name, pts)
    neq, d = compare(np.ascontiguousarray(got[pts]), exp, **TOL[name])
    assert neq == 0, f"{name}: {neq} sampled outputs differ from the oracle (max {d})"


def test_fullsize_band_sampled_parity():
    """Band 2 of 4 of Harris 6400x6400 (the bench.py --gpus 4 launch configuration of rank 2)."""
    import torch
    wl = PI.WORKLOADS["harris"]
    inp = wl.inputs()
    plan = pmg.Plan(pmg.Pipeline(wl.text), wl.params)
    o_r0, o_r1, i_r0, i_r1 = plan.band_rows(2, 4)
    ins = [to_device(inp["img"][i_r0:i_r1], "f32")]
    outs = [pmg.empty_pitched((o_r1 - o_r0, wl.params["W"]), "f32")]
    plan.run_band(2, 4, ins, outs)
    torch.cuda.synchronize()
    got = to_numpy(outs[0])
    rng = np.random.default_rng(3)
    ys = np.concatenate([rng.integers(o_r0, o_r1, size=64), [o_r0, o_r0, o_r1 - 1, o_r1 - 1]])
    xs = np.concatenate([rng.integers(0, wl.params["W"], size=64), [0, wl.params["W"] - 1, 0, wl.params["W"] - 1]])
    exp = evaluate_points(wl.text, wl.params, inp, "harris", (ys, xs))
    neq, d = compare(np.ascontiguousarray(got[ys - o_r0, xs]), exp, **TOL["harris"])
    assert neq == 0, f"{neq} sampled band outputs differ (max {d})"
