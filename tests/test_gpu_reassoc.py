"""GPU parity of the reassociation mode (pmg_sched_opts.reassoc = 1): rank-1 linear stencils
evaluated separably (factor.cpp) and a*b+c contracted to one fma.  f32 rounding differs from the written order,
so the bar is the north_star tolerance against the oracle on the pipeline AS WRITTEN: max abs error 1e-4 on
[0,1]-normalised images, relative 1e-5 (of the output range) on accumulation-derived outputs (Harris).

* small ragged sizes (several tiles + ragged tails, border / x-edge / interior kernels);
* the full C2 size (Harris 6400², whole image, bench.py's automatic schedule in this mode);
* N = 8 row bands stitched (bench.py's band launch configuration);
* unsharp and blur (already separable as written: fma contraction only)."""
import numpy as np
import pytest

import pmg_inputs as PI
from gpu_util import compare, run_gpu, to_device, to_numpy
from oracle import evaluate

pytestmark = pytest.mark.gpu

import paper_1909_07190_b200 as pmg  # noqa: E402

REL = 1e-5     # Harris: relative to max |output| (accumulations)
ABS = 1e-4     # [0,1] images


def _opts(**kw):
    return pmg.sched_opts(reassoc=True, **kw)


@pytest.mark.parametrize("W,H", [(300, 200), (517, 389), (130, 70), (1031, 97)])
def test_reassoc_harris_small(W, H):
    wl = PI.small("harris", W, H)
    inp = wl.inputs()
    exp = evaluate(wl.text, wl.params, inp)
    got, plan = run_gpu(wl.text, wl.params, inp, opts=_opts())
    assert plan.describe()["factored"] == ["Iy", "Ix", "Sxx", "Syy", "Sxy"]
    for k in exp:
        compare(got[k], exp[k], rel_range=REL)


@pytest.mark.parametrize("cfg", [dict(vec=4, chunks=1, rows=32, warps=1, prefetch=4),
                                 dict(vec=2, chunks=2, rows=16, warps=2, prefetch=4),
                                 dict(vec=1, chunks=4, rows=24, warps=1, prefetch=3)])
def test_reassoc_harris_configs(cfg):
    wl = PI.small("harris", 700, 333)
    inp = wl.inputs()
    exp = evaluate(wl.text, wl.params, inp)
    got, _ = run_gpu(wl.text, wl.params, inp, opts=_opts(**cfg))
    for k in exp:
        compare(got[k], exp[k], rel_range=REL)


@pytest.mark.parametrize("name", ["unsharp", "blur"])
def test_reassoc_other_float_pipelines(name):
    """Pipelines whose stencils are already separable as written: only fma contraction applies."""
    wl = (PI.Workload("ll", "local_laplacian_J4K4.pmg", {"W": 160, "H": 96}, 1005) if name == "local_laplacian"
          else PI.small(name, 260, 190))
    inp = wl.inputs()
    exp = evaluate(wl.text, wl.params, inp)
    got, _ = run_gpu(wl.text, wl.params, inp, opts=_opts())
    for k in exp:
        compare(got[k], exp[k], float_tol=ABS)


_FULL = {}


def _harris_full():
    if not _FULL:
        wl = PI.WORKLOADS["harris"]
        inp = wl.inputs()
        _FULL["v"] = (inp, evaluate(wl.text, wl.params, inp))
    return _FULL["v"]


def test_reassoc_harris_fullsize_whole_image():
    import torch
    wl = PI.WORKLOADS["harris"]
    inp, exp = _harris_full()
    plan = pmg.Plan(pmg.Pipeline(wl.text), wl.params, opts=_opts())
    outs = plan.run([to_device(inp[io.name], io.dtype) for io in plan.inputs])
    torch.cuda.synchronize()
    for io, t in zip(plan.outputs, outs):
        neq, d = compare(to_numpy(t), exp[io.name], rel_range=REL)
        print(f"harris 6400^2 reassoc: max |gpu - oracle| = {d:.3g}, {neq} elements not bit-identical")


def test_reassoc_harris_fullsize_bands():
    import torch
    nb = 8
    wl = PI.WORKLOADS["harris"]
    inp, exp = _harris_full()
    plan = pmg.Plan(pmg.Pipeline(wl.text), wl.params, opts=_opts(bands=nb))
    got = {o.name: np.zeros(o.shape, dtype=exp[o.name].dtype) for o in plan.outputs}
    ws = plan.workspace()
    for b in range(nb):
        o_r0, o_r1, i_r0, i_r1 = plan.band_rows(b, nb)
        ins = [to_device(inp[io.name][..., i_r0:i_r1, :], io.dtype) for io in plan.inputs]
        outs = [pmg.empty_pitched((o_r1 - o_r0, o.shape[-1]), o.dtype) for o in plan.outputs]
        plan.run_band(b, nb, ins, outs, ws)
        torch.cuda.synchronize()
        for o, t in zip(plan.outputs, outs):
            got[o.name][o_r0:o_r1, :] = to_numpy(t)
    for o in plan.outputs:
        compare(got[o.name], exp[o.name], rel_range=REL)
