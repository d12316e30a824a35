"""GPU parity at BASELINE.json's full sizes, WHOLE IMAGES, element by element, in the launch configurations
bench.py times:

* C2 Harris 6400², C3 unsharp 2048²×3, C4 camera 2528×1920, C5 local Laplacian 2560×1536×3, Pyramid Blend
  3840×2160×3 and Multiscale Interpolation 2560×1536 (RGBA) — automatic schedule, whole image, one run on the caller's stream (bench.py N=1);
* row bands (bench.py N>1, schedule for one band) — every band of N = 8 (Harris, local Laplacian) and N = 4
  (camera) run separately, stitched, compared with the whole-image oracle;
* C1 blur 128² as the 4096-frame batch (pmg_run_batch) of bench.py's per-config line.

The oracle is the whole-domain evaluator (oracle/pmg_oracle.py), each workload evaluated once per session.
Bar: bit-exact for every output, integer and float (reading R3 makes float results identical by
construction); the BASELINE tolerance is asserted as the ceiling as well."""
import numpy as np
import pytest

import pmg_inputs as PI
from gpu_util import compare, to_device, to_numpy
from oracle import evaluate, parse

pytestmark = pytest.mark.gpu

import paper_1909_07190_b200 as pmg  # noqa: E402

TOL = {"blur": dict(float_tol=1e-4), "unsharp": dict(float_tol=1e-4), "harris": dict(rel_range=1e-5),
       "local_laplacian": dict(float_tol=1e-4), "camera": {}, "pyramid_blend": dict(float_tol=1e-4),
       "multiscale_interp": dict(float_tol=1e-4)}
VARIANT = {"local_laplacian": "structured", "pyramid_blend": "structured", "multiscale_interp": "structured"}

_ORACLE = {}


def oracle_full(name):
    """(inputs, {liveout: oracle output}) of the full-size workload, computed once per session."""
    if name not in _ORACLE:
        wl = PI.WORKLOADS[name]
        inp = wl.inputs(VARIANT.get(name, "uniform"))
        _ORACLE[name] = (inp, evaluate(wl.text, wl.params, inp))
    return _ORACLE[name]


def assert_identical(name, got, exp, what=""):
    neq, d = compare(got, exp, **TOL[name])
    assert neq == 0, f"{name}{what}: {neq} of {exp.size} outputs differ from the oracle (max {d})"


@pytest.mark.parametrize("name", ["harris", "unsharp", "camera", "local_laplacian", "pyramid_blend", "multiscale_interp"])
def test_fullsize_whole_image_parity(name):
    import torch
    wl = PI.WORKLOADS[name]
    inp, exp = oracle_full(name)
    plan = pmg.Plan(pmg.Pipeline(wl.text), wl.params)              # automatic schedule, as bench.py
    ins = [to_device(inp[io.name], io.dtype, pitched=not io.is_table) for io in plan.inputs]
    outs = plan.run(ins)
    torch.cuda.synchronize()
    for io, out in zip(plan.outputs, outs):
        assert_identical(name, to_numpy(out), exp[io.name])


@pytest.mark.parametrize("name,nb", [("harris", 8), ("local_laplacian", 8), ("camera", 4), ("unsharp", 2)])
def test_fullsize_bands_stitched_parity(name, nb):
    """Every band of the bench's N-GPU launch configuration (schedule for one band, pmg_run_band on exactly the
    band's input rows), stitched, equals the whole-image oracle."""
    import torch
    wl = PI.WORKLOADS[name]
    inp, exp = oracle_full(name)
    plan = pmg.Plan(pmg.Pipeline(wl.text), wl.params, opts=pmg.sched_opts(bands=nb))
    got = {o.name: np.zeros(o.shape, dtype=exp[o.name].dtype) for o in plan.outputs}
    ws = plan.workspace()
    for b in range(nb):
        o_r0, o_r1, i_r0, i_r1 = plan.band_rows(b, nb)
        ins = [to_device(inp[io.name] if io.is_table else inp[io.name][..., i_r0:i_r1, :], io.dtype,
                         pitched=not io.is_table) for io in plan.inputs]
        outs = [pmg.empty_pitched((*o.shape[:-2], o_r1 - o_r0, o.shape[-1]), o.dtype) for o in plan.outputs]
        plan.run_band(b, nb, ins, outs, ws)
        torch.cuda.synchronize()
        for o, t in zip(plan.outputs, outs):
            got[o.name][..., o_r0:o_r1, :] = to_numpy(t)
    for o in plan.outputs:
        assert_identical(name, got[o.name], exp[o.name], f" ({nb} bands)")


def test_fullsize_blur_batch_4096():
    """C1 as bench.py's per-config line runs it: 4096 frames of 128x128 in one pmg_run_batch call; every frame
    equals the oracle of that frame."""
    import torch
    wl = PI.WORKLOADS["blur"]
    frames = PI.blur_frames(4096)
    plan = pmg.Plan(pmg.Pipeline(wl.text), wl.params)
    (io,) = plan.inputs
    x = pmg.empty_pitched((frames.shape[0], *io.shape), "f32", "cuda:0")
    x.copy_(torch.from_numpy(frames).to("cuda:0"))
    (out,) = plan.alloc_outputs(frames.shape[0])
    plan.run_batch([x], [out])
    torch.cuda.synchronize()
    got = to_numpy(out)
    prog = parse(wl.text)
    for f in range(frames.shape[0]):
        exp = evaluate(prog, wl.params, {"img": frames[f]})["blury"]
        assert_identical("blur", got[f], exp, f" frame {f}")
