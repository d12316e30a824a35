"""GPU: band and batch execution modes through the C ABI.

Band invariance: running band b of n for every b on one GPU and stitching the outputs gives the
full-image result bit for bit (global-row clamping inside bands).  Batch: pmg_run_batch over frames ==
per-frame oracle.  Workspace-using multi-group plans (camera, unfused) are included."""
import numpy as np
import pytest

import pmg_inputs as PI
from gpu_util import compare, run_gpu, to_device, to_numpy
from oracle import evaluate

pytestmark = pytest.mark.gpu

import paper_1909_07190_b200 as pmg  # noqa: E402


@pytest.mark.parametrize("name,W,H,n,fuse", [("harris", 300, 211, 4, True), ("unsharp", 160, 97, 3, True),
                                             ("blur", 128, 128, 8, True), ("harris", 120, 90, 3, False)])
# (camera and local Laplacian bands: test_gpu_fullsize.py::test_fullsize_bands_stitched_parity, full size)
def test_band_invariance(name, W, H, n, fuse):
    import torch
    wl = (PI.Workload("ll", "local_laplacian_J4K4.pmg", {"W": W, "H": H}, 1005) if name == "ll"
          else PI.small(name, W, H))
    inp = wl.inputs()
    full, plan = run_gpu(wl.text, wl.params, inp, opts=pmg.sched_opts(fuse=fuse))
    (key, ref), = full.items()
    exp = evaluate(wl.text, wl.params, inp)[key]
    compare(ref, exp, float_tol=1e-4, rel_range=1e-5 if name == "harris" else None)
    pieces = []
    for b in range(n):
        o_r0, o_r1, i_r0, i_r1 = plan.band_rows(b, n)
        ins = [to_device(inp[io.name][..., i_r0:i_r1, :] if not io.is_table else inp[io.name], io.dtype,
                         pitched=not io.is_table) for io in plan.inputs]
        outs = [pmg.empty_pitched((*o.shape[:-2], o_r1 - o_r0, o.shape[-1]), o.dtype) for o in plan.outputs]
        plan.run_band(b, n, ins, outs)
        torch.cuda.synchronize()
        pieces.append(to_numpy(outs[0]))
    stitched = np.concatenate(pieces, axis=-2)
    np.testing.assert_array_equal(stitched.view(np.uint8), ref.view(np.uint8))


@pytest.mark.parametrize("name,W,H", [("blur", 128, 128), ("unsharp", 64, 48), ("camera", 64, 48)])
def test_batch_frames(name, W, H):
    import torch
    wl = PI.small(name, W, H)
    frames = [PI.Workload(wl.name, wl.pipeline, wl.params, wl.seed + f).inputs() for f in range(5)]
    plan = pmg.Plan(pmg.Pipeline(wl.text), wl.params, opts=pmg.sched_opts(fuse=True))
    ins = []
    for io in plan.inputs:
        if io.is_table:
            ins.append(to_device(frames[0][io.name], io.dtype, pitched=False))
        else:
            t = pmg.empty_pitched(io.shape, io.dtype, frames=5)
            for f in range(5):
                t[f].copy_(to_device(frames[f][io.name], io.dtype))
            ins.append(t)
    outs = [pmg.empty_pitched(o.shape, o.dtype, frames=5) for o in plan.outputs]
    plan.run_batch(ins, outs)
    torch.cuda.synchronize()
    for f in range(5):
        exp = evaluate(wl.text, wl.params, frames[f])
        compare(to_numpy(outs[0][f]), exp[plan.outputs[0].name], float_tol=1e-4)


def test_misaligned_buffers_are_rejected():
    import torch
    wl = PI.small("blur", 64, 64)
    plan = pmg.Plan(pmg.Pipeline(wl.text), wl.params)
    base = torch.zeros(64 * 64 + 1, dtype=torch.float32, device="cuda")
    bad = base[1:].view(64, 64)                     # 4-byte offset: violates the 16-byte rule of pmg.h
    with pytest.raises(pmg.PmgError, match="aligned"):
        plan.run([bad])


def test_plan_describe_reports_kernels():
    wl = PI.small("harris", 256, 128)
    plan = pmg.Plan(pmg.Pipeline(wl.text), wl.params)
    d = plan.describe()
    assert plan.num_kernels == len(d["kernels"]) == 1
    k = d["kernels"][0]
    assert k["spill_stores"] == 0 and k["blocks_per_sm"] >= 1 and 0 < k["regs"] <= 255


@pytest.mark.parametrize("name,W,H,chunks", [("harris", 700, 301, 1), ("harris", 700, 301, 8), ("unsharp", 300, 170, 3),
                                             ("camera", 264, 130, 8)])
def test_run_host_equals_device_run(name, W, H, chunks):
    """pmg_run_host (pinned host buffers, row chunks pipelined over copy streams) == the device-buffer run,
    bit for bit; every input row is copied once and every output row comes back."""
    import torch
    wl = (PI.Workload("ll", "local_laplacian_J4K4.pmg", {"W": W, "H": H}, 1005) if name == "ll"
          else PI.small(name, W, H))
    inp = wl.inputs("structured") if name == "ll" else wl.inputs()
    ref, plan = run_gpu(wl.text, wl.params, inp)
    host_in = [torch.from_numpy(np.ascontiguousarray(inp[io.name]).view(
        {np.dtype(np.uint16): np.int16}.get(inp[io.name].dtype, inp[io.name].dtype))).pin_memory() for io in plan.inputs]
    host_out = [torch.full(o.shape, 7, dtype=pmg.pipeline._torch_dtype(o.dtype)).pin_memory() for o in plan.outputs]
    dev_in = [pmg.empty_pitched(io.shape, io.dtype) if not io.is_table else
              torch.empty(io.shape, dtype=pmg.pipeline._torch_dtype(io.dtype), device="cuda") for io in plan.inputs]
    dev_out = [pmg.empty_pitched(o.shape, o.dtype) for o in plan.outputs]
    plan.run_host(host_in, host_out, dev_in, dev_out, chunks=chunks)
    torch.cuda.synchronize()
    for o, h in zip(plan.outputs, host_out):
        got = h.view(torch.int16).numpy().view(np.uint16) if h.dtype == torch.uint16 else h.numpy()
        np.testing.assert_array_equal(got.view(np.uint8), ref[o.name].view(np.uint8))


def test_time_per_iter_microbenchmarks_feed_alg2():
    """NEXT-3 / PAPER.md l.890-898: TimePerIter measured on the device (each stage alone as one kernel) is the
    compute input of Alg. 2 (cost_model 1); the measured profile changes the cost, and the schedule it selects
    computes the same function (bit-exact)."""
    wl = PI.small("harris", 640, 480)
    pipe = pmg.Pipeline(wl.text)
    prof = pipe.profile_stages(wl.params)
    names = [s["name"] for s in prof["stages"]]
    assert sorted(names) == sorted(pipe.stages)
    assert all(s["us"] > 0 and s["time_per_iter"] > 0 and s["points"] == 640 * 480 for s in prof["stages"])
    tpi = [next(s["time_per_iter"] for s in prof["stages"] if s["name"] == n) for n in pipe.stages]
    static = pipe.schedule(wl.params, opts=pmg.sched_opts(cost_model=1))
    measured = pipe.schedule(wl.params, opts=pmg.sched_opts(cost_model=1, time_per_iter=tpi))
    ct = lambda sch: sum(g["cost"]["computeTime"] for g in sch["groups"])
    assert ct(static) != ct(measured)
    inp = wl.inputs()
    got, _ = run_gpu(wl.text, wl.params, inp, opts=pmg.sched_opts(cost_model=1, time_per_iter=tpi))
    compare(got["harris"], evaluate(wl.text, wl.params, inp)["harris"], rel_range=1e-5)
