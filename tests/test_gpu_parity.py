"""GPU parity: the CUDA path (through the C ABI) against the independent oracle, element by element, on
seeded inputs at sizes spanning several warp tiles with ragged tails; schedule sweeps (the result must not
depend on the schedule); edge shapes.  Bar: bit-exact (float results too, by construction — reading R3);
the BASELINE.json tolerance (1e-4 abs on [0,1] outputs, 1e-5 range-relative for Harris) is the ceiling
asserted."""
import numpy as np
import pytest

import pmg_inputs as PI
from gpu_util import compare, run_gpu
from oracle import evaluate

pytestmark = pytest.mark.gpu

import paper_1909_07190_b200 as pmg  # noqa: E402

TOL = {"blur": dict(float_tol=1e-4), "unsharp": dict(float_tol=1e-4), "harris": dict(rel_range=1e-5),
       "local_laplacian": dict(float_tol=1e-4), "camera": {}, "pyramid_blend": dict(float_tol=1e-4),
       "multiscale_interp": dict(float_tol=1e-4)}


def check(name, W, H, opts=None, variant="uniform", bit_exact=True):
    w = PI.small(name, W, H)
    inp = w.inputs(variant)
    exp = evaluate(w.text, w.params, inp)
    got, plan = run_gpu(w.text, w.params, inp, opts=opts)
    for k in exp:
        neq, d = compare(got[k], exp[k], **TOL[name])
        if bit_exact:
            assert neq == 0, f"{name} {W}x{H}: {neq} elements differ from the oracle (max {d})"
    return plan


def test_fig1_shuffle_selftest():
    """PAPER.md Fig. 1 (lines 252-260): lane 0 receives the warp sum 0+1+...+31 = 496."""
    assert pmg.selftest_shuffle(0) == 496


@pytest.mark.parametrize("W,H", [(128, 128), (1, 1), (33, 1), (127, 131), (4097, 3), (300, 257)])
def test_blur_parity(W, H):
    check("blur", W, H)


@pytest.mark.parametrize("W,H", [(256, 200), (1000, 37), (64, 64), (5, 3)])
def test_harris_parity(W, H):
    check("harris", W, H)


def test_harris_structured():
    check("harris", 500, 300, variant="structured")


@pytest.mark.parametrize("variant", ["uniform", "structured"])
def test_unsharp_parity(variant):
    check("unsharp", 300, 170, variant=variant)


SWEEP = [dict(vec=v, chunks=tx, rows=th, warps=nw, prefetch=pf)
         for (v, tx, th, nw, pf) in [(1, 1, 1, 1, 1), (2, 1, 3, 2, 2), (4, 1, 8, 4, 4), (4, 2, 32, 4, 2),
                                     (2, 4, 5, 8, 3), (1, 2, 64, 2, 4), (4, 4, 16, 1, 1)]]


@pytest.mark.parametrize("cfg", SWEEP, ids=lambda c: "V{vec}TX{chunks}TH{rows}NW{warps}P{prefetch}".format(**c))
@pytest.mark.parametrize("name", ["blur", "harris", "unsharp"])
def test_schedule_invariance(name, cfg):
    """Any (tile, block, prefetch) configuration computes the same function."""
    check(name, 211, 77, opts=pmg.sched_opts(**cfg, tx_size=32))


HYBRID = [dict(vec=4, chunks=2, smem_chunks=1, rows=16, warps=1, prefetch=4),
          dict(vec=2, chunks=4, smem_chunks=2, rows=8, warps=2, prefetch=3),
          dict(vec=4, chunks=1, smem_chunks=1, rows=32, warps=1, prefetch=4),
          dict(vec=1, chunks=2, smem_chunks=2, rows=5, warps=4, prefetch=2)]


@pytest.mark.parametrize("cfg", HYBRID, ids=lambda c: "V{vec}TX{chunks}S{smem_chunks}TH{rows}".format(**c))
@pytest.mark.parametrize("name", ["blur", "harris", "unsharp", "camera"])
def test_hybrid_tiling_parity(name, cfg):
    if name == "camera" and cfg["chunks"] != 1:
        pytest.skip("camera: one hybrid configuration (suite time; integer windows in smem follow the same code)")
    """Hybrid tiling (P:645-654): the S leftmost chunks keep their stage windows in shared memory, the rest in
    registers; the result must not change (interior kernel; border tiles stay in registers)."""
    check(name, 1200, 131, opts=pmg.sched_opts(**cfg, tx_size=32))   # wide enough for interior tiles


@pytest.mark.parametrize("name", ["blur", "harris", "unsharp"])
def test_unfused_equals_fused(name):
    """One kernel per stage (every intermediate through HBM) == the fused group."""
    check(name, 150, 90, opts=pmg.sched_opts(fuse=False))


def test_camera_parity():
    check("camera", 264, 130)


PARITY_SWEEP = [dict(vec=v, chunks=tx, rows=th, warps=1, prefetch=pf)
                for (v, tx, th, pf) in [(1, 1, 3, 2), (2, 1, 8, 4), (2, 2, 5, 3), (4, 1, 16, 4), (4, 2, 8, 2)]]


@pytest.mark.parametrize("cfg", PARITY_SWEEP, ids=lambda c: "V{vec}TX{chunks}TH{rows}P{prefetch}".format(**c))
@pytest.mark.parametrize("W,H", [(263, 131)])
def test_camera_schedules(cfg, W, H):
    """x-parity folding of `x % 2` / `x / 2` (even V) and the shift/mask forms of floor division: the camera
    pipe's interleave and deinterleave under every lane width, on even and odd extents."""
    check("camera", W, H, opts=pmg.sched_opts(**cfg, tx_size=32))


@pytest.mark.parametrize("cfg", PARITY_SWEEP[:3], ids=lambda c: "V{vec}TX{chunks}TH{rows}P{prefetch}".format(**c))
def test_local_laplacian_schedules(cfg):
    w = PI.Workload("ll", "local_laplacian_J4K4.pmg", {"W": 97, "H": 63}, 1005)
    inp = w.inputs("structured")
    exp = evaluate(w.text, w.params, inp)
    got, _ = run_gpu(w.text, w.params, inp, opts=pmg.sched_opts(**cfg, tx_size=32))
    neq, _ = compare(got["out"], exp["out"], float_tol=1e-4)
    assert neq == 0


def test_local_laplacian_small_parity():
    w = PI.Workload("ll", "local_laplacian_J4K4.pmg", {"W": 96, "H": 64}, 1005)
    inp = w.inputs("structured")
    exp = evaluate(w.text, w.params, inp)
    got, _ = run_gpu(w.text, w.params, inp)
    compare(got["out"], exp["out"], float_tol=1e-4)


SCALED = [dict(vec=v, chunks=tx, rows=th, warps=1, prefetch=pf)
          for (v, tx, th, pf) in [(1, 1, 3, 2), (2, 1, 8, 4), (2, 2, 5, 3), (4, 1, 16, 4), (4, 2, 8, 2), (4, 4, 4, 4)]]


@pytest.mark.parametrize("cfg", SCALED, ids=lambda c: "V{vec}TX{chunks}TH{rows}P{prefetch}".format(**c))
@pytest.mark.parametrize("W,H", [(97, 63), (256, 130), (1201, 77)])
def test_scaled_streams(cfg, W, H, monkeypatch):
    """Alignment & scaling: 2v+b and (v+b)/2 reads staged through the TMA ring as scaled streams
    (opt-in PMG_SCALED=1) on odd and even extents, every lane width; bit-exact against the oracle."""
    from pathlib import Path
    monkeypatch.setenv("PMG_SCALED", "1")
    text = (Path(__file__).parent / "golden" / "scaled_streams.pmg").read_text()
    img = PI.uniform((H, W), 77)
    exp = evaluate(text, {"W": W, "H": H}, {"img": img})
    got, plan = run_gpu(text, {"W": W, "H": H}, {"img": img}, opts=pmg.sched_opts(**cfg, tx_size=32))
    neq, _ = compare(got["u"], exp["u"], float_tol=1e-4)
    assert neq == 0
    assert any(s.get("scale", [0, 0, 0]) != [0, 0, 0] for g in plan.describe()["schedule"]["groups"]
               for s in g["config"]["streams"]), "no scaled stream in the plan"


@pytest.mark.parametrize("cfg,W,H", [(None, 97, 63), (PARITY_SWEEP[1], 97, 63), (PARITY_SWEEP[3], 97, 63)],
                         ids=lambda c: "auto" if c is None else c if isinstance(c, int) else "V{vec}TX{chunks}TH{rows}P{prefetch}".format(**c))
def test_pyramid_blend_parity(cfg, W, H):
    """Pyramid Blend (Table 2): three Gaussian pyramids, two Laplacian pyramids,
    per-level blend and collapse through scaled streams, inlined upsamplings and broadcast mask reads."""
    w = PI.Workload("pb", "pyramid_blend_J3.pmg", {"W": W, "H": H}, 1006)
    inp = w.inputs("structured")
    exp = evaluate(w.text, w.params, inp)
    got, _ = run_gpu(w.text, w.params, inp, opts=None if cfg is None else pmg.sched_opts(**cfg, tx_size=32))
    neq, _ = compare(got["out"], exp["out"], float_tol=1e-4)
    assert neq == 0


@pytest.mark.parametrize("name", ["camera"])
def test_scaled_streams_on_pipelines(name, monkeypatch):
    """The scaled-stream path on the camera pipe (Bayer phases: 2v+b in y and x) and the pyramid blend."""
    monkeypatch.setenv("PMG_SCALED", "1")
    w = PI.small(name, 263, 131) if name == "camera" else PI.Workload("pb", "pyramid_blend_J3.pmg", {"W": 97, "H": 63}, 1006)
    inp = w.inputs("structured") if name != "camera" else w.inputs()
    exp = evaluate(w.text, w.params, inp)
    got, plan = run_gpu(w.text, w.params, inp, opts=pmg.sched_opts(vec=2, chunks=2, rows=8, warps=1, prefetch=4, tx_size=32))
    for k in exp:
        neq, _ = compare(got[k], exp[k], float_tol=1e-4)
        assert neq == 0
    assert any(s.get("scale", [0, 0, 0]) != [0, 0, 0] for g in plan.describe()["schedule"]["groups"]
               for s in g["config"]["streams"])


@pytest.mark.parametrize("name,fuse", [("pyramid_blend", True), ("unsharp", False)])
def test_measured_selection(name, fuse, monkeypatch):
    """pmg_sched_opts.tune: the DP schedule and (greedily, round by round) each neighbour merge are compiled and
    timed on the device; the kept plan is the fastest candidate and computes the same function (bit-exact).
    Unfused starting points (one stage per group) make the merge rounds non-trivial."""
    monkeypatch.setenv("PMG_TUNE_GRID", "0")      # merge rounds only (the tile grid is exercised by bench.py)
    w = (PI.Workload("pb", "pyramid_blend_J3.pmg", {"W": 160, "H": 96}, 1006) if name == "pyramid_blend"
         else PI.small(name, 300, 200))
    inp = w.inputs("structured") if name == "pyramid_blend" else w.inputs()
    exp = evaluate(w.text, w.params, inp)
    got, plan = run_gpu(w.text, w.params, inp, opts=pmg.sched_opts(tune=True, fuse=fuse))
    for k in exp:
        neq, _ = compare(got[k], exp[k], **TOL[name])
        assert neq == 0
    t = plan.describe()["tune"]
    us = [c["us"] for c in t["candidates"]]
    assert us[t["chosen"]] == min(us)
    if not fuse:
        assert len(us) >= 2 and len(plan.describe()["schedule"]["groups"]) < len(plan.pipeline.stages)


@pytest.mark.parametrize("W,H,opts", [(24, 24, dict(vec=4, chunks=1, rows=8, warps=1, prefetch=4)),
                                      (77, 53, dict(vec=1, chunks=2, rows=5, warps=2, prefetch=2))])
def test_operator_table_parity(W, H, opts):
    """Reading R4 on the device: every operator / builtin / cast of tests/ops_table.py over all pairs of its
    edge-case values (shift counts outside [0, 31], zero and -1 divisors, INT_MIN, NaN, +-inf, out-of-range
    floats), bit-exact against the oracle (whose values are pinned by hand in test_oracle.py)."""
    import ops_table as OT
    inp = OT.inputs(W, H)
    with np.errstate(all="ignore"):
        exp = evaluate(OT.TEXT, {"W": W, "H": H}, inp)
    one = [0] * len(OT.STAGES)                    # one fused group with every stage a liveout (one compile)
    got, _ = run_gpu(OT.TEXT, {"W": W, "H": H}, inp, opts=pmg.sched_opts(**opts, group_of_stage=one))
    bad = []
    for k in OT.STAGES:
        g, e = got[k], exp[k]
        if e.dtype == np.float32:   # bit-exact, except that NaN payloads are unspecified (IEEE 754 6.2.3): both NaN
            diff = (g.view(np.uint32) != e.view(np.uint32)) & ~(np.isnan(g) & np.isnan(e))
        else:
            diff = g != e
        if np.any(diff):
            i = np.argwhere(diff)[0]
            bad.append((k, tuple(int(v) for v in i), inp["a"][tuple(i)], inp["b"][tuple(i)], inp["f"][tuple(i)],
                        g[tuple(i)], e[tuple(i)]))
    assert not bad, bad


XEDGE = [("harris", 512, 131, dict(vec=4, chunks=1, rows=16, warps=1, prefetch=4)),
         ("harris", 1024, 200, dict(vec=4, chunks=2, rows=24, warps=1, prefetch=4)),
         ("harris", 256, 96, dict(vec=2, chunks=1, rows=8, warps=2, prefetch=3)),
         ("unsharp", 1024, 77, dict(vec=4, chunks=1, rows=24, warps=1, prefetch=4)),
         ("unsharp", 1024, 60, dict(vec=2, chunks=2, rows=8, warps=1, prefetch=2)),
         ("blur", 512, 100, dict(vec=4, chunks=1, rows=32, warps=1, prefetch=4)),
         ("blur", 4096, 9, dict(vec=1, chunks=4, rows=3, warps=1, prefetch=2)),
         ("harris", 6400, 40, None)]


@pytest.mark.parametrize("name,W,H,cfg", XEDGE, ids=lambda v: str(v) if not isinstance(v, dict) else
                         "V{vec}TX{chunks}TH{rows}".format(**v))
def test_xedge_kernel_parity(name, W, H, cfg):
    """x-edge kernel: the first / last tile columns run the interior body with the halo elements
    beyond the image edge replaced by the edge column (reading R1 by selects), the first tile starting at x = 0,
    stores restricted to each tile's canonical columns; the interior tiling's last row is shifted to end at the
    image.  Widths divisible by V so the edge kernel is used (checked), bit-exact against the oracle."""
    plan = check(name, W, H, opts=pmg.sched_opts(**cfg, tx_size=32) if cfg else None)
    assert all(k["edge_regs"] > 0 for k in plan.describe()["kernels"]), plan.describe()["kernels"]


@pytest.mark.parametrize("cfg,W,H", [(None, 96, 64), (PARITY_SWEEP[2], 96, 64), (None, 160, 96)],
                         ids=lambda c: "auto" if c is None else c if isinstance(c, int) else "V{vec}TX{chunks}TH{rows}P{prefetch}".format(**c))
def test_multiscale_interp_parity(cfg, W, H):
    """Multiscale Interpolation (Table 2 l.1148; reading R23): premultiplied pull-push
    pyramid over sparse RGBA samples, J = 4 levels, bit-exact against the oracle."""
    w = PI.Workload("mi", "multiscale_interp_J4.pmg", {"W": W, "H": H}, 1007)
    inp = w.inputs("structured")
    exp = evaluate(w.text, w.params, inp)
    got, _ = run_gpu(w.text, w.params, inp, opts=None if cfg is None else pmg.sched_opts(**cfg, tx_size=32))
    neq, _ = compare(got["out"], exp["out"], float_tol=1e-4)
    assert neq == 0


def test_camera_interleave_fused(monkeypatch):
    """Interleave fusion (runtime.cpp detect_interleave): the camera's full-resolution interleave of its quad
    phases is not launched, the phases store straight into the liveout -- same bytes as the unfused plan and the
    oracle, two launches fewer."""
    w = PI.small("camera", 264, 130)
    inp = w.inputs()
    exp = evaluate(w.text, w.params, inp)
    fused, pf = run_gpu(w.text, w.params, inp)
    n_fused = pf.last_launches
    monkeypatch.setenv("PMG_ILV", "0")
    plain, pp = run_gpu(w.text, w.params, inp)
    for k in exp:
        assert np.array_equal(fused[k], exp[k]) and np.array_equal(plain[k], exp[k])
    assert n_fused < pp.last_launches
