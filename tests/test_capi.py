"""CPU tests of the C ABI (libpmg.so) and its host-side logic: symbol exports, parse-error taxonomy,
I/O descriptors, dependence vectors (§2.3), the §3/§4 worked examples and Alg. 2 arithmetic
(pinned by tests/golden/paper_worked_examples.json), DP fusion vs brute force, emitted-kernel census
(no block barrier: OTPW) and an NVRTC sm_100a compile with a SASS census."""
import itertools
import json
import re
import shutil
import subprocess
from pathlib import Path

import pytest

import paper_1909_07190_b200 as pmg
import pmg_inputs as PI
from paper_1909_07190_b200 import _binding as B

ROOT = Path(__file__).resolve().parents[1]
GOLD = json.loads((ROOT / "tests" / "golden" / "paper_worked_examples.json").read_text())
HDR = "param W, H\nimage img(H, W): f32\n"


def test_exports_every_declared_symbol():
    decl = set(re.findall(r"\b(pmg_[a-z_0-9]+)\s*\(", (ROOT / "include" / "pmg.h").read_text()))
    decl -= {"pmg_pipeline", "pmg_plan"}
    out = subprocess.run(["nm", "-D", "--defined-only", str(B.LIBPATH)], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (pmg_\w+)", out))
    assert decl <= exported, decl - exported
    assert decl <= set(B.EXPORTED), decl - set(B.EXPORTED)
    assert B.lib.pmg_version().decode().startswith("pmg-b200")


@pytest.mark.parametrize("text,frag", [
    (HDR + "stage a(y, x) [H, W]: f32 = img(y, x) +\nliveout a\n", "3:"),
    (HDR + "stage a(y, x) [H, W]: f32 = img(y, z)\nliveout a\n", "undeclared name"),
    (HDR + "stage a(y, x) [H, W]: f32 = imq(y, x)\nliveout a\n", "undeclared stage"),
    (HDR + "stage a(y, x) [H, W]: f32 = a(y, x-1)\nliveout a\n", "cyclic reference"),
    (HDR + "stage a(y, x) [H, W]: f32 = img(y, x)\nstage b(y, x) [H, W]: f32 = img(y, x)\nliveout b\n", "unreachable"),
    ("param W\nliveout a\n", "no stages"),
    (HDR + "stage a(y, x) [H, W]: f32 = img(x)\nliveout a\n", "dims"),
    (HDR + "stage a(y, x) [H, W]: f32 = img(y, x % 2.0)\nliveout a\n", "integer"),
])
def test_parse_errors(text, frag):
    with pytest.raises(pmg.PmgError, match=frag) as ei:
        pmg.Pipeline(text)
    assert ei.value.status == -1


def test_io_descriptors():
    p = pmg.Pipeline(PI.WORKLOADS["camera"].text)
    assert p.params == ["W", "H"]
    ins = p.inputs({"W": 2528, "H": 1920})
    assert [(i.name, i.dtype, i.shape, i.is_table) for i in ins] == [
        ("raw", "u16", (1920, 2528), False), ("ccm", "i32", (12,), True), ("curve", "u8", (1024,), True)]
    outs = p.outputs({"W": 2528, "H": 1920})
    assert [(o.name, o.dtype, o.shape) for o in outs] == [("curved", "u8", (3, 1920, 2528))]
    with pytest.raises(pmg.PmgError):
        p.inputs({"W": 2528})


def test_dependence_vectors_blur():
    """blury at (y, x) consumes blurx at (y-1, x), (y, x), (y+1, x): vectors (1,0,0,-1),(1,0,0,0),(1,0,0,1)
    (§2.3; stage component implicit)."""
    d = pmg.Pipeline(PI.WORKLOADS["blur"].text).describe({"W": 64, "H": 64})
    reads = [r for r in d["reads"] if r["consumer"] == "blury" and r["producer"] == "blurx"]
    assert sorted(r["offset"][1] for r in reads) == GOLD["dependence_vectors_blur"]["y_offsets"]
    assert all(r["form"][1:] == ["unit", "unit"] and r["offset"][2] == 0 for r in reads)
    cam = pmg.Pipeline(PI.WORKLOADS["camera"].text).describe({"W": 64, "H": 48})
    forms = {(r["consumer"], r["producer"]): r["form"] for r in cam["reads"]}
    assert forms[("g_gr", "denoised")][1:] == ["down2", "down2"]
    assert forms[("R", "r_gr")][1:] == ["up2", "up2"]


# ------------------------------------------------------------------ paper worked examples (§3, §4, Alg. 2)
def _analyze(text, params, stages, T, Bk, f=0.0, tx=128, regs=12, gpu="gtx1080ti"):
    return pmg.Pipeline(text).analyze_group(params, stages, T, Bk, frac_reg=f, tx_size=tx, regs_per_stage=regs,
                                            spec=pmg.gpu_spec(gpu), weights_=pmg.weights(gpu))


# the §3 blur walk-through tiles the dimension blury stencils over (reading R11)
BLUR_T = (HDR + "stage blurx(y, x) [H, W]: f32 = ((img(y-1, x) + img(y, x)) + img(y+1, x)) / 3.0\n"
          "stage blury(y, x) [H, W]: f32 = ((blurx(y, x-1) + blurx(y, x)) + blurx(y, x+1)) / 3.0\nliveout blury\n")
P4096 = {"W": 4096, "H": 4096}


def test_warp_sizes_and_warp_tile():
    g = GOLD["warp_sizes"]
    r = _analyze(BLUR_T, P4096, ["blurx", "blury"], GOLD["warp_tile"]["tile"], g["block"])
    assert r["warp"] == g["warp"] and r["warp_tile"] == GOLD["warp_tile"]["warp_tile"]
    for Bk, W in [((32, 1, 1), [32, 1, 1]), ((8, 8, 4), [8, 4, 1]), ((64, 4, 1), [32, 1, 1])]:
        assert _analyze(BLUR_T, P4096, ["blury"], [1, 1, 1], Bk)["warp"] == W


@pytest.mark.parametrize("key", ["blur_overlap_T8", "blur_overlap_T16"])
def test_overlap_fraction(key):
    g = GOLD[key]
    r = _analyze(BLUR_T, P4096, ["blurx", "blury"], [g["tile_x"], 1, 1], [64, 4, 1])
    assert (r["overlap_numerator"], r["overlap_denominator"]) == (g["numerator"], g["denominator"])
    assert round(100 * g["numerator"] / g["denominator"], 1) == g["percent_rounded"]
    assert r["stages"][0]["overlap"] == [2, 0, 0] and r["stages"][1]["overlap"] == [0, 0, 0]


def test_scratchpads_and_occupancy():
    g8, g16 = GOLD["blur_scratchpad_T8"], GOLD["blur_scratchpad_T16"]
    r8 = _analyze(BLUR_T, P4096, ["blurx", "blury"], g8["tile"], g8["block"])
    assert r8["stages"][0]["scratchpad"] == g8["floats"]
    r16 = _analyze(BLUR_T, P4096, ["blurx", "blury"], g16["tile"], g16["block"])
    assert r16["stages"][0]["scratchpad"] == g16["floats"]
    assert r16["cost"]["shMemPerTB"] == 4 * g16["floats"] > g16["bytes_over"]
    # 62.5 % occupancy shared-only, 100 % with half the tile in registers (24 + 8 regs)
    assert r16["cost"]["occupancy"] == GOLD["blur_occupancy_shared_T16"]["occupancy"]
    rh = _analyze(BLUR_T, P4096, ["blurx", "blury"], g16["tile"], g16["block"], f=0.5)
    assert rh["cost"]["regPerTh"] == 32 and rh["cost"]["occupancy"] == GOLD["blur_occupancy_hybrid_T16"]["occupancy"]


def test_alg2_arithmetic():
    r = _analyze(BLUR_T, P4096, ["blurx", "blury"], [8, 1, 1], [64, 4, 1])
    assert abs(r["cost"]["warpBW"] - GOLD["warp_bw_1080ti"]["bytes_per_s"]) < 1.0
    c = r["cost"]
    w = GOLD["weights"]["gtx1080ti"]
    ratio = c["memTime"] / c["computeTime"]
    exp = (w[0] * c["txsPerPoint"] + w[1] * (1 - c["occupancy"]) + w[2] * ratio + w[3] * c["unallocatedShMem"]
           + w[4] * c["unusedReg"] + w[5] * c["fracOverlap"] + w[6] * c["extraTBs"])
    assert abs(c["cost"] - exp) < 1e-9 * max(1, abs(exp))
    assert 0 <= c["occupancy"] <= 1 and 0 <= c["fracOverlap"] < 1
    # infinite cost when a hard limit is violated (Alg. 2, 961)
    big = _analyze(BLUR_T, P4096, ["blurx", "blury"], [32, 32, 1], [256, 4, 1])
    assert big["cost"]["infinite"] and big["cost"]["cost"] == "inf"
    regs = _analyze(BLUR_T, P4096, ["blurx", "blury"], [8, 1, 1], [64, 4, 1], regs=200)
    assert regs["cost"]["infinite"]


def test_non_constant_dependences_are_infinite():
    """A group across a x2 downsample edge is infeasible (Alg. 2)."""
    p = PI.WORKLOADS["camera"]
    r = _analyze(p.text, {"W": 64, "H": 48}, ["denoised", "g_gr"], [1, 1, 1], [32, 1, 1])
    assert r["cost"]["infinite"]


def test_presets_match_tables():
    for name in ("gtx1080ti", "teslav100"):
        s = pmg.gpu_spec(name).as_dict()
        for k, v in GOLD["gpu_tables"][name].items():
            assert s[k] == v, (name, k)
        assert list(pmg.weights(name).w) == GOLD["weights"][name]
    b = pmg.gpu_spec("b200").as_dict()
    assert b["nsms"] == 148 and b["gl_mem_bw"] == 6538.6e9 and b["max_shmem_per_tb"] == 227 * 1024
    with pytest.raises(pmg.PmgError):
        pmg.gpu_spec("h100")


# ------------------------------------------------------------------ selector: DP vs brute force
CHAIN = (HDR + "stage a(y, x) [H, W]: f32 = (img(y, x-1) + img(y, x)) + img(y, x+1)\n"
         "stage b(y, x) [H, W]: f32 = (a(y-1, x) + a(y, x)) + a(y+1, x)\n"
         "stage c(y, x) [H, W]: f32 = b(y, x) * 0.5\n"
         "stage d(y, x) [H, W]: f32 = (c(y, x-1) + c(y, x)) + c(y+1, x)\nliveout d\n")
DIAMOND = (HDR + "stage A(y, x) [H, W]: f32 = img(y, x) * 2.0\n"
           "stage B(y, x) [H, W]: f32 = A(y, x-1) + A(y, x+1)\n"
           "stage C(y, x) [H, W]: f32 = A(y-1, x) + A(y+1, x)\n"
           "stage D(y, x) [H, W]: f32 = B(y, x) + C(y, x)\nliveout D\n")


@pytest.mark.parametrize("text", [CHAIN, DIAMOND, PI.WORKLOADS["unsharp"].text])
def test_dp_fusion_equals_brute_force(text):
    """DP over contiguous topological runs == exhaustive enumeration of those partitions."""
    p = pmg.Pipeline(text)
    params = {"W": 512, "H": 512}
    kw = dict(vec=2, chunks=1, rows=16, warps=4, prefetch=4, tx_size=32, probe=False)
    dp = p.schedule(params, opts=pmg.sched_opts(**kw))
    order = [s for g in dp["groups"] for s in g["config"]["stages"]]   # topological order
    stages = p.stages
    n = len(order)
    best = None
    for cuts in itertools.product([0, 1], repeat=n - 1):
        gos, gid = [0] * len(stages), 0
        for i, s in enumerate(order):
            if i and cuts[i - 1]:
                gid += 1
            gos[stages.index(s)] = gid
        try:
            r = p.schedule(params, opts=pmg.sched_opts(group_of_stage=gos, **kw))
        except pmg.PmgError:
            continue
        if best is None or r["total_cost"] < best[0] - 1e-9:
            best = (r["total_cost"], [g["config"]["stages"] for g in r["groups"]])
    assert abs(dp["dp_cost"] - best[0]) < 1e-9 * max(1.0, abs(best[0]))
    assert [g["config"]["stages"] for g in dp["groups"]] == best[1]


def test_schedule_is_deterministic_and_fuses_blur():
    p = pmg.Pipeline(PI.WORKLOADS["blur"].text)
    o = pmg.sched_opts(probe=False)
    a, b = p.schedule({"W": 4096, "H": 4096}, opts=o), p.schedule({"W": 4096, "H": 4096}, opts=o)
    assert a == b
    assert len(a["groups"]) == 1 and a["groups"][0]["config"]["stages"] == ["blurx", "blury"]


def test_band_geometry_host():
    p = pmg.Pipeline(PI.WORKLOADS["harris"].text)
    o = pmg.sched_opts(probe=False)
    prm = {"W": 640, "H": 480}
    bands = [p.band_rows(prm, b, 4, opts=o) for b in range(4)]
    assert [b[:2] for b in bands] == [(0, 120), (120, 240), (240, 360), (360, 480)]
    assert [b[2:] for b in bands] == [(0, 122), (118, 242), (238, 362), (358, 480)]   # +-2 rows of halo


@pytest.mark.parametrize("wl,n", [
    (PI.Workload("ll", "local_laplacian_J4K4.pmg", {"W": 64, "H": 192}, 1005), 4),   # up/down + general y/2-1+2*(y%2)
    (PI.small("camera", 64, 96), 3),
    (PI.small("unsharp", 48, 64), 4),
])
def test_band_input_rows_suffice(wl, n):
    """Band geometry pinned against the oracle, not against itself: replacing every input row
    outside [in_r0, in_r1) by unrelated values must leave the band's output rows [out_r0, out_r1) unchanged.
    For the local Laplacian this exercises the interval analysis of the non-affine upsample row index."""
    import numpy as np
    from oracle import evaluate
    p = pmg.Pipeline(wl.text)
    inp = wl.inputs()
    full = evaluate(wl.text, wl.params, inp)
    (key, ref), = full.items()
    H = wl.params["H"]
    rng = np.random.default_rng(7)
    covered = []
    for b in range(n):
        o_r0, o_r1, i_r0, i_r1 = p.band_rows(wl.params, b, n, opts=pmg.sched_opts(probe=False))
        covered.append((o_r0, o_r1))
        pois = {}
        for name, v in inp.items():
            if v.ndim < 2:
                pois[name] = v
                continue
            w = v.copy()
            junk = (rng.integers(0, 1024, size=v.shape).astype(v.dtype) if v.dtype.kind in "iu"
                    else rng.random(v.shape).astype(v.dtype))
            w[..., :i_r0, :] = junk[..., :i_r0, :]
            w[..., i_r1:, :] = junk[..., i_r1:, :]
            pois[name] = w
        got = evaluate(wl.text, wl.params, pois)[key]
        np.testing.assert_array_equal(got[..., o_r0:o_r1, :].view(np.uint8), ref[..., o_r0:o_r1, :].view(np.uint8))
        if 0 < b < n - 1:
            assert i_r1 - i_r0 < H        # a middle band does not need the whole image
    assert covered[0][0] == 0 and covered[-1][1] == H
    assert all(covered[i][1] == covered[i + 1][0] for i in range(n - 1))


# ------------------------------------------------------------------ emitted kernels: OTPW synchronisation
@pytest.mark.parametrize("name", ["blur", "harris", "unsharp", "camera"])
def test_emitted_kernels_use_only_warp_synchronisation(name):
    """OTPW "does not employ thread block synchronization at all"."""
    wl = PI.WORKLOADS[name]
    pipe = pmg.Pipeline(wl.text)
    one = [0] * len(pipe.stages) if name == "harris" else None      # the fully fused Harris group
    e = pipe.emit(wl.params, opts=pmg.sched_opts(probe=False, group_of_stage=one))
    for g in e["groups"]:
        src = g["source"]
        assert "__syncthreads" not in src and "bar.sync" not in src
        if "pmg_mbar_wait" in src:       # groups staging inputs through the warp's TMA ring
            assert "__syncwarp" in src
    if name == "harris":
        assert any("pmg_shfl(" in g["source"] for g in e["groups"])   # load types (3)/(4): neighbour-lane registers


@pytest.mark.skipif(shutil.which("cuobjdump") is None, reason="cuobjdump not available")
def test_nvrtc_sm100a_sass_census(tmp_path):
    """Compile the Harris group for sm_100a on the host (NVRTC, no GPU) and inspect the SASS: TMA bulk
    copies (UBLKCP) + mbarriers (SYNCS), warp shuffles (SHFL), no block barrier (BAR.*), no spills."""
    wl = PI.WORKLOADS["harris"]
    pipe = pmg.Pipeline(wl.text)
    opts = pmg.sched_opts(vec=4, chunks=1, rows=24, warps=4, prefetch=8, probe=False, group_of_stage=[0] * len(pipe.stages))
    rep = pipe.precompile(wl.params, str(tmp_path), opts=opts)
    k = rep["kernels"][0]
    assert k["spill_stores"] == 0 and k["regs"] > 0
    cubins = list(tmp_path.glob("*.cubin"))
    assert cubins
    sass = subprocess.run(["cuobjdump", "-sass", str(cubins[0])], capture_output=True, text=True).stdout
    assert "UBLKCP" in sass and "SYNCS" in sass and "SHFL" in sass
    assert not re.search(r"\bBAR\.(SYNC|RED|ARV)", sass)


@pytest.mark.parametrize("wl", [PI.Workload("ll", "local_laplacian_J4K4.pmg", {"W": 96, "H": 64}, 1005),
                                PI.small("local_laplacian", 256, 128), PI.small("camera", 96, 64),
                                PI.small("harris", 64, 48), PI.Workload("pb", "pyramid_blend_J3.pmg", {"W": 64, "H": 48}, 1006)],
                         ids=lambda w: w.pipeline)
def test_inlining_preserves_the_definition(wl):
    """The inlining pass (inline.cpp) rewrites the pipeline text; the oracle evaluates the rewritten text and
    the text as written, and the liveouts must agree bit for bit (clamped substitution, stored-value casts)."""
    import numpy as np
    from oracle import evaluate
    p = pmg.Pipeline(wl.text)
    r = p.inlined(wl.params)
    inp = wl.inputs("structured") if "laplacian" in wl.pipeline else wl.inputs()
    a, b = evaluate(wl.text, wl.params, inp), evaluate(r["text"], wl.params, inp)
    assert a.keys() == b.keys()
    for k in a:
        np.testing.assert_array_equal(a[k].view(np.uint8), b[k].view(np.uint8))
    if "laplacian" in wl.pipeline:
        assert "gP0" in r["inlined"] and "lP0" in r["inlined"]      # the 8-plane full-resolution stages
        assert "gDx1/y" in r["split"]                               # phase split of the downsample pairs
    elif "pyramid" in wl.pipeline:
        assert "ADx1/y" in r["split"]
    else:
        assert r["inlined"] == []                                   # nothing data-expanding to substitute
    if "camera" in wl.pipeline:   # denoise -> quad-grid phases; R, G, B and their readers -> quad phases + interleave
        assert r["split"] == ["denoised/y", "denoised_ye/x", "denoised_yo/x", "R/up-yx", "corrected_ye_xe/planes",
                              "corrected_yo_xe/planes", "corrected_ye_xo/planes", "corrected_yo_xo/planes"]


PHASE = """param W, H
image img(H, W): f32
stage s(y, x) [H, W]: f32 = img(y, x) * 2.0 + img(y, x + 1)
stage c(y, x) [H / 2, W / 2]: f32 = ((((((s(2*y-3, 2*x) + 0.5 * s(2*y-2, 2*x+1)) + 0.25 * s(2*y-1, 2*x-1)) + s(2*y, 2*x) * 3.0) + s(2*y+1, 2*x+2)) + s(2*y+2, 2*x-2) * 0.125) + s(2*y+3, 2*x+3))
liveout c
"""


@pytest.mark.parametrize("W,H", [(2, 2), (4, 6), (10, 8), (6, 16), (12, 14)])
def test_phase_split_exact_at_every_edge(W, H):
    """Alignment & scaling by phase splitting (phase.cpp): a stage read only as s(2v + b) is replaced
    by its two phases; reads with b in [-3, 3] exercise both edge selects (q >= 1 at the high edge, q <= -1 at the
    low edge) in both dims at sizes down to 2 x 2.  The oracle must give the same bits for both texts."""
    import numpy as np
    from oracle import evaluate
    p = pmg.Pipeline(PHASE)
    r = p.inlined({"W": W, "H": H})
    assert r["split"] == ["s/y", "s_ye/x", "s_yo/x"]
    img = np.random.default_rng(W * 100 + H).random((H, W), dtype=np.float32)
    a = evaluate(PHASE, {"W": W, "H": H}, {"img": img})["c"]
    b = evaluate(r["text"], {"W": W, "H": H}, {"img": img})["c"]
    np.testing.assert_array_equal(a.view(np.uint32), b.view(np.uint32))


UPSPLIT = """param W, H
image lo(H / 2, W / 2): f32
image img(H, W): f32
stage up(y, x) [H, W]: f32 = select(y % 2 == 0, lo(y / 2, x / 2), lo((y + 1) / 2, (x - 1) / 2) * 0.5)
stage up2(y, x) [H, W]: f32 = lo((y - 1) / 2, x / 2) + select(x % 2 == 1, 1.0, 2.0)
stage c(y, x) [H, W]: f32 = ((((up(y - 1, x) + up(y + 2, x + 1)) + up(y, x - 2)) + up(y - 2, x + 2)) * img(y, x) + up(y + 1, x - 1)) + ((((up2(y, x - 2) + up2(y + 1, x)) + up2(y - 1, x + 1)) + up2(y, x)) * 0.5 + up2(y + 2, x - 1))
liveout c
"""


@pytest.mark.parametrize("W,H", [(4, 4), (6, 8), (10, 12), (16, 6)])
def test_up_split_exact_at_every_edge(W, H):
    """Upsampling edges (phase.cpp, reader split): stages using y, x only as (v + b) / 2 and (v + b) % 2 become four
    quad-resolution phases, their reader c too (reads at offsets -2..2 exercise the edge selects in both dims), and
    the liveout is rebuilt as the interleave of its phases.  The oracle must give the same bits for both texts."""
    import numpy as np
    from oracle import evaluate
    p = pmg.Pipeline(UPSPLIT)
    r = p.inlined({"W": W, "H": H})
    assert r["inlined"] == [] and r["split"] == ["up/up-yx"]
    rng = np.random.default_rng(W * 31 + H)
    inp = {"lo": rng.random((H // 2, W // 2), dtype=np.float32), "img": rng.random((H, W), dtype=np.float32)}
    a = evaluate(UPSPLIT, {"W": W, "H": H}, inp)["c"]
    b = evaluate(r["text"], {"W": W, "H": H}, inp)["c"]
    np.testing.assert_array_equal(a.view(np.uint32), b.view(np.uint32))
