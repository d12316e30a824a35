"""Pins for the independent oracle (oracle/pmg_oracle.py) against things other than itself:
brute-force loops on tiny images, closed forms, invariants, exact-arithmetic (f64) bounds and the
parse-error taxonomy of SPEC.md lines 40-47.  CPU only."""
import numpy as np
import pytest

import brute
import pmg_inputs as PI
from oracle import OracleError, evaluate, parse
from oracle.pmg_oracle import Evaluator

HDR = "param W, H\n"


def run(text, W, H, inputs, **kw):
    return evaluate(text, {"W": W, "H": H}, inputs, **kw)


# ----------------------------------------------------------------------------- brute force (bit-exact)
@pytest.mark.parametrize("W,H", [(1, 1), (2, 3), (7, 5), (13, 11)])
def test_blur_matches_bruteforce(W, H):
    w = PI.small("blur", W, H)
    img = w.inputs()["img"]
    got = evaluate(w.text, w.params, {"img": img})["blury"]
    np.testing.assert_array_equal(got, brute.blur(img))


@pytest.mark.parametrize("W,H", [(1, 1), (3, 2), (9, 7), (12, 10)])
def test_harris_matches_bruteforce(W, H):
    w = PI.small("harris", W, H)
    img = w.inputs()["img"]
    got = evaluate(w.text, w.params, {"img": img})["harris"]
    np.testing.assert_array_equal(got, brute.harris(img))


@pytest.mark.parametrize("variant", ["uniform", "structured"])
def test_unsharp_matches_bruteforce(variant):
    w = PI.small("unsharp", 11, 9)
    img = w.inputs(variant)["img"]
    got = evaluate(w.text, w.params, {"img": img})["masked"]
    np.testing.assert_array_equal(got, brute.unsharp(img))


def test_camera_matches_bruteforce():
    w = PI.small("camera", 14, 10)
    inp = w.inputs()
    got = evaluate(w.text, w.params, inp)["curved"]
    np.testing.assert_array_equal(got, brute.camera(inp["raw"], inp["ccm"], inp["curve"]))


# ----------------------------------------------------------------------------- closed forms / invariants
def test_blur_constant_and_integer_ramp_exact():
    w = PI.small("blur", 16, 12)
    c = np.full((12, 16), 0.375, np.float32)
    np.testing.assert_array_equal(evaluate(w.text, w.params, {"img": c})["blury"], c)
    yy, xx = np.mgrid[0:12, 0:16]
    ramp = (3 * xx + 6 * yy).astype(np.float32)       # sums of 3 small integers, /3 exact
    out = evaluate(w.text, w.params, {"img": ramp})["blury"]
    np.testing.assert_array_equal(out[1:-1, 1:-1], ramp[1:-1, 1:-1])


def test_blur_separable_equals_2d_kernel():
    """Separable blur == direct 3x3/9 kernel with clamped reads (f64 exact arithmetic)."""
    w = PI.small("blur", 23, 17)
    img = w.inputs()["img"]
    got64 = evaluate(w.text, w.params, {"img": img}, precision="f64")["blury"]
    p = np.pad(img.astype(np.float64), 1, mode="edge")
    direct = sum(p[1 + dy:1 + dy + 17, 1 + dx:1 + dx + 23] for dy in (-1, 0, 1) for dx in (-1, 0, 1)) / 9.0
    # interior: blurx(y±1) unclamped == direct; borders: both clamp-to-edge of img then of blurx.
    np.testing.assert_allclose(got64, direct, rtol=0, atol=1e-12)
    got32 = evaluate(w.text, w.params, {"img": img})["blury"]
    assert np.max(np.abs(got32 - direct)) < 3e-7


def test_intermediate_clamp_is_producer_clamp():
    """Reading blurx at x=-1 yields blurx(0) (producer clamp), not blurx computed from clamped img (R1)."""
    text = HDR + ("image img(H, W): f32\n"
                  "stage a(y, x) [H, W]: f32 = img(y, x-1) + 2.0 * img(y, x+1)\n"
                  "stage b(y, x) [H, W]: f32 = a(y, x-1)\n"
                  "liveout b\n")
    img = np.arange(5, dtype=np.float32)[None, :] + 1
    a = np.array([[1 + 4, 1 + 6, 2 + 8, 3 + 10, 4 + 10]], np.float32)   # img clamped inside a
    b = run(text, 5, 1, {"img": img})["b"]
    np.testing.assert_array_equal(b, np.array([[a[0, 0], a[0, 0], a[0, 1], a[0, 2], a[0, 3]]]))


def test_harris_constant_is_zero():
    """Constant image: every derivative sum cancels; exactly for dyadic constants (all partial sums
    exact), to within products of f32 rounding residuals otherwise."""
    w = PI.small("harris", 10, 9)
    for c in (0.0, 0.5, 0.375):
        out = evaluate(w.text, w.params, {"img": np.full((9, 10), c, np.float32)})["harris"]
        assert np.all(out == 0.0)
    for c in (0.1, 0.7391):
        out = evaluate(w.text, w.params, {"img": np.full((9, 10), c, np.float32)})["harris"]
        assert np.max(np.abs(out)) < 1e-30


def test_harris_ramp_closed_form():
    """Interior (>=2 px from the border) of img = a*x + b*y: Ix = 2a/3, Iy = 2b/3, det = 0,
    trace = 4(a^2+b^2), harris = -0.64 (a^2+b^2)^2 (exact arithmetic; k12 literal = 0.083333333)."""
    a, b = 0.013, -0.021
    yy, xx = np.mgrid[0:14, 0:15]
    img = (a * xx + b * yy).astype(np.float32)
    w = PI.small("harris", 15, 14)
    st = evaluate(w.text, w.params, {"img": img}, precision="f64", keep_all=True)
    ia, ib = img[2, 3] - img[2, 2], img[3, 2] - img[2, 2]      # the f32 ramp's actual slopes
    k = 0.083333333
    sl = (slice(2, -2), slice(2, -2))
    np.testing.assert_allclose(st["Ix"][sl], 8 * k * ia, rtol=2e-5)
    np.testing.assert_allclose(st["Iy"][sl], 8 * k * ib, rtol=2e-5)
    s = (8 * k) ** 2 * 9
    np.testing.assert_allclose(st["trace"][sl], s * (ia * ia + ib * ib), rtol=1e-4)
    assert np.max(np.abs(st["det"][sl])) < 1e-6 * s * s * (ia * ia + ib * ib) ** 2 + 1e-15
    np.testing.assert_allclose(st["harris"][sl], -0.04 * (s * (ia * ia + ib * ib)) ** 2, rtol=1e-3)


def test_unsharp_constant_and_ramp():
    w = PI.small("unsharp", 12, 10)
    c = np.full((3, 10, 12), 0.375, np.float32)
    np.testing.assert_array_equal(evaluate(w.text, w.params, {"img": c})["masked"], c)
    yy, xx = np.mgrid[0:10, 0:12]
    ramp = np.stack([(0.01 * xx + 0.02 * yy + 0.1 * k) for k in range(3)]).astype(np.float32)
    out = evaluate(w.text, w.params, {"img": ramp})["masked"]
    np.testing.assert_array_equal(out[:, 2:-2, 2:-2], ramp[:, 2:-2, 2:-2])   # blur preserves linear


def test_unsharp_select_branches_both_taken():
    w = PI.small("unsharp", 64, 48)
    img = w.inputs("structured")["img"]
    st = evaluate(w.text, w.params, {"img": img}, keep_all=True)
    take_img = np.abs(img - st["blury"]) < np.float32(0.001)
    assert take_img.any() and (~take_img).any()
    np.testing.assert_array_equal(st["masked"], np.where(take_img, img, st["sharpen"]))


def test_camera_flat_field_and_hot_pixel():
    w = PI.small("camera", 16, 12)
    ccm, curve = PI.camera_ccm(), PI.camera_curve()
    for v in (25, 300, 777, 1023):
        raw = np.full((12, 16), v, np.uint16)
        out = evaluate(w.text, w.params, {"raw": raw, "ccm": ccm, "curve": curve})["curved"]
        for c in range(3):
            exp = (int(ccm[4 * c + 3]) + (int(ccm[4 * c]) + int(ccm[4 * c + 1]) + int(ccm[4 * c + 2])) * v) >> 8
            assert np.all(out[c] == curve[min(max(exp, 0), 1023)])
        if v < 1023:
            hot = raw.copy()
            hot[5, 7] = 1023
            out2 = evaluate(w.text, w.params, {"raw": hot, "ccm": ccm, "curve": curve})["curved"]
            np.testing.assert_array_equal(out2, out)


def test_camera_demosaic_follows_edges():
    """A vertical edge in the green channel: green at R sites is interpolated along the edge (vertical)."""
    w = PI.small("camera", 16, 12)
    raw = np.full((12, 16), 200, np.uint16)
    raw[:, 8:] = 800
    st = evaluate(w.text, w.params, {"raw": raw, "ccm": PI.camera_ccm(), "curve": PI.camera_curve()},
                  keep_all=True)
    g_r = st["g_r"]
    assert np.all(g_r[:, :3] == 200) and np.all(g_r[:, 4:] == 800)


def _ll(J=4, K=4, W=64, H=48):
    from pathlib import Path
    import importlib.util
    spec = importlib.util.spec_from_file_location("genll", Path(PI.PIPELINES) / "gen_local_laplacian.py")
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m.generate(J, K), {"W": W, "H": H}


def test_local_laplacian_alpha0_is_pointwise():
    """alpha = 0, beta = 1: every processed plane equals gray, the Laplacian collapse telescopes back to
    gray, so out = clamp(gray (in + eps) / (gray + eps), 0, 1)  (exact arithmetic)."""
    text, p = _ll()
    inp = PI.uniform((3, 48, 64), 7)
    out = evaluate(text, p, {"inp": inp, "remap": np.zeros(2 * 3 * 256 + 1, np.float32)}, precision="f64")["out"]
    i = inp.astype(np.float64)
    gray = (0.299 * i[0] + 0.587 * i[1]) + 0.114 * i[2]      # f64 mode: literals are f64(decimal)
    exp = np.clip(gray * (i + 0.01) / (gray + 0.01), 0, 1)
    np.testing.assert_allclose(out, exp, rtol=0, atol=1e-12)


def test_local_laplacian_down_up_of_ramp():
    """Downsample of a ramp a*x is a*(2x+0.5); up(down(ramp)) == ramp >= 3 px from the border."""
    text, p = _ll()
    yy, xx = np.mgrid[0:48, 0:64]
    g = ((xx + 2 * yy) / 1024.0 + 0.125).astype(np.float32)        # dyadic: exact in f32
    inp = np.stack([g, g, g])
    st = evaluate(text, p, {"inp": inp, "remap": np.zeros(1537, np.float32)}, precision="f64", keep_all=True)
    s = (0.299 + 0.587) + 0.114                                     # gray = s * g exactly (f64 mode)
    xs = 2 * np.arange(32) + 0.5
    exp = s * ((xs[None, :] + 2 * np.arange(48)[:, None]) / 1024.0 + 0.125)
    np.testing.assert_allclose(st["inDx1"][:, 1:-1], exp[:, 1:-1], rtol=0, atol=1e-12)
    # lP0 = gP0 - up(gP1) vanishes on a ramp away from the border (up o down reproduces the ramp)
    assert np.max(np.abs(st["lP0"][:, 3:-3, 3:-3])) < 1e-12


def test_local_laplacian_shapes_and_stage_count():
    prog = parse((PI.PIPELINES / "local_laplacian.pmg").read_text())
    assert len(prog.stages) == 67
    ev = Evaluator(prog, {"W": 2560, "H": 1536})
    assert ev.shape_of("gP7") == (8, 12, 20) and ev.shape_of("out") == (3, 1536, 2560)


# ----------------------------------------------------------------------------- pyramid blend (NEXT-4)
def _pb(W=64, H=48):
    return (PI.PIPELINES / "pyramid_blend_J3.pmg").read_text(), {"W": W, "H": H}


@pytest.mark.parametrize("which", ["ones", "zeros"])
def test_pyramid_blend_constant_mask_reconstructs_one_image(which):
    """Mask == 1 (resp. 0): every blended level is lA_j (lB_j) exactly, and the Laplacian collapse
    telescopes back to A (B): oG_j = up(oG_{j+1}) + XG_j - up(XG_{j+1}) = XG_j by induction (exact
    arithmetic; f64 mode)."""
    text, p = _pb()
    A, B = PI.uniform((3, 48, 64), 3), PI.uniform((3, 48, 64), 4)
    M = np.full((48, 64), 1.0 if which == "ones" else 0.0, np.float32)
    out = evaluate(text, p, {"A": A, "B": B, "M": M}, precision="f64")["out"]
    np.testing.assert_allclose(out, (A if which == "ones" else B).astype(np.float64), rtol=0, atol=1e-12)


def test_pyramid_blend_identical_images_ignore_the_mask():
    text, p = _pb()
    A = PI.uniform((3, 48, 64), 5)
    out = evaluate(text, p, {"A": A, "B": A, "M": PI.uniform((48, 64), 6)}, precision="f64")["out"]
    np.testing.assert_allclose(out, A.astype(np.float64), rtol=0, atol=1e-12)


def test_pyramid_blend_down_up_of_ramp():
    """[1 3 3 1]/8 downsample of a ramp a*x is a*(2x+0.5); the (x+1)/2, (x-1)/2 linear upsample maps a
    coarse ramp back to a*(x-0.5)/2, so lA0 = AG0 - up(AG1) vanishes away from the border."""
    text, p = _pb()
    yy, xx = np.mgrid[0:48, 0:64]
    g = ((xx + 2 * yy) / 1024.0 + 0.125).astype(np.float32)
    A = np.stack([g, g, g])
    st = evaluate(text, p, {"A": A, "B": A, "M": np.zeros((48, 64), np.float32)}, precision="f64", keep_all=True)
    xs = 2 * np.arange(32) + 0.5
    np.testing.assert_allclose(st["ADx1"][0][:, 1:-1], ((xs[None, :] + 2 * np.arange(48)[:, None]) / 1024.0 + 0.125)[:, 1:-1],
                               rtol=0, atol=1e-12)
    assert np.max(np.abs(st["lA0"][:, 3:-3, 3:-3])) < 1e-12


def test_pyramid_blend_shapes_and_stage_count():
    prog = parse((PI.PIPELINES / "pyramid_blend.pmg").read_text())
    assert len(prog.stages) == 41
    ev = Evaluator(prog, {"W": 3840, "H": 2160})
    assert ev.shape_of("AG3") == (3, 270, 480) and ev.shape_of("MG3") == (270, 480)
    assert ev.shape_of("out") == (3, 2160, 3840)


# ----------------------------------------------------------------------------- multiscale interpolation (NEXT-4)
def _mi(W=96, H=64):
    return (PI.PIPELINES / "multiscale_interp_J4.pmg").read_text(), {"W": W, "H": H}


def test_multiscale_interp_full_alpha_is_identity():
    """alpha == 1 everywhere: I_0 = d_0 + (1 - 1) * up = d_0 = (c * 1, 1), so out = (c * 1) / 1 = c bit for bit
    (IEEE: x * 1 = x, 0 * finite = 0, x + 0 = x, x / 1 = x) whatever the pyramid holds."""
    text, p = _mi()
    rgb = PI.uniform((3, 64, 96), 11)
    inp = np.concatenate([rgb, np.ones((1, 64, 96), np.float32)])
    out = evaluate(text, p, {"inp": inp})["out"]
    np.testing.assert_array_equal(out.view(np.uint32), rgb.view(np.uint32))


def test_multiscale_interp_single_colour_fills_every_hole():
    """Every known sample has colour v: each premultiplied plane is v * alpha, every stage is linear in its
    inputs, so in exact arithmetic I_l(c) = v * I_l(3) at every level and out == v at every pixel (also in the
    holes); the f64 evaluation reaches it to rounding, the f32 one to 1e-5."""
    text, p = _mi()
    inp = PI.sparse_rgba(64, 96, 12)
    v = np.array([0.25, 0.5, 0.875], np.float32)
    inp[:3] = v[:, None, None]
    for prec, tol in [("f64", 1e-12), ("f32", 1e-5)]:
        out = evaluate(text, p, {"inp": inp}, precision=prec)["out"]
        assert np.max(np.abs(out - v[:, None, None])) < tol, prec


def test_multiscale_interp_keeps_known_samples_exactly_where_alpha_is_one():
    """Where alpha == 1, I_0 = d_0 + 0 * up_0 = (c, 1) exactly, so out(c) = c bit for bit at every sample."""
    text, p = _mi()
    inp = PI.sparse_rgba(64, 96, 13)
    out = evaluate(text, p, {"inp": inp})["out"]
    m = inp[3] == 1.0
    np.testing.assert_array_equal(out[:, m].view(np.uint32), inp[:3][:, m].view(np.uint32))


def test_multiscale_interp_shapes_and_stage_count():
    prog = parse((PI.PIPELINES / "multiscale_interp.pmg").read_text())
    assert len(prog.stages) == 47
    ev = Evaluator(prog, {"W": 2560, "H": 1536})
    assert ev.shape_of("pd9") == (4, 3, 5) and ev.shape_of("out") == (3, 1536, 2560)


# ----------------------------------------------------------------------------- f32 vs exact arithmetic
@pytest.mark.parametrize("name,W,H,tol", [("blur", 40, 30, 1e-6), ("unsharp", 40, 30, 1e-5),
                                          ("harris", 40, 30, None), ("pyramid_blend", 64, 48, 1e-5)])
def test_f32_within_tolerance_of_exact(name, W, H, tol):
    w = PI.small(name, W, H)
    inp = w.inputs()
    o32 = evaluate(w.text, w.params, inp)
    o64 = evaluate(w.text, w.params, inp, precision="f64")
    for k in o32:
        d = np.abs(o32[k].astype(np.float64) - o64[k])
        if tol is None:    # accumulation-derived liveout: range-relative bound
            assert d.max() <= 1e-5 * np.abs(o64[k]).max()
        else:
            assert d.max() <= tol


# ----------------------------------------------------------------------------- integer semantics (R4)
def test_integer_semantics():
    text = HDR + ("image img(H, W): i32\n"
                  "stage q(y, x) [H, W]: i32 = img(y, x) / 4\n"
                  "stage r(y, x) [H, W]: i32 = img(y, x) % 4\n"
                  "stage s(y, x) [H, W]: i32 = img(y, x) >> 1\n"
                  "stage t(y, x) [H, W]: u8 = img(y, x) * 3\n"
                  "stage u(y, x) [H, W]: i32 = i32(f32(img(y, x)) * 0.75)\n"
                  "stage v(y, x) [H, W]: i16 = ((((q(y,x) + r(y,x)) + s(y,x)) + t(y,x)) + u(y,x)) * 1000\n"
                  "liveout v, q, r, s, t, u\n")
    img = np.array([[-7, -1, 0, 5, 100]], np.int32)
    o = run(text, 5, 1, {"img": img})
    np.testing.assert_array_equal(o["q"], [[-2, -1, 0, 1, 25]])
    np.testing.assert_array_equal(o["r"], [[1, 3, 0, 1, 0]])
    np.testing.assert_array_equal(o["s"], [[-4, -1, 0, 2, 50]])
    np.testing.assert_array_equal(o["t"], np.array([[-21, -3, 0, 15, 300]]).astype(np.int64) % 256)
    np.testing.assert_array_equal(o["u"], [[-5, 0, 0, 3, 75]])
    tot = (np.array([[-2, -1, 0, 1, 25]]) + [[1, 3, 0, 1, 0]] + [[-4, -1, 0, 2, 50]]
           + (np.array([[-21, -3, 0, 15, 300]]) % 256) + [[-5, 0, 0, 3, 75]]) * 1000
    np.testing.assert_array_equal(o["v"], tot.astype(np.int16))


def test_builtins():
    text = HDR + ("image img(H, W): f32\n"
                  "stage a(y, x) [H, W]: f32 = lerp(img(y, x), 10.0, 0.25)\n"
                  "stage b(y, x) [H, W]: f32 = clamp(img(y, x), 0.5, 2.0) + min(img(y, x), 1.0) * max(img(y, x), 1.0)\n"
                  "stage c(y, x) [H, W]: f32 = select(img(y, x) > 1.0 && img(y, x) < 3.0, sqrt(img(y, x)), abs(0.0 - img(y, x)))\n"
                  "stage d(y, x) [H, W]: i32 = absd(i32(img(y, x)), 2) + sat_u8(i32(img(y, x)) * 100)\n"
                  "liveout a, b, c, d\n")
    x = np.array([[0.0, 0.25, 1.5, 2.0, 4.0]], np.float32)
    o = run(text, 5, 1, {"img": x})
    f = np.float32
    np.testing.assert_array_equal(o["a"], (x * (f(1) - f(0.25))) + f(10.0) * f(0.25))
    np.testing.assert_array_equal(o["b"], np.clip(x, 0.5, 2.0) + np.minimum(x, 1) * np.maximum(x, 1))
    np.testing.assert_array_equal(o["c"], np.where((x > 1) & (x < 3), np.sqrt(x), np.abs(x)))
    xi = x.astype(np.int32)
    np.testing.assert_array_equal(o["d"], np.abs(xi - 2) + np.clip(xi * 100, 0, 255))


# ----------------------------------------------------------------------------- structure / errors
def test_topo_order_declaration_ties():
    text = HDR + ("image img(H, W): f32\n"
                  "stage A(y, x) [H, W]: f32 = img(y, x)\n"
                  "stage B(y, x) [H, W]: f32 = A(y, x)\n"
                  "stage C(y, x) [H, W]: f32 = A(y, x)\n"
                  "stage D(y, x) [H, W]: f32 = B(y, x) + C(y, x)\n"
                  "liveout D\n")
    assert parse(text).topo_order() == ["A", "B", "C", "D"]
    prog = parse((PI.PIPELINES / "harris.pmg").read_text())
    order = prog.topo_order()
    for s in prog.stages:
        for p in prog.producers(s):
            assert order.index(p) < order.index(s)


@pytest.mark.parametrize("text,msg", [
    (HDR + "image img(H, W): f32\nstage a(y, x) [H, W]: f32 = img(y, x) +\nliveout a\n", "3:"),
    (HDR + "image img(H, W): f32\nstage a(y, x) [H, W]: f32 = img(y, z)\nliveout a\n", "undeclared name"),
    (HDR + "image img(H, W): f32\nstage a(y, x) [H, W]: f32 = imq(y, x)\nliveout a\n", "undeclared stage"),
    (HDR + "image img(H, W): f32\nstage a(y, x) [H, W]: f32 = a(y, x-1)\nliveout a\n", "cyclic reference"),
    (HDR + "image img(H, W): f32\nstage a(y, x) [H, W]: f32 = b(y, x)\n"
           "stage b(y, x) [H, W]: f32 = a(y, x)\nliveout b\n", "cyclic reference"),
    (HDR + "image img(H, W): f32\nstage a(y, x) [H, W]: f32 = img(y, x)\n"
           "stage b(y, x) [H, W]: f32 = img(y, x)\nliveout b\n", "unreachable"),
    (HDR + "image img(H, W): f32\nliveout a\n", "no stages"),
    (HDR + "image img(H, W): f32\nstage a(y, x) [H, W]: f32 = img(x)\nliveout a\n", "dims"),
    (HDR + "image img(H, W): f32\nstage a(y, x) [H, W]: f64 = img(y, x)\nliveout a\n", "element type"),
])
def test_parse_errors(text, msg):
    with pytest.raises(OracleError, match=msg):
        parse(text)


def test_shape_mismatch_is_an_error():
    w = PI.small("blur", 8, 8)
    with pytest.raises(OracleError, match="shape mismatch"):
        evaluate(w.text, w.params, {"img": np.zeros((8, 9), np.float32)})


def test_all_benchmark_pipelines_parse():
    for f in sorted(PI.PIPELINES.glob("*.pmg")):
        prog = parse(f.read_text())
        assert prog.liveouts


def test_golden_digests_unchanged():
    """Drift check: oracle outputs on seeded inputs match the recorded digests."""
    import json
    from pathlib import Path
    import importlib.util
    gdir = Path(__file__).with_name("golden")
    spec = importlib.util.spec_from_file_location("mk", gdir / "make_golden.py")
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    assert m.digests() == json.loads((gdir / "oracle_digests.json").read_text())


# ------------------------------------------------------------------ demand-driven (sampled) oracle
@pytest.mark.parametrize("wl", [PI.small("blur", 70, 50), PI.small("harris", 90, 61), PI.small("unsharp", 64, 40),
                                PI.small("camera", 96, 64),
                                PI.Workload("ll", "local_laplacian_J4K4.pmg", {"W": 96, "H": 64}, 1005),
                                PI.Workload("pb", "pyramid_blend_J3.pmg", {"W": 70, "H": 46}, 1006)],
                         ids=lambda w: w.pipeline)
def test_point_oracle_equals_whole_domain(wl):
    """oracle/points.py restates the definition at requested points only (used at BASELINE sizes); it must
    reproduce the whole-domain evaluation bit for bit, including corners, ragged edges and the data-dependent
    plane index of the local Laplacian."""
    from oracle import evaluate_points
    inp = wl.inputs("structured") if "laplacian" in wl.pipeline else wl.inputs()
    (key, ref), = evaluate(wl.text, wl.params, inp).items()
    rng = np.random.default_rng(1)
    pts = tuple(np.concatenate([rng.integers(0, n, size=40), [0, n - 1, n // 2]]) for n in ref.shape)
    got = evaluate_points(wl.text, wl.params, inp, key, pts)
    np.testing.assert_array_equal(got.view(np.uint8), np.ascontiguousarray(ref[pts]).view(np.uint8))


# ----------------------------------------------------------------------------- R4 operator table (hand values)
def test_integer_and_conversion_semantics_hand_values():
    """Reading R4: shift counts clamped to [0, 32], floor '/' and divisor-signed '%' with
    x/0 = x%0 = 0, int32 wrap-around, f32 -> int truncating + saturating with NaN -> 0, wrapping narrowing
    casts and stores, saturating sat_u8/sat_u16, 0/1 logical operators.  Every expected value in
    tests/ops_table.PINS is worked by hand from those definitions."""
    import ops_table as OT
    W = len(OT.PINS)
    a = np.array([[p[1] for p in OT.PINS]], dtype=np.int64).astype(np.int32)
    b = np.array([[p[2] for p in OT.PINS]], dtype=np.int64).astype(np.int32)
    f = np.array([[p[3] for p in OT.PINS]], dtype=np.float32)
    with np.errstate(all="ignore"):
        out = evaluate(OT.TEXT, {"W": W, "H": 1}, {"a": a, "b": b, "f": f})
    bad = [(p, int(out[p[0]][0, i])) for i, p in enumerate(OT.PINS) if int(out[p[0]][0, i]) != p[4]]
    assert not bad, bad


def test_ops_table_covers_every_operator():
    """The GPU operator-table parity test (tests/test_gpu_parity.py) exercises every binary operator,
    unary operator and builtin of the grammar."""
    import ops_table as OT
    text = OT.TEXT
    for op in ["<<", ">>", "/", "%", "||", "&&", "!", "+", "-", "*", "<", "==", ">="]:
        assert op in text, op
    for fn in ["abs", "absd", "min", "max", "clamp", "select", "sqrt", "f32", "i32", "i16", "u16", "u8",
               "sat_u8", "sat_u16"]:
        assert f"{fn}(" in text, fn
