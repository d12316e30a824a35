"""Host tests of the reassociation mode's separable rewrite (factor.cpp, pmg_pipeline_rewritten): the rewritten
text, evaluated by the ORACLE, agrees with the pipeline as written within the north_star f32 tolerance, at
every clamped edge (tiny and ragged images), and the rewrite fires exactly on rank-1 linear f32 stencils.

The pin is mathematical: sum_{dy,dx} u[dy] v[dx] Q(clamp(y+dy), clamp(x+dx)) = sum_dy u[dy] * (sum_dx v[dx]
Q(clamp(y+dy), clamp(x+dx))) holds exactly in real arithmetic because clamping acts per dimension; the two
f32 evaluations differ by rounding only (bounded by a few ulps of sum |terms|)."""
import re

import numpy as np
import pytest

import paper_1909_07190_b200 as pmg
import pmg_inputs as PI
from oracle import evaluate


def rewritten(text, params, **kw):
    return pmg.Pipeline(text).rewritten(params, pmg.sched_opts(reassoc=True, inline=False, **kw))


def close(a, b, rel=1e-6):
    a64, b64 = a.astype(np.float64), b.astype(np.float64)
    scale = max(1.0, float(np.max(np.abs(a64))))
    return float(np.max(np.abs(a64 - b64))) <= rel * scale


@pytest.mark.parametrize("W,H", [(67, 45), (130, 41), (5, 3), (1, 1), (2, 7), (33, 1)])
def test_harris_factored_text_agrees_with_written(W, H):
    wl = PI.small("harris", W, H)
    r = rewritten(wl.text, wl.params)
    assert r["factored"] == ["Iy", "Ix", "Sxx", "Syy", "Sxy"]
    assert sum(ln.startswith("stage ") for ln in r["text"].splitlines()) == 16
    inp = wl.inputs()
    a = evaluate(wl.text, wl.params, inp)["harris"]
    b = evaluate(r["text"], wl.params, inp)["harris"]
    assert close(a, b, rel=1e-5)


def _left_sum(terms):
    s = terms[0]
    for t in terms[1:]:
        s = f"({s} + {t})"
    return s


_U, _V = [1, 3, 1], [1, 4, 6, 4, 1]
_R1 = _left_sum([(f"{u * v}.0 * " if u * v != 1 else "") + f"I(y{dy:+d}, x{dx:+d})"
                 for dy, u in zip((-1, 0, 1), _U) for dx, v in zip((-2, -1, 0, 1, 2), _V)])
GEN = f"""param W, H
image I(H, W): f32
image C(3, H, W): f32
image N(H, W): i32
stage r1(y, x) [H, W]: f32 = {_R1} / 80.0
stage r2(y, x) [H, W]: f32 = ((((I(y-1, x-1) + I(y-1, x+1)) + I(y+1, x-1)) - I(y+1, x+1)) + I(y, x))
stage r3(c, y, x) [3, H, W]: f32 = (((((C(c, y-1, x-1) + 0.5 * C(c, y-1, x)) + C(c, y-1, x+1)) - C(c, y+1, x-1)) - 0.5 * C(c, y+1, x)) - C(c, y+1, x+1))
stage r4(y, x) [H, W]: i32 = (((N(y-1, x-1) + N(y-1, x)) + N(y+1, x-1)) + N(y+1, x))
stage out(y, x) [H, W]: f32 = (r1(y, x) + r2(y, x)) + (r3(0, y, x) + r3(2, y, x)) + f32(r4(y, x))
liveout out
"""


@pytest.mark.parametrize("W,H", [(23, 17), (4, 2), (1, 1)])
def test_factoring_fires_on_rank_one_only(W, H):
    params = {"W": W, "H": H}
    r = rewritten(GEN, params)
    # r1 is [1,3,1] x [1,4,6,4,1] / 80 (rank one), r3 is [1,0,-1] x [1,0.5,1] over planes (rank one);
    # r2 has rank two; r4 is an integer stage
    assert r["factored"] == ["r1", "r3"]
    rng = np.random.default_rng(7)
    inp = {"I": rng.random((H, W), dtype=np.float32), "C": rng.random((3, H, W), dtype=np.float32),
           "N": rng.integers(-1000, 1000, (H, W)).astype(np.int32)}
    a = evaluate(GEN, params, inp)["out"]
    b = evaluate(r["text"], params, inp)["out"]
    assert close(a, b, rel=1e-5)


def test_factoring_is_off_by_default():
    wl = PI.small("harris", 40, 30)
    r = pmg.Pipeline(wl.text).rewritten(wl.params, pmg.sched_opts(inline=False))
    assert r["factored"] == [] and sum(ln.startswith("stage ") for ln in r["text"].splitlines()) == 11


def test_factored_stages_save_operations():
    """The Sobel derivatives go from 5 to 3 operations per point and the box sums from 8 to 4 additions."""
    wl = PI.small("harris", 40, 30)
    text = rewritten(wl.text, wl.params)["text"]
    lines = {ln.split("(")[0].split()[1]: ln.split("=", 1)[1] for ln in text.splitlines() if ln.startswith("stage ")}
    def ops(s):   # arithmetic operators outside the read index lists
        s = re.sub(r"\b[A-Za-z_]\w*\((?:[^()]|\([^()]*\))*\)", "X", s)
        return s.count(" + ") + s.count(" - ") + s.count(" * ") + s.count(" / ")
    # box sums: the row sum pairs neighbouring columns (parity select: (Q(x)+Q(x+1)) is shared by columns x and
    # x+1), so each of its two branches has 2 additions of which one is shared; the column sum has 2
    assert lines["Sxx_h"].strip().startswith("select(((x % 2) == 0),")
    assert ops(lines["Sxx"]) == 2
    assert ops(lines["Ix_h"]) + ops(lines["Ix"]) <= 5
