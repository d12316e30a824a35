"""Brute-force, pure-Python-loop evaluators of the benchmark definitions — used only as oracle pins.

Written directly from the definitions (SURVEY §8(c) c.3 / pipelines/*.pmg comments), with explicit
per-read clamping to the producer's domain (reading R1) and np.float32 scalar arithmetic in the written
operand order (reading R3).  They share no code with oracle/pmg_oracle.py (no parser, no evaluator) and
are only run on tiny images.
"""
import numpy as np

f = np.float32


def _cl(v, n):
    return 0 if v < 0 else (n - 1 if v >= n else v)


def _get(a, y, x):
    H, W = a.shape
    return a[_cl(y, H), _cl(x, W)]


def blur(img):
    H, W = img.shape
    bx = np.zeros((H, W), np.float32)
    for y in range(H):
        for x in range(W):
            bx[y, x] = ((_get(img, y, x - 1) + _get(img, y, x)) + _get(img, y, x + 1)) / f(3.0)
    by = np.zeros((H, W), np.float32)
    for y in range(H):
        for x in range(W):
            by[y, x] = ((_get(bx, y - 1, x) + _get(bx, y, x)) + _get(bx, y + 1, x)) / f(3.0)
    return by


def harris(img):
    H, W = img.shape
    k12 = f(0.083333333)
    two = f(2.0)
    Ix = np.zeros((H, W), np.float32)
    Iy = np.zeros((H, W), np.float32)
    for y in range(H):
        for x in range(W):
            g = lambda dy, dx: _get(img, y + dy, x + dx)  # noqa: E731
            Iy[y, x] = ((((((-g(-1, -1) - two * g(-1, 0)) - g(-1, 1)) + g(1, -1)) + two * g(1, 0))
                         + g(1, 1)) * k12)
            Ix[y, x] = ((((((g(-1, 1) - g(-1, -1)) - two * g(0, -1)) + two * g(0, 1)) - g(1, -1))
                         + g(1, 1)) * k12)
    Ixx, Iyy, Ixy = Ix * Ix, Iy * Iy, Ix * Iy
    out = np.zeros((H, W), np.float32)
    for y in range(H):
        for x in range(W):
            S = []
            for P in (Ixx, Iyy, Ixy):
                acc = None
                for dy in (-1, 0, 1):
                    for dx in (-1, 0, 1):
                        v = _get(P, y + dy, x + dx)
                        acc = v if acc is None else acc + v
                S.append(acc)
            sxx, syy, sxy = S
            det = sxx * syy - sxy * sxy
            tr = sxx + syy
            out[y, x] = det - (f(0.04) * tr) * tr
    return out


def unsharp(img):
    C, H, W = img.shape
    out = np.zeros((C, H, W), np.float32)
    q = f(0.0625)
    for c in range(C):
        im = img[c]
        bx = np.zeros((H, W), np.float32)
        for y in range(H):
            for x in range(W):
                g = lambda dx: _get(im, y, x + dx)  # noqa: E731
                bx[y, x] = ((((g(-2) + f(4.0) * g(-1)) + f(6.0) * g(0)) + f(4.0) * g(1)) + g(2)) * q
        for y in range(H):
            for x in range(W):
                g = lambda dy: _get(bx, y + dy, x)  # noqa: E731
                by = ((((g(-2) + f(4.0) * g(-1)) + f(6.0) * g(0)) + f(4.0) * g(1)) + g(2)) * q
                sharpen = im[y, x] * f(4.0) - by * f(3.0)
                out[c, y, x] = im[y, x] if abs(im[y, x] - by) < f(0.001) else sharpen
    return out


def camera(raw, ccm, curve):
    """Integer camera pipe, looped pixel by pixel (definitions of pipelines/camera.pmg)."""
    H, W = raw.shape
    r = raw.astype(np.int64)
    den = np.zeros((H, W), np.int64)
    for y in range(H):
        for x in range(W):
            n = [_get(r, y - 2, x), _get(r, y + 2, x), _get(r, y, x - 2), _get(r, y, x + 2)]
            lo, hi = min(min(n[0], n[1]), min(n[2], n[3])), max(max(n[0], n[1]), max(n[2], n[3]))
            den[y, x] = np.int16(min(max(r[y, x], lo), hi))
    h, w = H // 2, W // 2
    q = {}
    q["g_gr"] = np.array([[_get(den, 2 * y, 2 * x) for x in range(w)] for y in range(h)])
    q["r_r"] = np.array([[_get(den, 2 * y, 2 * x + 1) for x in range(w)] for y in range(h)])
    q["b_b"] = np.array([[_get(den, 2 * y + 1, 2 * x) for x in range(w)] for y in range(h)])
    q["g_gb"] = np.array([[_get(den, 2 * y + 1, 2 * x + 1) for x in range(w)] for y in range(h)])

    def avg(a, b):
        return (a + b + 1) >> 1

    def st(fn):
        return np.array([[np.int16(fn(y, x)) for x in range(w)] for y in range(h)], dtype=np.int64)

    G = lambda n, y, x: _get(q[n], y, x)  # noqa: E731
    q["g_r"] = st(lambda y, x: avg(G("g_gr", y, x), G("g_gr", y, x + 1))
                  if abs(G("g_gr", y, x) - G("g_gr", y, x + 1)) < abs(G("g_gb", y - 1, x) - G("g_gb", y, x))
                  else avg(G("g_gb", y - 1, x), G("g_gb", y, x)))
    q["g_b"] = st(lambda y, x: avg(G("g_gb", y, x - 1), G("g_gb", y, x))
                  if abs(G("g_gb", y, x - 1) - G("g_gb", y, x)) < abs(G("g_gr", y, x) - G("g_gr", y + 1, x))
                  else avg(G("g_gr", y, x), G("g_gr", y + 1, x)))
    q["r_gr"] = st(lambda y, x: (G("g_gr", y, x) - avg(G("g_r", y, x - 1), G("g_r", y, x)))
                   + avg(G("r_r", y, x - 1), G("r_r", y, x)))
    q["b_gr"] = st(lambda y, x: (G("g_gr", y, x) - avg(G("g_b", y - 1, x), G("g_b", y, x)))
                   + avg(G("b_b", y - 1, x), G("b_b", y, x)))
    q["r_gb"] = st(lambda y, x: (G("g_gb", y, x) - avg(G("g_r", y, x), G("g_r", y + 1, x)))
                   + avg(G("r_r", y, x), G("r_r", y + 1, x)))
    q["b_gb"] = st(lambda y, x: (G("g_gb", y, x) - avg(G("g_b", y, x), G("g_b", y, x + 1)))
                   + avg(G("b_b", y, x), G("b_b", y, x + 1)))

    def rb(y, x):
        p = (G("g_b", y, x) - avg(G("g_r", y, x), G("g_r", y + 1, x - 1))) + avg(G("r_r", y, x), G("r_r", y + 1, x - 1))
        n = (G("g_b", y, x) - avg(G("g_r", y, x - 1), G("g_r", y + 1, x))) + avg(G("r_r", y, x - 1), G("r_r", y + 1, x))
        return p if abs(G("r_r", y, x) - G("r_r", y + 1, x - 1)) < abs(G("r_r", y, x - 1) - G("r_r", y + 1, x)) else n

    def br(y, x):
        p = (G("g_r", y, x) - avg(G("g_b", y - 1, x + 1), G("g_b", y, x))) + avg(G("b_b", y - 1, x + 1), G("b_b", y, x))
        n = (G("g_r", y, x) - avg(G("g_b", y - 1, x), G("g_b", y, x + 1))) + avg(G("b_b", y - 1, x), G("b_b", y, x + 1))
        return p if abs(G("b_b", y - 1, x + 1) - G("b_b", y, x)) < abs(G("b_b", y - 1, x) - G("b_b", y, x + 1)) else n

    q["r_b"] = st(rb)
    q["b_r"] = st(br)
    table = {"R": (("r_gr", "r_r"), ("r_b", "r_gb")), "G": (("g_gr", "g_r"), ("g_b", "g_gb")),
             "B": (("b_gr", "b_r"), ("b_b", "b_gb"))}
    full = {}
    for ch, ((ee, eo), (oe, oo)) in table.items():
        a = np.zeros((H, W), np.int64)
        for y in range(H):
            for x in range(W):
                n = (ee if x % 2 == 0 else eo) if y % 2 == 0 else (oe if x % 2 == 0 else oo)
                a[y, x] = np.int16(G(n, y // 2, x // 2))
        full[ch] = a
    out = np.zeros((3, H, W), np.uint8)
    m = ccm.astype(np.int64)
    for c in range(3):
        for y in range(H):
            for x in range(W):
                v = (m[4 * c + 3] + m[4 * c] * full["R"][y, x] + m[4 * c + 1] * full["G"][y, x]
                     + m[4 * c + 2] * full["B"][y, x]) >> 8
                out[c, y, x] = curve[min(max(int(v), 0), 1023)]
    return out
