"""Operator table for the integer / conversion semantics of reading R4 — test data only.

`TEXT` is a pipeline whose stages each apply one operator to two int32 images a, b and one f32 image f.
`inputs(W, H)` tiles the edge-case value lists below over the image (a varies with x, b with y, f with
x + y), so every (a, b) pair of the lists occurs.  `PINS` lists hand-computed results (from the R4
definitions, not from either evaluator): (stage, a, b, f, expected)."""
import numpy as np

INT_MIN, INT_MAX = -2147483648, 2147483647

A_VALS = [0, 1, -1, 5, -8, 7, -7, 300, 70000, -40000, 40000, 65536, 123456789, INT_MAX, INT_MIN, INT_MIN + 1,
          2, -2, 255, 256, 1 << 30, -(1 << 30), 13, -13]
B_VALS = [0, 1, -1, 2, -2, 3, -3, 5, 8, 15, 16, 30, 31, 32, 33, 40, 100, -5, -32, -33, INT_MAX, INT_MIN, 7, -7]
F_VALS = [0.0, -0.0, 0.5, -0.5, 1.5, -1.5, 2.9, -2.9, 255.5, 256.0, 65535.9, 65536.5, 70000.25, -1.0,
          40000.7, -40000.7, 3e9, -3e9, 2147483520.0, 2147483648.0, -2147483648.0, -2147483904.0, 1e10, -1e10,
          float("inf"), float("-inf"), float("nan"), 1e-45, 123.999, -123.999, 32767.5, -32768.9, 1e30]

_STAGES = [
    ("shl", "i32", "a(y, x) << b(y, x)"),
    ("shr", "i32", "a(y, x) >> b(y, x)"),
    ("shlc", "i32", "a(y, x) << 33"),
    ("shrc", "i32", "a(y, x) >> 40"),
    ("dv", "i32", "a(y, x) / b(y, x)"),
    ("md", "i32", "a(y, x) % b(y, x)"),
    ("dvc", "i32", "a(y, x) / -3"),
    ("mdc", "i32", "a(y, x) % -3"),
    ("dv4", "i32", "a(y, x) / 4"),
    ("md4", "i32", "a(y, x) % 4"),
    ("lor", "i32", "a(y, x) || b(y, x)"),
    ("land", "i32", "a(y, x) && b(y, x)"),
    ("lnot", "i32", "!a(y, x)"),
    ("fnot", "i32", "!f(y, x)"),
    ("flor", "i32", "f(y, x) || 0"),
    ("iadd", "i32", "a(y, x) + b(y, x)"),
    ("isub", "i32", "a(y, x) - b(y, x)"),
    ("imul", "i32", "a(y, x) * b(y, x)"),
    ("ineg", "i32", "-a(y, x)"),
    ("iabs", "i32", "abs(a(y, x))"),
    ("iabsd", "i32", "absd(a(y, x), b(y, x))"),
    ("imin", "i32", "min(a(y, x), b(y, x))"),
    ("iclamp", "i32", "clamp(a(y, x), -7, b(y, x))"),
    ("icmp", "i32", "(a(y, x) < b(y, x)) + 2 * (a(y, x) == b(y, x)) + 4 * (a(y, x) >= b(y, x))"),
    ("f2i", "i32", "i32(f(y, x))"),
    ("f2u16", "i32", "u16(f(y, x))"),
    ("f2i16", "i32", "i16(f(y, x))"),
    ("f2u8", "i32", "u8(f(y, x))"),
    ("i2u16", "i32", "u16(a(y, x))"),
    ("i2i16", "i32", "i16(a(y, x))"),
    ("i2u8", "i32", "u8(a(y, x))"),
    ("satu16", "i32", "sat_u16(a(y, x))"),
    ("satu8", "i32", "sat_u8(a(y, x))"),
    ("satu16f", "i32", "sat_u16(f(y, x))"),
    ("satu8f", "i32", "sat_u8(f(y, x))"),
    ("stu8", "u8", "a(y, x)"),
    ("stu16", "u16", "a(y, x)"),
    ("sti16", "i16", "f(y, x)"),
    ("sti32", "i32", "f(y, x)"),
    ("i2f", "f32", "f32(a(y, x))"),
    ("fmix", "f32", "a(y, x) + f(y, x)"),
    ("fmin", "f32", "min(f(y, x), 0.5)"),
    ("fmax", "f32", "max(f(y, x), -0.5)"),
    ("fsel", "f32", "select(f(y, x) < 1.0, f(y, x), -f(y, x))"),
    ("fdiv", "f32", "f(y, x) / a(y, x)"),
    ("fsqrt", "f32", "sqrt(f(y, x))"),
    ("fabsd", "f32", "absd(f(y, x), 0.25)"),
]

TEXT = "param W, H\nimage a(H, W): i32\nimage b(H, W): i32\nimage f(H, W): f32\n" + "".join(
    f"stage {n}(y, x) [H, W]: {t} = {e}\n" for n, t, e in _STAGES) + "".join(f"liveout {n}\n" for n, _, _ in _STAGES)

STAGES = [n for n, _, _ in _STAGES]


def inputs(W: int, H: int, seed: int = 7) -> dict:
    """a(y, x) = A_VALS[x mod |A|] (every 3rd row shifted by a seeded permutation), b(y, x) = B_VALS[y mod |B|],
    f(y, x) = F_VALS[(x + y) mod |F|] — every (a, b) pair of the lists occurs once the image is |A| x |B|."""
    rng = np.random.default_rng(seed)
    xs = np.arange(W)[None, :] + np.zeros((H, 1), dtype=np.int64)
    ys = np.arange(H)[:, None] + np.zeros((1, W), dtype=np.int64)
    perm = rng.permutation(len(A_VALS))
    ai = np.where(ys % 3 == 2, perm[xs % len(A_VALS)], xs % len(A_VALS))
    a = np.asarray(A_VALS, dtype=np.int64)[ai].astype(np.int32)
    b = np.asarray(B_VALS, dtype=np.int64)[ys % len(B_VALS)].astype(np.int32)
    f = np.asarray(F_VALS, dtype=np.float32)[(xs + ys) % len(F_VALS)]
    return {"a": a, "b": b, "f": f}


# (stage, a, b, f, expected) — each worked by hand from reading R4
PINS = [
    # shift counts clamped to [0, 32]: a << c == a * 2^c mod 2^32, a >> c == floor(a / 2^c)
    ("shl", 1, 33, 0.0, 0), ("shl", 1, 31, 0.0, INT_MIN), ("shl", 5, 1, 0.0, 10), ("shl", 5, -1, 0.0, 5),
    ("shl", -1, 32, 0.0, 0), ("shl", 3, 30, 0.0, -(1 << 30)), ("shl", 7, INT_MIN, 0.0, 7),
    ("shr", -8, 40, 0.0, -1), ("shr", 8, 40, 0.0, 0), ("shr", -8, 1, 0.0, -4), ("shr", -7, 1, 0.0, -4),
    ("shr", INT_MIN, 31, 0.0, -1), ("shr", INT_MAX, 32, 0.0, 0), ("shr", 13, -5, 0.0, 13), ("shr", 300, 8, 0.0, 1),
    ("shlc", 1, 0, 0.0, 0), ("shrc", -13, 0, 0.0, -1), ("shrc", 13, 0, 0.0, 0),
    # floor division, remainder with the divisor's sign, x/0 = x%0 = 0, INT_MIN / -1 wraps
    ("dv", -7, 2, 0.0, -4), ("dv", 7, -2, 0.0, -4), ("dv", -7, -2, 0.0, 3), ("dv", 7, 2, 0.0, 3), ("dv", 5, 0, 0.0, 0),
    ("dv", INT_MIN, -1, 0.0, INT_MIN), ("dv", INT_MAX, INT_MIN, 0.0, -1), ("dv", INT_MIN, INT_MIN, 0.0, 1),
    ("md", 7, -3, 0.0, -2), ("md", -7, 3, 0.0, 2), ("md", -7, -3, 0.0, -1), ("md", 7, 3, 0.0, 1), ("md", 5, 0, 0.0, 0),
    ("md", INT_MIN, -1, 0.0, 0), ("md", INT_MAX, INT_MIN, 0.0, -1), ("md", -1, INT_MAX, 0.0, INT_MAX - 1),
    ("dvc", 7, 0, 0.0, -3), ("dvc", -7, 0, 0.0, 2), ("mdc", 7, 0, 0.0, -2), ("mdc", -7, 0, 0.0, -1),
    ("dv4", -13, 0, 0.0, -4), ("md4", -13, 0, 0.0, 3), ("dv4", INT_MIN, 0, 0.0, -(1 << 29)), ("md4", INT_MIN + 1, 0, 0.0, 1),
    # logical operators give 0 / 1
    ("lor", 0, 0, 0.0, 0), ("lor", 0, -5, 0.0, 1), ("lor", 300, 0, 0.0, 1), ("land", 2, 0, 0.0, 0),
    ("land", -2, 7, 0.0, 1), ("lnot", 0, 0, 0.0, 1), ("lnot", INT_MIN, 0, 0.0, 0), ("fnot", 0, 0, -0.0, 1),
    ("fnot", 0, 0, 1e-45, 0), ("fnot", 0, 0, float("nan"), 0), ("flor", 0, 0, 0.5, 1), ("flor", 0, 0, -0.0, 0),
    # int32 wrap-around
    ("iadd", INT_MAX, 1, 0.0, INT_MIN), ("isub", INT_MIN, 1, 0.0, INT_MAX), ("imul", 70000, 70000, 0.0, 605032704),
    ("ineg", INT_MIN, 0, 0.0, INT_MIN), ("iabs", INT_MIN, 0, 0.0, INT_MIN), ("iabs", -13, 0, 0.0, 13),
    ("iabsd", INT_MIN, 1, 0.0, INT_MAX), ("iabsd", -7, 7, 0.0, 14), ("imin", -7, 7, 0.0, -7),
    ("iclamp", -40000, 0, 0.0, -7), ("iclamp", 300, 8, 0.0, 8), ("iclamp", 5, -33, 0.0, -33),
    ("icmp", 1, 2, 0.0, 1), ("icmp", 2, 2, 0.0, 6), ("icmp", 3, 2, 0.0, 4),
    # f32 -> int: truncate toward zero, saturate, NaN -> 0; then the narrowing casts wrap
    ("f2i", 0, 0, 3e9, INT_MAX), ("f2i", 0, 0, -3e9, INT_MIN), ("f2i", 0, 0, float("nan"), 0),
    ("f2i", 0, 0, float("inf"), INT_MAX), ("f2i", 0, 0, float("-inf"), INT_MIN), ("f2i", 0, 0, -2.9, -2),
    ("f2i", 0, 0, 2147483520.0, 2147483520), ("f2i", 0, 0, 2147483648.0, INT_MAX), ("f2i", 0, 0, -2147483648.0, INT_MIN),
    ("f2i", 0, 0, -0.5, 0), ("f2i", 0, 0, 123.999, 123),
    ("f2u16", 0, 0, 70000.25, 4464), ("f2u16", 0, 0, -1.0, 65535), ("f2u16", 0, 0, 65535.9, 65535),
    ("f2u16", 0, 0, 3e9, 65535), ("f2u16", 0, 0, -3e9, 0), ("f2u16", 0, 0, float("nan"), 0),
    ("f2i16", 0, 0, 40000.7, -25536), ("f2i16", 0, 0, -40000.7, 25536), ("f2i16", 0, 0, 32767.5, 32767),
    ("f2i16", 0, 0, -32768.9, -32768),
    ("f2u8", 0, 0, 255.5, 255), ("f2u8", 0, 0, 256.0, 0), ("f2u8", 0, 0, -1.5, 255), ("f2u8", 0, 0, 2.9, 2),
    ("i2u16", 70000, 0, 0.0, 4464), ("i2u16", -1, 0, 0.0, 65535), ("i2i16", 40000, 0, 0.0, -25536),
    ("i2i16", -40000, 0, 0.0, 25536), ("i2u8", 300, 0, 0.0, 44), ("i2u8", -1, 0, 0.0, 255), ("i2u8", 256, 0, 0.0, 0),
    # saturating casts
    ("satu16", -40000, 0, 0.0, 0), ("satu16", 70000, 0, 0.0, 65535), ("satu16", 40000, 0, 0.0, 40000),
    ("satu8", 300, 0, 0.0, 255), ("satu8", -7, 0, 0.0, 0), ("satu8", 13, 0, 0.0, 13),
    ("satu16f", 0, 0, 1e10, 65535), ("satu16f", 0, 0, -3e9, 0), ("satu16f", 0, 0, float("nan"), 0),
    ("satu16f", 0, 0, 65535.9, 65535), ("satu8f", 0, 0, 255.5, 255), ("satu8f", 0, 0, float("inf"), 255),
    ("satu8f", 0, 0, -0.5, 0), ("satu8f", 0, 0, 123.999, 123),
    # narrowing stores wrap like the casts; a float stored to an int stage converts like i32()
    ("stu8", 300, 0, 0.0, 44), ("stu8", -1, 0, 0.0, 255), ("stu16", 70000, 0, 0.0, 4464), ("stu16", -40000, 0, 0.0, 25536),
    ("sti16", 0, 0, 40000.7, -25536), ("sti16", 0, 0, float("nan"), 0), ("sti16", 0, 0, 1e10, -1),
    ("sti32", 0, 0, -3e9, INT_MIN), ("sti32", 0, 0, 1e30, INT_MAX),
]
