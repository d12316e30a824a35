"""Seeded synthetic inputs for the benchmark pipelines — shared by tests, bench.py and the oracle legs.

This module holds NONE of the method's arithmetic (no stage evaluation, no fusion, no tiling): it only
draws seeded input images and builds the workload's input tables (the camera tone curve and colour
matrix, the local-Laplacian remap LUT), which are inputs of the pipeline definitions, exactly like the
images.  Both the CUDA path and the oracle receive identical bytes from here.

Workload recipe (DESIGN.md §"Inputs"): shapes/dtypes are BASELINE.json's configs; values are
U[0,1) i.i.d. f32 for the float pipelines plus structured variants (gradients, rectangles, flat patches,
noise) where the pipeline has data-dependent control flow; camera raw is a GRBG mosaic of a synthetic
scene with sigma=8 DN noise and 0.01 % hot pixels, 10-bit.  Seeds: C1 1001, C2 1002, C3 1003, C4 1004,
C5 1005, PB 1006 (A) / 1007 (B).
"""
from __future__ import annotations

from dataclasses import dataclass
from pathlib import Path

import numpy as np

PIPELINES = Path(__file__).resolve().parent / "pipelines"


# ------------------------------------------------------------------------------------------ images
def uniform(shape, seed, dtype=np.float32):
    return np.random.default_rng(seed).random(shape, dtype=np.float32).astype(dtype)


def structured(shape, seed):
    """Smooth gradient + random axis-aligned flat rectangles + 2 % noise, in [0,1] (corners & flat areas)."""
    rng = np.random.default_rng(seed)
    *lead, h, w = shape
    y = np.linspace(0.0, 1.0, h, dtype=np.float64)[:, None]
    x = np.linspace(0.0, 1.0, w, dtype=np.float64)[None, :]
    out = np.empty(shape, dtype=np.float32)
    for idx in np.ndindex(*lead) if lead else [()]:
        img = 0.25 + 0.5 * (0.6 * x + 0.4 * y) + 0.0 * y * x
        for _ in range(max(4, (h * w) // 4096)):
            y0, x0 = rng.integers(0, h), rng.integers(0, w)
            hh, ww = rng.integers(1, max(2, h // 4)), rng.integers(1, max(2, w // 4))
            img[y0:y0 + hh, x0:x0 + ww] = rng.random()
        img = img + 0.02 * rng.standard_normal((h, w))
        # a fraction of exactly flat pixels so select() branches of unsharp mask both occur
        flat = rng.random((h, w)) < 0.05
        img = np.where(flat, 0.5, img)
        out[idx] = np.clip(img, 0.0, 1.0).astype(np.float32)
    return out


def sparse_rgba(h, w, seed, variant="uniform", density=0.1):
    """Multiscale Interpolation input: colour planes (uniform or structured) and an alpha plane that is 1 on a
    seeded ~10 % of the pixels (the known samples) and 0 elsewhere (at least one sample)."""
    rgb = structured((3, h, w), seed) if variant != "uniform" else uniform((3, h, w), seed)
    alpha = (np.random.default_rng(seed + 7).random((h, w)) < density).astype(np.float32)
    alpha[h // 2, w // 2] = 1.0
    return np.ascontiguousarray(np.concatenate([rgb, alpha[None]], axis=0))


def blend_mask(h, w):
    """Pyramid-blend mask: 0 on the left, 1 on the right, a linear ramp over the middle eighth of the width."""
    x = (np.arange(w, dtype=np.float64) - (w - 1) / 2.0) / max(1.0, w / 8.0) + 0.5
    return np.broadcast_to(np.clip(x, 0.0, 1.0)[None, :], (h, w)).astype(np.float32).copy()


def bayer_raw(h, w, seed, black=25, white=1023):
    """GRBG mosaic of a synthetic RGB scene, + sigma=8 DN noise, + 0.01 % hot pixels (value 1023)."""
    rng = np.random.default_rng(seed)
    y = np.linspace(0, 1, h)[:, None]
    x = np.linspace(0, 1, w)[None, :]
    scene = np.stack([0.2 + 0.6 * x + 0.0 * y, 0.3 + 0.5 * y + 0.0 * x, 0.8 - 0.6 * x * y])
    for _ in range(max(4, (h * w) // 20000)):
        y0, x0 = rng.integers(0, h), rng.integers(0, w)
        hh, ww = rng.integers(2, max(3, h // 6)), rng.integers(2, max(3, w // 6))
        scene[:, y0:y0 + hh, x0:x0 + ww] = rng.random((3, 1, 1))
    mosaic = np.empty((h, w))
    mosaic[0::2, 0::2] = scene[1, 0::2, 0::2]   # Gr
    mosaic[0::2, 1::2] = scene[0, 0::2, 1::2]   # R
    mosaic[1::2, 0::2] = scene[2, 1::2, 0::2]   # B
    mosaic[1::2, 1::2] = scene[1, 1::2, 1::2]   # Gb
    raw = black + mosaic * (white - black) + 8.0 * rng.standard_normal((h, w))
    raw = np.clip(np.rint(raw), 0, white).astype(np.uint16)
    hot = rng.random((h, w)) < 1e-4
    raw[hot] = white
    return raw


# ------------------------------------------------------------------------------------------ tables
def camera_curve(black=25, white=1023, gamma=2.0, contrast=50.0):
    """1024-entry u8 tone curve (Halide camera_pipe style), built in f64 and rounded once."""
    lut = np.zeros(1024, dtype=np.uint8)
    b = 2.0 - 2.0 ** (contrast / 100.0)
    a = 2.0 - 2.0 * b
    for v in range(1024):
        if v <= black:
            lut[v] = 0
            continue
        if v > white:
            lut[v] = 255
            continue
        xf = min(max((v - black) / (white - black), 0.0), 1.0)
        g = xf ** (1.0 / gamma)
        z = 1.0 - (a * (1.0 - g) * (1.0 - g) + b * (1.0 - g)) if g > 0.5 else a * g * g + b * g
        lut[v] = int(min(max(z * 256.0, 0.0), 255.0))
    return lut


def camera_ccm(color_temp=3700.0):
    """3x4 fixed-point (x256) colour matrix, rows [c][0..2] gains + [c][3] offset, as 12 int32."""
    m3200 = np.array([[1.6697, -0.2693, -0.4004, -42.4346],
                      [-0.3576, 1.0615, 1.5949, -37.1158],
                      [-0.2175, -1.8751, 6.9640, -26.6970]])
    m7000 = np.array([[2.2997, -0.4478, 0.1706, -39.0923],
                      [-0.3826, 1.5906, -0.2080, -25.4311],
                      [-0.0888, -0.7344, 2.2832, -20.0826]])
    alpha = (1.0 / color_temp - 1.0 / 3200) / (1.0 / 7000 - 1.0 / 3200)
    m = m3200 * (1 - alpha) + m7000 * alpha
    return np.rint(m * 256.0).astype(np.int32).reshape(-1)


def ll_remap(K=8, alpha=None):
    """remap[i + (K-1)*256] = alpha * (i/256) * exp(-(i/256)^2 / 2), i in [-(K-1)*256, (K-1)*256]."""
    top = (K - 1) * 256
    alpha = 1.0 / (K - 1) if alpha is None else alpha
    i = np.arange(-top, top + 1, dtype=np.float64) / 256.0
    return (alpha * i * np.exp(-i * i / 2.0)).astype(np.float32)


# ------------------------------------------------------------------------------------------ workloads
@dataclass
class Workload:
    name: str
    pipeline: str              # file under pipelines/
    params: dict
    seed: int
    note: str = ""

    @property
    def text(self) -> str:
        return (PIPELINES / self.pipeline).read_text()

    def inputs(self, variant: str = "uniform") -> dict:
        p, s = self.params, self.seed
        W, H = p["W"], p["H"]
        if self.pipeline == "camera.pmg":
            return {"raw": bayer_raw(H, W, s), "ccm": camera_ccm(), "curve": camera_curve()}
        if self.pipeline.startswith("local_laplacian"):
            K = 8 if self.pipeline == "local_laplacian.pmg" else int(self.pipeline.split("K")[-1].split(".")[0])
            img = structured((3, H, W), s) if variant != "uniform" else uniform((3, H, W), s)
            return {"inp": img, "remap": ll_remap(K)}
        if self.pipeline.startswith("multiscale_interp"):
            return {"inp": sparse_rgba(H, W, s, variant)}
        if self.pipeline.startswith("pyramid_blend"):
            return {"A": structured((3, H, W), s), "B": structured((3, H, W), s + 1) if variant != "uniform"
                    else uniform((3, H, W), s + 1), "M": blend_mask(H, W)}
        if self.pipeline == "unsharp.pmg":
            img = structured((3, H, W), s) if variant != "uniform" else uniform((3, H, W), s)
            return {"img": img}
        img = structured((H, W), s) if variant != "uniform" else uniform((H, W), s)
        return {"img": img}

    @property
    def out_pixels(self) -> int:
        """Spatial output pixels W*H (channels not multiplied; reading R20)."""
        return self.params["W"] * self.params["H"]


WORKLOADS = {
    "blur": Workload("blur", "blur.pmg", {"W": 128, "H": 128}, 1001, "C1 128x128 f32"),
    "harris": Workload("harris", "harris.pmg", {"W": 6400, "H": 6400}, 1002, "C2 6400x6400 f32"),
    "unsharp": Workload("unsharp", "unsharp.pmg", {"W": 2048, "H": 2048}, 1003, "C3 2048x2048x3 f32"),
    "camera": Workload("camera", "camera.pmg", {"W": 2528, "H": 1920}, 1004, "C4 2528x1920 u16 Bayer"),
    "local_laplacian": Workload("local_laplacian", "local_laplacian.pmg", {"W": 2560, "H": 1536}, 1005,
                                "C5 2560x1536x3 f32, J=8, K=8"),
    # PAPER.md Table 2 l.1148 (not a BASELINE.json config)
    "multiscale_interp": Workload("multiscale_interp", "multiscale_interp.pmg", {"W": 2560, "H": 1536}, 1007,
                                  "MI 2560x1536 RGBA -> 3 planes f32, J=10"),
    # PAPER.md Table 2 l.1150 (not a BASELINE.json config)
    "pyramid_blend": Workload("pyramid_blend", "pyramid_blend.pmg", {"W": 3840, "H": 2160}, 1006,
                              "PB 3840x2160x3 f32, J=4"),
}


def small(name: str, W: int, H: int) -> Workload:
    w = WORKLOADS[name]
    return Workload(w.name, w.pipeline, {"W": W, "H": H}, w.seed, w.note + f" (reduced to {W}x{H})")


def blur_frames(n: int, seed: int = 1001) -> np.ndarray:
    """C1 as a batch: n independent 128x128 f32 frames, U[0,1), frame-major [n][y][x]."""
    return uniform((n, 128, 128), seed)
