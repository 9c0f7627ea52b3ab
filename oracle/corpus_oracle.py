"""CPU restatement of slowness-model preparation -- TEST INFRASTRUCTURE ONLY.

The reference ships no code for it; the contract is SPEC.md `[MODULE] datagen`
(reference SPEC.md:404-417, 433-447): each corpus image -> bilinear resize to (n+1)^2 nodes ->
Gaussian smoothing (separable truncated Gaussian, radius ceil(3 sigma), edge-replicated;
sigma = 1 grid cell at n = 128, scaled with n / 128) -> affine normalisation onto [0.25, 1]
(a constant image maps to 0.25) -> SlownessModel.  Corpus files: 8-bit binary PGM (P5), or raw
little-endian float64 grids with a text sidecar ``<name>.hdr`` holding "rows cols".

The resize is corner-aligned (node grids: output node i samples input i (h_in - 1)/(h_out - 1)), a
documented choice (the SPEC names only "bilinear").  Evaluation orders match the GPU kernels
(paper_2306_17486_b200/csrc/prep.cu) so resize and normalisation agree bit for bit; smoothing taps
come from two exp implementations and agree to an ulp.

Only tests/ may use this module.
"""
from __future__ import annotations

import os

import numpy as np


def gaussian_taps(sigma: float) -> np.ndarray:
    if sigma <= 0:
        return np.ones(1)
    r = int(np.ceil(3.0 * sigma))
    t = np.arange(-r, r + 1, dtype=np.float64)
    k = np.exp(-0.5 * (t / sigma) * (t / sigma))
    return k / k.sum()


def gaussian_smooth(a: np.ndarray, sigma: float) -> np.ndarray:
    a = np.asarray(a, dtype=np.float64)
    k = gaussian_taps(sigma)
    r = len(k) // 2
    if r == 0:
        return a.copy()
    for axis in (0, 1):
        pad = [(0, 0), (0, 0)]
        pad[axis] = (r, r)
        p = np.pad(a, pad, mode="edge")
        acc = np.zeros_like(a)
        n = a.shape[axis]
        for i, w in enumerate(k):
            sl = [slice(None), slice(None)]
            sl[axis] = slice(i, i + n)
            acc = acc + w * p[tuple(sl)]
        a = acc
    return a


def resize_bilinear(a: np.ndarray, shape) -> np.ndarray:
    a = np.asarray(a, dtype=np.float64)
    hin, win = a.shape
    hout, wout = shape
    sy = (hin - 1) / (hout - 1) if hout > 1 else 0.0
    sx = (win - 1) / (wout - 1) if wout > 1 else 0.0
    y = np.arange(hout, dtype=np.float64) * sy
    x = np.arange(wout, dtype=np.float64) * sx
    y0 = np.minimum(np.floor(y).astype(int), hin - 1)
    x0 = np.minimum(np.floor(x).astype(int), win - 1)
    y1 = np.minimum(y0 + 1, hin - 1)
    x1 = np.minimum(x0 + 1, win - 1)
    fy = (y - y0)[:, None]
    fx = (x - x0)[None, :]
    gx, gy = 1.0 - fx, 1.0 - fy
    top = gx * a[y0][:, x0] + fx * a[y0][:, x1]
    bot = gx * a[y1][:, x0] + fx * a[y1][:, x1]
    return gy * top + fy * bot


def normalise(a: np.ndarray, lo: float = 0.25, hi: float = 1.0) -> np.ndarray:
    vmin, vmax = float(a.min()), float(a.max())
    if not (vmax - vmin > 0):
        return np.full(a.shape, lo)
    return lo + ((hi - lo) * (a - vmin)) / (vmax - vmin)


def sigma_for(n: int) -> float:
    return 1.0 * n / 128.0


def read_pgm(path: str) -> np.ndarray:
    with open(path, "rb") as f:
        data = f.read()
    toks, pos = [], 0
    while len(toks) < 4:  # magic, width, height, maxval (comments skipped)
        while data[pos:pos + 1].isspace():
            pos += 1
        if data[pos:pos + 1] == b"#":
            pos = data.index(b"\n", pos) + 1
            continue
        end = pos
        while not data[end:end + 1].isspace():
            end += 1
        toks.append(data[pos:end])
        pos = end
    if toks[0] != b"P5":
        raise ValueError(f"{path}: not a binary PGM")
    w, h, maxval = int(toks[1]), int(toks[2]), int(toks[3])
    if maxval > 255:
        raise ValueError(f"{path}: 16-bit PGM unsupported")
    pix = np.frombuffer(data[pos + 1:pos + 1 + w * h], dtype=np.uint8)
    return pix.reshape(h, w).astype(np.float64)


def read_f64(path: str) -> np.ndarray:
    with open(os.path.splitext(path)[0] + ".hdr") as f:
        rows, cols = (int(v) for v in f.read().split()[:2])
    return np.fromfile(path, dtype="<f8").reshape(rows, cols)


def prepare(image: np.ndarray, target_n: int) -> np.ndarray:
    """kappa^2 on (target_n + 1)^2 nodes."""
    n1 = target_n + 1
    return normalise(gaussian_smooth(resize_bilinear(image, (n1, n1)), sigma_for(target_n)))
