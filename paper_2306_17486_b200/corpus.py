"""Slowness-model preparation on the GPU.

The reference ships no code for it; its contract is SPEC.md `[MODULE] datagen` (reference
SPEC.md:404-417, 433-447; paper §4.3 "resized to the appropriate size, smoothed slightly by a
Gaussian kernel, and finally normalized"):

    load_slowness_corpus(path, target_n) -> list of SlownessModel: every image (8-bit binary PGM,
    or raw little-endian float64 with a ``.hdr`` sidecar "rows cols") -> bilinear resize to
    (target_n + 1)^2 nodes -> Gaussian smoothing, sigma = target_n / 128 grid cells -> affine
    normalisation onto [0.25, 1] (constant images map to 0.25) -> SlownessModel with the ABL and the
    ten-points-per-wavelength omega.

Resize, smoothing and normalisation run batched on the device (csrc/prep.cu, fp64); file reading
is host work.  The resize is corner-aligned (node grids), a documented choice.
"""
from __future__ import annotations

import glob
import os

import numpy as np

from .errors import ConfigurationError
from .fields import SlownessModel, slowness_model


def _lib():
    from . import _lib as L

    return L, L.load()


def resize_bilinear(fields, shape, return_device: bool = False):
    """(B, h, w) or (h, w) fp64 -> (B, *shape) corner-aligned bilinear, on the device."""
    import torch

    from .device import stream_handle, to_device

    L, lib = _lib()
    x = to_device(fields, torch.float64)
    squeeze = x.dim() == 2
    x = x.reshape(-1, *x.shape[-2:])
    out = torch.empty((x.shape[0], *shape), dtype=torch.float64, device=x.device)
    L.check(lib.hs_resize_bilinear(x.data_ptr(), out.data_ptr(), x.shape[0], x.shape[1], x.shape[2], shape[0],
                                   shape[1], stream_handle()), "resize")
    out = out[0] if squeeze else out
    return out if return_device else out.cpu().numpy()


def gaussian_smooth(fields, sigma: float, return_device: bool = False):
    """SPEC gaussian_smooth: separable truncated Gaussian (radius ceil(3 sigma)), edge-replicated."""
    import torch

    from .device import stream_handle, to_device

    if sigma < 0:
        raise ConfigurationError(f"sigma must be >= 0, got {sigma}")
    L, lib = _lib()
    x = to_device(fields, torch.float64)
    squeeze = x.dim() == 2
    x = x.reshape(-1, *x.shape[-2:]).contiguous()
    out, tmp = torch.empty_like(x), torch.empty_like(x)
    L.check(lib.hs_gaussian_smooth(x.data_ptr(), out.data_ptr(), tmp.data_ptr(), x.shape[0], x.shape[1], x.shape[2],
                                   float(sigma), stream_handle()), "gaussian_smooth")
    out = out[0] if squeeze else out
    return out if return_device else out.cpu().numpy()


def normalise(fields, lo: float = 0.25, hi: float = 1.0, return_device: bool = False):
    """Affine map of each field onto [lo, hi]; a constant field maps to lo (SPEC design decision)."""
    import torch

    from .device import stream_handle, to_device

    L, lib = _lib()
    x = to_device(fields, torch.float64)
    squeeze = x.dim() == 2
    x = x.reshape(-1, *x.shape[-2:]).contiguous()
    out = torch.empty_like(x)
    mm = torch.empty((x.shape[0], 2), dtype=torch.float64, device=x.device)
    L.check(lib.hs_normalise_range(x.data_ptr(), out.data_ptr(), mm.data_ptr(), x.shape[0], x.shape[1] * x.shape[2],
                                   float(lo), float(hi), stream_handle()), "normalise")
    out = out[0] if squeeze else out
    return out if return_device else out.cpu().numpy()


def sigma_for(target_n: int) -> float:
    """sigma = 1 grid cell at n = 128, scaled with n / 128."""
    return target_n / 128.0


def read_pgm(path: str) -> np.ndarray:
    """8-bit binary PGM (P5) -> float64 grid."""
    with open(path, "rb") as f:
        data = f.read()
    toks, pos = [], 0
    while len(toks) < 4:
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
    if toks[0] != b"P5" or int(toks[3]) > 255:
        raise ConfigurationError(f"{path}: not an 8-bit binary PGM")
    w, h = int(toks[1]), int(toks[2])
    return np.frombuffer(data[pos + 1:pos + 1 + w * h], dtype=np.uint8).reshape(h, w).astype(np.float64)


def read_f64(path: str) -> np.ndarray:
    """Raw little-endian float64 grid with a ``.hdr`` sidecar "rows cols"."""
    with open(os.path.splitext(path)[0] + ".hdr") as f:
        rows, cols = (int(v) for v in f.read().split()[:2])
    return np.fromfile(path, dtype="<f8").reshape(rows, cols)


def prepare(images, target_n: int):
    """kappa^2 fields on (target_n + 1)^2 nodes for a list of images (one device batch per input shape)."""
    n1 = target_n + 1
    out = [None] * len(images)
    by_shape = {}
    for i, im in enumerate(images):
        by_shape.setdefault(np.shape(im), []).append(i)
    for shape, idx in by_shape.items():
        x = resize_bilinear(np.stack([images[i] for i in idx]), (n1, n1), return_device=True)
        x = gaussian_smooth(x, sigma_for(target_n), return_device=True)
        k2 = normalise(x, return_device=True).cpu().numpy()
        for k, i in enumerate(idx):
            out[i] = k2[k]
    return out


def load_slowness_corpus(path: str, target_n: int, gamma0: float = 0.05, layer_width=None) -> list[SlownessModel]:
    """SPEC load_slowness_corpus: every *.pgm / *.f64 under ``path`` (sorted) -> SlownessModel."""
    files = sorted(glob.glob(os.path.join(path, "*.pgm")) + glob.glob(os.path.join(path, "*.f64")))
    if not files:
        raise ConfigurationError(f"empty corpus: {path}")
    images = []
    for f in files:
        try:
            images.append(read_pgm(f) if f.endswith(".pgm") else read_f64(f))
        except (OSError, ValueError) as e:
            raise ConfigurationError(f"unreadable corpus file {f}: {e}") from e
    return [slowness_model(k2, gamma0=gamma0, layer_width=layer_width) for k2 in prepare(images, target_n)]
