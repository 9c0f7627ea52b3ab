"""Seeded synthetic problem generators for the BASELINE configurations C1..C5.

The reference ships no data generator (its ``datagen`` module is missing, see
SURVEY.md §2.1 row 11), and the paper's datasets (OpenFWI, STL-10, CIFAR-10)
are not available here.  These host-side numpy generators stand in for them:
they reproduce the value range of the squared slowness (kappa^2 in [0.25, 1],
``/root/reference/SPEC.md:404-417``) and the paper's 10-points-per-wavelength
frequency rule (``fields.py:120-131``), with the shapes and absorbing-layer
widths that ``BASELINE.json`` names.  Every draw comes from
``numpy.random.default_rng(seed)`` so the oracle and the GPU path see the same
float64 inputs.

Node-count convention (``fields.py:26-28``): an external size n maps to n+1
nodes with h = 1/(max(nx, ny) - 1).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .fields import SlownessModel, slowness_model


def gaussian_kernel(sigma: float) -> np.ndarray:
    """Normalised 1D Gaussian taps truncated at radius ceil(3 sigma)."""
    if sigma <= 0:
        return np.ones(1)
    radius = int(np.ceil(3.0 * sigma))
    t = np.arange(-radius, radius + 1, dtype=np.float64)
    k = np.exp(-0.5 * (t / sigma) ** 2)
    return k / k.sum()


def gaussian_smooth(values: np.ndarray, sigma: float) -> np.ndarray:
    """Separable truncated-Gaussian smoothing with edge replication."""
    a = np.asarray(values, dtype=np.float64)
    k = gaussian_kernel(sigma)
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
            acc += w * p[tuple(sl)]
        a = acc
    return a


def normalise_range(values: np.ndarray, lo: float = 0.25, hi: float = 1.0) -> np.ndarray:
    """Affine map onto [lo, hi]; a constant field maps to lo."""
    vmin, vmax = float(values.min()), float(values.max())
    if vmax - vmin <= 0:
        return np.full(values.shape, lo)
    return lo + (hi - lo) * (values - vmin) / (vmax - vmin)


def smooth_random_kappa_sq(shape, sigma: float, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return normalise_range(gaussian_smooth(rng.uniform(0.0, 1.0, shape), sigma))


def layered_kappa_sq(shape, seed: int, layers: int = 8, noise: float = 0.1, sigma: float = 12.0):
    """Horizontal layers (along axis 0 = depth) plus 10% smoothed noise, clipped."""
    rng = np.random.default_rng(seed)
    nx, ny = shape
    cuts = np.sort(rng.choice(np.arange(1, nx), size=layers - 1, replace=False))
    values = rng.uniform(0.25, 1.0, layers)
    depth_index = np.searchsorted(cuts, np.arange(nx), side="right")
    background = values[depth_index][:, None] * np.ones((1, ny))
    perturb = normalise_range(gaussian_smooth(rng.uniform(0.0, 1.0, shape), sigma), -1.0, 1.0)
    return np.clip(background + noise * perturb, 0.25, 1.0)


def salt_kappa_sq(shape, seed: int, sigma: float = 24.0) -> np.ndarray:
    """Layered background with a smoothed elliptical kappa^2 = 0.25 inclusion."""
    rng = np.random.default_rng(seed)
    nx, ny = shape
    base = layered_kappa_sq(shape, seed + 1000, noise=0.05, sigma=sigma)
    cx, cy = rng.uniform(0.35, 0.65) * nx, rng.uniform(0.3, 0.7) * ny
    ax, ay = rng.uniform(0.1, 0.2) * nx, rng.uniform(0.1, 0.25) * ny
    ix = (np.arange(nx)[:, None] - cx) / ax
    iy = (np.arange(ny)[None, :] - cy) / ay
    mask = gaussian_smooth((ix**2 + iy**2 <= 1.0).astype(np.float64), sigma / 4)
    return np.clip(mask * 0.25 + (1.0 - mask) * np.maximum(base, 0.25 + 0.75 * 0.5), 0.25, 1.0)


def point_sources(shape, count: int, seed: int, margin: int) -> np.ndarray:
    """``count`` unit point sources at seeded nodes at least ``margin`` from the edge."""
    rng = np.random.default_rng(seed)
    nx, ny = shape
    out = np.zeros((count, nx, ny), dtype=np.complex128)
    xs = rng.integers(margin, nx - margin, count)
    ys = rng.integers(margin, ny - margin, count)
    out[np.arange(count), xs, ys] = 1.0
    return out


def complex_gaussian_rhs(shape, count: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.standard_normal((count,) + tuple(shape)) + 1j * rng.standard_normal(
        (count,) + tuple(shape)
    )


@dataclass
class ProblemSet:
    """A config: slowness models, right-hand sides and the solve settings."""

    name: str
    models: list[SlownessModel]
    rhs: np.ndarray  # (B, nx, ny) complex128
    model_of_rhs: np.ndarray  # (B,) int
    mg_levels: int
    cnn_channels: tuple[int, ...]
    restart: int
    tol: float = 1e-6
    max_iter: int = 2000
    jacobi_damping: tuple[float, float] = (0.8, 0.8)
    extra: dict = field(default_factory=dict)

    @property
    def shape(self):
        return self.models[0].shape


def make_config(name: str, rhs_per_model: int | None = None, models: int | None = None,
                seed_offset: int = 0) -> ProblemSet:
    """Build one of BASELINE.json's configs C1..C5.

    ``seed_offset`` shifts every seed (a distinct, same-sized instance per
    data-parallel rank); 0 gives the fixtures' inputs.
    """
    name = name.upper()
    so = 1000 * seed_offset
    if name == "C1":
        n, sig, abl, nm, nr = 129, 8.0, 16, 1, 4
        ks = [smooth_random_kappa_sq((n, n), sig, so)]
        lv, ch, rs = 3, (16, 32, 64), 10
    elif name == "C2":
        n, sig, abl, nm, nr = 257, 12.0, 20, 4, 32
        nm = models or nm
        ks = [smooth_random_kappa_sq((n, n), sig, s + so) for s in range(nm)]
        lv, ch, rs = 3, (16, 32, 64), 10
    elif name == "C3":
        shape, abl, nm, nr = (513, 1025), 32, 1, 64
        ks = [layered_kappa_sq(shape, so)]
        lv, ch, rs = 4, (16, 32, 64, 128), 20
    elif name == "C4":
        shape, abl, nm, nr = (1025, 2049), 32, 1, 128
        ks = [smooth_random_kappa_sq(shape, 24.0, so)]
        lv, ch, rs = 4, (16, 32, 64, 128), 20
    elif name == "C5":
        shape, abl, nm, nr = (2049, 4097), 48, 1, 256
        ks = [salt_kappa_sq(shape, so)]
        lv, ch, rs = 5, (16, 32, 64, 128, 128), 30
    else:
        raise ValueError(f"unknown config {name}")
    nr = rhs_per_model or nr
    mods = [slowness_model(k, gamma0=0.01, layer_width=abl) for k in ks]
    shape = mods[0].shape
    rhs, owner = [], []
    for m in range(len(mods)):
        if name == "C3":
            half = nr // 2
            rhs.append(point_sources(shape, half, 100 + m + so, abl))
            rhs.append(complex_gaussian_rhs(shape, nr - half, 200 + m + so))
        else:
            rhs.append(point_sources(shape, nr, 100 + m + so, abl))
        owner += [m] * nr
    return ProblemSet(
        name,
        mods,
        np.concatenate(rhs, axis=0),
        np.asarray(owner, dtype=np.int64),
        lv,
        ch,
        rs,
    )
