"""CPU restatement of the training-pair generator -- TEST INFRASTRUCTURE ONLY.

The reference ships no datagen code; its contract is SPEC.md `[MODULE] datagen`,
`[OP] generate_sample` (reference SPEC.md:418-426, paper Eq. (4.11), §4.3):

    draw x ~ standard complex normal per node; b = A x; k ~ uniform{2..20};
    x~ = FGMRES(A, M = V-cycle, b, x0 = 0, k iterations); e = x - x~; r = A e; return (r, e)

on models built with the training attenuation gamma0 = 0.05.  The operators are the oracle's
restatements (helm_oracle.helmholtz = fields.py:202-210, v_cycle = multigrid.py:247-274,
fgmres = krylov.py:39-146 with restart 10, the library default).  ``build_dataset`` deals samples
round-robin over the models.

The random draws follow one documented order so the GPU path (paper_2306_17486_b200/datagen.py)
reproduces them exactly: for sample i, model i % n_models; x = (N(0,1) + i N(0,1)) / sqrt(2) as two
``rng.standard_normal(shape)`` calls (real part first); then k = ``rng.integers(2, 21)``.

Only tests/ and bench.py's CPU leg may use this module.
"""
from __future__ import annotations

import numpy as np

from oracle import helm_oracle as ho

K_MIN, K_MAX = 2, 20
RESTART = 10
TRAINING_GAMMA0 = 0.05


def draw(rng: np.random.Generator, shape):
    """One sample's random inputs in the documented order: (x, k)."""
    re = rng.standard_normal(shape)
    im = rng.standard_normal(shape)
    x = (re + 1j * im) / np.sqrt(2.0)
    k = int(rng.integers(K_MIN, K_MAX + 1))
    return x, k


def generate_sample(model: ho.Model, rng: np.random.Generator, hier=None):
    """SPEC generate_sample: returns (r, e, k)."""
    x, k = draw(rng, model.kappa_sq.shape)
    return pair_from(model, x, k, hier)


def pair_from(model: ho.Model, x, k, hier=None):
    hier = hier or ho.build_hierarchy(model)
    A = lambda u: ho.helmholtz(u, model)  # noqa: E731
    b = A(x)
    # k iterations exactly: a tolerance no residual reaches
    xt, rep = ho.fgmres(A, lambda r: ho.v_cycle(r, None, hier), b, None, 1e-300, k, RESTART)
    assert rep.iterations == k
    e = x - xt
    return A(e), e, k


def build_dataset(models, samples: int, seed: int):
    """Round-robin over models, seeded: list of (r, e, k, model_id)."""
    if samples <= 0:
        raise ValueError("samples_per_epoch must be positive")
    rng = np.random.default_rng(seed)
    hiers = [ho.build_hierarchy(m) for m in models]
    out = []
    for i in range(samples):
        mid = i % len(models)
        x, k = draw(rng, models[mid].kappa_sq.shape)
        r, e, _ = pair_from(models[mid], x, k, hiers[mid])
        out.append((r, e, k, mid))
    return out


def high_frequency_fraction(e):
    """Share of e's energy in the top half of the Fourier modes (|freq| > N/4 on either axis)."""
    E = np.abs(np.fft.fft2(e)) ** 2
    nx, ny = e.shape
    fx = np.abs(np.fft.fftfreq(nx))[:, None]
    fy = np.abs(np.fft.fftfreq(ny))[None, :]
    hi = (fx > 0.25) | (fy > 0.25)
    return float(E[hi].sum() / E.sum())
