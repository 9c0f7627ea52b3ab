"""Parameter layout and seeded initialisation of the encoder-solver CNN (ARCH.md).

The reference never shipped its ``network`` module (``krylov.py:201``), so the
architecture is pinned in ``ARCH.md``; this file is its single source of
truth for parameter names, shapes and the seeded draw order, shared by the
GPU network (``network.py``) and the CPU oracle used by the tests.

Initialisation follows ``PAPER.md:574-575``: PyTorch-default Kaiming-uniform
for convolutions (bound ``1/sqrt(fan_in)`` for weights and biases), batch norm
scale 1 / offset 0 / running mean 0 / running var 1, and the implicit kernel
``L + iI`` (``green.py:24-30``).  All draws come, in list order, from one
``numpy.random.default_rng(seed)`` in float32.
"""
from __future__ import annotations

import numpy as np


def _conv(spec, name, co, ci, fan_in, transposed=False, bn=True, bias=True):
    shape = (ci, co, 3, 3) if transposed else (co, ci, 3, 3)
    spec.append((name + ".w", shape, "uniform", fan_in))
    if bias:
        spec.append((name + ".b", (co,), "uniform", fan_in))
    if bn:
        spec.append((name + ".bn.gamma", (co,), "one", 0))
        spec.append((name + ".bn.beta", (co,), "zero", 0))
        spec.append((name + ".bn.mean", (co,), "zero", 0))
        spec.append((name + ".bn.var", (co,), "one", 0))


def _res(spec, name, c):
    _conv(spec, name + ".a", c, c, 9 * c)
    _conv(spec, name + ".b", c, c, 9 * c, bn=False)


def param_spec(channels: tuple[int, ...]):
    """Ordered (name, shape, kind, fan_in) list for an L = len(channels) network."""
    L = len(channels)
    if L < 2:
        raise ValueError("the network needs at least two levels")
    if channels[-1] % 2:
        raise ValueError("coarsest channel count must be even (complex pairing)")
    spec = []
    for side in ("enc", "sol"):
        _conv(spec, f"{side}.stem", channels[0], 2, 18)
        _res(spec, f"{side}.res0", channels[0])
        for lv in range(1, L):
            _conv(spec, f"{side}.down{lv}", channels[lv], channels[lv - 1], 9 * channels[lv - 1])
            _res(spec, f"{side}.res{lv}", channels[lv])
    spec.append(("sol.implicit.w", (channels[-1] // 2, 3, 3), "implicit", 0))
    for lv in range(L - 1, 0, -1):
        _conv(spec, f"sol.up{lv}", channels[lv - 1], channels[lv], 9 * channels[lv - 1], transposed=True)
        _res(spec, f"sol.ures{lv - 1}", channels[lv - 1])
    _conv(spec, "sol.head", 2, channels[0], 9 * channels[0], bn=False)
    return spec


def init_params(channels: tuple[int, ...], seed: int = 0) -> dict[str, np.ndarray]:
    """Seeded float32 (complex64 for the implicit kernel) parameters."""
    rng = np.random.default_rng(seed)
    out = {}
    for name, shape, kind, fan_in in param_spec(tuple(channels)):
        if kind == "uniform":
            bound = 1.0 / np.sqrt(fan_in)
            out[name] = rng.uniform(-bound, bound, shape).astype(np.float32)
        elif kind == "one":
            out[name] = np.ones(shape, dtype=np.float32)
        elif kind == "zero":
            out[name] = np.zeros(shape, dtype=np.float32)
        elif kind == "implicit":
            k = np.zeros((3, 3), dtype=np.complex64)
            k[1, 1] = 4 + 1j
            k[0, 1] = k[2, 1] = k[1, 0] = k[1, 2] = -1
            out[name] = np.repeat(k[None], shape[0], axis=0)
        else:  # pragma: no cover
            raise AssertionError(kind)
    return out


def randomise_batchnorm(params: dict[str, np.ndarray], seed: int) -> dict[str, np.ndarray]:
    """Non-trivial BN statistics for tests (checks the BN fold, not used by configs)."""
    rng = np.random.default_rng(seed)
    out = dict(params)
    for name in sorted(params):
        if name.endswith(".bn.gamma"):
            out[name] = rng.uniform(0.5, 1.5, params[name].shape).astype(np.float32)
        elif name.endswith(".bn.beta"):
            out[name] = rng.uniform(-0.2, 0.2, params[name].shape).astype(np.float32)
        elif name.endswith(".bn.mean"):
            out[name] = rng.uniform(-0.2, 0.2, params[name].shape).astype(np.float32)
        elif name.endswith(".bn.var"):
            out[name] = rng.uniform(0.5, 2.0, params[name].shape).astype(np.float32)
    return out


def count_params(channels) -> int:
    return int(sum(int(np.prod(s)) for _, s, _, _ in param_spec(tuple(channels))))
