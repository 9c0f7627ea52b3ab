"""Error-residual training pairs on the GPU.

The reference ships no datagen module; this follows its contract, SPEC.md ``[MODULE] datagen``
(reference SPEC.md:395-437; paper Eq. (4.11), §4.3):

    generate_sample(model, rng) -> SamplePair: x ~ standard complex normal per node; b = A x;
    k ~ uniform{2..20}; x~ = FGMRES(A, M = V-cycle, b, x0 = 0, k iterations); e = x - x~; r = A e.

Models should carry the training attenuation gamma0 = 0.05 (SPEC precondition).  A batch of samples
is one device pass: b = A x in fp64 for all of them, then one batched FGMRES with a per-sample
iteration cap k (hs_solve_args_t.iter_cap) and the V-cycle preconditioner, then e and r = A e in fp64
on the device.  The random draws follow oracle/datagen_oracle.py's documented order, so a
seeded dataset is identical to the CPU restatement's up to the solver's rounding.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .fields import ComplexField, SlownessModel

K_MIN, K_MAX = 2, 20
RESTART = 10  # krylov.py's default window
TRAINING_GAMMA0 = 0.05


@dataclass(frozen=True)
class SamplePair:
    """(residual, true error, model) triple of Eq. (4.10); residual = A true_error."""
    residual: ComplexField
    true_error: ComplexField
    model_id: int
    iterations: int


def _draw(rng: np.random.Generator, shape):
    re = rng.standard_normal(shape)
    im = rng.standard_normal(shape)
    return (re + 1j * im) / np.sqrt(2.0), int(rng.integers(K_MIN, K_MAX + 1))


class PairGenerator:
    """Batched device generator over equal-shape models (hierarchies built once)."""

    def __init__(self, models, num_levels: int = 3, jacobi_damping=None, coarse_iters: int = 10):
        from .krylov import BatchSolver

        self.models = list(models)
        if len({m.shape for m in self.models}) != 1:
            raise ValueError("PairGenerator needs models of one shape")
        self.solver = BatchSolver(self.models, None, num_levels=num_levels, jacobi_damping=jacobi_damping,
                                  coarse_iters=coarse_iters)

    def pairs(self, x, k, model_of, return_device: bool = False):
        """x (B, nx, ny) complex, k (B,) iteration counts, model_of (B,) -> (r, e) complex128."""
        import torch

        from .device import to_device, to_host
        from .fields import apply_operator

        xd = to_device(x, torch.complex128)
        k = np.asarray(k, dtype=np.int64)
        owner = np.asarray(model_of, dtype=np.int64)
        if xd.shape[0] != len(k) or len(k) != len(owner):
            raise ValueError("x, k and model_of must have one entry per sample")
        if k.min(initial=K_MIN) < 1:
            raise ValueError("iteration counts must be >= 1")

        def per_model(fn, u):
            out = torch.empty_like(u, dtype=torch.complex128)
            for mid in np.unique(owner):
                sel = torch.from_numpy(np.nonzero(owner == mid)[0]).to(u.device)
                out[sel] = fn(u[sel], self.models[int(mid)])
            return out

        b = per_model(lambda u, m: apply_operator(u, m), xd)
        # one batched solve: a tolerance no residual reaches and a per-sample iteration cap k
        xt, _ = self.solver.solve(b, model_of=owner, tol=1e-300, max_iter=int(k.max()), restart=RESTART,
                                  return_device=True, iter_caps=k)
        e = xd - xt
        r = per_model(lambda u, m: apply_operator(u, m), e)
        if return_device:
            return r, e
        return to_host(r), to_host(e)


def generate_sample(model: SlownessModel, rng: np.random.Generator, generator: PairGenerator | None = None,
                    model_id: int = 0) -> SamplePair:
    """SPEC generate_sample for one model (a PairGenerator can be passed to reuse its set-up)."""
    gen = generator or PairGenerator([model])
    x, k = _draw(rng, model.shape)
    r, e = gen.pairs(x[None], [k], [0 if generator is None else model_id])
    return SamplePair(ComplexField(r[0], model.h), ComplexField(e[0], model.h), model_id, k)


def build_dataset(models, samples_per_epoch: int, seed: int, batch: int = 256):
    """Seeded, round-robin over models (SPEC build_dataset); eager list of SamplePairs."""
    if samples_per_epoch <= 0:
        raise ValueError("samples_per_epoch must be positive")
    rng = np.random.default_rng(seed)
    gen = PairGenerator(models)
    shape = gen.models[0].shape
    out = []
    for start in range(0, samples_per_epoch, batch):
        n = min(batch, samples_per_epoch - start)
        mids = [(start + i) % len(models) for i in range(n)]
        draws = [_draw(rng, shape) for _ in range(n)]
        x = np.stack([d[0] for d in draws])
        ks = [d[1] for d in draws]
        r, e = gen.pairs(x, ks, mids)
        h = gen.models[0].h
        out += [SamplePair(ComplexField(r[i], h), ComplexField(e[i], h), mids[i], ks[i]) for i in range(n)]
    return out
