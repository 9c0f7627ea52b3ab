"""Parity at the BENCHMARKED configurations (C2, C3) against reference-run goldens.

``oracle/make_golden_configs.py`` ran the REFERENCE's unmodified ``solve_helmholtz``
(``krylov.py:156-177``) and ``solve_with_learned_preconditioner`` (``krylov.py:180-246``,
the ARCH.md network composed from reference primitives injected as ``helmsolve.network``)
on the exact inputs ``bench.py`` solves (``problems.make_config``), and stored the
histories, iteration counts and solutions in ``tests/golden/configs_c{2,3}.npz``.

Here the device path solves the same RHS through the same public entry point the bench
times (``krylov.BatchSolver``) and must meet the north-star bar: iterations +-1, final
solution within 1e-4 relative L2 (C3: on the stored [::4, ::4] sub-grid), and residual
history within 1e-4 relative per iteration -- except where the REFERENCE'S OWN algorithm,
run in the BASELINE's complex64/fp32 precision class, already deviates from its complex128
run by more (``oracle/precision_envelope.py`` -> ``tests/golden/envelope_c*.npz``: fp32
V-cycle, complex64 Krylov bases, everything else complex128, as on the device).  There the
bar is 4x the running maximum of that envelope.  At C2 the envelope stays below 3e-6, so the
plain 1e-4 bar applies; at C3 the point-source RHS crosses a near-stagnation stretch around
iteration 240 where the envelope reaches 1.8e-2.

The network forward is also checked at the FULL bench shape (C2: 128 RHS, all active, so
the tcgen05 convolutions run their 32-row bands) against the numpy oracle on sampled RHS.
"""
import os

import numpy as np
import pytest

from conftest import GOLDEN, relerr

pytestmark = pytest.mark.gpu

from paper_2306_17486_b200 import krylov, netparams, network, problems  # noqa: E402
from oracle import network_oracle as no  # noqa: E402

HIST_TOL = 1e-4
X_TOL = 1e-4
ENV_FACTOR = 4.0  # allowed multiple of the precision envelope's running maximum


def load(cfg):
    p = os.path.join(GOLDEN, f"configs_{cfg}.npz")
    if not os.path.exists(p):
        pytest.fail(f"missing golden {p} (oracle/make_golden_configs.py)")
    return np.load(p)


def cases(g, prefix):
    return sorted({k.split(".")[0] for k in g.files if k.startswith(prefix)})


def history_bar(cfgname, case, n):
    """Per-iteration bar: max(1e-4, ENV_FACTOR x running max of the complex64 precision envelope)."""
    p = os.path.join(GOLDEN, f"envelope_{cfgname}.npz")
    bar = np.full(n, HIST_TOL)
    if os.path.exists(p):
        e = np.load(p)
        if f"{case}.env" in e.files:
            env = np.maximum.accumulate(e[f"{case}.env"])
            m = min(n, len(env))
            bar[:m] = np.maximum(HIST_TOL, ENV_FACTOR * env[:m])
            if m < n:
                bar[m:] = bar[m - 1]
            return bar
    if cfgname != "c2":
        pytest.fail(f"no precision envelope for {case} (oracle/precision_envelope.py)")
    return bar


def check_against(g, names, cfg, learned):
    idx = [int(g[f"{n}.idx"]) for n in names]
    rhs, owner = cfg.rhs[idx], cfg.model_of_rhs[idx]
    net = network.EncoderSolverNet.seeded(cfg.cnn_channels, seed=0) if learned else None
    solver = krylov.BatchSolver(cfg.models, net, jacobi_damping=cfg.jacobi_damping, num_levels=cfg.mg_levels)
    xs, reps = solver.solve(rhs, model_of=owner, tol=cfg.tol, max_iter=cfg.max_iter, restart=cfg.restart)
    worst = []
    for k, n in enumerate(names):
        it_ref = int(g[f"{n}.iterations"])
        href = g[f"{n}.hist"]
        rep = reps[k]
        h = np.asarray(rep.relative_residual_history)
        m = min(len(h), len(href))
        devs = np.abs(h[:m] - href[:m]) / href[:m]
        bar = history_bar(cfg.name.lower(), n, m)
        dev = float(devs.max())
        if f"{n}.x" in g.files:
            ex = relerr(xs[k], g[f"{n}.x"])
        else:
            ex = relerr(xs[k][::4, ::4], g[f"{n}.x_sub4"])
        worst.append((n, rep.iterations, it_ref, dev, ex))
        assert abs(rep.iterations - it_ref) <= 1, (n, rep.iterations, it_ref)
        assert rep.converged == bool(g[f"{n}.converged"]), n
        bad = np.nonzero(devs > bar)[0]
        assert bad.size == 0, (n, int(bad[0]), float(devs[bad[0]]), float(bar[bad[0]]))
        assert ex < X_TOL, (n, ex)
    print("\n".join(f"{n}: {a} it (ref {b}), hist dev {d:.2e}, x err {e:.2e}" for n, a, b, d, e in worst))


@pytest.mark.parametrize("kind", ["mg", "learned"])
def test_c2_matches_reference(kind):
    g = load("c2")
    names = cases(g, f"c2_{kind}_")
    assert len(names) == 4
    check_against(g, names, problems.make_config("C2"), kind == "learned")


@pytest.mark.parametrize("kind", ["mg", "learned"])
def test_c3_matches_reference(kind):
    g = load("c3")
    names = cases(g, f"c3_{kind}_")
    assert names, f"no c3_{kind} cases in the golden"
    check_against(g, names, problems.make_config("C3"), kind == "learned")


def _forward_check(cfgname, B, sample, tol=2e-5):
    import torch

    cfg = problems.make_config(cfgname)
    ch = cfg.cnn_channels
    L = len(ch)
    params = netparams.init_params(ch, seed=0)
    net = network.EncoderSolverNet(params, ch)
    models = cfg.models
    dn, enc = network.device_network(net, models, None, None)
    rng = np.random.default_rng(31)
    shape = models[0].shape
    r = (rng.standard_normal((B,) + shape) + 1j * rng.standard_normal((B,) + shape))
    r /= np.linalg.norm(r.reshape(B, -1), axis=1)[:, None, None]  # unit-norm Krylov vectors (krylov.py:94)
    owner = np.arange(B) * len(models) // B
    rd = torch.from_numpy(r.astype(np.complex64)).cuda()
    od = torch.from_numpy(owner.astype(np.int32)).cuda()
    dn.set_encodings(enc)
    u0 = dn.forward(rd, od).cpu().numpy()
    spec = no.spectrum_c64(params, L, shape)
    feats = {}
    for i in sample:
        m = models[int(owner[i])]
        if int(owner[i]) not in feats:
            feats[int(owner[i])] = no.encode(params, L, no.media_planes(m.kappa_sq, m.gamma, L))
        ref = no.preconditioner_estimate(params, L, feats[int(owner[i])], spec, r[i].astype(np.complex64), m.h)
        e = relerr(u0[i], ref)
        assert e < tol, (cfgname, i, e)


def test_network_forward_full_c2_shape():
    """C2 bench shape: 4 models x 32 RHS = 128 active RHS (32-row conv bands), 4 sampled RHS vs the oracle."""
    _forward_check("C2", 128, [0, 45, 77, 127])


def test_network_forward_c3_shape():
    """C3 shape (513x1025, CNN 16/32/64/128, implicit layer at 64x128), 16 RHS, 2 sampled vs the oracle."""
    _forward_check("C3", 16, [3, 14])
