"""Drop-in fidelity: reference settings outside the fused fast path, per-solver state, per-RHS failure.

The reference accepts any V(relax_pre, relax_post) cycle and coarse step count
(multigrid.py:185-193, 232-244), any restart window including ``restart=None``
(krylov.py:39-47, 79-83).  The fused batched solver implements V(1,1), <= 16 coarse steps and
windows <= 32; everything else runs the general device V-cycle / generic device FGMRES
(multigrid._v_cycle_general, krylov._generic_solve) and must still match the oracle.
"""
import numpy as np
import pytest

from conftest import complex_noise, history_dev, relerr

pytestmark = pytest.mark.gpu

from paper_2306_17486_b200 import fields, krylov, multigrid, network, problems  # noqa: E402
from oracle import helm_oracle as ho  # noqa: E402
from oracle import network_oracle as no  # noqa: E402


def model33(seed=1, n=33, lw=4):
    return fields.slowness_model(problems.smooth_random_kappa_sq((n, n), 3.0, seed), layer_width=lw)


def omodel(m):
    return ho.Model(m.kappa_sq, m.gamma, m.omega, m.h)


def test_jacobi_zero_sweeps_is_identity(rng):
    m = model33()
    H = multigrid.build_hierarchy(m)
    u = complex_noise(rng, m.shape)
    assert np.array_equal(multigrid.jacobi_relax(u, np.zeros_like(u), H.levels[0], 0), u)


@pytest.mark.parametrize("pre,post,ci", [(2, 3, 10), (0, 1, 10), (1, 1, 24)])
def test_general_vcycle_matches_oracle(rng, pre, post, ci):
    m = model33()
    H = multigrid.build_hierarchy(m, relax_pre=pre, relax_post=post, coarse_iters=ci, jacobi_damping=(0.8, 0.8))
    O = ho.build_hierarchy(omodel(m), relax_pre=pre, relax_post=post, coarse_iters=ci, damping=(0.8, 0.8))
    r = complex_noise(rng, m.shape)
    u0 = complex_noise(rng, m.shape, 1e-3)
    assert not multigrid.fused_cycle(H)
    assert relerr(multigrid.v_cycle(r, None, H), ho.v_cycle(r, None, O)) < 2e-5
    assert relerr(multigrid.v_cycle(r, u0, H), ho.v_cycle(r, u0, O)) < 2e-5


def test_long_coarse_solve_matches_oracle(rng):
    m = model33(2, 9, 2)
    H = multigrid.build_hierarchy(m, num_levels=1)
    O = ho.build_hierarchy(omodel(m), num_levels=1)
    b = complex_noise(rng, m.shape)
    x = multigrid.coarse_solve(b, H.levels[0], iters=40)
    assert relerr(x, ho.coarse_solve(b, O.levels[0], 40)) < 1e-8


@pytest.mark.parametrize("kw", [dict(restart=None, max_iter=120), dict(restart=40, max_iter=300)])
def test_long_restart_windows_match_oracle(rng, kw):
    m = model33(3)
    b = complex_noise(rng, m.shape)
    x, rep = krylov.solve_helmholtz(m, fields.ComplexField(b, m.h), tol=1e-7, **kw)
    xo, ro = ho.solve_vcycle(omodel(m), b, None, 1e-7, kw["max_iter"], kw["restart"])
    assert abs(rep.iterations - ro.iterations) <= 1
    assert history_dev(rep.relative_residual_history, ro.history) < 1e-4
    assert relerr(x.data, xo) < 1e-4


def test_general_cycle_solve_matches_oracle(rng):
    m = model33(4)
    H = multigrid.build_hierarchy(m, relax_pre=2, relax_post=2, coarse_iters=20)
    O = ho.build_hierarchy(omodel(m), relax_pre=2, relax_post=2, coarse_iters=20)
    b = complex_noise(rng, m.shape)
    x, rep = krylov.solve_helmholtz(m, fields.ComplexField(b, m.h), H, tol=1e-7, max_iter=200)
    xo, ro = ho.solve_vcycle(omodel(m), b, O, 1e-7, 200, 10)
    assert abs(rep.iterations - ro.iterations) <= 1
    assert history_dev(rep.relative_residual_history, ro.history) < 1e-4
    assert relerr(x.data, xo) < 1e-4


def test_learned_protocol_long_window_matches_oracle(rng):
    m = model33(5)
    net = network.EncoderSolverNet.seeded((8, 16, 16), seed=3)
    b = complex_noise(rng, m.shape)
    x, rep = krylov.solve_with_learned_preconditioner(m, fields.ComplexField(b, m.h), net, tol=1e-6,
                                                      max_iter=200, restart=40)
    L, p = 3, net.params
    feats = no.encode(p, L, no.media_planes(m.kappa_sq, m.gamma, L))
    spec = no.spectrum_c64(p, L, m.shape)
    xo, ro = ho.solve_learned(omodel(m), b, lambda r: no.preconditioner_estimate(p, L, feats, spec, r, m.h),
                              1e-6, 200, 40, 3)
    assert abs(rep.iterations - ro.iterations) <= 1
    assert history_dev(rep.relative_residual_history, ro.history) < 1e-4
    assert relerr(x.data, xo) < 1e-4


def test_two_solvers_on_one_net_keep_their_encodings(rng):
    # a DeviceNet is shared per (net, shape); each solver must re-bind its own encodings
    ms = [model33(s) for s in (6, 7, 8)]
    net = network.EncoderSolverNet.seeded((8, 16, 16), seed=4)
    rhs = complex_noise(rng, (2, 33, 33))
    s1 = krylov.BatchSolver(ms[:1], net)
    ref1 = s1.solve(rhs, tol=1e-6, max_iter=150)
    s3 = krylov.BatchSolver(ms, net)  # rebinds the shared DeviceNet to three models' encodings
    x3, r3 = s3.solve(rhs, model_of=[2, 1], tol=1e-6, max_iter=150)
    x1, r1 = s1.solve(rhs, tol=1e-6, max_iter=150)  # must still use model 6's encodings
    assert np.array_equal(x1, ref1[0])
    assert [r.relative_residual_history for r in r1] == [r.relative_residual_history for r in ref1[1]]
    fresh = krylov.BatchSolver(ms, net).solve(rhs, model_of=[2, 1], tol=1e-6, max_iter=150)
    assert np.array_equal(x3, fresh[0])


def test_nan_rhs_fails_only_its_own_solve(rng):
    # one RHS's failure (non-finite Krylov vector / coarse GMRES status) must not mark the
    # others failed; the reference raises per solve (krylov.py:96-99)
    from paper_2306_17486_b200.errors import NumericalError

    m = model33(9)
    rhs = complex_noise(rng, (3, 33, 33))
    rhs[1, 10, 10] = np.nan
    solver = krylov.BatchSolver([m])
    x, reps = solver.solve(rhs, tol=1e-6, max_iter=150, raise_errors=False)
    assert reps[0].converged and reps[2].converged and not reps[1].converged
    good = krylov.BatchSolver([m]).solve(rhs[[0, 2]], tol=1e-6, max_iter=150)
    assert np.array_equal(x[[0, 2]], good[0])
    with pytest.raises(NumericalError):
        solver.solve(rhs, tol=1e-6, max_iter=150)
