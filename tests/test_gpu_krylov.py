"""GPU parity of the FGMRES solve against the reference (golden fixtures) and the oracle.

The bar (BASELINE.json north_star): residual histories within 1e-4 relative
per iteration, final solutions within 1e-4 relative L2, iteration counts +-1.
"""
import numpy as np
import pytest

from conftest import complex_noise, golden, history_dev, relerr

pytestmark = pytest.mark.gpu

from paper_2306_17486_b200 import fields, krylov, multigrid  # noqa: E402
from paper_2306_17486_b200.errors import NumericalError, SolverError  # noqa: E402
from oracle import helm_oracle as ho  # noqa: E402

HIST_TOL = 1e-4
X_TOL = 1e-4


def test_solve_small_matches_reference():
    g = golden("solve_small.npz")
    for n in (33, 65):
        m = fields.slowness_model(g[f"kappa_sq_{n}"], layer_width=int(g[f"lw_{n}"]))
        x, rep = krylov.solve_helmholtz(m, fields.ComplexField(g[f"b_{n}"], m.h), tol=1e-7, max_iter=250)
        ref = g[f"hist_{n}"]
        assert abs(rep.iterations - (len(ref) - 1)) <= 1
        assert len(rep.relative_residual_history) == rep.iterations + 1
        assert history_dev(rep.relative_residual_history, ref) < HIST_TOL
        assert relerr(x.data, g[f"x_{n}"]) < X_TOL
        assert rep.converged and rep.relative_residual_history[-1] <= 1e-7


def test_c1_vcycle_batch_matches_reference():
    g = golden("solve_c1_vcycle.npz")
    m = fields.slowness_model(g["kappa_sq"], layer_width=16)
    xs, reps = krylov.solve_batch([m], g["rhs"], tol=1e-6, max_iter=2000, restart=10, jacobi_damping=(0.8, 0.8))
    for i, rep in enumerate(reps):
        it = int(g["iterations"][i])
        ref = g["hist"][i][: it + 1]
        assert abs(rep.iterations - it) <= 1, (rep.iterations, it)
        assert history_dev(rep.relative_residual_history, ref) < HIST_TOL
        assert relerr(xs[i], g["x"][i]) < X_TOL
        assert rep.converged


def test_multi_model_batch_matches_oracle(rng):
    ms = [fields.slowness_model(rng.uniform(0.25, 1.0, (33, 33)), layer_width=4) for _ in range(2)]
    rhs = complex_noise(rng, (3, 33, 33))
    owner = [1, 0, 1]
    xs, reps = krylov.solve_batch(ms, rhs, model_of=owner, tol=1e-6, max_iter=300, restart=10)
    for i in range(3):
        m = ms[owner[i]]
        om = ho.Model(m.kappa_sq, m.gamma, m.omega, m.h)
        xo, ro = ho.solve_vcycle(om, rhs[i], None, 1e-6, 300, 10)
        assert abs(reps[i].iterations - ro.iterations) <= 1
        assert history_dev(reps[i].relative_residual_history, ro.history) < HIST_TOL
        assert relerr(xs[i], xo) < X_TOL


def test_restart_windows_and_max_iter_cap(rng):
    m = fields.slowness_model(rng.uniform(0.25, 1.0, (33, 33)), layer_width=4)
    b = fields.ComplexField(complex_noise(rng, (33, 33)), m.h)
    x, rep = krylov.solve_helmholtz(m, b, tol=1e-12, max_iter=7, restart=3)
    assert rep.iterations == 7 and not rep.converged and len(rep.relative_residual_history) == 8
    om = ho.Model(m.kappa_sq, m.gamma, m.omega, m.h)
    xo, ro = ho.solve_vcycle(om, b.data, None, 1e-12, 7, 3)
    assert history_dev(rep.relative_residual_history, ro.history) < HIST_TOL
    assert relerr(x.data, xo) < X_TOL


def test_zero_rhs_and_tol_one(rng):
    m = fields.slowness_model(rng.uniform(0.25, 1.0, (17, 17)), layer_width=3)
    x, rep = krylov.solve_helmholtz(m, fields.ComplexField(np.zeros((17, 17)), m.h), tol=1e-8)
    assert rep.converged and rep.iterations == 0 and rep.relative_residual_history == [1.0, 0.0]
    assert np.all(x.data == 0)
    b = fields.ComplexField(complex_noise(rng, (17, 17)), m.h)
    x, rep = krylov.solve_helmholtz(m, b, tol=1.0)
    assert rep.converged and rep.iterations == 0 and rep.relative_residual_history == [1.0]


def test_report_fields(rng):
    # test_krylov.py:156-163
    m = fields.slowness_model(rng.uniform(0.25, 1.0, (17, 17)), layer_width=3)
    b = fields.ComplexField(complex_noise(rng, (17, 17)), m.h)
    _, rep = krylov.solve_helmholtz(m, b, tol=1e-6, max_iter=200)
    assert isinstance(rep, krylov.SolveReport)
    assert rep.wall_time > 0
    assert len(rep.relative_residual_history) == rep.iterations + 1
    assert rep.relative_residual_history[0] == 1.0


def test_true_residual_is_reported(rng):
    m = fields.slowness_model(rng.uniform(0.25, 1.0, (33, 33)), layer_width=4)
    b = complex_noise(rng, (33, 33))
    x, rep = krylov.solve_helmholtz(m, fields.ComplexField(b, m.h), tol=1e-8, max_iter=400)
    om = ho.Model(m.kappa_sq, m.gamma, m.omega, m.h)
    true_rel = np.linalg.norm(b - ho.helmholtz(x.data, om)) / np.linalg.norm(b)
    assert abs(true_rel - rep.relative_residual_history[-1]) <= 1e-9


# --------------------------------------------- generic callable fgmres (test_krylov.py)


def test_generic_identity_one_iteration(rng):
    b = complex_noise(rng, (30,))
    x, rep = krylov.fgmres(lambda v: v, lambda v: v, b, tol=1e-12, max_iter=10)
    assert rep.iterations == 1 and rep.converged and np.allclose(x, b)


def test_generic_dense_direct_solve(rng):
    n = 20
    A = complex_noise(rng, (n, n)) + 4 * np.eye(n)
    b = complex_noise(rng, (n,))
    x, rep = krylov.fgmres(lambda v: A @ v, lambda v: v, b, tol=1e-10, max_iter=n, restart=n)
    xd = np.linalg.solve(A, b)
    assert rep.converged and np.linalg.norm(x - xd) <= 1e-8 * np.linalg.norm(xd)


def test_generic_matches_oracle_and_textbook(rng):
    n = 16
    A = complex_noise(rng, (n, n)) + 4 * np.eye(n)
    M = np.linalg.inv(np.diag(np.diag(A)))
    b = complex_noise(rng, (n,))
    _, rep = krylov.fgmres(lambda v: A @ v, lambda v: M @ v, b, tol=1e-9, max_iter=12, restart=12)
    _, ro = ho.fgmres(lambda v: A @ v, lambda v: M @ v, b, None, 1e-9, 12, 12)
    assert history_dev(rep.relative_residual_history, ro.history) < 1e-10


def test_generic_nan_raises(rng):
    b = complex_noise(rng, (8,))

    def bad(v):
        out = v.copy()
        out[0] = np.nan
        return out

    with pytest.raises(NumericalError):
        krylov.fgmres(bad, lambda v: v, b, tol=1e-8, max_iter=4)


def test_generic_cap_and_2d(rng):
    n = 50
    A = complex_noise(rng, (n, n)) + 1.5 * np.eye(n)
    b = complex_noise(rng, (n,))
    _, rep = krylov.fgmres(lambda v: A @ v, lambda v: v, b, tol=1e-14, max_iter=7, restart=3)
    assert rep.iterations == 7 and not rep.converged
    b2 = complex_noise(rng, (6, 5))
    x, rep = krylov.fgmres(lambda v: 2 * v, lambda v: v, b2, tol=1e-12, max_iter=5)
    assert x.shape == (6, 5) and np.allclose(x, b2 / 2)


def test_bad_arguments():
    with pytest.raises(ValueError):
        krylov.fgmres(lambda v: v, lambda v: v, np.ones(3), tol=0.0)
    with pytest.raises(ValueError):
        krylov.fgmres(lambda v: v, lambda v: v, np.ones(3), max_iter=0)


def test_breakdown_raises_solver_error():
    # a Krylov space exhausted before tol: A = diag with 2 distinct values, tol unreachable
    A = np.diag([1.0, 1.0, 2.0, 2.0]).astype(complex)
    b = np.ones(4, dtype=complex)
    with pytest.raises(SolverError):
        krylov.fgmres(lambda v: A @ v, lambda v: v, b, tol=1e-300, max_iter=4, restart=4)
