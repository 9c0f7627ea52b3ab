"""GPU parity: operator, transfers, smoother, V-cycle and coarse solve vs the reference fixtures."""
import numpy as np
import pytest

from conftest import complex_noise, golden, relerr

pytestmark = pytest.mark.gpu

from paper_2306_17486_b200 import fields, multigrid, problems  # noqa: E402
from oracle import helm_oracle as ho  # noqa: E402


def fixture_model():
    g = golden("fields.npz")
    return g, fields.SlownessModel(g["kappa_sq"], g["gamma"], float(g["omega"]), float(g["h"]))


def test_operator_fp64_matches_reference():
    g, m = fixture_model()
    out = fields.apply_helmholtz_array(g["u"], m)
    assert out.dtype == np.complex128
    assert relerr(out, g["a_true"]) < 1e-14
    assert relerr(fields.apply_helmholtz_array(g["u"], m, fields.PRECONDITIONER_SHIFT), g["a_prec"]) < 1e-14


def test_operator_fp32_and_batched():
    import torch

    g, m = fixture_model()
    u = torch.from_numpy(np.stack([g["u"], 2 * g["u"]])).cuda()
    out = fields.apply_operator(u, m, precision="fp32")
    assert out.dtype == torch.complex64
    assert relerr(out[0].cpu().numpy(), g["a_true"]) < 2e-6
    assert relerr(out[1].cpu().numpy(), 2 * g["a_true"]) < 2e-6


def test_constant_field_interior():
    # test_fields.py:109-115
    h = 0.1
    lap = fields.neg_laplacian(np.full((7, 9), 3.0 + 0j), h)
    assert np.allclose(lap[1:-1, 1:-1], 0.0, atol=1e-9)
    assert lap[0, 0] == pytest.approx(2 * 3.0 / h**2)


@pytest.mark.parametrize("shape", [(9, 9), (16, 16), (9, 13), (12, 9), (33, 17)])
def test_transfers_fp64_and_fp32(shape):
    g = golden("transfers.npz")
    tag = f"{shape[0]}x{shape[1]}"
    assert relerr(multigrid.restrict_full_weighting(g[f"f_{tag}"]), g[f"r_{tag}"]) < 1e-14
    assert relerr(multigrid.prolong_bilinear(g[f"c_{tag}"], shape), g[f"p_{tag}"]) < 1e-14
    f32 = g[f"f_{tag}"].astype(np.complex64)
    assert relerr(multigrid.restrict_full_weighting(f32), g[f"r_{tag}"]) < 1e-6
    # real input stays real (restrict_media path of the reference)
    r = multigrid.restrict_full_weighting(g[f"f_{tag}"].real.copy())
    assert r.dtype == np.float64 and relerr(r, g[f"r_{tag}"].real) < 1e-14


def test_transfer_errors():
    from paper_2306_17486_b200.errors import DimensionError

    with pytest.raises(DimensionError):
        multigrid.restrict_full_weighting(np.zeros((3, 3), dtype=complex))
    with pytest.raises(DimensionError):
        multigrid.prolong_bilinear(np.zeros((4, 4), dtype=complex), (12, 12))


def _vcycle_cases():
    g = golden("vcycle.npz")
    return sorted({k[len("rhs_"):] for k in g.files if k.startswith("rhs_")})


@pytest.mark.parametrize("tag", _vcycle_cases())
def test_vcycle_matches_reference(tag):
    g = golden("vcycle.npz")
    m = fields.slowness_model(g[f"kappa_sq_{tag}"], layer_width=int(g[f"lw_{tag}"]))
    H = multigrid.build_hierarchy(m, jacobi_damping=tuple(g[f"damp_{tag}"]), num_levels=int(g[f"levels_{tag}"]))
    z0 = multigrid.v_cycle(g[f"rhs_{tag}"], None, H)
    z1 = multigrid.v_cycle(g[f"rhs_{tag}"], g[f"u0_{tag}"], H)
    # complex64 V-cycle vs the complex128 reference
    assert relerr(z0, g[f"z0_{tag}"]) < 2e-5
    assert relerr(z1, g[f"z1_{tag}"]) < 2e-5


def test_vcycle_homogeneity_and_zero(rng):
    # GMRES on the coarsest level makes the cycle homogeneous (v(a r) = a v(r)) but
    # not additive: the Krylov polynomial depends on the rhs (same in the reference).
    m = fields.slowness_model(rng.uniform(0.25, 1.0, (33, 33)), layer_width=4)
    H = multigrid.build_hierarchy(m)
    assert np.all(multigrid.v_cycle(np.zeros((33, 33), complex), None, H) == 0)
    a = complex_noise(rng, (33, 33))
    za = multigrid.v_cycle(a, None, H)
    assert relerr(multigrid.v_cycle((2.0 - 1j) * a, None, H), (2.0 - 1j) * za) < 1e-5


def test_batched_vcycle_over_two_models(rng):
    import torch

    from paper_2306_17486_b200.multigrid import DeviceHierarchy, run_vcycle

    ms = [fields.slowness_model(rng.uniform(0.25, 1.0, (33, 33)), layer_width=4) for _ in range(2)]
    Hs = [multigrid.build_hierarchy(m, jacobi_damping=(0.8, 0.8)) for m in ms]
    rhs = complex_noise(rng, (4, 33, 33))
    owner = np.array([0, 1, 1, 0], dtype=np.int32)
    dh = DeviceHierarchy(Hs)
    out = run_vcycle(dh, torch.from_numpy(rhs).cuda(), None, torch.from_numpy(owner).cuda()).cpu().numpy()
    for i in range(4):
        O = ho.build_hierarchy(ho.Model(ms[owner[i]].kappa_sq, ms[owner[i]].gamma, ms[owner[i]].omega,
                                        ms[owner[i]].h), damping=(0.8, 0.8))
        assert relerr(out[i], ho.v_cycle(rhs[i], None, O)) < 2e-5


def test_coarse_solve_matches_oracle(rng):
    m = fields.slowness_model(rng.uniform(0.25, 1.0, (16, 16)), layer_width=3)
    lv = multigrid.Level(m, fields.PRECONDITIONER_SHIFT)
    rhs = complex_noise(rng, (16, 16))
    x = multigrid.coarse_solve(rhs, lv, iters=10)
    xo = ho.coarse_solve(rhs, ho.Level(ho.Model(m.kappa_sq, m.gamma, m.omega, m.h), 1.0, 0.5), 10)
    assert relerr(x, xo) < 1e-4
    assert np.all(multigrid.coarse_solve(np.zeros((16, 16), complex), lv) == 0)


def test_jacobi_matches_oracle(rng):
    m = fields.slowness_model(rng.uniform(0.25, 1.0, (17, 17)), layer_width=3)
    H = multigrid.build_hierarchy(m, num_levels=2)
    lv = H.levels[1]
    u, r = complex_noise(rng, lv.model.shape), complex_noise(rng, lv.model.shape)
    O = ho.Level(ho.Model(lv.model.kappa_sq, lv.model.gamma, lv.model.omega, lv.model.h), 1.0, 0.5, lv.wall)
    assert relerr(multigrid.jacobi_relax(u, r, lv, 2, 0.8), ho.jacobi(u, r, O, 2, 0.8)) < 1e-5


@pytest.mark.parametrize("n,levels", [(257, 2), (129, 2)])
def test_vcycle_large_coarse_grid_matches_oracle(rng, n, levels):
    """Coarsest grids above the fast coarse kernel's 8192-node reach (C3 with 3 levels, C4, C5 use
    128 x 256) take the L2-basis coarse GMRES; 129^2 with 2 levels (64^2) takes the 4096-node tier."""
    import torch

    from paper_2306_17486_b200.multigrid import DeviceHierarchy, run_vcycle

    m = fields.slowness_model(problems.smooth_random_kappa_sq((n, n), 6.0, 11), layer_width=8)
    H = multigrid.build_hierarchy(m, jacobi_damping=(0.8, 0.8), num_levels=levels)
    rhs = complex_noise(rng, (2, n, n))
    u0 = complex_noise(rng, (2, n, n), 1e-3)
    dh = DeviceHierarchy([H])
    owner = torch.zeros(2, dtype=torch.int32, device="cuda")
    out = run_vcycle(dh, torch.from_numpy(rhs).cuda(), torch.from_numpy(u0).cuda(), owner).cpu().numpy()
    O = ho.build_hierarchy(ho.Model(m.kappa_sq, m.gamma, m.omega, m.h), damping=(0.8, 0.8), num_levels=levels)
    for i in range(2):
        assert relerr(out[i], ho.v_cycle(rhs[i], u0[i], O)) < 2e-5


@pytest.mark.parametrize("shape", [(64, 64), (64, 128), (65, 64), (45, 50)])
def test_coarse_solve_at_config_sizes_matches_oracle(rng, shape):
    # the coarsest grids of C2 / C3 (fast on-chip kernel, 4096 / 8192 nodes) and odd / irregular sizes
    # (the L2-basis kernel); batched, three RHS
    m = fields.slowness_model(rng.uniform(0.25, 1.0, shape), layer_width=4)
    H = multigrid.build_hierarchy(m, num_levels=1)
    O = ho.build_hierarchy(ho.Model(m.kappa_sq, m.gamma, m.omega, m.h), num_levels=1)
    b = complex_noise(rng, (3,) + shape)
    import torch

    out = multigrid.coarse_solve(torch.from_numpy(b).cuda(), H.levels[0], 10).cpu().numpy()
    for i in range(3):
        assert relerr(out[i], ho.coarse_solve(b[i], O.levels[0], 10)) < 2e-5
