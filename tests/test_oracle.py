"""The CPU oracle against the reference's golden vectors and known answers (no GPU).

Fixtures in tests/golden were produced by oracle/make_golden.py from the
reference itself; these tests re-pin the oracle anywhere.  Known-answer and
dense-matrix checks restate the reference's own tests (cited per test).
"""
import numpy as np
import pytest

from conftest import complex_noise, golden, history_dev, relerr
from oracle import helm_oracle as ho
from oracle import network_oracle as no


def test_operator_matches_reference_fixture():
    g = golden("fields.npz")
    m = ho.Model(g["kappa_sq"], g["gamma"], float(g["omega"]), float(g["h"]))
    assert relerr(ho.helmholtz(g["u"], m), g["a_true"]) < 1e-15
    assert relerr(ho.helmholtz(g["u"], m, 1.0, 0.5), g["a_prec"]) < 1e-15


def test_known_answers():
    g = golden("fields.npz")
    # test_fields.py:86-91
    assert ho.omega_10ppw(129, 1.0) == pytest.approx(80.384)
    assert ho.omega_10ppw(257, 1.0) == pytest.approx(160.768)
    assert ho.omega_10ppw(129, 0.5) == pytest.approx(160.768)
    assert np.array_equal(ho.abl_mask(12, 10, 4, 0.01), g["abl_12x10_w4"])
    # test_fields.py:56-62: one node in from the edge of a width-4 layer
    assert ho.abl_mask(20, 20, 4, 0.01)[1, 10] == pytest.approx(0.01 + 0.99 * (3 / 4) ** 2)
    # test_fields.py:109-115: constant field -> 4 - 4 = 0 interior of -Lap, edges see the wall
    lap = ho.neg_lap(np.ones((6, 6), dtype=complex), 1.0)
    assert np.allclose(lap[1:-1, 1:-1], 0.0) and lap[0, 0] == 2.0 and lap[0, 2] == 1.0


def dense_restriction(shape):
    nx, ny = shape
    cx, cy = ho.coarse_dims(shape)
    R = np.zeros((cx * cy, nx * ny))
    for K in range(cx):
        for L in range(cy):
            for a in range(3):
                for b in range(3):
                    i, j = 2 * K + a, 2 * L + b
                    if i < nx and j < ny:
                        R[K * cy + L, i * ny + j] = ho.FW[a, b]
    return R


@pytest.mark.parametrize("shape", [(9, 9), (16, 16), (9, 13), (12, 9), (33, 17)])
def test_transfers_fixture_and_dense_oracle(shape):
    g = golden("transfers.npz")
    tag = f"{shape[0]}x{shape[1]}"
    assert relerr(ho.restrict(g[f"f_{tag}"]), g[f"r_{tag}"]) < 1e-15
    assert relerr(ho.prolong(g[f"c_{tag}"], shape), g[f"p_{tag}"]) < 1e-15
    R = dense_restriction(shape)  # test_multigrid.py:31-56, :79-86
    assert relerr(ho.restrict(g[f"f_{tag}"]).ravel(), R @ g[f"f_{tag}"].ravel()) < 1e-13
    assert relerr(ho.prolong(g[f"c_{tag}"], shape).ravel(), 4 * R.T @ g[f"c_{tag}"].ravel()) < 1e-13


def test_hierarchy_fixture():
    g = golden("hierarchy.npz")
    for n in (33, 34):
        m = ho.Model(g[f"k2_{n}_0"], g[f"gamma_{n}_0"], 0.0, 0.0)
        lw = 4
        model = ho.make_model(g[f"kappa_sq_{n}"], layer_width=lw)
        H = ho.build_hierarchy(model)
        for li, lv in enumerate(H.levels):
            assert relerr(lv.diag, g[f"diag_{n}_{li}"]) < 1e-14
            wall = np.zeros(lv.model.shape) if lv.wall is None else lv.wall
            assert np.allclose(wall, g[f"wall_{n}_{li}"])
        del m


def _vcycle_cases():
    g = golden("vcycle.npz")
    return sorted({k[len("rhs_"):] for k in g.files if k.startswith("rhs_")})


@pytest.mark.parametrize("tag", _vcycle_cases())
def test_vcycle_fixture(tag):
    g = golden("vcycle.npz")
    model = ho.make_model(g[f"kappa_sq_{tag}"], layer_width=int(g[f"lw_{tag}"]))
    H = ho.build_hierarchy(model, damping=tuple(g[f"damp_{tag}"]), num_levels=int(g[f"levels_{tag}"]))
    assert relerr(ho.v_cycle(g[f"rhs_{tag}"], None, H), g[f"z0_{tag}"]) < 1e-12
    assert relerr(ho.v_cycle(g[f"rhs_{tag}"], g[f"u0_{tag}"], H), g[f"z1_{tag}"]) < 1e-12


def test_poisson_vcycle_contracts():
    # test_multigrid.py:248-257: omega = 0, 33x33, spectral radius of V(1,1) < 0.25
    model = ho.make_model(np.ones((33, 33)), gamma0=0.0, layer_width=4, omega=0.0)
    H = ho.build_hierarchy(model, coarse_iters=10)
    rng = np.random.default_rng(3)
    e = complex_noise(rng, (33, 33))
    for _ in range(30):
        e_new = e - ho.v_cycle(ho.helmholtz(e, model, 1.0, 0.5) * 0 + H.levels[0].apply(e), None, H)
        rho = np.linalg.norm(e_new) / np.linalg.norm(e)
        e = e_new / np.linalg.norm(e_new)
    assert rho < 0.3


def textbook_gmres(A, M, b, tol, max_iter, restart):
    """test_krylov.py:12-46 restated: right-preconditioned GMRES via lstsq."""
    n = len(b)
    x = np.zeros(n, dtype=complex)
    r = b.copy()
    beta0 = np.linalg.norm(r)
    norms = [1.0]
    while True:
        beta = np.linalg.norm(r)
        V = [r / beta]
        Hm = np.zeros((restart + 1, restart), dtype=complex)
        for j in range(restart):
            w = A @ (M @ V[j])
            for k in range(j + 1):
                Hm[k, j] = np.vdot(V[k], w)
                w = w - Hm[k, j] * V[k]
            Hm[j + 1, j] = np.linalg.norm(w)
            V.append(w / Hm[j + 1, j])
            e1 = np.zeros(j + 2, dtype=complex)
            e1[0] = beta
            y = np.linalg.lstsq(Hm[: j + 2, : j + 1], e1, rcond=None)[0]
            est = np.linalg.norm(e1 - Hm[: j + 2, : j + 1] @ y) / beta0
            norms.append(est)
            if est <= tol or len(norms) - 1 >= max_iter:
                return norms


def test_oracle_fgmres_matches_textbook_gmres(rng):
    n = 16
    A = complex_noise(rng, (n, n)) + 4 * np.eye(n)
    M = np.linalg.inv(np.diag(np.diag(A)))
    b = complex_noise(rng, (n,))
    _, rep = ho.fgmres(lambda v: A @ v, lambda v: M @ v, b, None, 1e-9, 12, 12)
    ref = textbook_gmres(A, M, b, 1e-9, 12, 12)
    assert history_dev(rep.history, ref) < 1e-8


def test_oracle_solves_small_fixture():
    g = golden("solve_small.npz")
    for n in (33, 65):
        model = ho.make_model(g[f"kappa_sq_{n}"], layer_width=int(g[f"lw_{n}"]))
        x, rep = ho.solve_vcycle(model, g[f"b_{n}"], None, 1e-7, 250, 10)
        assert rep.iterations == len(g[f"hist_{n}"]) - 1
        assert history_dev(rep.history, g[f"hist_{n}"]) < 1e-8
        assert relerr(x, g[f"x_{n}"]) < 1e-9


def test_oracle_c1_first_rhs_fixture():
    g = golden("solve_c1_vcycle.npz")
    model = ho.make_model(g["kappa_sq"], layer_width=16)
    H = ho.build_hierarchy(model, damping=(0.8, 0.8))
    x, rep = ho.solve_vcycle(model, g["rhs"][0], H, 1e-6, 2000, 10)
    assert rep.iterations == int(g["iterations"][0])
    ref = g["hist"][0][: rep.iterations + 1]
    assert history_dev(rep.history, ref) < 1e-8
    assert relerr(x, g["x"][0]) < 1e-6


def test_cnn_primitives_fixture():
    g = golden("cnn_primitives.npz")
    assert relerr(no.conv2d(g["x"], g["w"], g["bias"]), g["conv_s1"]) < 1e-6
    assert relerr(no.conv2d(g["x"], g["w"], g["bias"], 2), g["conv_s2"]) < 1e-6
    assert relerr(no.conv_transpose2d(g["x"], g["wt"], g["bias"][:1].repeat(5)), g["tconv"]) < 1e-6
    assert relerr(no.batchnorm_infer(g["x"], g["bn_g"], g["bn_b"], g["bn_mu"], g["bn_var"]), g["bn"]) < 1e-6
    assert relerr(no.softplus(g["x"] * 10), g["softplus"]) < 1e-7
    for tag in ("8x8", "16x16", "8x16"):
        hh, ww = map(int, tag.split("x"))
        assert relerr(no.green_function(g[f"gk_{tag}"], (hh, ww)), g[f"spec_{tag}"]) < 1e-6
        assert relerr(no.implicit_apply(g[f"ix_{tag}"], g[f"spec_{tag}"].astype(np.complex64)), g[f"iy_{tag}"]) < 1e-6


def test_green_regression_ratio():
    # test_green.py:73-80: |G[16,16]| / |G[0,0]| ~= 1.137e-8 (+-5%)
    S = no.green_function(no.laplacian_plus_i(1), (16, 16))
    resp = np.fft.ifft2(S[0])
    assert np.abs(resp[16, 16]) / np.abs(resp[0, 0]) == pytest.approx(1.137e-8, rel=0.05)
    assert float(golden("cnn_primitives.npz")["green_ratio"]) == pytest.approx(1.137e-8, rel=0.05)


@pytest.mark.parametrize("L", [2, 3])
def test_network_oracle_matches_reference_primitive_composition(L):
    from paper_2306_17486_b200 import netparams

    g = golden("network.npz")
    tag = f"L{L}"
    ch = (16, 32, 64) if L == 3 else (8, 16)
    p = netparams.randomise_batchnorm(netparams.init_params(ch, seed=5), seed=6)
    media = no.media_planes(g[f"kappa_sq_{tag}"], g[f"gamma_{tag}"], L)
    feats = no.encode(p, L, media)
    for i, f in enumerate(feats):
        assert relerr(f, g[f"enc{i}_{tag}"]) < 2e-6
    r = g[f"r_{tag}"]
    (ix, iy), _ = no.cnn_dims(r.shape, L)
    r2 = np.stack([r[:ix, :iy].real, r[:ix, :iy].imag])[None].astype(np.float32)
    y = no.solve(p, L, r2, feats, no.spectrum_c64(p, L, r.shape))
    assert relerr(y, g[f"y_{tag}"]) < 2e-5
