"""Training step, CPU side: the oracle against the reference autodiff's golden.

tests/golden/train.npz holds, for two small networks (L = 2 and L = 3), the loss, every parameter
gradient and the updated running statistics of one training step computed by the REFERENCE's own
autodiff (oracle/make_golden.py fx_train, float64).  Adam has no reference implementation, so the
oracle's Adam is pinned to torch.optim.Adam.
"""
import numpy as np
import pytest
import torch

from conftest import golden, relerr
from oracle import train_oracle as to
from paper_2306_17486_b200 import netparams
from paper_2306_17486_b200 import train as tr
from paper_2306_17486_b200.errors import ConfigurationError, DimensionError


def fixture(tag):
    g = golden("train.npz")
    names = [n for n, *_ in netparams.param_spec(tuple(int(c) for c in g[f"channels_{tag}"]))]
    params = {n: g[f"p_{tag}_{n}"].copy() for n in names}
    grads = {n: g[f"g_{tag}_{n}"] for n in names if to.trainable(n)}
    stats = {n: g[f"s_{tag}_{n}"] for n in names if not to.trainable(n)}
    return g, params, grads, stats


@pytest.mark.parametrize("tag", ["a", "b"])
def test_oracle_matches_reference_autodiff(tag):
    g, params, grads, stats = fixture(tag)
    L = int(g[f"levels_{tag}"])
    loss, og, _ = to.loss_and_grads(params, L, g[f"media_{tag}"], g[f"r_{tag}"], g[f"e_{tag}"], float(g[f"h_{tag}"]))
    assert loss == pytest.approx(float(g[f"loss_{tag}"]), rel=1e-12)
    for k, ref in grads.items():
        if np.linalg.norm(ref) > 1e-12:
            assert relerr(og[k], ref) < 1e-9, k
        else:
            assert np.abs(og[k] - ref).max() < 1e-12, k
    for k, ref in stats.items():  # running statistics updated in place (autodiff.py:575-579)
        assert relerr(params[k], ref) < 1e-12, k


def test_adam_matches_torch():
    rng = np.random.default_rng(3)
    p = {"a.w": rng.standard_normal((3, 4)), "k": rng.standard_normal((2, 3)) + 1j * rng.standard_normal((2, 3))}
    tp = {k: torch.tensor(v, requires_grad=True) for k, v in p.items()}
    opt_t = torch.optim.Adam(list(tp.values()), lr=1e-2)
    opt = to.Adam(p, lr=1e-2)
    for _ in range(4):
        g = {k: rng.standard_normal(v.shape) + (1j * rng.standard_normal(v.shape) if np.iscomplexobj(v) else 0)
             for k, v in p.items()}
        for k, t in tp.items():
            t.grad = torch.tensor(g[k])
        opt_t.step()
        p = opt.step(p, g)
    for k in p:
        assert np.allclose(p[k], tp[k].detach().numpy(), rtol=1e-12, atol=1e-14), k


def test_lr_zero_leaves_parameters():
    g, params, _, _ = fixture("a")
    before = {k: v.copy() for k, v in params.items()}
    opt = to.Adam(params, lr=0.0)
    to.train_step(params, int(g["levels_a"]), g["media_a"], g["r_a"], g["e_a"], float(g["h_a"]), opt)
    for k in before:
        if to.trainable(k):
            assert np.array_equal(params[k], before[k]), k


def test_flat_layout_round_trip():
    ch = (16, 32, 64)
    p = netparams.init_params(ch, seed=2)
    vec = tr.flatten(p, ch)
    n_complex = int(np.prod(p["sol.implicit.w"].shape))
    assert vec.size == netparams.count_params(ch) + n_complex
    back = tr.unflatten(vec, ch)
    for k in p:
        assert np.array_equal(back[k], p[k]), k
    with pytest.raises(DimensionError):
        tr.unflatten(vec[:-1], ch)


def test_mse_loss_spec_examples():
    z = np.zeros((1, 2, 2), dtype=complex)
    assert tr.mse_loss(z, z) == 0.0
    assert tr.mse_loss(np.ones((1, 2, 2), dtype=complex), z) == 4.0
    with pytest.raises(DimensionError):
        tr.mse_loss(np.ones((1, 2, 2)), np.ones((1, 2, 3)))


def test_train_config_invariants():
    tr.TrainConfig(sizes=(65, 129), samples_per_epoch=(2000, 500))
    with pytest.raises(ConfigurationError):
        tr.TrainConfig(sizes=(129, 65), samples_per_epoch=(10, 10))
    with pytest.raises(ConfigurationError):
        tr.TrainConfig(sizes=(65, 129), samples_per_epoch=(10, 20))


def test_abi_param_count_matches_layout():
    import ctypes

    from paper_2306_17486_b200 import _lib

    lib = _lib.load()
    for ch in [(4, 8), (16, 32, 64), (16, 32, 64, 128)]:
        d = _lib.HsTrainDesc()
        d.levels = len(ch)
        for i, c in enumerate(ch):
            d.channels[i] = c
        d.nx = d.ny = 129
        d.batch = 2
        d.h = 1.0 / 128
        n = int(lib.hs_train_param_count(ctypes.byref(d)))
        assert n == tr.flatten(netparams.init_params(ch, 0), ch).size
