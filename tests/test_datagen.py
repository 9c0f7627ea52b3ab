"""CPU checks of the training-pair oracle against the SPEC's own examples.

The reference has no datagen code, so its contract's examples pin the restatement: residual
consistency r = A e, k covering {2..20}, spectral smoothing of e with k, seeded determinism, and the
zero-sample error.
"""
import numpy as np
import pytest

from oracle import datagen_oracle as dg
from oracle import helm_oracle as ho


def model(n=33, seed=0):
    k2 = np.random.default_rng(seed).uniform(0.25, 1.0, (n, n))
    return ho.make_model(k2, gamma0=dg.TRAINING_GAMMA0, layer_width=4)


def test_residual_consistency_and_k_range():
    m = model()
    rng = np.random.default_rng(1)
    ks = set()
    for _ in range(6):
        r, e, k = dg.generate_sample(m, rng)
        assert 2 <= k <= 20
        ks.add(k)
        ref = ho.helmholtz(e, m)
        assert np.linalg.norm(r - ref) <= 1e-10 * np.linalg.norm(ref)
    # the draw covers the whole range over many samples
    rng = np.random.default_rng(2)
    draws = {dg.draw(rng, (2, 2))[1] for _ in range(400)}
    assert draws == set(range(2, 21))


def test_spectral_smoothing_with_iterations():
    # SPEC example: e's top-half Fourier energy is lower for k = 20 than for k = 2 (averaged over draws)
    m = model()
    hier = ho.build_hierarchy(m)
    rng = np.random.default_rng(3)
    f2, f20 = [], []
    for _ in range(10):
        x, _ = dg.draw(rng, m.kappa_sq.shape)
        f2.append(dg.high_frequency_fraction(dg.pair_from(m, x, 2, hier)[1]))
        f20.append(dg.high_frequency_fraction(dg.pair_from(m, x, 20, hier)[1]))
    assert np.mean(f20) < np.mean(f2)


def test_seeded_determinism_and_round_robin():
    ms = [model(seed=s) for s in range(3)]
    a = dg.build_dataset(ms, 5, seed=7)
    b = dg.build_dataset(ms, 5, seed=7)
    assert [s[3] for s in a] == [0, 1, 2, 0, 1]
    for sa, sb in zip(a, b):
        assert np.array_equal(sa[0], sb[0]) and np.array_equal(sa[1], sb[1]) and sa[2] == sb[2]
    with pytest.raises(ValueError):
        dg.build_dataset(ms, 0, seed=7)
