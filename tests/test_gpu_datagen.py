"""GPU training-pair generator (paper_2306_17486_b200/datagen.py) against the CPU restatement.

Same seeded draws on both sides; the bar is the north-star tolerance on the iterate (1e-4 relative),
applied to e = x - x~ and r = A e, plus exact residual consistency of the GPU pairs in fp64.
"""
import numpy as np
import pytest

from conftest import relerr

pytestmark = pytest.mark.gpu

from paper_2306_17486_b200 import datagen, fields  # noqa: E402
from oracle import datagen_oracle as dg  # noqa: E402
from oracle import helm_oracle as ho  # noqa: E402


def models(n, count=2):
    out = []
    for s in range(count):
        k2 = np.random.default_rng(s).uniform(0.25, 1.0, (n, n))
        out.append(fields.slowness_model(k2, gamma0=datagen.TRAINING_GAMMA0, layer_width=4))
    return out


def oracle_model(m):
    return ho.Model(m.kappa_sq, m.gamma, m.omega, m.h)


@pytest.mark.parametrize("n", [33, 65])
def test_pairs_match_oracle(n):
    ms = models(n)
    gen = datagen.PairGenerator(ms)
    rng = np.random.default_rng(11)
    x, ks, mids = [], [], []
    for i in range(12):
        xi, ki = dg.draw(rng, ms[0].shape)
        x.append(xi)
        ks.append(ki if i >= 2 else (2 if i == 0 else 20))  # both ends of the range
        mids.append(i % 2)
    r, e = gen.pairs(np.stack(x), ks, mids)
    for i in range(len(ks)):
        om = oracle_model(ms[mids[i]])
        ro, eo, _ = dg.pair_from(om, x[i], ks[i])
        assert relerr(e[i], eo) < 1e-4, (i, ks[i], relerr(e[i], eo))
        assert relerr(r[i], ro) < 1e-4, (i, ks[i], relerr(r[i], ro))
        # residual consistency of the GPU pair in fp64 (SPEC invariant, 1e-10)
        ref = ho.helmholtz(e[i], om)
        assert np.linalg.norm(r[i] - ref) <= 1e-10 * np.linalg.norm(ref)


def test_dataset_seeded_round_robin():
    ms = models(33, 3)
    a = datagen.build_dataset(ms, 7, seed=5, batch=4)
    b = datagen.build_dataset(ms, 7, seed=5, batch=4)
    assert [p.model_id for p in a] == [0, 1, 2, 0, 1, 2, 0]
    for pa, pb in zip(a, b):
        assert pa.iterations == pb.iterations
        assert np.array_equal(pa.true_error.data, pb.true_error.data)
    # same draws as the oracle's dataset
    o = dg.build_dataset([oracle_model(m) for m in ms], 7, seed=5)
    for pa, po in zip(a, o):
        assert pa.iterations == po[2] and pa.model_id == po[3]
        assert relerr(pa.true_error.data, po[1]) < 1e-4
