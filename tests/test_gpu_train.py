"""Training step on the GPU against the reference autodiff and the oracle.

Bar (fp32 device arithmetic against float64 references): loss to 1e-5 relative; every parameter
gradient to 2e-4 relative (tensor norm) where the reference gradient is significant; the pre-BN
conv biases, whose exact gradient is zero (batch norm removes a constant), to an absolute 1e-6 of
the largest gradient; running statistics to 1e-5.
"""
import numpy as np
import pytest

from conftest import golden, relerr

pytestmark = pytest.mark.gpu

from oracle import train_oracle as to  # noqa: E402
from paper_2306_17486_b200 import netparams, network, problems  # noqa: E402
from paper_2306_17486_b200 import train as tr  # noqa: E402


def fixture(tag):
    g = golden("train.npz")
    ch = tuple(int(c) for c in g[f"channels_{tag}"])
    names = [n for n, *_ in netparams.param_spec(ch)]
    params = {n: g[f"p_{tag}_{n}"] for n in names}
    return g, ch, params


def f32(params):
    return {k: (v.astype(np.complex64) if np.iscomplexobj(v) else v.astype(np.float32)) for k, v in params.items()}


def pre_bn_bias(name, params):
    return name.endswith(".b") and (name[:-2] + ".bn.gamma") in params


def compare_grads(gpu, ref, params, rel=2e-4):
    scale = max(np.abs(v).max() for k, v in ref.items() if to.trainable(k))
    worst = 0.0
    for k, r in ref.items():
        if not to.trainable(k):
            continue
        if pre_bn_bias(k, params):
            assert np.abs(gpu[k] - r).max() < 1e-6 * scale, k
            continue
        e = relerr(gpu[k], r)
        worst = max(worst, e)
        assert e < rel, (k, e)
    return worst


@pytest.mark.parametrize("tag", ["a", "b"])
def test_gradients_match_reference_autodiff(tag):
    g, ch, params = fixture(tag)
    B, n = g[f"r_{tag}"].shape[:2]
    net = network.EncoderSolverNet(f32(params), ch)
    t = tr.Trainer(net, (n, n), float(g[f"h_{tag}"]), B)
    loss = t.step(g[f"media_{tag}"], g[f"r_{tag}"], g[f"e_{tag}"], model_of=np.arange(B), update=False)
    assert loss == pytest.approx(float(g[f"loss_{tag}"]), rel=1e-5)
    gg = t.grads()
    ref = {k: g[f"g_{tag}_{k}"] for k in params if to.trainable(k)}
    compare_grads(gg, ref, params)
    after = t.params()
    for k in params:
        if not to.trainable(k):
            assert relerr(after[k], g[f"s_{tag}_{k}"]) < 1e-5, k


def oracle_setup(ch, n, B, seed):
    rng = np.random.default_rng(seed)
    models = [problems.make_config("C1").models[0]] if n == 129 else None
    if models is None:
        from paper_2306_17486_b200 import fields
        models = [fields.slowness_model(problems.smooth_random_kappa_sq((n, n), 3.0, s), layer_width=max(2, n // 8))
                  for s in (1, 2)]
    params = netparams.randomise_batchnorm(netparams.init_params(ch, seed=seed), seed=seed + 1)
    owner = np.arange(B) % len(models)
    media = tr.media_planes(models, len(ch))
    r = rng.standard_normal((B, n, n)) + 1j * rng.standard_normal((B, n, n))
    e = 0.01 * (rng.standard_normal((B, n, n)) + 1j * rng.standard_normal((B, n, n)))
    return params, models, owner, media, r, e


def test_gradients_match_oracle_production_channels():
    # (16, 32, 64) channels on a 65^2 grid (coarse 16^2), batch 4 over two models
    ch, n, B = (16, 32, 64), 65, 4
    params, models, owner, media, r, e = oracle_setup(ch, n, B, 11)
    h = models[0].h
    po = to.as_float64(params)
    loss, og, _ = to.loss_and_grads(po, len(ch), media[owner].astype(np.float64), r, e, h)
    t = tr.Trainer(network.EncoderSolverNet(params, ch), (n, n), h, B)
    lg = t.step(media, r, e, model_of=owner, update=False)
    assert lg == pytest.approx(loss, rel=1e-5)
    compare_grads(t.grads(), og, po)


def test_adam_steps_match_oracle():
    g, ch, params = fixture("b")
    B, n = g["r_b"].shape[:2]
    h = float(g["h_b"])
    t = tr.Trainer(network.EncoderSolverNet(f32(params), ch), (n, n), h, B, lr=1e-3)
    po = {k: v.copy() for k, v in params.items()}
    opt = to.Adam(po, lr=1e-3)
    for _ in range(3):
        lo, _ = to.train_step(po, 3, g["media_b"], g["r_b"], g["e_b"], h, opt)
        lg = t.step(g["media_b"], g["r_b"], g["e_b"], model_of=np.arange(B))
        assert lg == pytest.approx(lo, rel=1e-4)
    got = t.params()
    for k, v in po.items():
        if pre_bn_bias(k, params):
            continue  # zero-gradient parameters: Adam normalises rounding noise (|update| <= 3 lr)
        d_ref = v - params[k]
        d_gpu = got[k] - params[k].astype(got[k].dtype)
        if to.trainable(k):
            assert relerr(d_gpu, d_ref) < 2e-2, k
        else:
            assert relerr(got[k], v) < 1e-5, k


def test_lr_zero_keeps_parameters():
    g, ch, params = fixture("a")
    B, n = g["r_a"].shape[:2]
    p32 = f32(params)
    t = tr.Trainer(network.EncoderSolverNet(p32, ch), (n, n), float(g["h_a"]), B, lr=0.0)
    t.step(g["media_a"], g["r_a"], g["e_a"], model_of=np.arange(B))
    got = t.params()
    for k in params:
        if to.trainable(k):
            assert np.array_equal(got[k], p32[k]), k


def test_overfit_one_batch_and_checkpoint_round_trip(tmp_path):
    ch, n, B = (8, 16), 33, 4
    params, models, owner, media, r, e = oracle_setup(ch, n, B, 21)
    h = models[0].h
    # a representable target on the u0 scale (h^2/64): a constant field on the network grid
    e = np.zeros((B, n, n), dtype=complex)
    e[:, : n - 1, : n - 1] = (h * h / 64.0) * (0.4 - 0.3j)
    t = tr.Trainer(network.EncoderSolverNet(params, ch), (n, n), h, B, lr=1e-2)
    losses = [t.step(media, r, e, owner) for _ in range(40)]
    assert losses[-1] < 0.5 * losses[0], (losses[0], losses[-1])
    # checkpoint: save, restore into a fresh trainer, continue identically (deterministic reductions)
    path = str(tmp_path / "ck.npz")
    tr.save_checkpoint(path, t.state(), ch)
    st = tr.load_checkpoint(path)
    t2 = tr.Trainer(network.EncoderSolverNet(params, ch), (n, n), h, B, lr=1e-2)
    t2.load_state(st)
    a = t.step(media, r, e, owner)
    b = t2.step(media, r, e, owner)
    assert a == b
    pa, pb = t.params(), t2.params()
    for k in pa:
        assert np.array_equal(pa[k], pb[k]), k


def test_deterministic_gradients():
    ch, n, B = (8, 16), 33, 3
    params, models, owner, media, r, e = oracle_setup(ch, n, B, 5)
    g1 = tr.Trainer(network.EncoderSolverNet(params, ch), (n, n), models[0].h, B)
    g2 = tr.Trainer(network.EncoderSolverNet(params, ch), (n, n), models[0].h, B)
    g1.step(media, r, e, owner, update=False)
    g2.step(media, r, e, owner, update=False)
    a, b = g1.grads(), g2.grads()
    for k in a:
        assert np.array_equal(a[k], b[k]), k


def test_gradients_match_oracle_four_levels_nonsquare():
    # C3-style network (16, 32, 64, 128): 4 levels, implicit layer on a 4 x 8 coarse grid, 33 x 65 nodes
    ch, B = (16, 32, 64, 128), 2
    rng = np.random.default_rng(31)
    from paper_2306_17486_b200 import fields

    models = [fields.slowness_model(problems.smooth_random_kappa_sq((33, 65), 3.0, s), layer_width=4) for s in (1, 2)]
    params = netparams.randomise_batchnorm(netparams.init_params(ch, seed=3), seed=4)
    owner = np.arange(B) % 2
    media = tr.media_planes(models, len(ch))
    r = rng.standard_normal((B, 33, 65)) + 1j * rng.standard_normal((B, 33, 65))
    e = 0.01 * (rng.standard_normal((B, 33, 65)) + 1j * rng.standard_normal((B, 33, 65)))
    h = models[0].h
    po = to.as_float64(params)
    loss, og, _ = to.loss_and_grads(po, len(ch), media[owner].astype(np.float64), r, e, h)
    t = tr.Trainer(network.EncoderSolverNet(params, ch), (33, 65), h, B)
    lg = t.step(media, r, e, model_of=owner, update=False)
    assert lg == pytest.approx(loss, rel=1e-5)
    compare_grads(t.grads(), og, po)


def test_split_step_equals_fused_step():
    # the data-parallel sequence (backward, gradients out / in around an all-reduce, Adam) is the fused step
    import ctypes

    import torch

    from paper_2306_17486_b200 import _lib
    from paper_2306_17486_b200.device import stream_handle

    g, ch, params = fixture("a")
    B, n = g["r_a"].shape[:2]
    a = tr.Trainer(network.EncoderSolverNet(f32(params), ch), (n, n), float(g["h_a"]), B)
    b = tr.Trainer(network.EncoderSolverNet(f32(params), ch), (n, n), float(g["h_a"]), B)
    la = a.step(g["media_a"], g["r_a"], g["e_a"], model_of=np.arange(B))
    lb = b.step(g["media_a"], g["r_a"], g["e_a"], model_of=np.arange(B), update=False)
    lib = _lib.load()
    buf = torch.empty(b.n, dtype=torch.float32, device="cuda")
    _lib.check(lib.hs_trainer_grads(b.handle, buf.data_ptr(), 0, stream_handle()), "out")
    _lib.check(lib.hs_trainer_grads(b.handle, buf.data_ptr(), 1, stream_handle()), "in")
    _lib.check(lib.hs_trainer_apply(b.handle, ctypes.byref(b.adam), stream_handle()), "apply")
    assert la == lb
    pa, pb = a.params(), b.params()
    for k in pa:
        assert np.array_equal(pa[k], pb[k]), k
