"""Generate tests/golden/*.npz from the REFERENCE and pin the oracle against it.

Run in this container only (it imports ``/root/reference/pkg/src`` in place):

    PYTHONDONTWRITEBYTECODE=1 python oracle/make_golden.py [--quick]

For every fixture it (1) runs the reference, (2) runs the oracle restatement
on the same inputs and asserts agreement, and (3) stores inputs + reference
outputs.  ``tests/test_oracle.py`` re-checks the oracle against the stored
fixtures anywhere (no reference needed), and the GPU parity tests compare the
CUDA path against the same fixtures.

The encoder-solver network is missing from the reference (krylov.py:201), so
for the learned protocol this script composes ARCH.md's architecture from the
reference's own autodiff/green primitives and injects it as
``helmsolve.network`` into the reference's unmodified
``solve_with_learned_preconditioner``.
"""
from __future__ import annotations

import argparse
import os
import sys
import types

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/pkg/src"
OUT = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)
sys.path.insert(0, REF)

from helmsolve import autodiff as ad  # noqa: E402  (reference)
from helmsolve import fields as rf  # noqa: E402
from helmsolve import green as rg  # noqa: E402
from helmsolve import krylov as rk  # noqa: E402
from helmsolve import multigrid as rm  # noqa: E402

from oracle import helm_oracle as ho  # noqa: E402
from oracle import network_oracle as no  # noqa: E402
from paper_2306_17486_b200 import netparams, problems  # noqa: E402


def relerr(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def save(name, **arrays):
    os.makedirs(OUT, exist_ok=True)
    np.savez_compressed(os.path.join(OUT, name), **arrays)
    print(f"wrote {name}: " + ", ".join(f"{k}{tuple(np.shape(v))}" for k, v in arrays.items()))


def noise(rng, shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def omodel(m):
    return ho.Model(m.kappa_sq, m.gamma, m.omega, m.h)


# ------------------------------------------------------------------- fixtures


def fx_fields():
    rng = np.random.default_rng(11)
    k2 = rng.uniform(0.25, 1.0, (9, 7))
    m = rf.slowness_model(k2, layer_width=2)
    u = noise(rng, (9, 7))
    a_true = rf.apply_helmholtz_array(u, m, rf.TRUE_SHIFT)
    a_prec = rf.apply_helmholtz_array(u, m, rf.PRECONDITIONER_SHIFT)
    om = omodel(m)
    assert relerr(ho.helmholtz(u, om), a_true) < 1e-15
    assert relerr(ho.helmholtz(u, om, 1.0, 0.5), a_prec) < 1e-15
    assert relerr(ho.make_model(k2, layer_width=2).gamma, m.gamma) == 0.0
    kat = np.array([rf.wavenumber_for_grid(129, 1.0), rf.wavenumber_for_grid(257, 1.0),
                    rf.wavenumber_for_grid(129, 0.5)])
    assert np.allclose(kat, [ho.omega_10ppw(129, 1.0), ho.omega_10ppw(257, 1.0), ho.omega_10ppw(129, 0.5)])
    abl = rf.build_abl(12, 10, 4, 0.01)
    assert np.array_equal(abl, ho.abl_mask(12, 10, 4, 0.01))
    save("fields.npz", kappa_sq=k2, gamma=m.gamma, omega=m.omega, h=m.h, u=u, a_true=a_true, a_prec=a_prec,
         omega_kat=kat, abl_12x10_w4=abl)


def fx_transfers():
    rng = np.random.default_rng(12)
    out = {}
    for shape in [(9, 9), (16, 16), (9, 13), (12, 9), (33, 17)]:
        tag = f"{shape[0]}x{shape[1]}"
        f = noise(rng, shape)
        c = noise(rng, rm.coarse_shape(shape))
        r = rm.restrict_full_weighting(f)
        p = rm.prolong_bilinear(c, shape)
        assert relerr(ho.restrict(f), r) < 1e-15 and relerr(ho.prolong(c, shape), p) < 1e-15
        out.update({f"f_{tag}": f, f"r_{tag}": r, f"c_{tag}": c, f"p_{tag}": p})
    save("transfers.npz", **out)


def fx_hierarchy():
    rng = np.random.default_rng(13)
    out = {}
    for n, lw in [(33, 4), (34, 4)]:
        m = rf.slowness_model(rng.uniform(0.25, 1.0, (n, n)), layer_width=lw)
        H = rm.build_hierarchy(m)
        O = ho.build_hierarchy(omodel(m))
        out[f"kappa_sq_{n}"] = m.kappa_sq
        for li, (a, b) in enumerate(zip(H.levels, O.levels)):
            assert relerr(b.diag, a.diag) < 1e-14
            out[f"diag_{n}_{li}"] = a.diag
            out[f"wall_{n}_{li}"] = np.zeros(a.model.shape) if a.wall is None else a.wall
            out[f"k2_{n}_{li}"] = a.model.kappa_sq
            out[f"gamma_{n}_{li}"] = a.model.gamma
    save("hierarchy.npz", **out)


def fx_vcycle():
    rng = np.random.default_rng(14)
    out = {}
    for n, lw, damp, nl in [(33, 4, rm.CHEBYSHEV_DAMPING, 3), (65, 8, (0.8, 0.8), 3), (66, 8, (0.8, 0.8), 3),
                            (33, 4, (0.8, 0.8), 1), (129, 16, (0.8, 0.8), 4)]:
        tag = f"{n}_{nl}_{damp[0]}"
        m = rf.slowness_model(problems.smooth_random_kappa_sq((n, n), 4.0, n), layer_width=lw)
        H = rm.build_hierarchy(m, jacobi_damping=damp, num_levels=nl)
        O = ho.build_hierarchy(omodel(m), damping=damp, num_levels=nl)
        rhs = noise(rng, (n, n))
        u0 = 1e-5 * noise(rng, (n, n))
        z0 = rm.v_cycle(rhs, None, H)
        z1 = rm.v_cycle(rhs, u0, H)
        assert relerr(ho.v_cycle(rhs, None, O), z0) < 1e-12 and relerr(ho.v_cycle(rhs, u0, O), z1) < 1e-12
        out.update({f"kappa_sq_{tag}": m.kappa_sq, f"rhs_{tag}": rhs, f"u0_{tag}": u0, f"z0_{tag}": z0,
                    f"z1_{tag}": z1, f"lw_{tag}": lw, f"damp_{tag}": np.array(damp), f"levels_{tag}": nl})
    save("vcycle.npz", **out)


def fx_solve_c1():
    """C1 V-cycle-only with the reference's own solve_helmholtz."""
    cfg = problems.make_config("C1")
    m = cfg.models[0]
    H = rm.build_hierarchy(m, jacobi_damping=(0.8, 0.8))
    O = ho.build_hierarchy(omodel(m), damping=(0.8, 0.8))
    hists, iters, xs = [], [], []
    for i in range(cfg.rhs.shape[0]):
        b = rf.ComplexField(cfg.rhs[i], m.h)
        x, rep = rk.solve_helmholtz(m, b, H, tol=1e-6, max_iter=2000, restart=10)
        xo, ro = ho.solve_vcycle(omodel(m), cfg.rhs[i], O, 1e-6, 2000, 10)
        assert ro.iterations == rep.iterations, (ro.iterations, rep.iterations)
        assert max(abs(a - c) / c for a, c in zip(ro.history, rep.relative_residual_history)) < 1e-8
        assert relerr(xo, x.data) < 1e-9
        hists.append(np.array(rep.relative_residual_history))
        iters.append(rep.iterations)
        xs.append(x.data.astype(np.complex64))
        print(f"  C1 rhs {i}: {rep.iterations} iterations, final {rep.relative_residual_history[-1]:.3e}")
    L = max(len(h) for h in hists)
    H2 = np.full((len(hists), L), np.nan)
    for i, h in enumerate(hists):
        H2[i, : len(h)] = h
    save("solve_c1_vcycle.npz", kappa_sq=m.kappa_sq, rhs=cfg.rhs, hist=H2, iterations=np.array(iters),
         x=np.stack(xs))


def fx_solve_small():
    """33x33 and 65x65 solves, default Chebyshev damping, tol 1e-7 (test_krylov.py:148-154 style)."""
    rng = np.random.default_rng(15)
    out = {}
    for n, lw in [(33, 4), (65, 8)]:
        m = rf.slowness_model(rng.uniform(0.25, 1.0, (n, n)), layer_width=lw)
        b = noise(rng, (n, n))
        x, rep = rk.solve_helmholtz(m, rf.ComplexField(b, m.h), tol=1e-7, max_iter=250)
        xo, ro = ho.solve_vcycle(omodel(m), b, None, 1e-7, 250, 10)
        assert ro.iterations == rep.iterations
        assert relerr(xo, x.data) < 1e-9
        out.update({f"kappa_sq_{n}": m.kappa_sq, f"b_{n}": b, f"hist_{n}": np.array(rep.relative_residual_history),
                    f"x_{n}": x.data, f"lw_{n}": lw})
        print(f"  {n}^2 solve: {rep.iterations} iterations")
    save("solve_small.npz", **out)


def fx_cnn_primitives():
    rng = np.random.default_rng(16)
    out = {}
    with ad.no_grad():
        x = rng.standard_normal((2, 3, 8, 10)).astype(np.float32)
        w = rng.standard_normal((4, 3, 3, 3)).astype(np.float32)
        bias = rng.standard_normal(4).astype(np.float32)
        y1 = ad.conv2d(ad.Tensor(x), ad.Tensor(w), ad.Tensor(bias)).data
        y2 = ad.conv2d(ad.Tensor(x), ad.Tensor(w), ad.Tensor(bias), stride=2).data
        assert relerr(no.conv2d(x, w, bias), y1) < 1e-6 and relerr(no.conv2d(x, w, bias, 2), y2) < 1e-6
        wt = rng.standard_normal((3, 5, 3, 3)).astype(np.float32)
        yt = ad.conv_transpose2d(ad.Tensor(x), ad.Tensor(wt), ad.Tensor(bias[:1].repeat(5))).data
        assert relerr(no.conv_transpose2d(x, wt, bias[:1].repeat(5)), yt) < 1e-6
        g, be = rng.uniform(0.5, 1.5, 3).astype(np.float32), rng.uniform(-1, 1, 3).astype(np.float32)
        mu, var = rng.uniform(-1, 1, 3).astype(np.float32), rng.uniform(0.5, 2, 3).astype(np.float32)
        ybn = ad.batchnorm2d(ad.Tensor(x), ad.Tensor(g), ad.Tensor(be), mu.copy(), var.copy(), False).data
        assert relerr(no.batchnorm_infer(x, g, be, mu, var), ybn) < 1e-6
        ysp = ad.softplus(ad.Tensor(x * 10)).data
        assert relerr(no.softplus(x * 10), ysp) < 1e-7
        z = ad.pack_complex(ad.Tensor(x[:, :2])).data
        assert np.array_equal(no.pack_complex(x[:, :2]), z)
        out.update(x=x, w=w, bias=bias, conv_s1=y1, conv_s2=y2, wt=wt, tconv=yt, bn_g=g, bn_b=be, bn_mu=mu,
                   bn_var=var, bn=ybn, softplus=ysp, packed=z)
        for hh, ww in [(8, 8), (16, 16), (8, 16)]:
            k = rg.laplacian_plus_i_kernel(2) + (0.1 * noise(rng, (2, 3, 3))).astype(np.complex64)
            S = rg.green_function(k, (hh, ww))
            So = no.green_function(k, (hh, ww))
            assert S.dtype == So.dtype == np.complex128 and relerr(So, S) < 1e-6, relerr(So, S)
            xi = noise(rng, (3, 2, hh, ww)).astype(np.complex64)
            yi = rg.implicit_apply(xi, S.astype(np.complex64))
            assert relerr(no.implicit_apply(xi, S.astype(np.complex64)), yi) < 1e-6
            tag = f"{hh}x{ww}"
            out.update({f"gk_{tag}": k, f"spec_{tag}": S, f"ix_{tag}": xi, f"iy_{tag}": yi})
        kl = rg.laplacian_plus_i_kernel(1)
        G = rg.green_function(kl, (16, 16))
        resp = np.fft.ifft2(G[0])
        out["green_ratio"] = np.abs(resp[16, 16]) / np.abs(resp[0, 0])
    save("cnn_primitives.npz", **out)


# ---------------------------------------- ARCH.md network on reference primitives


def ref_cbs(p, pre, x, stride=1, transposed=False, out_hw=None):
    T = ad.Tensor
    if transposed:
        y = ad.conv_transpose2d(x, T(p[pre + ".w"]), T(p[pre + ".b"]), stride=2, pad=1, out_hw=out_hw)
    else:
        y = ad.conv2d(x, T(p[pre + ".w"]), T(p[pre + ".b"]), stride=stride)
    y = ad.batchnorm2d(y, T(p[pre + ".bn.gamma"]), T(p[pre + ".bn.beta"]), p[pre + ".bn.mean"].copy(),
                       p[pre + ".bn.var"].copy(), training=False)
    return ad.softplus(y)


def ref_res(p, pre, x):
    return ad.add(x, ad.conv2d(ref_cbs(p, pre + ".a", x), ad.Tensor(p[pre + ".b.w"]), ad.Tensor(p[pre + ".b.b"])))


def ref_encode(p, L, media):
    e = ref_res(p, "enc.res0", ref_cbs(p, "enc.stem", ad.Tensor(media)))
    out = [e]
    for lv in range(1, L):
        e = ref_res(p, f"enc.res{lv}", ref_cbs(p, f"enc.down{lv}", e, stride=2))
        out.append(e)
    return out


class RefNet:
    """ARCH.md network built only from reference primitives (under no_grad)."""

    def __init__(self, params, levels):
        self.p, self.L = params, levels
        self.implicit = rg.ImplicitKernel(params["sol.implicit.w"].shape[0], weights=params["sol.implicit.w"])

    def solve(self, r2, feats):
        p, L = self.p, self.L
        x = ad.add(ref_cbs(p, "sol.stem", ad.Tensor(r2)), feats[0])
        x = ref_res(p, "sol.res0", x)
        skips = [x]
        for lv in range(1, L):
            x = ad.add(ref_cbs(p, f"sol.down{lv}", x, stride=2), feats[lv])
            x = ref_res(p, f"sol.res{lv}", x)
            skips.append(x)
        z = ad.pack_complex(x)
        spec = self.implicit.spectrum(z.data.shape[-2:])
        # ARCH.md: the cached spectrum is applied in complex64 (GPU precision class)
        z = rg.implicit_apply(z, ad.Tensor(spec.data.astype(np.complex64) if hasattr(spec, "data") else
                                           np.asarray(spec).astype(np.complex64)))
        x = ad.unpack_complex(z)
        for lv in range(L - 1, 0, -1):
            s = skips[lv - 1]
            x = ad.add(ref_cbs(p, f"sol.up{lv}", x, transposed=True, out_hw=s.data.shape[-2:]), s)
            x = ref_res(p, f"sol.ures{lv - 1}", x)
        return ad.conv2d(x, ad.Tensor(p["sol.head.w"]), ad.Tensor(p["sol.head.b"])).data


def install_ref_network():
    """Inject helmsolve.network = ARCH.md on reference primitives (krylov.py:201)."""
    mod = types.ModuleType("helmsolve.network")

    def precompute_encodings(net, model):
        with ad.no_grad():
            return ref_encode(net.p, net.L, no.media_planes(model.kappa_sq, model.gamma, net.L))

    def preconditioner_estimate(net, enc, r):
        (ix, iy), _ = no.cnn_dims(r.shape, net.L)
        rc = np.asarray(r)[:ix, :iy]
        r2 = np.stack([rc.real, rc.imag])[None].astype(np.float32)
        with ad.no_grad():
            out = net.solve(r2, enc)
        scale = np.float32(net.h * net.h / 64.0)
        u0 = np.zeros(r.shape, dtype=np.complex64)
        u0[:ix, :iy] = scale * out[0, 0] + 1j * (scale * out[0, 1])
        return u0

    mod.precompute_encodings = precompute_encodings
    mod.preconditioner_estimate = preconditioner_estimate
    sys.modules["helmsolve.network"] = mod
    import helmsolve

    helmsolve.network = mod


def fx_network():
    """Network forward at I = 32 (33^2 grid): reference-primitive composition vs oracle."""
    out = {}
    rng = np.random.default_rng(17)
    for L, ch, n in [(3, (16, 32, 64), 33), (2, (8, 16), 17)]:
        params = netparams.randomise_batchnorm(netparams.init_params(ch, seed=5), seed=6)
        m = rf.slowness_model(problems.smooth_random_kappa_sq((n, n), 3.0, 1), layer_width=max(2, n // 8))
        media = no.media_planes(m.kappa_sq, m.gamma, L)
        net = RefNet(params, L)
        with ad.no_grad():
            feats_ref = ref_encode(params, L, media)
        feats_or = no.encode(params, L, media)
        for a, b in zip(feats_or, feats_ref):
            assert relerr(a, b.data) < 2e-6, relerr(a, b.data)
        (ix, iy), coarse = no.cnn_dims((n, n), L)
        r = noise(rng, (n, n))
        r /= np.linalg.norm(r)
        r2 = np.stack([r[:ix, :iy].real, r[:ix, :iy].imag])[None].astype(np.float32)
        with ad.no_grad():
            y_ref = net.solve(r2, feats_ref)
        spec = no.spectrum_c64(params, L, (n, n))
        y_or = no.solve(params, L, r2, feats_or, spec)
        e = relerr(y_or, y_ref)
        assert e < 2e-5, e
        tag = f"L{L}"
        out.update({f"kappa_sq_{tag}": m.kappa_sq, f"gamma_{tag}": m.gamma, f"r_{tag}": r, f"y_{tag}": y_ref,
                    f"spec_{tag}": spec})
        for i, f in enumerate(feats_ref):
            out[f"enc{i}_{tag}"] = f.data
        print(f"  network L={L}: oracle vs reference-primitive composition {e:.2e}")
    save("network.npz", **out)


def fx_learned_c1(n_rhs):
    """Reference solve_with_learned_preconditioner (unmodified) at C1 with the ARCH.md net injected."""
    install_ref_network()
    cfg = problems.make_config("C1")
    m = cfg.models[0]
    L, ch = 3, (16, 32, 64)
    params = netparams.init_params(ch, seed=0)
    net = RefNet(params, L)
    net.h = m.h
    H = rm.build_hierarchy(m, jacobi_damping=(0.8, 0.8))
    enc = sys.modules["helmsolve.network"].precompute_encodings(net, m)
    O = ho.build_hierarchy(omodel(m), damping=(0.8, 0.8))
    feats = no.encode(params, L, no.media_planes(m.kappa_sq, m.gamma, L))
    spec = no.spectrum_c64(params, L, m.shape)
    hists, iters, xs = [], [], []
    for i in range(n_rhs):
        b = rf.ComplexField(cfg.rhs[i], m.h)
        x, rep = rk.solve_with_learned_preconditioner(m, b, net, enc, tol=1e-6, max_iter=400, restart=10,
                                                      hierarchy=H)
        xo, ro = ho.solve_learned(omodel(m), cfg.rhs[i],
                                  lambda r: no.preconditioner_estimate(params, L, feats, spec, r, m.h),
                                  1e-6, 400, 10, 3, O)
        dev = max(abs(a - c) / c for a, c in zip(ro.history, rep.relative_residual_history))
        print(f"  learned C1 rhs {i}: ref {rep.iterations} it, oracle {ro.iterations} it, hist dev {dev:.2e}")
        assert abs(ro.iterations - rep.iterations) <= 1 and dev < 1e-5
        hists.append(np.array(rep.relative_residual_history))
        iters.append(rep.iterations)
        xs.append(x.data.astype(np.complex64))
    Lh = max(len(h) for h in hists)
    H2 = np.full((len(hists), Lh), np.nan)
    for i, h in enumerate(hists):
        H2[i, : len(h)] = h
    save("learned_c1.npz", hist=H2, iterations=np.array(iters), x=np.stack(xs), rhs=cfg.rhs[:n_rhs],
         kappa_sq=m.kappa_sq)


# ---------------------------------------- training step on reference autodiff


def fx_train():
    """Loss + every parameter gradient of one training step, from the reference's autodiff.

    ARCH.md network composed from reference primitives with gradients ON, training-mode batch
    norm (running buffers updated in place, autodiff.py:570-580), the Green spectrum built from
    the trainable kernel Tensor (green.py:55-82), float64 throughout; loss = SPEC mse_loss of
    u0 = (h^2/64) net(r) (zero-padded) against e.  Pins oracle/train_oracle.py.
    """
    from oracle import train_oracle as to

    out = {}
    rng = np.random.default_rng(29)
    for tag, L, ch, n, B in [("a", 2, (4, 8), 17, 3), ("b", 3, (4, 8, 8), 33, 2)]:
        params = to.as_float64(netparams.randomise_batchnorm(netparams.init_params(ch, seed=7), seed=8))
        models = [rf.slowness_model(problems.smooth_random_kappa_sq((n, n), 3.0, s), layer_width=max(2, n // 8))
                  for s in (1, 2)]
        owner = np.arange(B) % 2
        media = np.concatenate([no.media_planes(models[o].kappa_sq, models[o].gamma, L) for o in owner]
                               ).astype(np.float64)
        r = noise(rng, (B, n, n))
        e = noise(rng, (B, n, n)) * 0.01
        h = 1.0 / (n - 1)
        T = ad.Tensor
        tp = {k: T(v.copy(), requires_grad=True) for k, v in params.items() if to.trainable(k)}
        stats = {k: v.copy() for k, v in params.items() if not to.trainable(k)}

        def cbs(pre, x, stride=1, transposed=False, out_hw=None):
            if transposed:
                y = ad.conv_transpose2d(x, tp[pre + ".w"], tp[pre + ".b"], stride=2, pad=1, out_hw=out_hw)
            else:
                y = ad.conv2d(x, tp[pre + ".w"], tp[pre + ".b"], stride=stride)
            y = ad.batchnorm2d(y, tp[pre + ".bn.gamma"], tp[pre + ".bn.beta"], stats[pre + ".bn.mean"],
                               stats[pre + ".bn.var"], training=True)
            return ad.softplus(y)

        def res(pre, x):
            return ad.add(x, ad.conv2d(cbs(pre + ".a", x), tp[pre + ".b.w"], tp[pre + ".b.b"]))

        e0 = res("enc.res0", cbs("enc.stem", T(media)))
        feats = [e0]
        for lv in range(1, L):
            e0 = res(f"enc.res{lv}", cbs(f"enc.down{lv}", e0, stride=2))
            feats.append(e0)
        (ix, iy), coarse = no.cnn_dims((n, n), L)
        r2 = np.stack([r[:, :ix, :iy].real, r[:, :ix, :iy].imag], axis=1)
        x = res("sol.res0", ad.add(cbs("sol.stem", T(r2)), feats[0]))
        skips = [x]
        for lv in range(1, L):
            x = res(f"sol.res{lv}", ad.add(cbs(f"sol.down{lv}", x, stride=2), feats[lv]))
            skips.append(x)
        spec = rg.green_function(tp["sol.implicit.w"], coarse)
        x = ad.unpack_complex(rg.implicit_apply(ad.pack_complex(x), spec))
        for lv in range(L - 1, 0, -1):
            s = skips[lv - 1]
            x = res(f"sol.ures{lv - 1}", ad.add(cbs(f"sol.up{lv}", x, transposed=True, out_hw=s.data.shape[-2:]), s))
        y = ad.conv2d(x, tp["sol.head.w"], tp["sol.head.b"])
        sc = h * h / 64.0
        tgt = np.stack([e[:, :ix, :iy].real, e[:, :ix, :iy].imag], axis=1)
        d = ad.sub(ad.mul(y, sc), T(tgt))
        pad = float(np.sum(np.abs(e) ** 2) - np.sum(np.abs(e[:, :ix, :iy]) ** 2))
        loss = ad.add(ad.mul(ad.tsum(ad.mul(d, d)), 1.0 / B), pad / B)
        loss.backward()
        ref_grads = {k: t.grad for k, t in tp.items()}
        # oracle restatement on the same inputs
        po = {k: v.copy() for k, v in params.items()}
        lo, go, _ = to.loss_and_grads(po, L, media, r, e, h)
        el = abs(lo - float(loss.data)) / abs(float(loss.data))
        assert el < 1e-12, el
        worst = 0.0
        for k, g in ref_grads.items():
            er = relerr(go[k], g) if np.linalg.norm(g) > 1e-12 else float(np.abs(go[k] - g).max())
            worst = max(worst, er)
            assert er < 1e-9, (k, er)
        for k in stats:
            assert relerr(po[k], stats[k]) < 1e-12, k
        print(f"  train {tag}: loss {float(loss.data):.6e}, oracle grads within {worst:.1e}")
        out.update({f"media_{tag}": media, f"r_{tag}": r, f"e_{tag}": e, f"h_{tag}": h, f"loss_{tag}": float(loss.data),
                    f"levels_{tag}": L, f"channels_{tag}": np.array(ch)})
        for k, v in params.items():
            out[f"p_{tag}_{k}"] = v
        for k, g in ref_grads.items():
            out[f"g_{tag}_{k}"] = g
        for k, v in stats.items():
            out[f"s_{tag}_{k}"] = v
    save("train.npz", **out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    ap.add_argument("--learned-rhs", type=int, default=2)
    a = ap.parse_args()
    todo = {
        "fields": fx_fields, "transfers": fx_transfers, "hierarchy": fx_hierarchy, "vcycle": fx_vcycle,
        "solve_small": fx_solve_small, "solve_c1": fx_solve_c1, "cnn": fx_cnn_primitives, "network": fx_network,
        "learned": lambda: fx_learned_c1(a.learned_rhs), "train": fx_train,
    }
    for name, fn in todo.items():
        if a.only and name not in a.only.split(","):
            continue
        print(f"[{name}]")
        fn()


if __name__ == "__main__":
    main()
