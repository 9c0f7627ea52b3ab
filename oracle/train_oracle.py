"""CPU restatement of one network training step -- TEST INFRASTRUCTURE ONLY.

The reference ships no trainer; its contract is SPEC.md ``[MODULE] trainer`` (reference
SPEC.md:454-507): MSE training (paper Eq. 4.10) of the encoder and solver jointly, Adam,
training-mode batch norm.  The gradients follow the reference's own autodiff
(``autodiff.py``), restated here by hand in float64 numpy:

* conv2d backward            -- autodiff.py:472-507 (``_corr_t`` :442-469, ``_corr_wgrad`` :424-439)
* conv_transpose2d backward  -- autodiff.py:510-544
* batchnorm2d (training)     -- autodiff.py:547-592: batch statistics, unbiased running-var update,
                                momentum 0.1, backward ``inv (dxh - s1/m - xh s2/m)``
* softplus backward          -- autodiff.py:243-252 (logistic ``0.5 (1 + tanh(x/2))``)
* pack/unpack_complex        -- autodiff.py:343-372
* implicit_apply backward    -- green.py:85-107 through fft2/ifft2/mul (autodiff.py:375-399, 188-196)
* green_function backward    -- green.py:55-82 (mul/div/conj/add chain, autodiff.py:166-216)

and the complex-gradient convention of autodiff.py:3-12 (grad = dL/dRe + i dL/dIm).

The loss is the SPEC ``mse_loss`` on the preconditioner's estimate: with the network output
``out`` and ``u0 = (h^2/64)(out_0 + i out_1)`` zero-padded to the node grid (ARCH.md),
``loss = (1/B) sum_b ||u0_b - e_b||^2`` (complex norm).  Adam is PyTorch's default
(betas 0.9/0.999, eps 1e-8, bias-corrected, complex parameters per real component).

Pinning: ``oracle/make_golden.py fx_train`` builds the same network from the reference's
autodiff/green primitives with gradients on, runs the loss backward and stores loss, every
parameter gradient and the updated running statistics in ``tests/golden/train.npz``;
``tests/test_train.py`` checks this module against that fixture.
Only ``tests/`` and ``bench.py``'s CPU legs may import this module.
"""
from __future__ import annotations

import numpy as np

from oracle import network_oracle as no

BN_EPS = 1e-5
BN_MOMENTUM = 0.1
SPECTRUM_EPS = 1e-5


# ------------------------------------------------------------------ conv primitives


def conv_bwd(x, w, g, stride):
    """Gradients of conv2d (3x3, pad 1) for x, w, bias (autodiff.py:501-507)."""
    n, ci, hh, ww = x.shape
    _, _, ho, wo = g.shape
    xp = np.zeros((n, ci, hh + 2, ww + 2), dtype=x.dtype)
    xp[:, :, 1:-1, 1:-1] = x
    dxp = np.zeros_like(xp)
    dw = np.zeros_like(w)
    for u in range(3):
        for v in range(3):
            sl = (slice(None), slice(None), slice(u, u + stride * (ho - 1) + 1, stride),
                  slice(v, v + stride * (wo - 1) + 1, stride))
            dw[:, :, u, v] = np.einsum("nohw,nchw->oc", g, xp[sl], optimize=True)
            dxp[sl] += np.einsum("nohw,oc->nchw", g, w[:, :, u, v], optimize=True)
    return dxp[:, :, 1:-1, 1:-1], dw, g.sum(axis=(0, 2, 3))


def tconv_bwd(x, w, g, stride=2):
    """Gradients of conv_transpose2d (weight (ci, co, 3, 3), pad 1) (autodiff.py:535-541)."""
    n, ci, hh, ww = x.shape
    _, co, oh, ow = g.shape
    fh, fw = stride * (hh - 1) + 3, stride * (ww - 1) + 3
    gf = np.zeros((n, co, max(fh, oh + 1), max(fw, ow + 1)), dtype=g.dtype)
    gf[:, :, 1 : 1 + oh, 1 : 1 + ow] = g
    dx = np.zeros_like(x)
    dw = np.zeros_like(w)
    for u in range(3):
        for v in range(3):
            gs = gf[:, :, u : u + stride * (hh - 1) + 1 : stride, v : v + stride * (ww - 1) + 1 : stride]
            dx += np.einsum("nohw,co->nchw", gs, w[:, :, u, v], optimize=True)
            dw[:, :, u, v] = np.einsum("nchw,nohw->co", x, gs, optimize=True)
    return dx, dw, g.sum(axis=(0, 2, 3))


# ------------------------------------------------------------------ batch norm + softplus


def bn_train_fwd(z, gamma, beta, rmean, rvar):
    """Training batch norm; returns (a, cache) and updates rmean / rvar in place (autodiff.py:570-580)."""
    axes = (0, 2, 3)
    m = z.shape[0] * z.shape[2] * z.shape[3]
    mean = z.mean(axis=axes)
    var = z.var(axis=axes)
    inv = 1.0 / np.sqrt(var + BN_EPS)
    xh = (z - mean.reshape(1, -1, 1, 1)) * inv.reshape(1, -1, 1, 1)
    rmean *= 1.0 - BN_MOMENTUM
    rmean += BN_MOMENTUM * mean
    rvar *= 1.0 - BN_MOMENTUM
    rvar += BN_MOMENTUM * var * (m / max(m - 1, 1))
    a = gamma.reshape(1, -1, 1, 1) * xh + beta.reshape(1, -1, 1, 1)
    return a, (xh, inv, m, gamma)


def bn_train_bwd(g, cache):
    xh, inv, m, gamma = cache
    axes = (0, 2, 3)
    dgamma = (g * xh).sum(axis=axes)
    dbeta = g.sum(axis=axes)
    dxh = g * gamma.reshape(1, -1, 1, 1)
    s1 = dxh.sum(axis=axes).reshape(1, -1, 1, 1)
    s2 = (dxh * xh).sum(axis=axes).reshape(1, -1, 1, 1)
    return inv.reshape(1, -1, 1, 1) * (dxh - s1 / m - xh * s2 / m), dgamma, dbeta


def softplus_grad(a):
    return 0.5 * (1.0 + np.tanh(0.5 * a))


# ------------------------------------------------------------------ Green spectrum + implicit layer


def _corner_rc(bh, bw):
    return (bh - 1, 0, 1), (bw - 1, 0, 1)


def green_fwd(k, coarse):
    """green.py:55-82 in complex128; returns (spectrum, cache)."""
    hh, ww = coarse
    gh, gw = 2 * hh, 2 * ww
    bh, bw = 3 * gh, 3 * gw
    S = np.fft.fft2(no.kernel_corners(k.astype(np.complex128), (bh, bw)), axes=(-2, -1))
    D = (S * np.conj(S)).real + SPECTRUM_EPS
    delta = np.zeros((bh, bw))
    delta[bh // 2, bw // 2] = 1.0
    dhat = np.fft.fft2(delta)
    R = np.fft.ifft2(np.conj(S) / D * dhat, axes=(-2, -1))
    oy, ox = bh // 2 - gh // 2, bw // 2 - gw // 2
    T = R[..., oy : oy + gh, ox : ox + gw]
    G = np.fft.fft2(np.fft.ifftshift(T, axes=(-2, -1)), axes=(-2, -1))
    return G, (S, D, dhat, (gh, gw, bh, bw, oy, ox))


def green_bwd(gG, cache):
    """Gradient of the kernel weights from the spectrum gradient (convention autodiff.py:3-12)."""
    S, D, dhat, (gh, gw, bh, bw, oy, ox) = cache
    gU = gh * gw * np.fft.ifft2(gG, axes=(-2, -1))  # fft2 backward: N ifft
    gT = np.fft.fftshift(gU, axes=(-2, -1))  # ifftshift backward
    gR = np.zeros(S.shape, dtype=np.complex128)
    gR[..., oy : oy + gh, ox : ox + gw] = gT  # crop backward
    gQ = np.fft.fft2(gR, axes=(-2, -1)) / (bh * bw)  # ifft2 backward: fft / N
    gP = gQ * np.conj(dhat)
    # P = conj(S) / D, D = S conj(S) + eps (real): Wirtinger chain through conj/mul/div
    gS = np.conj(gP) * SPECTRUM_EPS / D**2 - gP * S * S / D**2
    gkp = bh * bw * np.fft.ifft2(gS, axes=(-2, -1))
    rows, cols = _corner_rc(bh, bw)
    gk = np.empty(gkp.shape[:-2] + (3, 3), dtype=np.complex128)
    for a in range(3):
        for b in range(3):
            gk[..., a, b] = gkp[..., rows[a], cols[b]]
    return gk


def implicit_fwd(z, G):
    n, c, hh, ww = z.shape
    sh, sw = G.shape[-2:]
    zp = np.zeros((n, c, sh, sw), dtype=np.complex128)
    zp[..., :hh, :ww] = z
    X = np.fft.fft2(zp, axes=(-2, -1))
    y = np.fft.ifft2(X * G[None], axes=(-2, -1))[..., :hh, :ww]
    return y, X


def implicit_bwd(gy, X, G):
    """(dz, dG): dz = implicit_apply(gy, conj G); dG = sum_b conj(X) fft2(pad gy) / N."""
    n, c, hh, ww = gy.shape
    sh, sw = G.shape[-2:]
    gp = np.zeros((n, c, sh, sw), dtype=np.complex128)
    gp[..., :hh, :ww] = gy
    Gf = np.fft.fft2(gp, axes=(-2, -1)) / (sh * sw)
    dG = (np.conj(X) * Gf).sum(axis=0)
    dz = (sh * sw) * np.fft.ifft2(Gf * np.conj(G)[None], axes=(-2, -1))[..., :hh, :ww]
    return dz, dG


# ------------------------------------------------------------------ network forward / backward


class Tape:
    def __init__(self, params, levels):
        self.p = params
        self.L = levels
        self.grads = {k: np.zeros_like(v) for k, v in params.items()}
        self.caches = {}

    # conv (+bias) -> training BN -> softplus
    def cbs(self, pre, x, stride=1, transposed=False, out_hw=None):
        p = self.p
        if transposed:
            z = no.conv_transpose2d(x, p[pre + ".w"], p[pre + ".b"], 2, out_hw)
        else:
            z = no.conv2d(x, p[pre + ".w"], p[pre + ".b"], stride)
        a, bnc = bn_train_fwd(z, p[pre + ".bn.gamma"], p[pre + ".bn.beta"], p[pre + ".bn.mean"], p[pre + ".bn.var"])
        self.caches[pre] = (x, a, bnc, stride, transposed)
        return no.softplus(a)

    def cbs_bwd(self, pre, gy):
        x, a, bnc, stride, transposed = self.caches[pre]
        ga = gy * softplus_grad(a)
        gz, dgamma, dbeta = bn_train_bwd(ga, bnc)
        self.grads[pre + ".bn.gamma"] += dgamma
        self.grads[pre + ".bn.beta"] += dbeta
        if transposed:
            dx, dw, db = tconv_bwd(x, self.p[pre + ".w"], gz)
        else:
            dx, dw, db = conv_bwd(x, self.p[pre + ".w"], gz, stride)
        self.grads[pre + ".w"] += dw
        self.grads[pre + ".b"] += db
        return dx

    def res(self, pre, x):
        t = self.cbs(pre + ".a", x)
        self.caches[pre + ".b"] = t
        return x + no.conv2d(t, self.p[pre + ".b.w"], self.p[pre + ".b.b"])

    def res_bwd(self, pre, gy):
        t = self.caches[pre + ".b"]
        dt, dw, db = conv_bwd(t, self.p[pre + ".b.w"], gy, 1)
        self.grads[pre + ".b.w"] += dw
        self.grads[pre + ".b.b"] += db
        return gy + self.cbs_bwd(pre + ".a", dt)

    def forward(self, media, r2, coarse):
        p, L = self.p, self.L
        e = self.res("enc.res0", self.cbs("enc.stem", media))
        feats = [e]
        for lv in range(1, L):
            e = self.res(f"enc.res{lv}", self.cbs(f"enc.down{lv}", e, stride=2))
            feats.append(e)
        x = self.res("sol.res0", self.cbs("sol.stem", r2) + feats[0])
        skips = [x]
        for lv in range(1, L):
            x = self.res(f"sol.res{lv}", self.cbs(f"sol.down{lv}", x, stride=2) + feats[lv])
            skips.append(x)
        G, gcache = green_fwd(p["sol.implicit.w"], coarse)
        y, X = implicit_fwd(no.pack_complex(x), G)
        self.caches["implicit"] = (X, G, gcache)
        x = no.unpack_complex(y)
        for lv in range(L - 1, 0, -1):
            s = skips[lv - 1]
            x = self.res(f"sol.ures{lv - 1}", self.cbs(f"sol.up{lv}", x, transposed=True, out_hw=s.shape[-2:]) + s)
        self.caches["head"] = x
        return no.conv2d(x, p["sol.head.w"], p["sol.head.b"])

    def backward(self, gout):
        L = self.L
        x = self.caches["head"]
        gx, dw, db = conv_bwd(x, self.p["sol.head.w"], gout, 1)
        self.grads["sol.head.w"] += dw
        self.grads["sol.head.b"] += db
        gskip = [None] * L
        for lv in range(1, L):
            gs = self.res_bwd(f"sol.ures{lv - 1}", gx)
            gskip[lv - 1] = gs.copy()
            gx = self.cbs_bwd(f"sol.up{lv}", gs)
        X, G, gcache = self.caches["implicit"]
        gz, dG = implicit_bwd(no.pack_complex(gx), X, G)
        self.grads["sol.implicit.w"] += green_bwd(dG, gcache)
        gx = no.unpack_complex(gz)
        gfeat = [None] * L
        for lv in range(L - 1, 0, -1):
            g = self.res_bwd(f"sol.res{lv}", gx)
            gfeat[lv] = g
            gx = self.cbs_bwd(f"sol.down{lv}", g) + gskip[lv - 1]
        g = self.res_bwd("sol.res0", gx)
        gfeat[0] = g
        self.cbs_bwd("sol.stem", g)
        ge = gfeat[L - 1]
        for lv in range(L - 1, 0, -1):
            g = self.res_bwd(f"enc.res{lv}", ge)
            ge = self.cbs_bwd(f"enc.down{lv}", g) + gfeat[lv - 1]
        self.cbs_bwd("enc.stem", self.res_bwd("enc.res0", ge))


# ------------------------------------------------------------------ loss, step, Adam


def as_float64(params):
    return {k: (v.astype(np.complex128) if np.iscomplexobj(v) else v.astype(np.float64)) for k, v in params.items()}


def loss_and_grads(params, levels, media, r, e, h):
    """Forward (training BN), MSE loss, backward.

    media (B, 2, Ix, Iy) per sample, r and e (B, nx, ny) complex.  ``params`` running statistics
    are updated in place.  Returns (loss, grads dict, network output).
    """
    B, nx, ny = r.shape
    (ix, iy), coarse = no.cnn_dims((nx, ny), levels)
    r2 = np.stack([r[:, :ix, :iy].real, r[:, :ix, :iy].imag], axis=1)
    tape = Tape(params, levels)
    out = tape.forward(np.asarray(media, dtype=np.float64), r2, coarse)
    s = h * h / 64.0
    pred = np.zeros((B, nx, ny), dtype=np.complex128)
    pred[:, :ix, :iy] = s * out[:, 0] + 1j * (s * out[:, 1])
    d = pred - e
    loss = float(np.sum(d.real**2 + d.imag**2) / B)
    gout = np.stack([d[:, :ix, :iy].real, d[:, :ix, :iy].imag], axis=1) * (2.0 * s / B)
    tape.backward(gout)
    return loss, tape.grads, out


def trainable(name):
    return not (name.endswith(".bn.mean") or name.endswith(".bn.var"))


class Adam:
    """torch.optim.Adam defaults; complex parameters per real component."""

    def __init__(self, params, lr=1e-3, betas=(0.9, 0.999), eps=1e-8):
        self.lr, self.b1, self.b2, self.eps = lr, betas[0], betas[1], eps
        self.t = 0
        self.m = {k: np.zeros_like(v) for k, v in params.items() if trainable(k)}
        self.v = {k: np.zeros(v.shape + ((2,) if np.iscomplexobj(v) else ()), dtype=np.float64)
                  for k, v in params.items() if trainable(k)}

    def step(self, params, grads):
        self.t += 1
        c1 = 1.0 - self.b1**self.t
        c2 = 1.0 - self.b2**self.t
        for k in self.m:
            g = grads[k]
            self.m[k] = self.b1 * self.m[k] + (1.0 - self.b1) * g
            gr = np.stack([g.real, g.imag], axis=-1) if np.iscomplexobj(g) else g
            self.v[k] = self.b2 * self.v[k] + (1.0 - self.b2) * gr * gr
            den = np.sqrt(self.v[k] / c2) + self.eps
            if np.iscomplexobj(g):
                mr = self.m[k]
                params[k] = params[k] - self.lr * ((mr.real / c1) / den[..., 0] + 1j * ((mr.imag / c1) / den[..., 1]))
            else:
                params[k] = params[k] - self.lr * (self.m[k] / c1) / den
        return params


def train_step(params, levels, media, r, e, h, opt: Adam):
    loss, grads, _ = loss_and_grads(params, levels, media, r, e, h)
    opt.step(params, grads)
    return loss, grads
