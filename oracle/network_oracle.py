"""CPU ORACLE (test infrastructure only) for the encoder-solver CNN and the
implicit (Green's-function) layer.

The reference ships the CNN's primitives but not the network itself
(``krylov.py:201`` imports a ``helmsolve.network`` that does not exist; SURVEY.md
§0.3).  This module restates, in numpy float32/complex64, the forward semantics
of the reference primitives the network is built from, and composes them into
the architecture pinned in ``ARCH.md``:

* ``conv2d``            — ``autodiff.py:472-507`` (``_corr`` ``:407-421``), pad 1
* ``conv_transpose2d``  — ``autodiff.py:510-541`` (``_corr_t`` ``:442-469``)
* ``batchnorm_infer``   — ``autodiff.py:595-607`` (inference branch)
* ``softplus``          — ``autodiff.py:243-252``
* ``pack/unpack``       — ``autodiff.py:343-372``
* ``green_function``    — ``green.py:55-82`` (dtype flow of numpy 2 kept: c128 out)
* ``implicit_apply``    — ``green.py:85-107``

Pinning: ``oracle/make_golden.py`` runs the same inputs through the reference
primitives (and through the reference's own ``solve_with_learned_preconditioner``
with this network injected as ``helmsolve.network``) and stores the results as
fixtures under ``tests/golden/``.  The composed network is a reconstruction, so
its end-to-end parity is pinned at the primitive level plus that protocol run.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this module.
"""
from __future__ import annotations

import numpy as np

SPECTRUM_EPS = 1e-5  # green.py:19
BN_EPS = 1e-5  # autodiff.py:555


# ----------------------------------------------------------- forward primitives


def conv2d(x, w, b=None, stride=1):
    """3x3 cross-correlation, zero pad 1 (autodiff.py:472-507)."""
    n, ci, hh, ww = x.shape
    co = w.shape[0]
    ho, wo = (hh - 1) // stride + 1, (ww - 1) // stride + 1
    xp = np.zeros((n, ci, hh + 2, ww + 2), dtype=x.dtype)
    xp[:, :, 1:-1, 1:-1] = x
    out = np.zeros((n, co, ho, wo), dtype=np.result_type(x.dtype, w.dtype))
    for u in range(3):
        for v in range(3):
            tap = xp[:, :, u : u + stride * (ho - 1) + 1 : stride, v : v + stride * (wo - 1) + 1 : stride]
            out += np.einsum("nchw,oc->nohw", tap, w[:, :, u, v], optimize=True)
    if b is not None:
        out += b.reshape(1, -1, 1, 1)
    return out


def conv_transpose2d(x, w, b=None, stride=2, out_hw=None):
    """Transposed 3x3 conv, pad 1, weight (c_in, c_out, 3, 3) (autodiff.py:510-541).

    Scatter form of the adjoint of the stride-2 correlation: input pixel i
    lands on output 2i - 1 + k for tap k.
    """
    n, ci, hh, ww = x.shape
    co = w.shape[1]
    oh, ow = out_hw or (stride * hh, stride * ww)
    fh, fw = stride * (hh - 1) + 3, stride * (ww - 1) + 3
    full = np.zeros((n, co, max(fh, oh + 1), max(fw, ow + 1)), dtype=np.result_type(x.dtype, w.dtype))
    for u in range(3):
        for v in range(3):
            full[:, :, u : u + stride * (hh - 1) + 1 : stride, v : v + stride * (ww - 1) + 1 : stride] += (
                np.einsum("nchw,co->nohw", x, w[:, :, u, v], optimize=True)
            )
    out = np.ascontiguousarray(full[:, :, 1 : 1 + oh, 1 : 1 + ow])
    if b is not None:
        out += b.reshape(1, -1, 1, 1)
    return out


def batchnorm_infer(x, gamma, beta, mean, var, eps=BN_EPS):
    """Inference batch norm with running statistics (autodiff.py:595-607)."""
    inv = 1.0 / np.sqrt(var + eps)
    scale = (gamma * inv).reshape(1, -1, 1, 1)
    return scale * (x - mean.reshape(1, -1, 1, 1)) + beta.reshape(1, -1, 1, 1)


def softplus(x):
    """log(1 + e^x), overflow safe (autodiff.py:243-252)."""
    return np.logaddexp(np.zeros((), dtype=x.dtype), x)


def pack_complex(x):
    """Real channels (2i, 2i+1) -> complex channel i (autodiff.py:343-357)."""
    ct = np.complex64 if x.dtype == np.float32 else np.complex128
    return (x[:, 0::2] + 1j * x[:, 1::2]).astype(ct)


def unpack_complex(z):
    """Complex channel i -> real channels (2i, 2i+1) (autodiff.py:360-372)."""
    rt = np.float32 if z.dtype == np.complex64 else np.float64
    out = np.empty((z.shape[0], 2 * z.shape[1]) + z.shape[2:], dtype=rt)
    out[:, 0::2] = z.real
    out[:, 1::2] = z.imag
    return out


# ---------------------------------------------------------------- green.py


def laplacian_plus_i(channels: int) -> np.ndarray:
    """green.py:24-30: the 5-point stencil with +i at the centre, per channel."""
    k = np.zeros((3, 3), dtype=np.complex64)
    k[1, 1] = 4 + 1j
    k[0, 1] = k[2, 1] = k[1, 0] = k[1, 2] = -1
    return np.repeat(k[None], channels, axis=0)


def kernel_corners(k, size):
    """autodiff.py:323-337: kernel centre to (0,0), neighbours wrapped."""
    hh, ww = size
    out = np.zeros(k.shape[:-2] + (hh, ww), dtype=k.dtype)
    for a, r in enumerate((hh - 1, 0, 1)):
        for b, c in enumerate((ww - 1, 0, 1)):
            out[..., r, c] = k[..., a, b]
    return out


def _as(dtype_src, arr):
    ct = np.complex64 if dtype_src in (np.float32, np.complex64) else np.complex128
    return arr.astype(ct)


def green_function(kernel, coarse_size, eps=SPECTRUM_EPS):
    """green.py:55-82 with the reference's numpy-2 dtype flow.

    S = fft2(corner-embedded kernel on 6h x 6w) is rounded to the kernel's
    complex dtype; ``S conj(S)`` is formed in that dtype and then promoted to
    complex128 by ``+ eps`` (a 0-d float64 array under NEP 50); the point-source
    spectrum is rounded to S's dtype; everything after that is complex128.
    """
    hh, ww = coarse_size
    k = np.asarray(kernel)
    gh, gw = 2 * hh, 2 * ww
    bh, bw = 3 * gh, 3 * gw
    S = _as(k.dtype, np.fft.fft2(kernel_corners(k, (bh, bw)), axes=(-2, -1)))
    denom = (S * np.conj(S)) + np.asarray(eps)  # promotes to complex128
    delta = np.zeros((bh, bw))
    delta[bh // 2, bw // 2] = 1.0
    dhat = np.fft.fft2(delta).astype(S.dtype)
    resp = (np.conj(S) / denom) * dhat
    resp = np.fft.ifft2(resp, axes=(-2, -1)).astype(np.complex128)
    oy, ox = bh // 2 - gh // 2, bw // 2 - gw // 2
    crop = resp[..., oy : oy + gh, ox : ox + gw]
    return np.fft.fft2(np.fft.ifftshift(crop, axes=(-2, -1)), axes=(-2, -1)).astype(np.complex128)


def implicit_apply(x, spectrum):
    """green.py:85-107: zero-pad to (2h, 2w) at the high end, FFT, multiply, IFFT, crop."""
    n, c, hh, ww = x.shape
    sh, sw = spectrum.shape[-2:]
    padded = np.zeros((n, c, sh, sw), dtype=x.dtype)
    padded[..., :hh, :ww] = x
    X = _as(x.dtype, np.fft.fft2(padded, axes=(-2, -1)))
    Y = X * spectrum[None]
    y = _as(Y.dtype, np.fft.ifft2(Y, axes=(-2, -1)))
    return np.ascontiguousarray(y[..., :hh, :ww])


# ------------------------------------------------------ the network (ARCH.md)


def _cbs(p, pre, x, stride=1, transposed=False, out_hw=None):
    """conv (+bias) -> batchnorm -> softplus (paper Fig. 1 caption)."""
    if transposed:
        y = conv_transpose2d(x, p[pre + ".w"], p[pre + ".b"], 2, out_hw)
    else:
        y = conv2d(x, p[pre + ".w"], p[pre + ".b"], stride)
    y = batchnorm_infer(y, p[pre + ".bn.gamma"], p[pre + ".bn.beta"], p[pre + ".bn.mean"], p[pre + ".bn.var"])
    return softplus(y)


def _res(p, pre, x):
    """x + K_b softplus(BN(K_a x)) (paper eq. 3.8, ResNet step)."""
    return x + conv2d(_cbs(p, pre + ".a", x), p[pre + ".b.w"], p[pre + ".b.b"])


def encode(p, levels: int, media):
    """Encoder: media (N, 2, Ix, Iy) float32 (kappa^2, gamma) -> list of L features."""
    e = _res(p, "enc.res0", _cbs(p, "enc.stem", media))
    feats = [e]
    for lv in range(1, levels):
        e = _res(p, f"enc.res{lv}", _cbs(p, f"enc.down{lv}", e, stride=2))
        feats.append(e)
    return feats


def solve(p, levels: int, r2, feats, spectrum):
    """Solver U-Net: r2 (N, 2, Ix, Iy) float32 -> (N, 2, Ix, Iy) float32."""
    x = _cbs(p, "sol.stem", r2) + feats[0]
    x = _res(p, "sol.res0", x)
    skips = [x]
    for lv in range(1, levels):
        x = _cbs(p, f"sol.down{lv}", x, stride=2) + feats[lv]
        x = _res(p, f"sol.res{lv}", x)
        skips.append(x)
    x = unpack_complex(implicit_apply(pack_complex(x), spectrum))
    for lv in range(levels - 1, 0, -1):
        skip = skips[lv - 1]
        x = _cbs(p, f"sol.up{lv}", x, transposed=True, out_hw=skip.shape[-2:]) + skip
        x = _res(p, f"sol.ures{lv - 1}", x)
    return conv2d(x, p["sol.head.w"], p["sol.head.b"])


def cnn_dims(shape, levels):
    """Network grid (Ix, Iy) = (nx-1, ny-1) and the coarsest size (ARCH.md)."""
    ix, iy = shape[0] - 1, shape[1] - 1
    f = 2 ** (levels - 1)
    return (ix, iy), (ix // f, iy // f)


def media_planes(kappa_sq, gamma, levels):
    (ix, iy), _ = cnn_dims(kappa_sq.shape, levels)
    return np.stack([kappa_sq[:ix, :iy], gamma[:ix, :iy]])[None].astype(np.float32)


def spectrum_c64(p, levels, shape):
    _, coarse = cnn_dims(shape, levels)
    return green_function(p["sol.implicit.w"], coarse).astype(np.complex64)


def preconditioner_estimate(p, levels, feats, spectrum, r, h):
    """u0 = (h^2/64) net(r[:Ix, :Iy]) zero-padded to r's shape (ARCH.md)."""
    (ix, iy), _ = cnn_dims(r.shape, levels)
    rc = np.asarray(r)[:ix, :iy]
    r2 = np.stack([rc.real, rc.imag])[None].astype(np.float32)
    out = solve(p, levels, r2, feats, spectrum)
    scale = np.float32(h * h / 64.0)
    u0 = np.zeros(r.shape, dtype=np.complex64)
    u0[:ix, :iy] = scale * out[0, 0] + 1j * (scale * out[0, 1])
    return u0
