"""GPU parity of the CNN primitives, the implicit layer, the network and the learned solve."""
import ctypes

import numpy as np
import pytest

from conftest import complex_noise, golden, history_dev, relerr

pytestmark = pytest.mark.gpu

from paper_2306_17486_b200 import fields, green, krylov, netparams, network  # noqa: E402
from oracle import helm_oracle as ho  # noqa: E402
from oracle import network_oracle as no  # noqa: E402


def run_conv(x_nchw, w, b, stride=1, transposed=False, softplus=False, addend=None, residual=None):
    """One hs_conv2d call on NCHW numpy data (weights in the reference's layout)."""
    import torch

    from paper_2306_17486_b200 import _lib
    from paper_2306_17486_b200.device import stream_handle

    wt = w.transpose(1, 0, 2, 3) if transposed else w
    cout, cin = wt.shape[:2]
    wd = torch.from_numpy(np.ascontiguousarray(wt.transpose(0, 2, 3, 1)).astype(np.float32)).cuda()
    bd = torch.from_numpy(b.astype(np.float32)).cuda()
    xd = torch.from_numpy(np.ascontiguousarray(x_nchw.transpose(0, 2, 3, 1))).cuda()
    B, H, W = x_nchw.shape[0], x_nchw.shape[2], x_nchw.shape[3]
    Ho, Wo = (2 * H, 2 * W) if transposed else ((H - 1) // stride + 1, (W - 1) // stride + 1)
    y = torch.empty((B, Ho, Wo, cout), dtype=torch.float32, device="cuda")
    c = _lib.HsConv(cin, cout, stride if not transposed else 2, int(transposed), int(softplus), wd.data_ptr(),
                    bd.data_ptr())
    ad = None if addend is None else torch.from_numpy(np.ascontiguousarray(addend.transpose(0, 2, 3, 1))).cuda()
    rd = None if residual is None else torch.from_numpy(np.ascontiguousarray(residual.transpose(0, 2, 3, 1))).cuda()
    _lib.check(_lib.load().hs_conv2d(xd.data_ptr(), ctypes.byref(c), None if ad is None else ad.data_ptr(),
                                     None if rd is None else rd.data_ptr(), y.data_ptr(), B, H, W, stream_handle()),
               "conv")
    return y.cpu().numpy().transpose(0, 3, 1, 2)


def test_conv_primitives_match_reference():
    g = golden("cnn_primitives.npz")
    x, w, b = g["x"], g["w"], g["bias"]
    assert relerr(run_conv(x, w, b), g["conv_s1"]) < 1e-6
    assert relerr(run_conv(x, w, b, stride=2), g["conv_s2"]) < 1e-6
    assert relerr(run_conv(x, g["wt"], b[:1].repeat(5), transposed=True), g["tconv"]) < 1e-6


@pytest.mark.parametrize("cin,cout,stride,hw", [(2, 16, 1, (32, 32)), (16, 16, 1, (64, 40)), (16, 32, 2, (64, 64)),
                                                (32, 64, 2, (32, 48)), (64, 64, 1, (16, 16)), (64, 128, 2, (16, 32)),
                                                (16, 2, 1, (32, 32)), (128, 128, 1, (8, 16))])
def test_conv_shapes_and_epilogue(rng, cin, cout, stride, hw):
    x = rng.standard_normal((2, cin, *hw)).astype(np.float32)
    w = (rng.standard_normal((cout, cin, 3, 3)) / np.sqrt(9 * cin)).astype(np.float32)
    b = rng.standard_normal(cout).astype(np.float32)
    ho, wo = (hw[0] - 1) // stride + 1, (hw[1] - 1) // stride + 1
    add = rng.standard_normal((2, cout, ho, wo)).astype(np.float32)
    y = run_conv(x, w, b, stride=stride, softplus=True, addend=add)
    ref = no.softplus(no.conv2d(x, w, b, stride)) + add
    assert relerr(y, ref) < 2e-6
    y2 = run_conv(x, w, b, stride=stride, residual=add)
    assert relerr(y2, no.conv2d(x, w, b, stride) + add) < 2e-6


@pytest.mark.parametrize("cin,cout,hw", [(64, 32, (8, 8)), (32, 16, (16, 24)), (128, 64, (4, 8))])
def test_tconv_shapes(rng, cin, cout, hw):
    x = rng.standard_normal((2, cin, *hw)).astype(np.float32)
    w = (rng.standard_normal((cin, cout, 3, 3)) / np.sqrt(9 * cout)).astype(np.float32)
    b = rng.standard_normal(cout).astype(np.float32)
    skip = rng.standard_normal((2, cout, 2 * hw[0], 2 * hw[1])).astype(np.float32)
    y = run_conv(x, w, b, transposed=True, softplus=True, addend=skip)
    assert relerr(y, no.softplus(no.conv_transpose2d(x, w, b)) + skip) < 2e-6


@pytest.mark.parametrize("cin,cout,mode,hw", [(16, 16, 0, (6, 128)), (16, 16, 0, (5, 256)), (16, 16, 0, (70, 128)),
                                               # tcgen05.shift kernel (conv_shift.cu): any width -- partial last
                                               # segment / tile, one-segment images, bands of 1 and 33+ rows
                                               (16, 16, 0, (7, 100)), (16, 16, 0, (1, 33)), (16, 16, 0, (33, 30)),
                                               (16, 16, 0, (3, 121)), (16, 16, 0, (40, 250)),
                                               (32, 32, 0, (7, 100)), (32, 32, 0, (1, 33)), (32, 32, 0, (35, 150)),
                                               (32, 32, 0, (9, 256)),
                                               # stride-2 tcgen05.shift kernel: odd and even sizes, partial segments
                                               (16, 32, 1, (7, 100)), (16, 32, 1, (1, 33)), (16, 32, 1, (34, 63)),
                                               (16, 32, 1, (9, 129)), (16, 32, 1, (66, 250)),
                                               # transposed tcgen05.shift kernel: partial segments, one-row and 33-row inputs
                                               (32, 16, 2, (5, 50)), (32, 16, 2, (1, 31)), (32, 16, 2, (33, 65)),
                                               (32, 16, 2, (7, 125)),
                                               (64, 32, 2, (5, 50)), (64, 32, 2, (1, 31)), (64, 32, 2, (33, 65)),
                                               (64, 32, 2, (4, 128)),
                                               (32, 32, 0, (4, 128)),
                                               (16, 32, 1, (6, 256)), (32, 16, 2, (3, 128)), (32, 16, 2, (2, 256)),
                                               # M = 64 tiles (64-wide levels) and cout split across CTAs
                                               (16, 16, 0, (5, 64)), (32, 32, 0, (3, 64)), (64, 64, 0, (4, 64)),
                                               (64, 64, 0, (3, 192)), (32, 64, 1, (5, 128)), (16, 32, 1, (4, 128)),
                                               (64, 32, 2, (3, 64)), (32, 16, 2, (2, 64)),
                                               # K-streamed wide kernel (conv_wide.cu): >= 64 channels, widths
                                               # multiples of 128; odd row counts leave partial passes
                                               (64, 64, 0, (5, 128)), (64, 64, 0, (9, 256)), (128, 128, 0, (5, 128)),
                                               (128, 128, 0, (3, 256)), (64, 128, 1, (7, 256)), (128, 128, 1, (5, 256)),
                                               (128, 64, 2, (3, 128)), (128, 128, 2, (3, 128)), (128, 64, 2, (2, 256)),
                                               (32, 64, 1, (7, 256)), (32, 64, 1, (4, 512))])
def test_tcgen05_conv_matches_oracle(rng, cin, cout, mode, hw):
    """The tcgen05 BF16x3 paths (conv_tc.cu at widths that are multiples of 64, conv_wide.cu for the
    >= 64-channel layers at multiples of 128) against the fp64 oracle, and the SIMT fp32 path."""
    from paper_2306_17486_b200 import _lib

    x = rng.standard_normal((3, cin, *hw)).astype(np.float32)
    if mode == 2:
        w = (rng.standard_normal((cin, cout, 3, 3)) / np.sqrt(9 * cout)).astype(np.float32)
        out_hw = (2 * hw[0], 2 * hw[1])
    else:
        w = (rng.standard_normal((cout, cin, 3, 3)) / np.sqrt(9 * cin)).astype(np.float32)
        s = 2 if mode == 1 else 1
        out_hw = ((hw[0] - 1) // s + 1, (hw[1] - 1) // s + 1)
    b = rng.standard_normal(cout).astype(np.float32)
    add = rng.standard_normal((3, cout, *out_hw)).astype(np.float32)
    lib = _lib.load()
    errs = {}
    try:
        for tc in (1, 0):
            lib.hs_set_conv_path(tc)
            if mode == 2:
                y = run_conv(x, w, b, transposed=True, softplus=True, addend=add)
                ref = no.softplus(no.conv_transpose2d(x.astype(np.float64), w.astype(np.float64), b)) + add
            else:
                y = run_conv(x, w, b, stride=2 if mode == 1 else 1, softplus=True, addend=add)
                ref = no.softplus(no.conv2d(x.astype(np.float64), w.astype(np.float64), b,
                                            2 if mode == 1 else 1)) + add
            y2 = run_conv(x, w, b, stride=2 if mode == 1 else 1, transposed=mode == 2, residual=add)
            ref2 = (no.conv_transpose2d(x.astype(np.float64), w.astype(np.float64), b) if mode == 2 else
                    no.conv2d(x.astype(np.float64), w.astype(np.float64), b, 2 if mode == 1 else 1)) + add
            errs[tc] = (relerr(y, ref), relerr(y2, ref2))
    finally:
        lib.hs_set_conv_path(1)
    print(f"conv {cin}->{cout} mode {mode} {hw}: tcgen05 {errs[1]}, SIMT fp32 {errs[0]}")
    # fp32-class: the SIMT path is plain fp32 (K = 9 cin products per output); the tensor-core path may not
    # exceed 2e-6 or twice the plain-fp32 error of the same layer, whichever is larger
    for k in range(2):
        assert errs[0][k] < 4e-6, errs
        assert errs[1][k] < max(2e-6, 2.0 * errs[0][k]), errs


def test_green_function_and_implicit_apply_match_reference():
    g = golden("cnn_primitives.npz")
    for tag in ("8x8", "16x16", "8x16"):
        hh, ww = map(int, tag.split("x"))
        S = green.green_function(g[f"gk_{tag}"], (hh, ww))
        assert S.dtype == np.complex128
        assert relerr(S, g[f"spec_{tag}"]) < 1e-6
        y = green.implicit_apply(g[f"ix_{tag}"], g[f"spec_{tag}"].astype(np.complex64))
        assert relerr(y, g[f"iy_{tag}"]) < 2e-6


@pytest.mark.parametrize("hh,ww", [(32, 32), (64, 64), (32, 64), (64, 32), (128, 64), (64, 128), (128, 128), (32, 128),
                                   (128, 256)])
def test_fused_implicit_layer_matches_oracle(hh, ww):
    # the fused one-kernel path (implicit.cu) and, at 128 x 256 (the C4 / C5 coarsest level), the batched
    # cuFFT path; the oracle is green.py's pad/fft2/ifft2/crop
    rng = np.random.default_rng(hh * 1000 + ww)
    x = (rng.standard_normal((3, 5, hh, ww)) + 1j * rng.standard_normal((3, 5, hh, ww))).astype(np.complex64)
    spec = (rng.standard_normal((5, 2 * hh, 2 * ww)) + 1j * rng.standard_normal((5, 2 * hh, 2 * ww)))
    spec = spec.astype(np.complex64)
    y = green.implicit_apply(x, spec)
    ref = no.implicit_apply(x.astype(np.complex128), spec.astype(np.complex128))
    assert relerr(y, ref) < 2e-6


def test_green_regression_ratio_on_device():
    # test_green.py:73-80
    S = green.green_function(green.laplacian_plus_i_kernel(1), (16, 16))
    resp = np.fft.ifft2(S[0])
    assert np.abs(resp[16, 16]) / np.abs(resp[0, 0]) == pytest.approx(1.137e-8, rel=0.05)


def test_implicit_kernel_cache():
    k = green.ImplicitKernel(2)
    s1 = k.spectrum((8, 8))
    assert k.spectrum((8, 8)) is s1
    k.weights[0, 1, 1] += 0.5
    k.bump_version()
    assert k.spectrum((8, 8)) is not s1
    # the reference's form (test_green.py:210-220): weights is a versioned tensor, the cache key
    # (size, weights.version)
    s2 = k.spectrum((8, 8))
    k.weights.data[1, 1, 1] += 0.25
    k.weights.bump_version()
    assert k._cache_key == ((8, 8), 1)
    s3 = k.spectrum((8, 8))
    assert s3 is not s2 and k._cache_key == ((8, 8), 2)
    assert relerr(s3, no.green_function(k.weights.data, (8, 8))) < 1e-6


@pytest.mark.parametrize("eps", [1e-3, 0.0])
def test_green_function_eps(eps):
    # green.py:55 green_function(kernel, coarse_size, eps=SPECTRUM_EPS): any regulariser
    rng = np.random.default_rng(41)
    kern = (green.laplacian_plus_i_kernel(3) + 0.1 * (rng.standard_normal((3, 3, 3)) +
                                                      1j * rng.standard_normal((3, 3, 3)))).astype(np.complex64)
    S = green.green_function(kern, (8, 16), eps=eps)
    assert relerr(S, no.green_function(kern, (8, 16), eps=eps)) < 1e-6


@pytest.mark.parametrize("L", [2, 3])
def test_network_matches_reference_composition(L):
    g = golden("network.npz")
    tag = f"L{L}"
    ch = (16, 32, 64) if L == 3 else (8, 16)
    p = netparams.randomise_batchnorm(netparams.init_params(ch, seed=5), seed=6)
    k2, gm = g[f"kappa_sq_{tag}"], g[f"gamma_{tag}"]
    n = k2.shape[0]
    m = fields.SlownessModel(k2, gm, 10.0, 1.0 / (n - 1))
    net = network.EncoderSolverNet(p, ch)
    enc = network.precompute_encodings(net, m)
    for lv in range(L):
        e = enc.tensors[lv].cpu().numpy().transpose(0, 3, 1, 2)
        assert relerr(e, g[f"enc{lv}_{tag}"]) < 1e-5
    r = g[f"r_{tag}"]
    u0 = network.preconditioner_estimate(net, enc, r)
    (ix, iy), _ = no.cnn_dims(r.shape, L)
    y = g[f"y_{tag}"][0]
    s = np.float32(m.h * m.h / 64.0)
    ref = np.zeros(r.shape, np.complex64)
    ref[:ix, :iy] = s * y[0] + 1j * (s * y[1])
    assert relerr(u0, ref) < 2e-5


def test_preconditioner_estimate_matches_oracle_batched(rng):
    n, L, ch = 65, 3, (16, 32, 64)
    m = fields.slowness_model(rng.uniform(0.25, 1.0, (n, n)), layer_width=8)
    net = network.EncoderSolverNet.seeded(ch, seed=3)
    enc = network.precompute_encodings(net, m)
    r = complex_noise(rng, (3, n, n)).astype(np.complex64)
    u0 = network.preconditioner_estimate(net, enc, r)
    feats = no.encode(net.params, L, no.media_planes(m.kappa_sq, m.gamma, L))
    spec = no.spectrum_c64(net.params, L, m.shape)
    for i in range(3):
        assert relerr(u0[i], no.preconditioner_estimate(net.params, L, feats, spec, r[i], m.h)) < 2e-5


def test_learned_c1_matches_reference():
    g = golden("learned_c1.npz")
    m = fields.slowness_model(g["kappa_sq"], layer_width=16)
    net = network.EncoderSolverNet.seeded((16, 32, 64), seed=0)
    xs, reps = krylov.solve_batch([m], g["rhs"], net=net, tol=1e-6, max_iter=400, restart=10,
                                  jacobi_damping=(0.8, 0.8))
    for i, rep in enumerate(reps):
        it = int(g["iterations"][i])
        assert abs(rep.iterations - it) <= 1, (rep.iterations, it)
        assert history_dev(rep.relative_residual_history, g["hist"][i][: it + 1]) < 1e-4
        assert relerr(xs[i], g["x"][i]) < 1e-4
        assert rep.converged


def test_learned_entry_point_single_rhs(rng):
    n = 33
    m = fields.slowness_model(rng.uniform(0.25, 1.0, (n, n)), layer_width=4)
    net = network.EncoderSolverNet.seeded((8, 16), seed=1)
    b = fields.ComplexField(complex_noise(rng, (n, n)), m.h)
    x, rep = krylov.solve_with_learned_preconditioner(m, b, net, tol=1e-6, max_iter=300)
    om = ho.Model(m.kappa_sq, m.gamma, m.omega, m.h)
    feats = no.encode(net.params, 2, no.media_planes(m.kappa_sq, m.gamma, 2))
    spec = no.spectrum_c64(net.params, 2, m.shape)
    xo, ro = ho.solve_learned(om, b.data, lambda r: no.preconditioner_estimate(net.params, 2, feats, spec, r, m.h),
                              1e-6, 300, 10, 3)
    assert abs(rep.iterations - ro.iterations) <= 1
    assert history_dev(rep.relative_residual_history, ro.history) < 1e-4
    assert relerr(x.data, xo) < 1e-4
    # tol = 1 returns after the warm-up's first check
    x1, rep1 = krylov.solve_with_learned_preconditioner(m, b, net, tol=1.0)
    assert rep1.converged and rep1.iterations == 0
