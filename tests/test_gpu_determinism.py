"""Race detectors: the warp-specialised kernels must give bit-identical results on every run.

The 16-channel tcgen05 conv runs two converter-warp groups on alternate input rows and its
epilogue on another eight warps; the V-cycle legs stream rows through cp.async rings; the fast
coarse GMRES keeps its vectors in shared memory.  A missing barrier in any of them shows up as
run-to-run differences long before it shows up as a wrong answer.
"""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.mark.parametrize("cin,cout,H,W,stride", [(16, 16, 256, 256, 1), (32, 32, 128, 128, 1), (64, 64, 64, 64, 1),
                                                  (16, 32, 256, 256, 2), (16, 16, 250, 250, 1), (32, 16, 128, 128, -2), (64, 32, 64, 64, -2)])
def test_tc_conv_bitwise_repeatable(cin, cout, H, W, stride):
    transposed = stride < 0  # stride -2: transposed conv, output 2H x 2W
    stride = abs(stride)
    from paper_2306_17486_b200 import _lib
    from paper_2306_17486_b200.device import stream_handle

    lib = _lib.load()
    g = torch.Generator(device="cuda").manual_seed(3)
    B = 128
    x = torch.randn(B, H, W, cin, device="cuda", generator=g)
    w = torch.randn(cout, 3, 3, cin, device="cuda", generator=g) / np.sqrt(9 * cin)
    b = torch.randn(cout, device="cuda", generator=g)
    Ho, Wo = (2 * H, 2 * W) if transposed else ((H - 1) // stride + 1, (W - 1) // stride + 1)
    add = torch.randn(B, Ho, Wo, cout, device="cuda", generator=g)
    y = torch.empty_like(add)
    c = _lib.HsConv(cin, cout, stride, int(transposed), 1, w.data_ptr(), b.data_ptr())
    ref = None
    for _ in range(8):
        y.fill_(float("nan"))
        _lib.check(lib.hs_conv2d(x.data_ptr(), ctypes.byref(c), add.data_ptr(), None, y.data_ptr(), B, H, W,
                                 stream_handle()), "conv")
        torch.cuda.synchronize()
        assert torch.isfinite(y).all()
        if ref is None:
            ref = y.clone()
        else:
            assert torch.equal(y, ref)


def test_vcycle_bitwise_repeatable():
    from paper_2306_17486_b200 import fields, multigrid, problems
    from paper_2306_17486_b200.multigrid import DeviceHierarchy, run_vcycle

    n = 257
    ms = [fields.slowness_model(problems.smooth_random_kappa_sq((n, n), 12.0, s), layer_width=20) for s in range(2)]
    Hs = [multigrid.build_hierarchy(m, jacobi_damping=(0.8, 0.8)) for m in ms]
    dh = DeviceHierarchy(Hs)
    rng = np.random.default_rng(5)
    rhs = (rng.standard_normal((64, n, n)) + 1j * rng.standard_normal((64, n, n))).astype(np.complex64)
    u0 = (1e-3 * rng.standard_normal((64, n, n))).astype(np.complex64)
    owner = torch.from_numpy(np.repeat(np.arange(2), 32).astype(np.int32)).cuda()
    r, u = torch.from_numpy(rhs).cuda(), torch.from_numpy(u0).cuda()
    outs = [run_vcycle(dh, r, u, owner).clone() for _ in range(4)]
    outs += [run_vcycle(dh, r, None, owner).clone() for _ in range(2)]
    for o in outs[1:4]:
        assert torch.equal(o, outs[0])
    assert torch.equal(outs[4], outs[5])
