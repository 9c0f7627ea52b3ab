"""Where do repeated runs of the 16->16 tcgen05.shift conv differ?  (race hunting; prints position histograms)"""
import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_17486_b200 import _lib
from paper_2306_17486_b200.device import stream_handle
if os.environ.get('HS_LIB'):
    _lib.LIB_PATH = os.environ['HS_LIB']
lib = _lib.load()
B, H, W = int(sys.argv[1]) if len(sys.argv) > 1 else 128, 256, 256
g = torch.Generator(device="cuda").manual_seed(3)
x = torch.randn(B, H, W, 16, device="cuda", generator=g)
w = torch.randn(16, 3, 3, 16, device="cuda", generator=g) / 12
b = torch.randn(16, device="cuda", generator=g)
add = torch.randn(B, H, W, 16, device="cuda", generator=g)
y = torch.empty_like(add)
c = _lib.HsConv(16, 16, 1, 0, 1, w.data_ptr(), b.data_ptr())
lib.hs_set_conv_path(0)
_lib.check(lib.hs_conv2d(x.data_ptr(), ctypes.byref(c), add.data_ptr(), None, y.data_ptr(), B, H, W, stream_handle()), "conv")
torch.cuda.synchronize()
simt = y.clone()
lib.hs_set_conv_path(1)
for it in range(8):
    y.fill_(float("nan"))
    _lib.check(lib.hs_conv2d(x.data_ptr(), ctypes.byref(c), add.data_ptr(), None, y.data_ptr(), B, H, W, stream_handle()), "conv")
    torch.cuda.synchronize()
    d = (y - simt).abs()
    bad = (d > 1e-4) | ~torch.isfinite(y)
    n = int(bad.sum())
    print(f"run {it}: max |y - simt| {float(d.max()):.3e}, bad elements {n}")
    if n:
        idx = bad.any(dim=3).nonzero()
        bb, yy, xx = idx[:, 0].cpu().numpy(), idx[:, 1].cpu().numpy(), idx[:, 2].cpu().numpy()
        print("  pixels", len(bb), "images", np.unique(bb)[:10], "rows", np.unique(yy)[:20], "row%32", np.unique(yy % 32))
        print("  x", np.unique(xx)[:40], "x%30", np.unique(xx % 30))
        ev = {}
        for i in range(len(bb)):
            ev.setdefault((int(bb[i]), int(yy[i])), []).append(int(xx[i]))
        for k in sorted(ev)[:40]:
            xs = ev[k]
            print("   image %d row %d: x %d..%d (%d px)" % (k[0], k[1], min(xs), max(xs), len(xs)))
