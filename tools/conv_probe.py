"""Time one network convolution shape through hs_conv2d (CUDA events); used for ncu captures."""
import argparse
import ctypes
import sys
import os

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_17486_b200 import _lib  # noqa: E402
from paper_2306_17486_b200.device import stream_handle  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=128)
ap.add_argument("--H", type=int, default=256)
ap.add_argument("--W", type=int, default=256)
ap.add_argument("--cin", type=int, default=16)
ap.add_argument("--cout", type=int, default=16)
ap.add_argument("--stride", type=int, default=1)
ap.add_argument("--transposed", type=int, default=0)
ap.add_argument("--tc", type=int, default=1)
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--side", default="addend", choices=["addend", "residual", "none"])
ap.add_argument("--softplus", type=int, default=1)
ap.add_argument("--lib", default="", help="a measurement variant (tools/_variants/*.so) instead of the product")
a = ap.parse_args()
if a.lib:
    _lib.LIB_PATH = a.lib
lib = _lib.load()
lib.hs_set_conv_path(a.tc)
dev = torch.device("cuda")
x = torch.randn(a.B, a.H, a.W, a.cin, device=dev)
w = torch.randn(a.cout, 3, 3, a.cin, device=dev) / np.sqrt(9 * a.cin)
b = torch.randn(a.cout, device=dev)
Ho, Wo = (2 * a.H, 2 * a.W) if a.transposed else ((a.H - 1) // a.stride + 1, (a.W - 1) // a.stride + 1)
y = torch.empty(a.B, Ho, Wo, a.cout, device=dev)
add = torch.randn_like(y)
c = _lib.HsConv(a.cin, a.cout, a.stride if not a.transposed else 2, a.transposed, a.softplus, w.data_ptr(),
                b.data_ptr())
addp = add.data_ptr() if a.side == "addend" else None
resp = add.data_ptr() if a.side == "residual" else None
def run():
    _lib.check(lib.hs_conv2d(x.data_ptr(), ctypes.byref(c), addp, resp, y.data_ptr(), a.B, a.H, a.W,
                             stream_handle()), "conv")
print("launch", flush=True)
for _ in range(3):
    run()
torch.cuda.synchronize()
print("synced", flush=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
best = []
for _ in range(3):  # best of three batches (clocks vary under the power cap)
    e0.record()
    for _ in range(a.iters):
        run()
    e1.record()
    torch.cuda.synchronize()
    best.append(e0.elapsed_time(e1) / a.iters)
print("synced", flush=True)
if os.environ.get("HS_DBG"):
    print("dbg y[0:4]", y.flatten()[:4].tolist())
ms = min(best)
pix = (a.B * a.H * a.W) if a.transposed else (a.B * Ho * Wo)
flops = 2 * 9 * a.cin * a.cout * pix
byts = 4 * (a.B * a.H * a.W * a.cin + (1 + (a.side != "none")) * a.B * Ho * Wo * a.cout)
print(f"cin {a.cin} cout {a.cout} s{a.stride} t{a.transposed} tc{a.tc}: {ms:.3f} ms  {flops / ms / 1e9:.1f} TFLOP/s  "
      f"{byts / ms / 1e6:.0f} GB/s (x + {a.side} + y)")
