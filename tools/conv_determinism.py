"""Run one tcgen05 conv shape many times on the same input and count bitwise mismatches (race detector)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_17486_b200 import _lib  # noqa: E402
from paper_2306_17486_b200.device import stream_handle  # noqa: E402

cin, cout, B, H, W, reps = (int(v) for v in (sys.argv[1:] + ["16", "16", "128", "256", "256", "30"])[:6])
lib = _lib.load()
torch.manual_seed(0)
x = torch.randn(B, H, W, cin, device="cuda")
w = torch.randn(cout, 3, 3, cin, device="cuda") / np.sqrt(9 * cin)
b = torch.randn(cout, device="cuda")
y = torch.empty(B, H, W, cout, device="cuda")
add = torch.randn_like(y)
c = _lib.HsConv(cin, cout, 1, 0, 1, w.data_ptr(), b.data_ptr())
ref = None
bad = 0
for i in range(reps):
    y.fill_(float("nan"))
    _lib.check(lib.hs_conv2d(x.data_ptr(), ctypes.byref(c), add.data_ptr(), None, y.data_ptr(), B, H, W,
                             stream_handle()), "conv")
    torch.cuda.synchronize()
    if ref is None:
        ref = y.clone()
    elif not torch.equal(y, ref):
        bad += 1
        d = (y - ref).abs()
        print(f"run {i}: mismatch, max abs diff {d.max().item():.3e}, elements {(d > 0).sum().item()}", flush=True)
print(f"cin {cin} cout {cout}: {bad} of {reps - 1} repeats differ")
