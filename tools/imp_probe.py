"""Time the fused implicit layer (hs_implicit_apply path) at the C2 coarse size: B x C complex channels."""
import argparse
import sys
import os

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2306_17486_b200 import _lib  # noqa: E402
from paper_2306_17486_b200.device import stream_handle  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=128)
ap.add_argument("--C", type=int, default=32)
ap.add_argument("--h", type=int, default=64)
ap.add_argument("--w", type=int, default=64)
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--lib", default="", help="a measurement variant instead of the product library")
a = ap.parse_args()
if a.lib:
    _lib.LIB_PATH = os.path.abspath(a.lib)
lib = _lib.load()
x = torch.randn(a.B, a.C, a.h, a.w, dtype=torch.complex64, device="cuda")
spec = torch.randn(a.C, 2 * a.h, 2 * a.w, dtype=torch.complex64, device="cuda")
y = torch.empty_like(x)
for _ in range(2):
    _lib.check(lib.hs_implicit_apply(x.data_ptr(), spec.data_ptr(), y.data_ptr(), a.B, a.C, a.h, a.w, stream_handle()),
               "implicit")
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.iters):
    lib.hs_implicit_apply(x.data_ptr(), spec.data_ptr(), y.data_ptr(), a.B, a.C, a.h, a.w, stream_handle())
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.iters
print(f"implicit B={a.B} C={a.C} {a.h}x{a.w}: {ms:.3f} ms per call (includes spectrum permute + alloc)")
