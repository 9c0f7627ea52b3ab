"""Time the network forward alone (hs_net_forward) at a config's shape: CUDA events, no profiling tags.

    python tools/cnn_probe.py [--config C3] [--B 64] [--iters 10]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2306_17486_b200 import _lib, network, problems  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--B", type=int, default=64)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--profile", action="store_true", help="also report the per-tag breakdown (events per launch)")
    ap.add_argument("--lib", default="", help="a measurement variant instead of the product library")
    a = ap.parse_args()
    if a.lib:
        _lib.LIB_PATH = os.path.abspath(a.lib)
    cfg = problems.make_config(a.config)
    net = network.EncoderSolverNet.seeded(cfg.cnn_channels, seed=0)
    dn, enc = network.device_network(net, cfg.models, None, None)
    shape = cfg.models[0].shape
    rng = np.random.default_rng(1)
    r = (rng.standard_normal((a.B,) + shape) + 1j * rng.standard_normal((a.B,) + shape)).astype(np.complex64)
    rd = torch.from_numpy(r).cuda()
    od = torch.zeros(a.B, dtype=torch.int32, device="cuda")
    dn.set_encodings(enc)
    for _ in range(3):
        dn.forward(rd, od)
    torch.cuda.synchronize()
    lib = _lib.load()
    best = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.iters):
            dn.forward(rd, od)
        e1.record()
        torch.cuda.synchronize()
        best.append(e0.elapsed_time(e1) / a.iters)
    print(f"{a.config} network forward, {a.B} RHS: {min(best):.2f} ms per application (best of 3 x {a.iters})")
    if a.profile:
        tags = {"convs": _lib.PROF_CONV, "l0": _lib.PROF_CONV_L0, "wide": _lib.PROF_CONV_WIDE, "cnn": _lib.PROF_CNN,
                "implicit": _lib.PROF_IMPLICIT}
        lib.hs_profile_reset()
        lib.hs_profile_enable(sum(1 << t for t in tags.values()))
        for _ in range(a.iters):
            dn.forward(rd, od)
        torch.cuda.synchronize()
        for n, t in tags.items():
            ms, work, cnt = _lib.profile_query(t)
            print(f"  {n}: {ms / a.iters:.2f} ms per application ({cnt // a.iters} launches)")
        lib.hs_profile_enable(0)
        # per layer (label = cin * 100000 + cout * 100 + mode): hot time per launch, CUDA events
        lib.hs_profile_reset()
        lib.hs_profile_enable(1 << _lib.PROF_CONV)
        for _ in range(a.iters):
            dn.forward(rd, od)
        torch.cuda.synchronize()
        lib.hs_profile_enable(0)
        recs = _lib.profile_records()
        per = len(recs) // a.iters
        print(f"  per layer ({per} convs per application, mean of {a.iters}):")
        for k in range(per):
            _, lab, _ = recs[k]
            ms = sum(recs[i * per + k][2] for i in range(a.iters)) / a.iters
            cin, cout, mode = lab // 100000, (lab // 100) % 1000, lab % 100
            print(f"    {k:2d}  {cin:3d} -> {cout:3d} {('s1', 's2', 't')[mode]:>2}  {ms:.3f} ms")


if __name__ == "__main__":
    main()
