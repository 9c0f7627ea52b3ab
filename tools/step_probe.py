"""One truncated batched solve of a config (for ncu launch lists / captures of the bench's kernels).

    python tools/step_probe.py [--config C3] [--precond learned] [--iters 6] [--rhs 64] [--repeat 1]

Runs krylov.BatchSolver.solve on the config's first --rhs RHS with max_iter = --iters (3 V-cycle warm-up
iterations, then the learned protocol), --repeat times, and prints the wall time of the last repeat.
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2306_17486_b200 import krylov, network, problems  # noqa: E402
from paper_2306_17486_b200.device import to_device  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--precond", default="learned")
    ap.add_argument("--iters", type=int, default=6)
    ap.add_argument("--rhs", type=int, default=0)
    ap.add_argument("--repeat", type=int, default=1)
    ap.add_argument("--profile", action="store_true",
                    help="after the timed repeats, one more solve with the tags on: ms per step by kernel group")
    a = ap.parse_args()
    cfg = problems.make_config(a.config)
    n = a.rhs or cfg.rhs.shape[0]
    net = network.EncoderSolverNet.seeded(cfg.cnn_channels, seed=0) if a.precond == "learned" else None
    solver = krylov.BatchSolver(cfg.models, net, jacobi_damping=cfg.jacobi_damping, num_levels=cfg.mg_levels)
    b = to_device(cfg.rhs[:n], torch.complex128)
    kw = dict(model_of=cfg.model_of_rhs[:n], tol=cfg.tol, max_iter=a.iters, restart=cfg.restart, return_device=True,
              raise_errors=False)
    for _ in range(a.repeat):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        solver.solve(b, **kw)
        torch.cuda.synchronize()
    print(f"{a.config} {a.precond} {n} RHS, {a.iters} iterations: {1e3 * (time.perf_counter() - t0):.1f} ms")
    if a.profile:
        from paper_2306_17486_b200 import _lib

        lib = _lib.load()
        tags = {_lib.PROF_CNN: "network", _lib.PROF_VCYCLE: "V-cycle", _lib.PROF_ARNOLDI: "Gram-Schmidt dot",
                _lib.PROF_KRYLOV: "krylov"}
        names = {1: "orth + re-dot (fused)", 5: "orth + re-dot (fused, 20-vector chunk)", 2: "re-dot", 3: "second orth",
             4: "orth", 10: "givens", 11: "x update",
                 12: "residual"}
        lib.hs_profile_reset()
        lib.hs_profile_enable(sum(1 << t for t in tags))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        solver.solve(b, **kw)
        torch.cuda.synchronize()
        wall = 1e3 * (time.perf_counter() - t0)
        lib.hs_profile_enable(0)
        agg = {}
        for tag, lab, ms in _lib.profile_records():
            key = tags[tag] if tag != _lib.PROF_KRYLOV else "krylov: " + names.get(lab, str(lab))
            agg[key] = agg.get(key, 0.0) + ms
        print(f"  profiled solve {wall:.1f} ms wall; per iteration ({a.iters}):")
        for k, v in sorted(agg.items(), key=lambda kv: -kv[1]):
            print(f"    {k:28s} {v / a.iters:8.3f} ms")
        print(f"    {'(untagged: launches, polls, other)':28s} {(wall - sum(agg.values())) / a.iters:8.3f} ms")


if __name__ == "__main__":
    main()
