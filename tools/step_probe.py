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


if __name__ == "__main__":
    main()
