"""Full solves of a config's first RHS on one GPU: iterations, converged, wall time, true residual.

    python tools/config_probe.py --config C4 --rhs 1 --precond learned
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from oracle import helm_oracle as ho  # noqa: E402
from paper_2306_17486_b200 import krylov, network, problems  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--rhs", type=int, default=1)
    ap.add_argument("--precond", default="learned")
    ap.add_argument("--max-iter", type=int, default=0)
    a = ap.parse_args()
    cfg = problems.make_config(a.config, rhs_per_model=a.rhs)
    net = network.EncoderSolverNet.seeded(cfg.cnn_channels, seed=0) if a.precond == "learned" else None
    t0 = time.perf_counter()
    solver = krylov.BatchSolver(cfg.models, net, jacobi_damping=cfg.jacobi_damping, num_levels=cfg.mg_levels)
    torch.cuda.synchronize()
    setup = time.perf_counter() - t0
    t0 = time.perf_counter()
    xs, reps = solver.solve(cfg.rhs, model_of=cfg.model_of_rhs, tol=cfg.tol, max_iter=a.max_iter or cfg.max_iter,
                            restart=cfg.restart)
    el = time.perf_counter() - t0
    m = cfg.models[0]
    om = ho.Model(m.kappa_sq, m.gamma, m.omega, m.h)
    for i, r in enumerate(reps):
        rt = float(np.linalg.norm(cfg.rhs[i] - ho.helmholtz(xs[i], om)) / np.linalg.norm(cfg.rhs[i]))
        print(f"{a.config} {a.precond} rhs {i}: {r.iterations} it, converged {r.converged}, "
              f"final {r.relative_residual_history[-1]:.3e}, true residual {rt:.3e}")
    print(f"{a.config} {a.precond} {len(reps)} RHS: setup {setup:.2f}s, solve {el:.2f}s, "
          f"max mem {torch.cuda.max_memory_allocated() / 2**30:.1f} GiB")


if __name__ == "__main__":
    main()
