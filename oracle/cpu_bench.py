"""CPU ORACLE timing (bench.py's cpu_baseline leg and --impl reference arm only).

Test/measurement infrastructure, never the product path.  Times the numpy
restatement of the reference path (oracle/helm_oracle.py + oracle/network_oracle.py;
the reference itself is pure numpy) on the host cores: P worker
processes, each running a bounded number of FGMRES iterations of one RHS of the
workload with the same preconditioner protocol as the GPU run
(``krylov.py:156-177`` / ``:180-246``).

Throughput in RHS/s is extrapolated from seconds per iteration and the
iterations per RHS that the REFERENCE itself needed on the same seeded inputs
(``tests/golden/configs_c{2,3}.npz``, written by ``oracle/make_golden_configs.py``),
so no GPU-measured number enters the CPU baseline.
"""
from __future__ import annotations

import os
import time

import numpy as np

_STATE = {}
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def reference_iterations(config: str, learned: bool):
    """(mean iterations per RHS, how many reference solves it averages) from the committed goldens."""
    p = os.path.join(ROOT, "tests", "golden", f"configs_{config.lower()}.npz")
    kind = "learned" if learned else "mg"
    try:
        g = np.load(p)
    except OSError:
        return None, 0
    its = [int(g[k]) for k in g.files if k.startswith(f"{config.lower()}_{kind}_") and k.endswith(".iterations")]
    return (float(np.mean(its)), len(its)) if its else (None, 0)


def _setup(config: str, learned: bool):
    from oracle import helm_oracle as ho
    from oracle import network_oracle as no
    from paper_2306_17486_b200 import netparams, problems

    cfg = problems.make_config(config)
    models = [ho.Model(m.kappa_sq, m.gamma, m.omega, m.h) for m in cfg.models]
    hiers = [ho.build_hierarchy(m, damping=cfg.jacobi_damping, num_levels=cfg.mg_levels) for m in models]
    nets = None
    if learned:
        L = len(cfg.cnn_channels)
        p = netparams.init_params(cfg.cnn_channels, seed=0)
        spec = no.spectrum_c64(p, L, cfg.shape)
        nets = [(p, L, no.encode(p, L, no.media_planes(m.kappa_sq, m.gamma, L)), spec) for m in models]
    _STATE.update(cfg=cfg, models=models, hiers=hiers, nets=nets, key=(config, learned))


def _worker(args):
    config, learned, index, iters, warm = args
    # one BLAS/FFT thread per worker process: the pool itself provides the parallelism
    from threadpoolctl import threadpool_limits

    threadpool_limits(1)
    if _STATE.get("key") != (config, learned):
        _setup(config, learned)
    from oracle import helm_oracle as ho
    from oracle import network_oracle as no

    cfg = _STATE["cfg"]
    b = cfg.rhs[index % cfg.rhs.shape[0]]
    mi = int(cfg.model_of_rhs[index % cfg.rhs.shape[0]])
    m, H = _STATE["models"][mi], _STATE["hiers"][mi]
    A = lambda u: ho.helmholtz(u, m)  # noqa: E731
    # phase 1: V-cycle-only iterations (the whole solve, or the learned protocol's warm-up)
    t0 = time.perf_counter()
    x1, r1 = ho.fgmres(A, lambda r: ho.v_cycle(r, None, H), b, None, 1e-30, max(warm if learned else iters, 1),
                       cfg.restart)
    t_v = (time.perf_counter() - t0) / max(r1.iterations, 1)
    if not learned or iters == 0:
        return t_v, 0.0
    # phase 2: net -> V-cycle iterations (krylov.py:225-236)
    p, L, feats, spec = _STATE["nets"][mi]
    t0 = time.perf_counter()
    _, r2 = ho.fgmres(A, lambda r: ho.v_cycle(r, no.preconditioner_estimate(p, L, feats, spec, r, m.h), H),
                      b, x1, 1e-30, iters, cfg.restart)
    return t_v, (time.perf_counter() - t0) / max(r2.iterations, 1)


class CpuArm:
    """A persistent pool of ``workers`` single-threaded oracle processes (set-up paid once)."""

    def __init__(self, config: str, learned: bool, workers: int):
        import multiprocessing as mp

        self.config, self.learned, self.workers = config, learned, workers
        self.pool = mp.get_context("fork").Pool(workers)

    def sample(self, iters: int, warm: int = 3):
        """(seconds per V-cycle iteration, seconds per learned iteration) with every worker busy."""
        args = [(self.config, self.learned, i, iters, warm) for i in range(self.workers)]
        res = self.pool.map(_worker, args)
        return float(np.mean([r[0] for r in res])), float(np.mean([r[1] for r in res]))

    def close(self):
        self.pool.close()
        self.pool.join()


def rhs_per_second(t_v: float, t_l: float, workers: int, mean_iters: float, learned: bool, warmup: int = 3):
    """Extrapolated whole-RHS throughput of `workers` concurrent processes."""
    per_rhs = (warmup * t_v + max(mean_iters - warmup, 0.0) * t_l) if learned else mean_iters * t_v
    return workers / per_rhs
