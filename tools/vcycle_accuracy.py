"""Accuracy of the device V-cycle against the complex128 oracle and an ideal fp32 V-cycle (numpy), per part.

    python tools/vcycle_accuracy.py [--config C3]

Prints relative L2 errors of: the full V-cycle, the coarse solve alone (one-level hierarchy), one Jacobi
sweep, restriction and prolongation, on a unit-norm complex Gaussian vector of the config's finest grid.
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import helm_oracle as ho  # noqa: E402
from oracle.precision_envelope import V32  # noqa: E402
from paper_2306_17486_b200 import multigrid, problems  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - b) / np.linalg.norm(b))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    a = ap.parse_args()
    cfg = problems.make_config(a.config, rhs_per_model=1)
    m = cfg.models[0]
    om = ho.Model(m.kappa_sq, m.gamma, m.omega, m.h)
    O = ho.build_hierarchy(om, num_levels=cfg.mg_levels, damping=cfg.jacobi_damping)
    H = multigrid.build_hierarchy(m, num_levels=cfg.mg_levels, jacobi_damping=cfg.jacobi_damping)
    rng = np.random.default_rng(3)
    r = rng.standard_normal(m.shape) + 1j * rng.standard_normal(m.shape)
    r /= np.linalg.norm(r)
    ref = ho.v_cycle(r, None, O)
    print(f"{a.config} V-cycle: device {rel(multigrid.v_cycle(r, None, H), ref):.2e}, "
          f"numpy fp32 {rel(V32(O)(r), ref):.2e}")
    # point-source-like residual (smooth) as well
    r2 = cfg.rhs[0] / np.linalg.norm(cfg.rhs[0])
    ref2 = ho.v_cycle(r2, None, O)
    print(f"  point-source rhs: device {rel(multigrid.v_cycle(r2, None, H), ref2):.2e}, "
          f"numpy fp32 {rel(V32(O)(r2), ref2):.2e}")
    # coarse solve alone at the coarsest level
    Lc = O.levels[-1]
    rc = rng.standard_normal(Lc.model.kappa_sq.shape) + 1j * rng.standard_normal(Lc.model.kappa_sq.shape)
    refc = ho.coarse_solve(rc, Lc, O.coarse_iters)
    dc = multigrid.coarse_solve(rc, H.levels[-1], O.coarse_iters)
    print(f"  coarse solve {Lc.model.kappa_sq.shape}: device {rel(dc, refc):.2e}")
    # one Jacobi sweep at the finest level
    u = rng.standard_normal(m.shape) + 1j * rng.standard_normal(m.shape)
    print(f"  jacobi sweep: device {rel(multigrid.jacobi_relax(u, r, H.levels[0], 1, 0.8), ho.jacobi(u, r, O.levels[0], 1, 0.8)):.2e}")
    print(f"  restrict: device {rel(multigrid.restrict_full_weighting(r), ho.restrict(r)):.2e}")
    cs = ho.restrict(r)
    print(f"  prolong: device {rel(multigrid.prolong_bilinear(cs, m.shape), ho.prolong(cs, m.shape)):.2e}")


if __name__ == "__main__":
    main()
