"""Reference-run goldens at the BENCHMARKED configurations (C2 and C3), for the GPU parity tests.

Test infrastructure only (like the rest of ``oracle/``): it imports the REFERENCE
(``/root/reference/pkg/src``) in place and runs its unmodified solve entry points on
the exact inputs ``bench.py`` uses (``problems.make_config``):

* ``solve_helmholtz`` (``krylov.py:156-177``) -- the multigrid-only preconditioner;
* ``solve_with_learned_preconditioner`` (``krylov.py:180-246``) with the ARCH.md
  network composed from the reference's own autodiff/green primitives and injected
  as ``helmsolve.network`` (``make_golden.install_ref_network``), seed-0 weights.

Cases (one process each, run in parallel; ``--jobs``):

    c2_mg_m{0..3}       C2, first RHS of each of the 4 models, MG3 (0.8/0.8), FGMRES(10), tol 1e-6
    c2_learned_m{0..3}  the same RHS through the learned protocol (CNN 16/32/64)
    c3_mg_{0,32}        C3 RHS 0 (point source) and 32 (complex Gaussian), MG4, FGMRES(20)
    c3_learned_{0,32}   the same RHS through the learned protocol (CNN 16/32/64/128);
                        about 7 s per network application on one core, ~1 h per RHS

The C2 multigrid cases are also solved by the oracle (``helm_oracle.solve_vcycle``)
and asserted equal (iterations, history to 1e-8), which pins the oracle at C2.

Output: ``tests/golden/configs_c2.npz`` and ``tests/golden/configs_c3.npz`` with
per case the RHS index, history, iteration count and the solution (C2 full, C3 on
the [::4, ::4] sub-grid plus its full-grid norm, to keep the fixture small).

    PYTHONDONTWRITEBYTECODE=1 python oracle/make_golden_configs.py --jobs 8
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PARTS = os.path.join(ROOT, "oracle", "_ref", "golden_parts")
OUT = os.path.join(ROOT, "tests", "golden")

CASES = ([f"c2_mg_m{m}" for m in range(4)] + [f"c2_learned_m{m}" for m in range(4)]
         + ["c3_mg_0", "c3_mg_32", "c3_learned_0", "c3_learned_32"])


def case_spec(case):
    """(config name, rhs index, learned)."""
    parts = case.split("_")
    cfg, kind, tag = parts[0].upper(), parts[1], parts[2]
    idx = 32 * int(tag[1:]) if tag.startswith("m") else int(tag)
    return cfg, idx, kind == "learned"


def run_case(case):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    sys.path.insert(0, ROOT)
    import make_golden as mg  # reference imported in place by make_golden

    from oracle import helm_oracle as ho
    from paper_2306_17486_b200 import netparams, problems

    cfgname, idx, learned = case_spec(case)
    cfg = problems.make_config(cfgname)
    m = cfg.models[int(cfg.model_of_rhs[idx])]
    b = cfg.rhs[idx]
    H = mg.rm.build_hierarchy(m, num_levels=cfg.mg_levels, jacobi_damping=cfg.jacobi_damping)
    t0 = time.time()
    if learned:
        mg.install_ref_network()
        ch = cfg.cnn_channels
        net = mg.RefNet(netparams.init_params(ch, seed=0), len(ch))
        net.h = m.h
        enc = sys.modules["helmsolve.network"].precompute_encodings(net, m)
        x, rep = mg.rk.solve_with_learned_preconditioner(
            m, mg.rf.ComplexField(b, m.h), net, enc, tol=cfg.tol, max_iter=cfg.max_iter, restart=cfg.restart,
            hierarchy=H)
    else:
        x, rep = mg.rk.solve_helmholtz(m, mg.rf.ComplexField(b, m.h), H, tol=cfg.tol, max_iter=cfg.max_iter,
                                       restart=cfg.restart)
        if cfgname == "C2":  # pin the oracle restatement at C2 as well
            O = ho.build_hierarchy(mg.omodel(m), num_levels=cfg.mg_levels, damping=cfg.jacobi_damping)
            xo, ro = ho.solve_vcycle(mg.omodel(m), b, O, cfg.tol, cfg.max_iter, cfg.restart)
            assert ro.iterations == rep.iterations, (ro.iterations, rep.iterations)
            assert max(abs(a - c) / c for a, c in zip(ro.history, rep.relative_residual_history)) < 1e-8
            assert mg.relerr(xo, x.data) < 1e-9
    el = time.time() - t0
    xd = np.asarray(x.data)
    out = {"idx": idx, "iterations": rep.iterations, "converged": rep.converged,
           "hist": np.asarray(rep.relative_residual_history), "x_norm": float(np.linalg.norm(xd)), "seconds": el}
    if cfgname == "C2":
        out["x"] = xd.astype(np.complex64)
    else:
        out["x_sub4"] = xd[::4, ::4].astype(np.complex64)
    os.makedirs(PARTS, exist_ok=True)
    np.savez(os.path.join(PARTS, case + ".npz"), **out)
    print(json.dumps({"case": case, "iterations": rep.iterations, "converged": rep.converged,
                      "final": rep.relative_residual_history[-1], "seconds": round(el, 1)}), flush=True)


def merge():
    for cfg in ("c2", "c3"):
        arrays = {}
        for case in CASES:
            if not case.startswith(cfg):
                continue
            p = os.path.join(PARTS, case + ".npz")
            if not os.path.exists(p):
                print(f"missing {case}; not merged")
                continue
            g = np.load(p)
            for k in g.files:
                if k != "seconds":
                    arrays[f"{case}.{k}"] = g[k]
        if arrays:
            np.savez_compressed(os.path.join(OUT, f"configs_{cfg}.npz"), **arrays)
            print(f"wrote configs_{cfg}.npz ({len(arrays)} arrays)")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default=",".join(CASES))
    ap.add_argument("--jobs", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--merge-only", action="store_true")
    ap.add_argument("--one", default="", help="run a single case in this process")
    a = ap.parse_args()
    if a.one:
        return run_case(a.one)
    if not a.merge_only:
        import subprocess

        todo = [c for c in a.cases.split(",") if c]
        # longest first
        todo.sort(key=lambda c: (not c.startswith("c3_learned"), not c.startswith("c2_learned")))
        procs = []
        while todo or procs:
            while todo and len(procs) < a.jobs:
                c = todo.pop(0)
                procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__), "--one", c]))
            time.sleep(2)
            procs = [p for p in procs if p.poll() is None]
    merge()


if __name__ == "__main__":
    main()
