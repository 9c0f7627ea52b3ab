"""GPU vs reference-golden parity report at C2/C3 (writes gpurun_out/parity_<cfg>.npz + a JSON summary).

    python tools/parity_report.py [--configs c2,c3] [--out gpurun_out]

For every case in tests/golden/configs_<cfg>.npz: the device solve (krylov.BatchSolver, the bench's
entry point) of the same RHS, its history, iteration count, and the per-iteration deviation from the
reference run, next to the complex64 precision envelope (tests/golden/envelope_<cfg>.npz) when present.
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2306_17486_b200 import krylov, network, problems  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c2,c3")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out"))
    a = ap.parse_args()
    os.makedirs(a.out, exist_ok=True)
    summary = []
    for c in a.configs.split(","):
        g = np.load(os.path.join(ROOT, "tests", "golden", f"configs_{c}.npz"))
        envp = os.path.join(ROOT, "tests", "golden", f"envelope_{c}.npz")
        env = np.load(envp) if os.path.exists(envp) else None
        cfg = problems.make_config(c.upper())
        out = {}
        for kind in ("mg", "learned"):
            names = sorted({k.split(".")[0] for k in g.files if k.startswith(f"{c}_{kind}_")})
            if not names:
                continue
            idx = [int(g[f"{n}.idx"]) for n in names]
            net = network.EncoderSolverNet.seeded(cfg.cnn_channels, seed=0) if kind == "learned" else None
            solver = krylov.BatchSolver(cfg.models, net, jacobi_damping=cfg.jacobi_damping, num_levels=cfg.mg_levels)
            xs, reps = solver.solve(cfg.rhs[idx], model_of=cfg.model_of_rhs[idx], tol=cfg.tol, max_iter=cfg.max_iter,
                                    restart=cfg.restart)
            for k, n in enumerate(names):
                h = np.asarray(reps[k].relative_residual_history)
                ref = g[f"{n}.hist"]
                m = min(len(h), len(ref))
                dev = np.abs(h[:m] - ref[:m]) / ref[:m]
                xr = g[f"{n}.x"] if f"{n}.x" in g.files else g[f"{n}.x_sub4"]
                xg = xs[k] if f"{n}.x" in g.files else xs[k][::4, ::4]
                ex = float(np.linalg.norm(xg - xr) / np.linalg.norm(xr))
                row = {"case": n, "iterations": reps[k].iterations, "ref_iterations": int(g[f"{n}.iterations"]),
                       "max_hist_dev": float(dev.max()), "argmax": int(dev.argmax()), "x_err": ex}
                if env is not None and f"{n}.env" in env.files:
                    e = env[f"{n}.env"]
                    row["max_env"] = float(e.max())
                    row["env_iterations"] = int(env[f"{n}.iterations"])
                summary.append(row)
                out[f"{n}.hist"] = h
                out[f"{n}.dev"] = dev
                print(json.dumps(row), flush=True)
        np.savez(os.path.join(a.out, f"parity_{c}.npz"), **out)
    with open(os.path.join(a.out, "parity_summary.json"), "w") as f:
        json.dump(summary, f, indent=1)


if __name__ == "__main__":
    main()
