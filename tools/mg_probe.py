"""Hot timing of the multigrid-only pieces at a config's shape (CUDA events, back to back, no profiling tags):
one batched V-cycle (hs_vcycle) and a truncated MG-only FGMRES solve.

    python tools/mg_probe.py [--config C3] [--rhs 64] [--iters 40] [--lib tools/_variants/x.so ...]

With several --lib values each library is timed in its own subprocess (variants side by side).
"""
import argparse
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(a):
    import numpy as np
    import torch

    from paper_2306_17486_b200 import _lib, krylov, multigrid, problems
    from paper_2306_17486_b200.device import stream_handle, to_device, workspace

    if a.lib:
        _lib.LIB_PATH = os.path.abspath(a.lib[0])
    lib = _lib.load()
    cfg = problems.make_config(a.config)
    n = a.rhs or cfg.rhs.shape[0]
    H = multigrid.build_hierarchy(cfg.models[0], num_levels=cfg.mg_levels, jacobi_damping=cfg.jacobi_damping)
    dh = multigrid.DeviceHierarchy([H])
    rng = np.random.default_rng(3)
    r = torch.from_numpy((rng.standard_normal((n,) + cfg.shape) + 1j * rng.standard_normal((n,) + cfg.shape))
                         .astype(np.complex64)).cuda()
    out = torch.empty_like(r)
    ws_bytes = dh.workspace_bytes(n)
    ws = workspace(ws_bytes)
    status = torch.zeros(n, dtype=torch.int32, device="cuda")

    def vc():
        _lib.check(lib.hs_vcycle(ctypes.byref(dh.hs), r.data_ptr(), None, out.data_ptr(), None, n, ws.data_ptr(),
                                 ws_bytes, status.data_ptr(), stream_handle()), "v_cycle")

    def timed(fn, reps):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        best = 1e30
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                fn()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) / reps)
        return best

    t_vc = timed(vc, 20)
    solver = krylov.BatchSolver(cfg.models, None, jacobi_damping=cfg.jacobi_damping, num_levels=cfg.mg_levels)
    b = to_device(cfg.rhs[:n], torch.complex128)
    kw = dict(model_of=cfg.model_of_rhs[:n], tol=cfg.tol, max_iter=a.iters, restart=cfg.restart,
              return_device=True, raise_errors=False)
    t_solve = timed(lambda: solver.solve(b, **kw), 2)
    name = os.path.basename(a.lib[0]) if a.lib else "product"
    print(f"{name}: {a.config} {n} RHS  V-cycle {t_vc:.3f} ms   MG-only solve of {a.iters} iterations "
          f"{t_solve:.1f} ms ({t_solve / a.iters:.3f} ms/it)", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--rhs", type=int, default=0)
    ap.add_argument("--iters", type=int, default=40)
    ap.add_argument("--lib", action="append", default=[])
    a = ap.parse_args()
    if len(a.lib) > 1:
        for lib in a.lib:
            subprocess.run([sys.executable, __file__, "--config", a.config, "--rhs", str(a.rhs), "--iters",
                            str(a.iters), "--lib", lib])
        return
    run(a)


if __name__ == "__main__":
    main()
