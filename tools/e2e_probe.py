"""Where the end-to-end (host buffers) solve spends its time beyond the device solve (C2 learned)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_17486_b200 import krylov, network, problems  # noqa: E402
from paper_2306_17486_b200.device import to_device  # noqa: E402

pre = sys.argv[1] if len(sys.argv) > 1 else "learned"
cfg = problems.make_config("C2")
net = network.EncoderSolverNet.seeded(cfg.cnn_channels, seed=0) if pre == "learned" else None
solver = krylov.BatchSolver(cfg.models, net, jacobi_damping=cfg.jacobi_damping, num_levels=cfg.mg_levels)
kw = dict(model_of=cfg.model_of_rhs, tol=cfg.tol, max_iter=cfg.max_iter, restart=cfg.restart)
rhs_dev = to_device(cfg.rhs, torch.complex128)
rhs_pin = torch.from_numpy(np.ascontiguousarray(cfg.rhs)).pin_memory()
for _ in range(2):
    solver.solve(rhs_dev, return_device=True, **kw)
torch.cuda.synchronize()


def t(label, fn, n=3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        r = fn()
    torch.cuda.synchronize()
    print(f"{label}: {(time.perf_counter() - t0) / n * 1e3:.1f} ms", flush=True)
    return r


t("device in, device out", lambda: solver.solve(rhs_dev, return_device=True, **kw))
t("pinned in, device out", lambda: solver.solve(rhs_pin, return_device=True, **kw))
t("pinned in, host out", lambda: solver.solve(rhs_pin, return_device=False, **kw))
x, _ = solver.solve(rhs_dev, return_device=True, **kw)
t("x.cpu() alone", lambda: x.cpu())
t("h2d pinned alone", lambda: rhs_pin.to("cuda"))
