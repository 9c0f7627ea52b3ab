"""Flexible GMRES and the solve protocols (mirror of ``helmsolve.krylov``).

* ``fgmres`` keeps the reference's callable interface (``krylov.py:39-146``)
  for arbitrary operators: the Krylov basis, Gram-Schmidt and the iterate live
  on the GPU, the user callables are invoked once per iteration (with numpy
  arrays if ``b`` was numpy, CUDA tensors otherwise).
* ``solve_helmholtz`` / ``solve_with_learned_preconditioner``
  (``krylov.py:156-246``) and ``solve_batch`` route to the native batched
  engine (``hs_fgmres_solve``), which runs whole solves on the device.
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np

from .errors import DimensionError, NumericalError, SolverError
from .fields import TRUE_SHIFT, ComplexField, SlownessModel


@dataclass
class SolveReport:
    """Iterations and relative-residual trace of one solve (krylov.py:19-26)."""

    iterations: int
    relative_residual_history: list[float] = field(repr=False)
    converged: bool = False
    wall_time: float = 0.0


def _givens(a: complex, b: float):
    """(c, s, r): [c s; -conj(s) c] maps (a, b) to (r, 0), complex a, real b >= 0 (krylov.py:29-36)."""
    if a == 0:
        return 0.0, 1.0 + 0.0j, b
    mag = abs(a)
    t = math.hypot(mag, b)
    return mag / t, (a / mag) * (b / t), (a / mag) * t


def _solve_upper(R, g):
    """Back substitution on the rotated Hessenberg matrix (krylov.py:149-153)."""
    n = len(g)
    y = np.zeros(n, dtype=np.complex128)
    for i in range(n - 1, -1, -1):
        y[i] = (g[i] - R[i, i + 1 :] @ y[i + 1 :]) / R[i, i]
    return y


def fgmres(apply_A, apply_M, b, x0=None, tol: float = 1e-7, max_iter: int = 250, restart: int | None = 10):
    """Restarted, right-preconditioned flexible GMRES on arrays of any shape (krylov.py:39-146).

    Stops when ||b - A x|| / ||b - A x0|| <= tol or after ``max_iter``
    preconditioner applications.  Same control flow as the reference: CGS
    with a conditional second pass, complex Givens rotations, the estimate
    relative to the initial residual, and the drift guard at window ends.
    """
    import torch

    from .device import require_cuda

    if tol <= 0:
        raise ValueError(f"tol must be positive, got {tol}")
    if max_iter < 1:
        raise ValueError(f"max_iter must be >= 1, got {max_iter}")
    start = time.perf_counter()
    dev = require_cuda()
    host = not isinstance(b, torch.Tensor)
    bd = (torch.from_numpy(np.asarray(b, dtype=np.complex128)) if host else b).to(dev, torch.complex128)
    shape = tuple(bd.shape)
    n = bd.numel()

    def call(fn, v):
        out = fn(v.reshape(shape).cpu().numpy() if host else v.reshape(shape))
        t = torch.from_numpy(np.asarray(out, dtype=np.complex128)) if host else out
        return t.to(dev, torch.complex128).reshape(-1)

    if x0 is None:
        x = torch.zeros(n, dtype=torch.complex128, device=dev)
        r = bd.reshape(-1).clone()
    else:
        if tuple(np.shape(x0)) != shape:
            raise DimensionError(f"x0 {tuple(np.shape(x0))} does not match b {shape}")
        x = (torch.from_numpy(np.asarray(x0, dtype=np.complex128)) if host else x0).to(dev, torch.complex128)
        x = x.reshape(-1).clone()
        r = bd.reshape(-1) - call(apply_A, x)
    beta0 = float(torch.linalg.vector_norm(r))
    history = [1.0]

    def result(xv, it, conv):
        out = xv.reshape(shape)
        return (out.cpu().numpy() if host else out), SolveReport(it, history, conv, time.perf_counter() - start)

    if beta0 == 0.0:
        history.append(0.0)
        return result(x, 0, True)
    if 1.0 <= tol:
        return result(x, 0, True)
    window = max_iter if restart is None else min(restart, max_iter)
    iterations, converged = 0, False
    while iterations < max_iter and not converged:
        m = min(window, max_iter - iterations)
        beta = float(torch.linalg.vector_norm(r))
        V = torch.empty((m + 1, n), dtype=torch.complex128, device=dev)
        Z = torch.empty((m, n), dtype=torch.complex128, device=dev)
        H = np.zeros((m + 1, m), dtype=np.complex128)
        rot = []
        g = np.zeros(m + 1, dtype=np.complex128)
        g[0] = beta
        V[0] = r / beta
        j = 0
        while j < m:
            z = call(apply_M, V[j])
            w = call(apply_A, z)
            if not bool(torch.isfinite(w).all()):
                raise NumericalError(f"non-finite Krylov vector at iteration {iterations + 1}")
            Z[j] = z
            before = float(torch.linalg.vector_norm(w))
            coeffs = V[: j + 1].conj() @ w
            w = w - coeffs @ V[: j + 1]
            h_next = float(torch.linalg.vector_norm(w))
            if h_next < 0.25 * before:
                extra = V[: j + 1].conj() @ w
                coeffs = coeffs + extra
                w = w - extra @ V[: j + 1]
                h_next = float(torch.linalg.vector_norm(w))
            col = coeffs.cpu().numpy()
            for k, (c, s) in enumerate(rot):
                col[k], col[k + 1] = c * col[k] + s * col[k + 1], -np.conj(s) * col[k] + c * col[k + 1]
            c, s, rr = _givens(col[j], h_next)
            rot.append((c, s))
            col[j] = rr
            H[: j + 1, j] = col
            gj = g[j]
            g[j], g[j + 1] = c * gj, -np.conj(s) * gj
            iterations += 1
            j += 1
            estimate = abs(g[j]) / beta0
            history.append(estimate)
            if estimate <= tol:
                converged = True
                break
            if h_next <= 1e-14 * max(1.0, before):
                raise SolverError(
                    f"Arnoldi breakdown at iteration {iterations} with relative residual {estimate:.3e}"
                )
            V[j] = w / h_next
        y = torch.from_numpy(_solve_upper(H[:j, :j], g[:j])).to(dev)
        x = x + y @ Z[:j]
        r = bd.reshape(-1) - call(apply_A, x)
        true_rel = float(torch.linalg.vector_norm(r)) / beta0
        if converged and true_rel > tol:
            converged = False  # the estimate drifted below tol early; keep iterating
        if converged:
            history[-1] = true_rel
    return result(x, iterations, converged)


# -------------------------------------------------------------- solve entry points

MAX_FUSED_WINDOW = 32  # engine.MAX_WINDOW: the batched device solver's per-RHS Hessenberg


def _needs_generic(hierarchy, restart, max_iter) -> bool:
    """Settings the fused batched solver does not implement (the reference accepts them all).

    Restart windows beyond 32 vectors (``restart=None`` means one window of ``max_iter``) and V-cycles
    other than V(1,1) with <= 16 coarse steps run the generic device FGMRES above with the device
    operator and V-cycle as its callables -- the reference's own composition (krylov.py:170-176,
    :215-236), on the GPU, one RHS at a time.
    """
    from .multigrid import fused_cycle

    window = max_iter if restart is None else min(restart, max_iter)
    return window > MAX_FUSED_WINDOW or (hierarchy is not None and not fused_cycle(hierarchy))


def _generic_solve(model, b, hierarchy, tol, max_iter, restart, net=None, encodings=None, warmup_iters=3):
    """solve_helmholtz / solve_with_learned_preconditioner through ``fgmres`` with device callables.

    ``b`` is a complex128 CUDA tensor (nx, ny); returns (x tensor, SolveReport).
    """
    import torch

    from .fields import apply_operator
    from .multigrid import v_cycle

    def A(v):
        return apply_operator(v, model)

    if net is None:
        return fgmres(A, lambda r: v_cycle(r, None, hierarchy), b, None, tol, max_iter, restart)
    from .network import preconditioner_estimate

    x1, r1 = fgmres(A, lambda r: v_cycle(r, None, hierarchy), b, None, tol, min(warmup_iters, max_iter), restart)
    if r1.converged or r1.iterations >= max_iter:
        return x1, r1
    rel1 = float(torch.linalg.vector_norm(b - A(x1)) / torch.linalg.vector_norm(b))

    def M(r):
        return v_cycle(r, preconditioner_estimate(net, encodings, r).to(torch.complex128), hierarchy)

    x2, r2 = fgmres(A, M, b, x1, tol / rel1, max_iter - r1.iterations, restart)
    hist = r1.relative_residual_history + [e * rel1 for e in r2.relative_residual_history[1:]]
    return x2, SolveReport(r1.iterations + r2.iterations, hist, r2.converged)


def _engine_for(model: SlownessModel, hierarchy, net=None):
    from .engine import Engine
    from .multigrid import DeviceHierarchy, build_hierarchy

    if hierarchy is None:
        hierarchy = build_hierarchy(model)
    key = ("_engine", id(model), id(net))
    cached = hierarchy.__dict__.get(key)
    if cached is None or cached[0] is not model:
        dh = DeviceHierarchy([hierarchy], true_models=[model])
        cached = (model, Engine(dh, net))
        hierarchy.__dict__[key] = cached
    return cached[1]


def solve_helmholtz(model: SlownessModel, b: ComplexField, hierarchy=None, tol: float = 1e-7, max_iter: int = 250,
                    restart: int | None = 10) -> tuple[ComplexField, SolveReport]:
    """FGMRES on the true operator with the V-cycle preconditioner (krylov.py:156-177)."""
    import torch

    from .device import to_host
    from .engine import raise_for_status

    if tol <= 0:
        raise ValueError(f"tol must be positive, got {tol}")
    if max_iter < 1:
        raise ValueError(f"max_iter must be >= 1, got {max_iter}")
    start = time.perf_counter()
    if _needs_generic(hierarchy, restart, max_iter):
        from .device import to_device
        from .multigrid import build_hierarchy

        H = hierarchy if hierarchy is not None else build_hierarchy(model)
        x, rep = _generic_solve(model, to_device(np.asarray(b.data), torch.complex128), H, tol, max_iter, restart)
        rep.wall_time = time.perf_counter() - start
        return ComplexField(to_host(x), b.h), rep
    eng = _engine_for(model, hierarchy)
    bd = torch.from_numpy(np.array(b.data))[None]
    res = eng.fgmres(bd, None, tol, max_iter, restart)
    raise_for_status(res)
    x = to_host(res.x[0])
    rep = SolveReport(int(res.iterations[0]), res.histories[0], bool(res.converged[0]), time.perf_counter() - start)
    return ComplexField(x, b.h), rep


def solve_with_learned_preconditioner(model: SlownessModel, b: ComplexField, net, encodings=None, tol: float = 1e-7,
                                      max_iter: int = 250, restart: int | None = 10, warmup_iters: int = 3,
                                      hierarchy=None) -> tuple[ComplexField, SolveReport]:
    """V-cycle warm-up, then FGMRES with M(r) = v_cycle(r, net(r)) (krylov.py:180-246)."""
    from .network import precompute_encodings

    start = time.perf_counter()
    if encodings is None:
        encodings = precompute_encodings(net, model)
    xs, reports = solve_batch([model], np.asarray(b.data)[None], net=net, encodings=[encodings], tol=tol,
                              max_iter=max_iter, restart=restart, warmup_iters=warmup_iters,
                              hierarchies=None if hierarchy is None else [hierarchy])
    reports[0].wall_time = time.perf_counter() - start
    return ComplexField(xs[0], b.h), reports[0]


class BatchSolver:
    """Device-resident solver for many RHS over one or more equal-shape slowness models.

    Setup (hierarchies, device media, network encodings and Green spectrum)
    happens once here; ``solve`` then runs the whole batch on the GPU.
    ``net is None`` gives the V-cycle-only protocol of ``solve_helmholtz``;
    otherwise the warm-up + net->V-cycle protocol of
    ``solve_with_learned_preconditioner`` (krylov.py:214-245) for every RHS.
    """

    def __init__(self, models, net=None, encodings=None, hierarchies=None, num_levels: int = 3,
                 jacobi_damping=None, coarse_iters: int = 10):
        from .engine import Engine
        from .multigrid import CHEBYSHEV_DAMPING, DeviceHierarchy, build_hierarchy

        self.models = list(models)
        if hierarchies is None:
            damp = CHEBYSHEV_DAMPING if jacobi_damping is None else jacobi_damping
            hierarchies = [build_hierarchy(m, num_levels=num_levels, jacobi_damping=damp,
                                           coarse_iters=coarse_iters) for m in self.models]
        self.hierarchies = list(hierarchies)
        self.dh = DeviceHierarchy(self.hierarchies, true_models=self.models)
        self.net = net
        net_dev, net_enc = None, None
        if net is not None:
            from .network import device_network

            # the DeviceNet is shared by every solver on this (net, shape); this solver keeps its own
            # stacked encodings and the engine re-binds them before each solve
            net_dev, net_enc = device_network(net, self.models, encodings, self.dh)
        self.engine = Engine(self.dh, net_dev, net_enc)
        self._encodings = encodings
        self._enc_cache = {}

    def _encodings_for(self, m: int):
        """Encodings of model m for the generic (unfused) path."""
        from .network import precompute_encodings

        if self._encodings is not None and self._encodings[m] is not None:
            return self._encodings[m]
        if m not in self._enc_cache:
            self._enc_cache[m] = precompute_encodings(self.net, self.models[m])
        return self._enc_cache[m]

    def solve(self, rhs, model_of=None, tol: float = 1e-7, max_iter: int = 250, restart: int | None = 10,
              warmup_iters: int = 3, return_device: bool = False, raise_errors: bool = True, iter_caps=None):
        """x (B, nx, ny) complex128 and one SolveReport per RHS.

        ``iter_caps`` (V-cycle protocol only): a per-RHS iteration cap <= max_iter, so samples that
        need different iteration counts share one batched solve (training-pair generation).
        """
        import torch

        from .device import require_cuda, to_device, to_host
        from .engine import BatchResult, raise_for_status
        from .fields import apply_operator

        if tol <= 0:
            raise ValueError(f"tol must be positive, got {tol}")
        if max_iter < 1:
            raise ValueError(f"max_iter must be >= 1, got {max_iter}")
        start = time.perf_counter()
        dev = require_cuda()
        bd = to_device(rhs, torch.complex128)
        B = bd.shape[0]
        owner = np.zeros(B, dtype=np.int32) if model_of is None else np.asarray(model_of, dtype=np.int32)
        if _needs_generic(self.hierarchies[0], restart, max_iter):
            if iter_caps is not None:
                raise ValueError("iter_caps needs the fused solver (restart <= 32, V(1,1), <= 16 coarse steps)")
            from .network import precompute_encodings

            xs, reports = [], []
            for i in range(B):
                m = int(owner[i])
                enc = None
                if self.net is not None:
                    enc = self._encodings_for(m)
                x, rep = _generic_solve(self.models[m], bd[i], self.hierarchies[m], tol, max_iter, restart,
                                        self.net, enc, warmup_iters)
                xs.append(x)
                reports.append(rep)
            x = torch.stack(xs)
            wall = time.perf_counter() - start
            for rep in reports:
                rep.wall_time = wall
            return (x if return_device else to_host(x)), reports
        owner_d = torch.from_numpy(owner).to(dev)
        eng = self.engine
        if iter_caps is not None and self.net is not None:
            raise ValueError("iter_caps applies to the V-cycle protocol only")
        if self.net is None:
            res = eng.fgmres(bd, None, tol, max_iter, restart, owner_d, iter_caps=iter_caps)
            reports = [SolveReport(int(res.iterations[i]), res.histories[i], bool(res.converged[i]), 0.0)
                       for i in range(B)]
            status, x = res.status, res.x
        else:
            # phase 1: V-cycle warm-up from zero (krylov.py:215-220)
            r1 = eng.fgmres(bd, None, tol, min(warmup_iters, max_iter), restart, owner_d)
            x = r1.x
            status = r1.status.copy()
            reports = [SolveReport(int(r1.iterations[i]), r1.histories[i], bool(r1.converged[i]), 0.0)
                       for i in range(B)]
            cont = [i for i in range(B) if not (r1.converged[i] or r1.iterations[i] >= max_iter) and not status[i]]
            if cont:
                idx = torch.tensor(cont, device=dev)
                # rel1 = ||b - A x1|| / ||b|| in fp64 on the device (krylov.py:222-223)
                # (one batched operator application per slowness model)
                num = torch.empty(len(cont), dtype=torch.float64, device=dev)
                cont_a = np.asarray(cont)
                for m in np.unique(owner[cont_a]):
                    sel = np.nonzero(owner[cont_a] == m)[0]
                    ii = torch.from_numpy(cont_a[sel]).to(dev)
                    res = bd[ii] - apply_operator(x[ii], self.models[int(m)])
                    num[torch.from_numpy(sel).to(dev)] = torch.linalg.vector_norm(res.reshape(len(sel), -1), dim=1)
                den = torch.linalg.vector_norm(bd[idx].reshape(len(cont), -1), dim=1)
                rel1 = (num / den).cpu().numpy()
                it1 = int(r1.iterations[cont[0]])
                r2 = eng.fgmres(bd[idx], x[idx], tol / rel1, max_iter - it1, restart, owner_d[idx], use_net=True)
                x[idx] = r2.x
                for k, i in enumerate(cont):
                    reports[i] = SolveReport(
                        reports[i].iterations + int(r2.iterations[k]),
                        reports[i].relative_residual_history + [e * rel1[k] for e in r2.histories[k][1:]],
                        bool(r2.converged[k]), 0.0)
                    status[i] = r2.status[k]
        wall = time.perf_counter() - start
        for rep in reports:
            rep.wall_time = wall
        if raise_errors:
            chk = BatchResult(x, [r.relative_residual_history for r in reports],
                              np.array([r.iterations for r in reports]), None, np.asarray(status))
            for i in range(B):
                raise_for_status(chk, i)
        return (x if return_device else to_host(x)), reports


def solve_batch(models, rhs, model_of=None, net=None, encodings=None, tol: float = 1e-7, max_iter: int = 250,
                restart: int | None = 10, warmup_iters: int = 3, hierarchies=None, num_levels: int = 3,
                jacobi_damping=None, coarse_iters: int = 10, return_device: bool = False, raise_errors=True):
    """Data-parallel solve of many RHS (see BatchSolver); returns (x, reports)."""
    solver = BatchSolver(models, net, encodings, hierarchies, num_levels, jacobi_damping, coarse_iters)
    return solver.solve(rhs, model_of, tol, max_iter, restart, warmup_iters, return_device, raise_errors)
