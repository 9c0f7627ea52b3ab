"""CPU ORACLE (test infrastructure only) for the Helmholtz FGMRES hot path.

This module is a numpy restatement of the reference package ``helmsolve``
(``/root/reference/pkg/src/helmsolve``) for the north-star path: the 5-point
Helmholtz operator, the shifted-Laplacian V-cycle and flexible GMRES.  It is
the checker for the CUDA path and the CPU baseline leg of ``bench.py``; only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The product package never does.

Pinning: ``oracle/make_golden.py`` imports the reference in place (this
container only), checks every function here against it, and writes the
fixtures under ``tests/golden/`` that ``tests/test_oracle.py`` re-checks on any
machine.  Arithmetic is complex128/float64, exactly as the reference.

Each function cites the reference ``file:line`` it restates.
"""
from __future__ import annotations

import math

import numpy as np

PPW = 0.628  # fields.py:23
FW = np.array([[1.0, 2.0, 1.0], [2.0, 4.0, 2.0], [1.0, 2.0, 1.0]]) / 16.0  # multigrid.py:49
CHEB = (0.5617, 1.3895)  # multigrid.py:52


class OracleError(Exception):
    def __init__(self, kind: str, msg: str):
        super().__init__(msg)
        self.kind = kind


# ----------------------------------------------------------------- fields.py


def spacing(nx: int, ny: int) -> float:
    """fields.py:26-28."""
    return 1.0 / (max(nx, ny) - 1)


def omega_10ppw(n: int, kappa_max: float) -> float:
    """fields.py:120-131: omega * kappa_max * h == PPW with h = 1/(n-1)."""
    return PPW * (n - 1) / kappa_max


def abl_mask(nx: int, ny: int, width: int, gamma0: float) -> np.ndarray:
    """fields.py:134-154: gamma0 + (1-gamma0) * clip((W-d)/W, 0)^2, d = distance to edge."""
    dx = np.minimum(np.arange(nx), np.arange(nx)[::-1])
    dy = np.minimum(np.arange(ny), np.arange(ny)[::-1])
    d = np.minimum(dx[:, None], dy[None, :]).astype(np.float64)
    ramp = np.maximum((width - d) / width, 0.0)
    return gamma0 + (1.0 - gamma0) * ramp * ramp


def layer_width_default(n_ext: int) -> int:
    """fields.py:157-159."""
    return max(2, round(16 * n_ext / 128))


class Model:
    """kappa^2, gamma, omega, h of one problem (fields.py:75-117)."""

    def __init__(self, kappa_sq, gamma, omega, h):
        self.kappa_sq = np.asarray(kappa_sq, dtype=np.float64)
        self.gamma = np.asarray(gamma, dtype=np.float64)
        self.omega = float(omega)
        self.h = float(h)

    @property
    def shape(self):
        return self.kappa_sq.shape


def make_model(kappa_sq, gamma0=0.01, layer_width=None, omega=None) -> Model:
    """fields.py:162-183 (validation omitted; the product checks it)."""
    k = np.asarray(kappa_sq, dtype=np.float64)
    nx, ny = k.shape
    n = max(nx, ny)
    if layer_width is None:
        layer_width = layer_width_default(n - 1)
    if omega is None:
        omega = omega_10ppw(n, math.sqrt(k.max()))
    return Model(k, abl_mask(nx, ny, layer_width, gamma0), omega, spacing(nx, ny))


def mass(model: Model, alpha: float, beta: float) -> np.ndarray:
    """fields.py:186-188: c = omega^2 kappa^2 (alpha - i (beta + gamma))."""
    return (model.omega**2 * model.kappa_sq) * (alpha - 1j * (beta + model.gamma))


def neg_lap(u: np.ndarray, h: float) -> np.ndarray:
    """fields.py:191-199: (4u - sum of the 4 neighbours, zero outside) / h^2."""
    out = 4.0 * u
    out[:-1, :] -= u[1:, :]  # x+1, x-1, y+1, y-1: the reference's summation order
    out[1:, :] -= u[:-1, :]
    out[:, :-1] -= u[:, 1:]
    out[:, 1:] -= u[:, :-1]
    return out / (h * h)


def helmholtz(u: np.ndarray, model: Model, alpha=1.0, beta=0.0) -> np.ndarray:
    """fields.py:202-210: A u = -Lap u - c u, in complex128."""
    u = np.asarray(u, dtype=np.complex128)
    return neg_lap(u, model.h) - mass(model, alpha, beta) * u


def diagonal(model: Model, alpha: float, beta: float) -> np.ndarray:
    """fields.py:222-224."""
    return 4.0 / model.h**2 - mass(model, alpha, beta)


# -------------------------------------------------------------- multigrid.py


def coarse_dims(shape):
    """multigrid.py:55-56: n -> n // 2 (coarse K sits on fine 2K+1)."""
    return shape[0] // 2, shape[1] // 2


def restrict(fine: np.ndarray) -> np.ndarray:
    """multigrid.py:64-78: 3x3 full weighting centred on fine 2K+1, zero outside."""
    nx, ny = fine.shape
    if nx < 5 or ny < 5:
        raise OracleError("dimension", f"grid {nx}x{ny} too small to coarsen")
    cx, cy = coarse_dims(fine.shape)
    padded = np.zeros((2 * cx + 1, 2 * cy + 1), dtype=fine.dtype)
    padded[: min(nx, 2 * cx + 1), : min(ny, 2 * cy + 1)] = fine[: 2 * cx + 1, : 2 * cy + 1]
    out = np.zeros((cx, cy), dtype=fine.dtype)
    for a in range(3):
        for b in range(3):
            out += FW[a, b] * padded[a : a + 2 * cx : 2, b : b + 2 * cy : 2]
    return out


def prolong(coarse: np.ndarray, fine_shape) -> np.ndarray:
    """multigrid.py:81-114: P = 4 R^T (bilinear, zero beyond the coarse grid)."""
    cx, cy = coarse.shape
    nx, ny = fine_shape
    if not (2 * cx <= nx <= 2 * cx + 1 and 2 * cy <= ny <= 2 * cy + 1):
        raise OracleError("dimension", f"cannot prolong {coarse.shape} onto {fine_shape}")
    # scatter form of 4 R^T: every coarse node K spreads 4*FW onto fine 2K+1 +- 1
    full = np.zeros((2 * cx + 1, 2 * cy + 1), dtype=coarse.dtype)
    for a in range(3):
        for b in range(3):
            full[a : a + 2 * cx : 2, b : b + 2 * cy : 2] += (4.0 * FW[a, b]) * coarse
    return full[:nx, :ny]


def restrict_media(values: np.ndarray) -> np.ndarray:
    """multigrid.py:117-125: weight-renormalised full weighting."""
    return restrict(values) / restrict(np.ones_like(values))


class Level:
    """One level: model, shift, wall term, diagonal (multigrid.py:128-150)."""

    def __init__(self, model: Model, alpha: float, beta: float, wall=None):
        self.model, self.alpha, self.beta, self.wall = model, alpha, beta, wall
        d = diagonal(model, alpha, beta)
        self.diag = d if wall is None else d + wall

    def apply(self, u):
        out = helmholtz(u, self.model, self.alpha, self.beta)
        if self.wall is not None:
            out = out + self.wall * u
        return out


def wall_term(shape, d_hi, h):
    """multigrid.py:153-163: (1-d)/d/h^2 on the high edge of each short axis."""
    if d_hi[0] >= 1.0 and d_hi[1] >= 1.0:
        return None
    w = np.zeros(shape)
    if d_hi[0] < 1.0:
        w[-1, :] += (1.0 - d_hi[0]) / d_hi[0] / h**2
    if d_hi[1] < 1.0:
        w[:, -1] += (1.0 - d_hi[1]) / d_hi[1] / h**2
    return w


class Hierarchy:
    def __init__(self, levels, relax_pre, relax_post, damping, coarse_iters):
        self.levels = levels
        self.relax_pre, self.relax_post = relax_pre, relax_post
        self.damping = tuple(damping)
        self.coarse_iters = coarse_iters


def build_hierarchy(model: Model, alpha=1.0, beta=0.5, num_levels=3, relax_pre=1,
                    relax_post=1, damping=CHEB, coarse_iters=10) -> Hierarchy:
    """multigrid.py:185-215: rediscretised media, h doubling, wall re-alignment."""
    levels = [Level(model, alpha, beta)]
    k2, g, h = model.kappa_sq, model.gamma, model.h
    d_hi = (1.0, 1.0)
    for _ in range(num_levels - 1):
        parent = k2.shape
        k2 = restrict_media(k2)
        g = np.clip(restrict_media(g), 0.0, 1.0)
        h *= 2.0
        d_hi = ((d_hi[0] + parent[0] % 2) / 2, (d_hi[1] + parent[1] % 2) / 2)
        levels.append(Level(Model(k2, g, model.omega, h), alpha, beta, wall_term(k2.shape, d_hi, h)))
    return Hierarchy(levels, relax_pre, relax_post, damping, coarse_iters)


def jacobi(u, rhs, level: Level, sweeps: int, w: float):
    """multigrid.py:218-229."""
    for _ in range(sweeps):
        u = u + w * ((rhs - level.apply(u)) / level.diag)
    return u


def coarse_solve(rhs, level: Level, iters=10, w=0.8):
    """multigrid.py:232-244: GMRES + one damped Jacobi sweep as preconditioner."""
    s = w / level.diag
    x, _ = fgmres(level.apply, lambda r: s * r, rhs, None, 1e-12, iters, iters)
    return x


def v_cycle(rhs, u0, hier: Hierarchy):
    """multigrid.py:247-274: V(relax_pre, relax_post) recursion."""
    rhs = np.asarray(rhs, dtype=np.complex128)
    u = np.zeros_like(rhs) if u0 is None else np.asarray(u0)
    return _cycle(rhs, u, hier, 0)


def _cycle(rhs, u, hier, depth):
    level = hier.levels[depth]
    if depth == len(hier.levels) - 1:
        return coarse_solve(rhs, level, hier.coarse_iters)
    u = jacobi(u, rhs, level, hier.relax_pre, hier.damping[0])
    coarse_rhs = restrict(rhs - level.apply(u))
    e = _cycle(coarse_rhs, np.zeros_like(coarse_rhs), hier, depth + 1)
    u = u + prolong(e, rhs.shape)
    return jacobi(u, rhs, level, hier.relax_post, hier.damping[1])


# ----------------------------------------------------------------- krylov.py


class Report:
    def __init__(self, iterations, history, converged):
        self.iterations, self.history, self.converged = iterations, history, converged


def _rotation(a: complex, b: float):
    """krylov.py:29-36: (c, s, r) with [c s; -conj(s) c] (a, b) = (r, 0)."""
    if a == 0:
        return 0.0, 1.0 + 0.0j, b
    mag = abs(a)
    t = math.hypot(mag, b)
    phase = a / mag
    return mag / t, phase * (b / t), phase * t


def _back_substitute(R, g):
    """krylov.py:149-153."""
    n = len(g)
    y = np.zeros(n, dtype=np.complex128)
    for i in reversed(range(n)):
        y[i] = (g[i] - R[i, i + 1 :] @ y[i + 1 :]) / R[i, i]
    return y


def fgmres(apply_A, apply_M, b, x0=None, tol=1e-7, max_iter=250, restart=10, store=None):
    """krylov.py:39-146: restarted flexible GMRES, CGS + conditional second pass.

    ``store`` (precision-envelope experiments only) rounds every basis vector as it is stored in V / Z.
    """
    st = store or (lambda v: v)
    if tol <= 0 or max_iter < 1:
        raise ValueError("bad tol / max_iter")
    b = np.asarray(b, dtype=np.complex128)
    shape, n = b.shape, b.size
    if x0 is None:
        x = np.zeros(shape, dtype=np.complex128)
        r = b.copy()
    else:
        x = np.asarray(x0, dtype=np.complex128).copy()
        r = b - apply_A(x)
    beta0 = np.linalg.norm(r)
    hist = [1.0]
    if beta0 == 0.0:
        return x, Report(0, hist + [0.0], True)
    if tol >= 1.0:
        return x, Report(0, hist, True)
    window = max_iter if restart is None else min(restart, max_iter)
    it, done = 0, False
    while it < max_iter and not done:
        m = min(window, max_iter - it)
        beta = np.linalg.norm(r)
        V = np.empty((m + 1, n), dtype=np.complex128)
        Z = np.empty((m, n), dtype=np.complex128)
        H = np.zeros((m + 1, m), dtype=np.complex128)
        cs, sn = [], []
        g = np.zeros(m + 1, dtype=np.complex128)
        g[0] = beta
        V[0] = st(r.ravel() / beta)
        j = 0
        while j < m:
            z = np.asarray(apply_M(V[j].reshape(shape)), dtype=np.complex128).ravel()
            w = np.asarray(apply_A(z.reshape(shape)), dtype=np.complex128).ravel()
            if not np.isfinite(w).all():
                raise OracleError("nonfinite", f"non-finite Krylov vector at iteration {it + 1}")
            Z[j] = st(z)
            wn = np.linalg.norm(w)
            hcol = V[: j + 1].conj() @ w
            w = w - hcol @ V[: j + 1]
            hn = np.linalg.norm(w)
            if hn < 0.25 * wn:
                extra = V[: j + 1].conj() @ w
                hcol = hcol + extra
                w = w - extra @ V[: j + 1]
                hn = np.linalg.norm(w)
            for k in range(j):
                a, bb = hcol[k], hcol[k + 1]
                hcol[k] = cs[k] * a + sn[k] * bb
                hcol[k + 1] = -np.conj(sn[k]) * a + cs[k] * bb
            c, s, rr = _rotation(hcol[j], hn)
            cs.append(c)
            sn.append(s)
            hcol[j] = rr
            H[: j + 1, j] = hcol
            gj = g[j]
            g[j] = c * gj
            g[j + 1] = -np.conj(s) * gj
            it += 1
            j += 1
            est = abs(g[j]) / beta0
            hist.append(est)
            if est <= tol:
                done = True
                break
            if hn <= 1e-14 * max(1.0, wn):
                raise OracleError(
                    "breakdown",
                    f"Arnoldi breakdown at iteration {it} with relative residual {est:.3e}",
                )
            V[j] = st(w / hn)
        y = _back_substitute(H[:j, :j], g[:j])
        x = x + (y @ Z[:j]).reshape(shape)
        r = b - apply_A(x)
        true_rel = np.linalg.norm(r) / beta0
        if done and true_rel > tol:
            done = False
        if done:
            hist[-1] = true_rel
    return x, Report(it, hist, done)


def solve_vcycle(model: Model, b, hier=None, tol=1e-7, max_iter=250, restart=10):
    """krylov.py:156-177."""
    hier = hier or build_hierarchy(model)
    return fgmres(
        lambda u: helmholtz(u, model),
        lambda r: v_cycle(r, None, hier),
        b, None, tol, max_iter, restart,
    )


def solve_learned(model: Model, b, net_apply, tol=1e-7, max_iter=250, restart=10,
                  warmup_iters=3, hier=None, round_z=None, vcycle=None, store=None):
    """krylov.py:180-246: V-cycle warm-up, then M(r) = v_cycle(r, u0 = net(r)).

    ``round_z`` / ``vcycle`` (precision-envelope experiments only, oracle/precision_envelope.py)
    post-process every preconditioner output z / replace the V-cycle ``vcycle(r, u0)``.
    """
    hier = hier or build_hierarchy(model)
    A = lambda u: helmholtz(u, model)  # noqa: E731
    rz = round_z or (lambda z: z)
    vc = vcycle or (lambda r, u0: v_cycle(r, u0, hier))
    x1, r1 = fgmres(A, lambda r: rz(vc(r, None)), b, None, tol,
                    min(warmup_iters, max_iter), restart, store)
    if r1.converged or r1.iterations >= max_iter:
        return x1, r1
    rel1 = np.linalg.norm(b - A(x1)) / np.linalg.norm(b)
    x2, r2 = fgmres(A, lambda r: rz(vc(r, net_apply(r))), b, x1, tol / rel1,
                    max_iter - r1.iterations, restart, store)
    return x2, Report(r1.iterations + r2.iterations,
                      r1.history + [e * rel1 for e in r2.history[1:]], r2.converged)
