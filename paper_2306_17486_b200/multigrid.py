"""Shifted-Laplacian geometric multigrid (mirror of ``helmsolve.multigrid``).

The hierarchy is built on the host in float64 exactly as the reference does
(rediscretised media, h doubling, coarse node K at fine 2K+1, wall
re-alignment term on even-parent levels; ``multigrid.py:1-31, 117-215``) and
uploaded once per slowness model: each level's mass term as complex64.  The
cycle itself runs on the GPU (``hs_vcycle``): two fused shared-memory kernels
per level plus an on-device GMRES-Jacobi coarse solve.  Following the
precision recipe the V-cycle computes in complex64; public
functions return complex128 arrays like the reference.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from .errors import ConfigurationError, DimensionError, SingularityError
from .fields import (
    PRECONDITIONER_SHIFT,
    HelmholtzShift,
    SlownessModel,
    apply_operator,
    mass_coefficient,
    stencil_diagonal,
)

#: Full-weighting stencil; prolongation is 4x its transpose (multigrid.py:48-49).
TRANSFER_KERNEL = np.outer([1.0, 2.0, 1.0], [1.0, 2.0, 1.0]) / 16.0

#: Pre/post Jacobi dampings: reciprocal degree-2 Chebyshev roots on [1/2, 2] (multigrid.py:51-52).
CHEBYSHEV_DAMPING = (0.5617, 1.3895)


def coarse_shape(shape: tuple[int, int]) -> tuple[int, int]:
    """n nodes coarsen to n // 2 (coarse K sits on fine 2K+1), multigrid.py:55-56."""
    return shape[0] // 2, shape[1] // 2


def _check_coarsenable(nx: int, ny: int):
    if nx < 5 or ny < 5:
        raise DimensionError(f"grid {nx}x{ny} too small to coarsen")


# ------------------------------------------------------- host setup (float64)


def _fw_host(fine: np.ndarray) -> np.ndarray:
    """Host float64 full weighting, used only while building a hierarchy."""
    nx, ny = fine.shape
    _check_coarsenable(nx, ny)
    cx, cy = coarse_shape(fine.shape)
    ext = np.zeros((2 * cx + 1, 2 * cy + 1), dtype=fine.dtype)
    ext[: min(nx, 2 * cx + 1), : min(ny, 2 * cy + 1)] = fine[: 2 * cx + 1, : 2 * cy + 1]
    out = np.zeros((cx, cy), dtype=fine.dtype)
    for a in range(3):
        for b in range(3):
            out += TRANSFER_KERNEL[a, b] * ext[a : a + 2 * cx : 2, b : b + 2 * cy : 2]
    return out


def restrict_media(values: np.ndarray) -> np.ndarray:
    """Weight-renormalised full weighting of kappa^2 / gamma (multigrid.py:117-125)."""
    values = np.asarray(values, dtype=np.float64)
    return _fw_host(values) / _fw_host(np.ones_like(values))


@dataclass(frozen=True)
class Level:
    """One level: rediscretised medium, shift, wall term and diagonal (multigrid.py:128-150)."""

    model: SlownessModel
    shift: HelmholtzShift
    wall: np.ndarray | None = field(repr=False, default=None)
    diag: np.ndarray = field(repr=False, default=None)

    def __post_init__(self):
        if self.diag is None:
            d = stencil_diagonal(self.model, self.shift)
            object.__setattr__(self, "diag", d if self.wall is None else d + self.wall)
        if (np.abs(self.diag) < 1e-300).any():
            raise SingularityError("stencil diagonal has (near-)zero entries")

    @property
    def wall_edges(self) -> tuple[float, float]:
        """(wall on row nx-1, wall on column ny-1); the only pattern _wall_term builds."""
        if self.wall is None:
            return 0.0, 0.0
        w = np.asarray(self.wall)
        wx, wy = float(w[-1, 0]), float(w[0, -1])
        expect = np.zeros_like(w)
        expect[-1, :] += wx
        expect[:, -1] += wy
        if not np.array_equal(expect, w):
            raise ConfigurationError("wall term must be constant on the high edges (multigrid.py:153-163)")
        return wx, wy

    def apply(self, u):
        """Level operator incl. wall term, fp64 on the GPU (multigrid.py:146-150)."""
        import torch

        from .device import to_device

        if isinstance(u, torch.Tensor):
            return apply_operator(u, self.model, self.shift, self.wall_edges)
        out = apply_operator(to_device(np.asarray(u), torch.complex128), self.model, self.shift, self.wall_edges)
        return out.cpu().numpy()


def _wall_term(shape, d_hi, h):
    """(1-d)/d/H^2 on the high edge of each axis whose wall sits d*H past the last node."""
    if min(d_hi) >= 1.0:
        return None
    w = np.zeros(shape)
    if d_hi[0] < 1.0:
        w[-1, :] += (1.0 - d_hi[0]) / d_hi[0] / h**2
    if d_hi[1] < 1.0:
        w[:, -1] += (1.0 - d_hi[1]) / d_hi[1] / h**2
    return w


@dataclass(frozen=True)
class GridHierarchy:
    """Immutable per-level operators for the V-cycle (multigrid.py:166-182)."""

    levels: tuple[Level, ...]
    relax_pre: int = 1
    relax_post: int = 1
    jacobi_damping: tuple[float, float] = CHEBYSHEV_DAMPING
    coarse_iters: int = 10

    @property
    def num_levels(self) -> int:
        return len(self.levels)

    @property
    def shape(self) -> tuple[int, int]:
        return self.levels[0].model.shape


def build_hierarchy(model: SlownessModel, shift: HelmholtzShift = PRECONDITIONER_SHIFT, num_levels: int = 3,
                    relax_pre: int = 1, relax_post: int = 1,
                    jacobi_damping: tuple[float, float] = CHEBYSHEV_DAMPING,
                    coarse_iters: int = 10) -> GridHierarchy:
    """Restrict the medium level by level (multigrid.py:185-215)."""
    levels = [Level(model, shift)]
    k2, gm, h = model.kappa_sq, model.gamma, model.h
    d_hi = (1.0, 1.0)
    for _ in range(num_levels - 1):
        _check_coarsenable(*k2.shape)
        parent = k2.shape
        k2 = restrict_media(k2)
        gm = np.clip(restrict_media(gm), 0.0, 1.0)
        h = 2.0 * h
        d_hi = tuple((d + (n % 2)) / 2 for d, n in zip(d_hi, parent))
        levels.append(Level(SlownessModel(k2, gm, model.omega, h), shift, _wall_term(k2.shape, d_hi, h)))
    return GridHierarchy(tuple(levels), relax_pre=relax_pre, relax_post=relax_post,
                         jacobi_damping=tuple(jacobi_damping), coarse_iters=coarse_iters)


# ------------------------------------------------------------ device hierarchy


class DeviceHierarchy:
    """Device-resident hierarchy for one or more slowness models of equal shape.

    Level l's mass term of every model is stacked into one complex64
    (n_models, nx_l, ny_l) tensor; the finest level also keeps the TRUE
    operator's mass in complex128 for the outer matvec.  ``hs`` is the
    hs_hierarchy_t handed to the C ABI.
    """

    def __init__(self, hierarchies, true_models=None):
        import torch

        from . import _lib
        from .device import to_device

        hierarchies = list(hierarchies)
        first = hierarchies[0]
        for g in hierarchies[1:]:
            if [lv.model.shape for lv in g.levels] != [lv.model.shape for lv in first.levels]:
                raise DimensionError("all hierarchies of a batch need identical level shapes")
            if (g.relax_pre, g.relax_post, tuple(g.jacobi_damping), g.coarse_iters) != (
                first.relax_pre, first.relax_post, tuple(first.jacobi_damping), first.coarse_iters):
                raise ConfigurationError("all hierarchies of a batch need identical cycle settings")
        if first.num_levels > 8:
            raise ConfigurationError("at most 8 levels")
        self.hierarchies = hierarchies
        self.n_models = len(hierarchies)
        self.shape = first.shape
        self.mass = []
        hs = _lib.HsHierarchy()
        hs.num_levels = first.num_levels
        hs.n_models = self.n_models
        for li, lv in enumerate(first.levels):
            stack = np.stack([mass_coefficient(g.levels[li].model, g.levels[li].shift) for g in hierarchies])
            t = to_device(stack, torch.complex64)
            self.mass.append(t)
            walls = [g.levels[li].wall_edges for g in hierarchies]
            if len(set(walls)) != 1:
                raise ConfigurationError("wall terms differ between models")
            hs.levels[li].nx, hs.levels[li].ny = lv.model.shape
            hs.levels[li].h = lv.model.h
            hs.levels[li].wall_x, hs.levels[li].wall_y = walls[0]
            hs.levels[li].mass = t.data_ptr()
        hs.relax_pre, hs.relax_post = first.relax_pre, first.relax_post
        hs.damping_pre, hs.damping_post = map(float, first.jacobi_damping)
        hs.coarse_iters = first.coarse_iters
        hs.coarse_damping = 0.8  # coarse_solve default (multigrid.py:233)
        self.hs = hs
        if true_models is None:
            true_models = [g.levels[0].model for g in hierarchies]
        from .fields import TRUE_SHIFT

        self.c_true = to_device(np.stack([mass_coefficient(m, TRUE_SHIFT) for m in true_models]),
                                torch.complex128)

    def workspace_bytes(self, B: int) -> int:
        from . import _lib

        return int(_lib.load().hs_vcycle_workspace_bytes(ctypes.byref(self.hs), B))


def device_hierarchy(hierarchy: GridHierarchy) -> DeviceHierarchy:
    """Cached DeviceHierarchy of a single GridHierarchy (uploaded on first use)."""
    cached = hierarchy.__dict__.get("_device")
    if cached is None:
        cached = DeviceHierarchy([hierarchy])
        object.__setattr__(hierarchy, "_device", cached)
    return cached


def run_vcycle(dh: DeviceHierarchy, rhs, u0=None, model_of=None):
    """Batched V-cycle on CUDA tensors: rhs/u0 (B, nx, ny) -> complex64 (B, nx, ny)."""
    import torch

    from . import _lib
    from .device import stream_handle, workspace

    rhs = rhs.to(torch.complex64).contiguous()
    B = rhs.shape[0]
    out = torch.empty_like(rhs)
    u0c = None if u0 is None else u0.to(torch.complex64).contiguous()
    ws_bytes = dh.workspace_bytes(B)
    ws = workspace(ws_bytes)
    status = torch.zeros(B, dtype=torch.int32, device=rhs.device)  # per RHS
    lib = _lib.load()
    _lib.check(
        lib.hs_vcycle(ctypes.byref(dh.hs), rhs.data_ptr(), None if u0c is None else u0c.data_ptr(),
                      out.data_ptr(), None if model_of is None else model_of.data_ptr(), B, ws.data_ptr(),
                      ws_bytes, status.data_ptr(), stream_handle()),
        "v_cycle",
    )
    codes = status.cpu().numpy()
    code = int(codes[np.nonzero(codes)[0][0]]) if codes.any() else 0
    if code:
        _lib.check(code, "coarse-grid GMRES")
    return out


# ----------------------------------------------------------- public functions


def _as_device_complex(a, dtype):
    import torch

    from .device import to_device

    return a.to(dtype).contiguous() if isinstance(a, torch.Tensor) else to_device(np.asarray(a), dtype)


def restrict_full_weighting(fine):
    """Full weighting centred on fine 2K+1, zero outside (multigrid.py:64-78), on the GPU.

    float64/complex128 inputs use the fp64 kernel, float32/complex64 the fp32
    one; real inputs return real outputs.
    """
    import torch

    from . import _lib
    from .device import stream_handle

    was_np = not isinstance(fine, torch.Tensor)
    arr = np.asarray(fine) if was_np else fine
    nx, ny = arr.shape[-2:]
    _check_coarsenable(nx, ny)
    f64 = arr.dtype in (np.float64, np.complex128, torch.float64, torch.complex128)
    real = arr.dtype in (np.float64, np.float32, torch.float64, torch.float32)
    ct = torch.complex128 if f64 else torch.complex64
    src = _as_device_complex(arr, ct)
    B = int(np.prod(src.shape[:-2])) if src.dim() > 2 else 1
    cx, cy = coarse_shape((nx, ny))
    out = torch.empty(tuple(src.shape[:-2]) + (cx, cy), dtype=ct, device=src.device)
    _lib.check(_lib.load().hs_restrict(src.data_ptr(), out.data_ptr(), B, nx, ny, int(f64), stream_handle()),
               "restrict_full_weighting")
    if real:
        out = out.real.contiguous()
    return out.cpu().numpy() if was_np else out


def prolong_bilinear(coarse, fine_shape):
    """Bilinear interpolation P = 4 R^T (multigrid.py:81-114), on the GPU."""
    import torch

    from . import _lib
    from .device import stream_handle

    was_np = not isinstance(coarse, torch.Tensor)
    arr = np.asarray(coarse) if was_np else coarse
    cx, cy = arr.shape[-2:]
    nx, ny = fine_shape
    if not (2 * cx <= nx <= 2 * cx + 1 and 2 * cy <= ny <= 2 * cy + 1):
        raise DimensionError(f"cannot prolong {tuple(arr.shape)} onto {tuple(fine_shape)}; expected about 2x")
    f64 = arr.dtype in (np.float64, np.complex128, torch.float64, torch.complex128)
    real = arr.dtype in (np.float64, np.float32, torch.float64, torch.float32)
    ct = torch.complex128 if f64 else torch.complex64
    src = _as_device_complex(arr, ct)
    B = int(np.prod(src.shape[:-2])) if src.dim() > 2 else 1
    out = torch.empty(tuple(src.shape[:-2]) + (nx, ny), dtype=ct, device=src.device)
    _lib.check(_lib.load().hs_prolong(src.data_ptr(), out.data_ptr(), B, cx, cy, nx, ny, int(f64), stream_handle()),
               "prolong_bilinear")
    if real:
        out = out.real.contiguous()
    return out.cpu().numpy() if was_np else out


def jacobi_relax(u, rhs, level: Level, sweeps: int, damping: float = 0.8):
    """Damped Jacobi u <- u + w D^-1 (rhs - A u), ``sweeps`` times (multigrid.py:218-229); complex64 on the GPU."""
    import torch

    from . import _lib
    from .device import stream_handle

    was_np = not isinstance(u, torch.Tensor)
    if sweeps <= 0:  # the reference loop body never runs: u comes back unchanged
        return u
    cur = _as_device_complex(u, torch.complex64)
    r = _as_device_complex(rhs, torch.complex64)
    if tuple(cur.shape[-2:]) != tuple(level.model.shape):
        raise DimensionError(f"field {tuple(cur.shape[-2:])} does not match level {level.model.shape}")
    B = int(np.prod(cur.shape[:-2])) if cur.dim() > 2 else 1
    mass = torch.from_numpy(mass_coefficient(level.model, level.shift)).to(cur.device, torch.complex64)
    lv = _lib.HsLevel()
    lv.nx, lv.ny = level.model.shape
    lv.h = level.model.h
    lv.wall_x, lv.wall_y = level.wall_edges
    lv.mass = mass.data_ptr()
    lib = _lib.load()
    for _ in range(sweeps):
        nxt = torch.empty_like(cur)
        _lib.check(lib.hs_jacobi(cur.data_ptr(), r.data_ptr(), nxt.data_ptr(), ctypes.byref(lv), None, B,
                                 float(damping), stream_handle()), "jacobi_relax")
        cur = nxt
    out = cur.to(torch.complex128)
    return out.cpu().numpy() if was_np else out


COARSE_MAX_ITERS = 16  # hs::kCoarseMaxIters (csrc/vcycle.h)


def fused_cycle(hierarchy: GridHierarchy) -> bool:
    """Whether the fused device V-cycle (csrc/vcycle.cu) implements these cycle settings.

    It fuses exactly one pre- and one post-smoothing sweep into the down / up legs and keeps the
    coarse GMRES basis on chip for up to 16 steps (BASELINE: V(1,1), 10 coarse steps).  Any other
    ``relax_pre`` / ``relax_post`` / ``coarse_iters`` the reference accepts (multigrid.py:185-193)
    runs the general device cycle below instead.
    """
    return hierarchy.relax_pre == 1 and hierarchy.relax_post == 1 and 1 <= hierarchy.coarse_iters <= COARSE_MAX_ITERS


def _v_cycle_general(rhs, u0, hierarchy: GridHierarchy):
    """V(relax_pre, relax_post) cycle from the device primitives, any sweep / coarse-step counts.

    The reference's recursion (multigrid.py:264-274) on CUDA tensors: damped Jacobi (hs_jacobi), the
    level operator in fp64 (hs_helm_apply), full-weighting restriction and bilinear prolongation
    (hs_restrict / hs_prolong), the coarse solve (fused kernel or, beyond 16 steps, the generic device
    FGMRES).  Batched (B, nx, ny) or single (nx, ny) complex128 tensors in and out.
    """
    import torch

    def cycle(r, u, depth):
        lv = hierarchy.levels[depth]
        if depth == len(hierarchy.levels) - 1:
            return coarse_solve(r, lv, hierarchy.coarse_iters)
        w0, w1 = hierarchy.jacobi_damping
        u = jacobi_relax(u, r, lv, hierarchy.relax_pre, w0).to(torch.complex128)
        rc = restrict_full_weighting(r - lv.apply(u)).to(torch.complex128)
        e = cycle(rc, torch.zeros_like(rc), depth + 1)
        u = u + prolong_bilinear(e, tuple(r.shape[-2:])).to(torch.complex128)
        return jacobi_relax(u, r, lv, hierarchy.relax_post, w1).to(torch.complex128)

    if len(hierarchy.levels) == 1:  # multigrid.py:266-267: u0 ignored
        return coarse_solve(rhs, hierarchy.levels[0], hierarchy.coarse_iters)
    return cycle(rhs, torch.zeros_like(rhs) if u0 is None else u0, 0)


def coarse_solve(rhs, level: Level, iters: int = 10, damping: float = 0.8):
    """GMRES(iters) with a damped-Jacobi preconditioner, zero guess (multigrid.py:232-244)."""
    import torch

    was_np = not isinstance(rhs, torch.Tensor)
    if iters > COARSE_MAX_ITERS:
        # The fused coarse kernel keeps its GMRES basis on chip for up to 16 steps.  Longer runs (the
        # reference's own tests use 20-40, test_multigrid.py:201-229) take the generic device FGMRES
        # (krylov.fgmres: complex128 basis on the GPU, the level operator in fp64) with the same
        # arguments as multigrid.py:243: tol 1e-12, max_iter = restart = iters, M = damping / diag.
        from .device import to_device
        from .krylov import fgmres

        s = to_device(damping / np.asarray(level.diag), torch.complex128)
        b = rhs if not was_np else to_device(np.asarray(rhs), torch.complex128)
        b = b.to(torch.complex128)
        if b.dim() > 2:
            x = torch.stack([coarse_solve(bi, level, iters, damping) for bi in b])
        else:
            x, _ = fgmres(level.apply, lambda r: s * r, b, None, 1e-12, iters, iters)
        return x.cpu().numpy() if was_np else x
    one = GridHierarchy((level,), coarse_iters=iters)
    dh = DeviceHierarchy([one])
    dh.hs.coarse_damping = float(damping)
    r = _as_device_complex(rhs, torch.complex64)
    batched = r.dim() > 2
    out = run_vcycle(dh, r if batched else r[None])
    out = (out if batched else out[0]).to(torch.complex128)
    return out.cpu().numpy() if was_np else out


def v_cycle(rhs, u0, hierarchy: GridHierarchy):
    """One V(relax_pre, relax_post) cycle on the shifted operator (multigrid.py:247-274).

    Linear in (rhs, u0); u0 = None means a zero initial guess.  numpy in ->
    numpy complex128 out; CUDA tensors (optionally batched (B, nx, ny)) stay
    on the device.
    """
    import torch

    if tuple(np.shape(rhs)[-2:]) != tuple(hierarchy.shape):
        raise DimensionError(f"rhs {tuple(np.shape(rhs))} does not match hierarchy finest grid {hierarchy.shape}")
    if u0 is not None and tuple(np.shape(u0)) != tuple(np.shape(rhs)):
        raise DimensionError(f"u0 {tuple(np.shape(u0))} does not match rhs {tuple(np.shape(rhs))}")
    was_np = not isinstance(rhs, torch.Tensor)
    if not fused_cycle(hierarchy):
        out = _v_cycle_general(_as_device_complex(rhs, torch.complex128),
                               None if u0 is None else _as_device_complex(u0, torch.complex128), hierarchy)
        return out.cpu().numpy() if was_np else out
    r = _as_device_complex(rhs, torch.complex64)
    u = None if u0 is None else _as_device_complex(u0, torch.complex64)
    batched = r.dim() > 2
    if not batched:
        r = r[None]
        u = None if u is None else u[None]
    out = run_vcycle(device_hierarchy(hierarchy), r, u)
    out = (out if batched else out[0]).to(torch.complex128)
    return out.cpu().numpy() if was_np else out
