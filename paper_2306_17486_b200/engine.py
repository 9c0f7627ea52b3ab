"""Batched solve engine: many right-hand sides (and slowness models) per call.

This is the data-parallel core behind ``krylov.solve_helmholtz`` and
``krylov.solve_with_learned_preconditioner``: one ``hs_fgmres_solve`` call runs
the reference's flexible GMRES (``krylov.py:39-146``) for every RHS of the
batch at once, device resident, with per-RHS windows, histories and stopping.
The host only allocates buffers and reads the results back at the end.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .device import require_cuda, stream_handle, workspace

MAX_WINDOW = 32  # hs::kMaxRestart (csrc/krylov.h): per-RHS Hessenberg / Givens state lives in RhsState


@dataclass
class BatchResult:
    """Device iterate plus host copies of the per-RHS reports."""

    x: torch.Tensor  # (B, nx, ny) complex128, device
    histories: list  # list[list[float]]
    iterations: np.ndarray
    converged: np.ndarray
    status: np.ndarray


class Engine:
    """FGMRES over a DeviceHierarchy, optionally with the device network."""

    def __init__(self, dh, net=None, net_encodings=None):
        self.dh = dh
        self.net = net
        # this engine's own per-level encodings (n_models, h_l, w_l, c_l): the DeviceNet is shared per
        # (net, shape), so another solver may have pointed it at a different model set since
        self.net_encodings = net_encodings
        self._ws = None

    def _workspace(self, nbytes: int) -> torch.Tensor:
        if self._ws is None or self._ws.numel() < nbytes:
            self._ws = workspace(nbytes)
        return self._ws

    def fgmres(self, b: torch.Tensor, x0: torch.Tensor | None, tol, max_iter: int, restart: int | None,
               model_of: torch.Tensor | None = None, use_net: bool = False, iter_caps=None) -> BatchResult:
        """One batched hs_fgmres_solve; ``iter_caps`` (B,) optionally caps each RHS below max_iter."""
        dev = require_cuda()
        b = b.to(device=dev, dtype=torch.complex128).contiguous()
        B = b.shape[0]
        nx, ny = b.shape[-2:]
        if (nx, ny) != tuple(self.dh.shape):
            from .errors import DimensionError

            raise DimensionError(f"rhs {(nx, ny)} does not match hierarchy {self.dh.shape}")
        window = max_iter if restart is None else min(restart, max_iter)
        if window > MAX_WINDOW:
            from .errors import ConfigurationError

            raise ConfigurationError(
                f"FGMRES window {window} (restart={restart}, max_iter={max_iter}) exceeds the device solver's "
                f"{MAX_WINDOW}-vector Hessenberg; pass restart <= {MAX_WINDOW} (BASELINE uses 10/20/30)")
        tol_t = torch.as_tensor(np.broadcast_to(np.asarray(tol, dtype=np.float64), (B,)).copy(), device=dev)
        x = torch.empty_like(b)
        x0c = None if x0 is None else x0.to(device=dev, dtype=torch.complex128).contiguous()
        hist = torch.zeros((B, max_iter + 2), dtype=torch.float64, device=dev)
        ints = torch.zeros((4, B), dtype=torch.int32, device=dev)
        args = _lib.HsSolveArgs()
        args.B, args.max_iter, args.restart = B, int(max_iter), int(window)
        args.b, args.x0, args.x = b.data_ptr(), None if x0c is None else x0c.data_ptr(), x.data_ptr()
        args.tol = tol_t.data_ptr()
        args.c_true = self.dh.c_true.data_ptr()
        args.model_of = None if model_of is None else model_of.data_ptr()
        args.hist = hist.data_ptr()
        args.hist_len, args.iterations = ints[0].data_ptr(), ints[1].data_ptr()
        args.converged, args.status = ints[2].data_ptr(), ints[3].data_ptr()
        caps = None
        if iter_caps is not None:
            caps = torch.as_tensor(np.asarray(iter_caps, dtype=np.int32), device=dev)
            args.iter_cap = caps.data_ptr()
        net_handle = self.net.handle if (use_net and self.net is not None) else None
        if net_handle is not None and self.net_encodings is not None:
            self.net.set_encodings(self.net_encodings)
        lib = _lib.load()
        nbytes = int(lib.hs_fgmres_workspace_bytes(ctypes.byref(self.dh.hs), net_handle, B, nx, ny,
                                                   int(window), int(max_iter)))
        if nbytes == 0:
            _lib.check(_lib.HS_ECONFIG, "fgmres workspace")
        ws = self._workspace(nbytes)
        _lib.check(lib.hs_fgmres_solve(ctypes.byref(self.dh.hs), net_handle, ctypes.byref(args), ws.data_ptr(),
                                       nbytes, stream_handle()), "fgmres")
        ints_h = ints.cpu().numpy()
        hist_h = hist.cpu().numpy()
        histories = [hist_h[i, : ints_h[0, i]].tolist() for i in range(B)]
        return BatchResult(x, histories, ints_h[1].copy(), ints_h[2].astype(bool), ints_h[3].copy())


def raise_for_status(res: BatchResult, index: int = 0):
    """Raise the reference's exception for a failed RHS (krylov.py:96-99, :130-134)."""
    from .errors import NumericalError, SolverError

    code = int(res.status[index])
    if code == _lib.HS_ENONFINITE:
        raise NumericalError(f"non-finite Krylov vector at iteration {int(res.iterations[index]) + 1}")
    if code == _lib.HS_EBREAKDOWN:
        it = int(res.iterations[index])
        est = res.histories[index][-1] if res.histories[index] else float("nan")
        raise SolverError(f"Arnoldi breakdown at iteration {it} with relative residual {est:.3e}")
    if code:
        _lib.check(code, "fgmres")
