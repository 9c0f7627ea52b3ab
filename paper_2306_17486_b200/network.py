"""The encoder-solver network -- the ``helmsolve.network`` module the reference
imports (``krylov.py:201``) but never shipped.

Architecture: ARCH.md (parameter layout and seeded init in ``netparams``).
The two functions the reference protocol calls keep their names and roles:

* ``precompute_encodings(net, model)`` -- the encoder, once per slowness
  model (``krylov.py:205-206``);
* ``preconditioner_estimate(net, encodings, r)`` -- the solver U-Net applied to
  a Krylov vector, returning the V-cycle's initial guess
  ``u0 = (h^2/64) net(r[:nx-1, :ny-1])`` zero-padded (``krylov.py:225-226``).

Both run on the GPU through the C ABI (``hs_net_encode`` / ``hs_net_forward``):
float32 NHWC activations, batch norm folded into the convolutions, fused
epilogues, the implicit layer through the FFT.
"""
from __future__ import annotations

import ctypes

import numpy as np

from .errors import DimensionError
from .netparams import init_params

BN_EPS = 1e-5


class EncoderSolverNet:
    """Host-side parameters of one network (ARCH.md); ``levels = len(channels)``."""

    def __init__(self, params: dict, channels):
        self.params = {k: np.asarray(v) for k, v in params.items()}
        self.channels = tuple(int(c) for c in channels)
        self.levels = len(self.channels)
        self._device = {}

    @classmethod
    def seeded(cls, channels=(16, 32, 64), seed: int = 0) -> "EncoderSolverNet":
        return cls(init_params(tuple(channels), seed), channels)

    def dims(self, shape):
        ix, iy = shape[0] - 1, shape[1] - 1
        f = 2 ** (self.levels - 1)
        if ix % f or iy % f:
            raise DimensionError(f"network grid {(ix, iy)} not divisible by {f}")
        return ix, iy


def _fold(params, name, transposed=False, bn=True):
    """conv (+bias) -> BN(inference) folded into [cout][3][3][cin] weights and a bias."""
    w = params[name + ".w"].astype(np.float64)
    b = params[name + ".b"].astype(np.float64)
    if transposed:
        w = w.transpose(1, 0, 2, 3)  # (cin, cout, 3, 3) -> (cout, cin, 3, 3)
    if bn:
        scale = params[name + ".bn.gamma"].astype(np.float64) / np.sqrt(
            params[name + ".bn.var"].astype(np.float64) + BN_EPS)
        w = w * scale[:, None, None, None]
        b = (b - params[name + ".bn.mean"]) * scale + params[name + ".bn.beta"]
    return np.ascontiguousarray(w.transpose(0, 2, 3, 1)).astype(np.float32), b.astype(np.float32)


class DeviceNet:
    """A network prepared for one grid shape: folded weights, Green spectrum, hs_net_t."""

    def __init__(self, net: EncoderSolverNet, shape, h: float):
        import torch

        from . import _lib
        from .device import require_cuda, stream_handle

        self.net = net
        self.shape = tuple(shape)
        ix, iy = net.dims(shape)
        dev = require_cuda()
        self._keep = []
        d = _lib.HsNetDesc()
        d.levels = net.levels
        for i, c in enumerate(net.channels):
            d.channels[i] = c
        d.ix, d.iy = ix, iy
        d.nx, d.ny = shape
        d.out_scale = float(np.float32(h * h / 64.0))
        p = net.params

        def conv(slot, name, cin, cout, stride=1, transposed=False, bn=True, act=True):
            w, b = _fold(p, name, transposed, bn)
            wt, bt = torch.from_numpy(w).to(dev), torch.from_numpy(b).to(dev)
            self._keep += [wt, bt]
            slot.cin, slot.cout, slot.stride = cin, cout, stride
            slot.transposed, slot.softplus = int(transposed), int(act)
            slot.w, slot.b = wt.data_ptr(), bt.data_ptr()

        C = net.channels
        for side, stem, ra, rb, down in (("enc", d.enc_stem, d.enc_res_a, d.enc_res_b, d.enc_down),
                                         ("sol", d.sol_stem, d.sol_res_a, d.sol_res_b, d.sol_down)):
            conv(stem, f"{side}.stem", 2, C[0])
            for lv in range(net.levels):
                if lv:
                    conv(down[lv], f"{side}.down{lv}", C[lv - 1], C[lv], stride=2)
                conv(ra[lv], f"{side}.res{lv}.a", C[lv], C[lv])
                conv(rb[lv], f"{side}.res{lv}.b", C[lv], C[lv], bn=False, act=False)
        for lv in range(1, net.levels):
            conv(d.sol_up[lv], f"sol.up{lv}", C[lv], C[lv - 1], stride=2, transposed=True)
            conv(d.sol_ures_a[lv - 1], f"sol.ures{lv - 1}.a", C[lv - 1], C[lv - 1])
            conv(d.sol_ures_b[lv - 1], f"sol.ures{lv - 1}.b", C[lv - 1], C[lv - 1], bn=False, act=False)
        conv(d.sol_head, "sol.head", C[0], 2, bn=False, act=False)
        kw = torch.from_numpy(np.ascontiguousarray(p["sol.implicit.w"].astype(np.complex64))).to(dev)
        self._keep.append(kw)
        d.implicit_w = kw.data_ptr()
        self.desc = d
        handle = ctypes.c_void_p()
        _lib.check(_lib.load().hs_net_create(ctypes.byref(handle), ctypes.byref(d), stream_handle()), "hs_net_create")
        self.handle = handle
        self.encodings = None
        self.ix, self.iy = ix, iy

    def __del__(self):
        try:
            from . import _lib

            if getattr(self, "handle", None):
                _lib.load().hs_net_destroy(self.handle)
        except Exception:  # pragma: no cover - interpreter shutdown
            pass

    def encode(self, models):
        """Encoder on (kappa^2, gamma) of each model -> per-level NHWC float32 tensors."""
        import torch

        from . import _lib
        from .device import require_cuda, stream_handle, workspace

        dev = require_cuda()
        media = np.stack([np.stack([m.kappa_sq[: self.ix, : self.iy], m.gamma[: self.ix, : self.iy]], axis=-1)
                          for m in models]).astype(np.float32)
        md = torch.from_numpy(np.ascontiguousarray(media)).to(dev)
        M = len(models)
        enc = [torch.empty((M, self.ix >> lv, self.iy >> lv, c), dtype=torch.float32, device=dev)
               for lv, c in enumerate(self.net.channels)]
        ptrs = (ctypes.c_void_p * 8)(*[e.data_ptr() for e in enc])
        lib = _lib.load()
        nb = int(lib.hs_net_encode_workspace_bytes(self.handle, M))
        ws = workspace(nb)
        _lib.check(lib.hs_net_encode(self.handle, md.data_ptr(), M, ctypes.cast(ptrs, ctypes.c_void_p), ws.data_ptr(),
                                     nb, stream_handle()),
                   "precompute_encodings")
        self.encodings = enc
        return enc

    def set_encodings(self, enc):
        """Point the network at stacked per-level encodings (n_models, h_l, w_l, c_l) (recomputes no-op)."""
        from . import _lib

        lib = _lib.load()
        ptrs = (ctypes.c_void_p * 8)(*[e.data_ptr() for e in enc])
        _lib.check(lib.hs_net_set_encodings(self.handle, len(enc), ctypes.cast(ptrs, ctypes.c_void_p)),
                   "set encodings")
        self.encodings = enc

    def forward(self, r, model_of=None):
        """u0 = (h^2/64) net(r): r complex64 CUDA tensor (B, nx, ny) -> complex64 (B, nx, ny)."""
        import torch

        from . import _lib
        from .device import stream_handle, workspace

        r = r.to(torch.complex64).contiguous()
        B = r.shape[0]
        u0 = torch.empty_like(r)
        lib = _lib.load()
        nb = int(lib.hs_net_workspace_bytes(self.handle, B))
        ws = workspace(nb)
        _lib.check(lib.hs_net_forward(self.handle, r.data_ptr(), u0.data_ptr(),
                                      None if model_of is None else model_of.data_ptr(), B, ws.data_ptr(), nb,
                                      stream_handle()), "preconditioner_estimate")
        return u0


class Encodings:
    """Encoder output for one slowness model (device NHWC tensors per level)."""

    def __init__(self, model, tensors, device_net):
        self.model = model
        self.tensors = tensors
        self.device_net = device_net


def _device_net(net: EncoderSolverNet, model) -> DeviceNet:
    key = (tuple(model.shape), float(model.h))
    dn = net._device.get(key)
    if dn is None:
        dn = DeviceNet(net, model.shape, model.h)
        net._device[key] = dn
    return dn


def precompute_encodings(net: EncoderSolverNet, model) -> Encodings:
    """Encoder applied once per slowness model (krylov.py:205-206)."""
    dn = _device_net(net, model)
    return Encodings(model, [t[0:1].clone() for t in dn.encode([model])], dn)


def preconditioner_estimate(net: EncoderSolverNet, encodings: Encodings, r):
    """The network's error estimate for residual r, used as the V-cycle's u0 (krylov.py:225-226)."""
    import torch

    from .device import to_device

    was_np = not isinstance(r, torch.Tensor)
    rd = to_device(r, torch.complex64)
    batched = rd.dim() == 3
    dn = encodings.device_net
    dn.set_encodings(encodings.tensors)
    out = dn.forward(rd if batched else rd[None])
    out = out if batched else out[0]
    return out.cpu().numpy() if was_np else out


def device_network(net: EncoderSolverNet, models, encodings, dh) -> DeviceNet:
    """DeviceNet with the stacked encodings of every model of a batch (engine use)."""
    import torch

    dn = _device_net(net, models[0])
    if encodings is None or any(e is None for e in encodings):
        dn.encode(models)
    else:
        dn.set_encodings([torch.cat([e.tensors[lv] for e in encodings], dim=0).contiguous()
                          for lv in range(net.levels)])
    return dn, list(dn.encodings)
