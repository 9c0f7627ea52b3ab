"""Network training on the GPU (SPEC.md ``[MODULE] trainer``, reference SPEC.md:454-507).

The reference ships no trainer, only the autodiff it would run on (``autodiff.py``) and the
contract in SPEC.md.  One ``Trainer.step`` is one device pass through the C ABI
(``hs_trainer_step``): forward with training-mode batch norm, the SPEC ``mse_loss`` of the
preconditioner estimate ``u0 = (h^2/64) net(r)`` against the true error ``e`` (paper Eq. 4.10),
the backward pass with the reference autodiff's rules (conv / transposed conv / batch norm /
softplus / implicit layer / Green function), and Adam (torch.optim.Adam defaults).  Encoder and
solver are trained jointly (PAPER §4.1).  ``train`` runs the SPEC schedule: round-robin over grid
sizes in blocks of ``epochs_per_size_block`` epochs, learning rate divided by 10 every
``lr_decay_epochs`` epochs, per-epoch train / validation MSE.

The CPU restatement used by the tests is ``oracle/train_oracle.py``.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import dist as hdist
from . import netparams
from .errors import ConfigurationError, DimensionError, NumericalError
from .network import EncoderSolverNet

WHICH_PARAMS, WHICH_GRADS, WHICH_M, WHICH_V = range(4)


def flatten(params: dict, channels) -> np.ndarray:
    """netparams.param_spec order -> one float32 vector (complex as (re, im) pairs)."""
    parts = []
    for name, shape, _, _ in netparams.param_spec(tuple(channels)):
        v = np.asarray(params[name])
        if v.shape != tuple(shape):
            raise DimensionError(f"{name}: shape {v.shape} != {shape}")
        if np.iscomplexobj(v):
            v = np.stack([v.real, v.imag], axis=-1)
        parts.append(np.ascontiguousarray(v, dtype=np.float32).ravel())
    return np.concatenate(parts)


def unflatten(vec: np.ndarray, channels) -> dict:
    spec = netparams.param_spec(tuple(channels))
    need = sum(int(np.prod(s)) * (2 if k == "implicit" else 1) for _, s, k, _ in spec)
    if vec.size != need:
        raise DimensionError(f"parameter vector has {vec.size} floats, layout needs {need}")
    out, off = {}, 0
    for name, shape, kind, _ in spec:
        n = int(np.prod(shape))
        if kind == "implicit":
            pr = vec[off : off + 2 * n].reshape(tuple(shape) + (2,))
            out[name] = (pr[..., 0] + 1j * pr[..., 1]).astype(np.complex64)
            off += 2 * n
        else:
            out[name] = vec[off : off + n].reshape(shape).astype(np.float32)
            off += n
    return out


def media_planes(models, levels: int) -> np.ndarray:
    """(n_models, 2, Ix, Iy) float32 (kappa^2, gamma) on the network grid (ARCH.md)."""
    ix, iy = models[0].shape[0] - 1, models[0].shape[1] - 1
    return np.stack([np.stack([m.kappa_sq[:ix, :iy], m.gamma[:ix, :iy]]) for m in models]).astype(np.float32)


def mse_loss(pred, target) -> float:
    """SPEC ``mse_loss``: (1/m) sum_i ||pred_i - target_i||^2, complex norm (host reference form)."""
    pred, target = np.asarray(pred), np.asarray(target)
    if pred.shape != target.shape:
        raise DimensionError(f"mse_loss shapes {pred.shape} vs {target.shape}")
    d = pred - target
    return float(np.sum(d.real**2 + d.imag**2) / pred.shape[0])


class Trainer:
    """Device training state for one grid shape and batch size (parameters, gradients, Adam moments)."""

    def __init__(self, net: EncoderSolverNet, shape, h: float, batch: int, lr: float = 1e-3,
                 betas=(0.9, 0.999), eps: float = 1e-8):
        from . import _lib
        from .device import require_cuda, stream_handle

        require_cuda()
        self.channels = tuple(net.channels)
        self.shape = tuple(int(s) for s in shape)
        self.h = float(h)
        self.batch = int(batch)
        self.adam = _lib.HsAdam(lr, betas[0], betas[1], eps)
        d = _lib.HsTrainDesc()
        d.levels = len(self.channels)
        for i, c in enumerate(self.channels):
            d.channels[i] = c
        d.nx, d.ny = self.shape
        d.batch = self.batch
        d.h = self.h
        self._desc = d
        lib = _lib.load()
        self.n = int(lib.hs_train_param_count(ctypes.byref(d)))
        vec = flatten(net.params, self.channels)
        if vec.size != self.n:
            raise DimensionError(f"parameter vector {vec.size} != library layout {self.n}")
        handle = ctypes.c_void_p()
        _lib.check(lib.hs_trainer_create(ctypes.byref(handle), ctypes.byref(d), vec.ctypes.data, stream_handle()),
                   "trainer create")
        self.handle = handle
        self.steps = 0

    def __del__(self):
        try:
            from . import _lib

            if getattr(self, "handle", None):
                _lib.load().hs_trainer_destroy(self.handle)
        except Exception:  # pragma: no cover - interpreter shutdown
            pass

    @property
    def lr(self) -> float:
        return float(self.adam.lr)

    @lr.setter
    def lr(self, value: float):
        self.adam.lr = float(value)

    def step(self, media, r, e, model_of=None, update: bool = True) -> float:
        """One step on a batch: media (n_models, 2, Ix, Iy), r / e (batch, nx, ny) complex -> loss."""
        import torch

        from . import _lib
        from .device import stream_handle, to_device

        md = media if isinstance(media, torch.Tensor) and media.dtype == torch.float32 else to_device(media, torch.float32)
        md = md.contiguous()
        rd = to_device(r, torch.complex128)
        ed = to_device(e, torch.complex128)
        if rd.shape != (self.batch,) + self.shape or ed.shape != rd.shape:
            raise DimensionError(f"batch shape {tuple(rd.shape)} / {tuple(ed.shape)} != {(self.batch,) + self.shape}")
        owner = np.zeros(self.batch, dtype=np.int32) if model_of is None else np.asarray(model_of, dtype=np.int32)
        owner = np.ascontiguousarray(owner)
        loss = ctypes.c_double()
        lib = _lib.load()
        data_parallel = update and hdist.world_size() > 1
        _lib.check(lib.hs_trainer_step(self.handle, md.data_ptr(), int(md.shape[0]), owner.ctypes.data,
                                       rd.data_ptr(), ed.data_ptr(),
                                       ctypes.byref(self.adam) if update and not data_parallel else None,
                                       ctypes.byref(loss), stream_handle()), "training step")
        value = float(loss.value)
        if data_parallel:
            # data-parallel step: average the gradient vector over ranks (NCCL), then Adam
            if getattr(self, "_gbuf", None) is None:
                self._gbuf = torch.empty(self.n, dtype=torch.float32, device=rd.device)
            _lib.check(lib.hs_trainer_grads(self.handle, self._gbuf.data_ptr(), 0, stream_handle()), "grads out")
            hdist.allreduce_mean(self._gbuf)
            _lib.check(lib.hs_trainer_grads(self.handle, self._gbuf.data_ptr(), 1, stream_handle()), "grads in")
            _lib.check(lib.hs_trainer_apply(self.handle, ctypes.byref(self.adam), stream_handle()), "adam")
            value = hdist.reduce_scalar(value, "sum") / hdist.world_size()
        if update:
            self.steps += 1
        return value

    def _read(self, which: int) -> np.ndarray:
        from . import _lib
        from .device import stream_handle

        out = np.empty(self.n, dtype=np.float32)
        _lib.check(_lib.load().hs_trainer_read(self.handle, which, out.ctypes.data, stream_handle()), "trainer read")
        return out

    def _write(self, which: int, vec: np.ndarray, step: int = -1):
        from . import _lib
        from .device import stream_handle

        vec = np.ascontiguousarray(vec, dtype=np.float32)
        if vec.size != self.n:
            raise DimensionError(f"state vector {vec.size} != {self.n}")
        _lib.check(_lib.load().hs_trainer_write(self.handle, which, vec.ctypes.data, int(step), stream_handle()),
                   "trainer write")

    def params(self) -> dict:
        return unflatten(self._read(WHICH_PARAMS), self.channels)

    def grads(self) -> dict:
        """Gradients of the last step (running-statistics entries are zero)."""
        return unflatten(self._read(WHICH_GRADS), self.channels)

    def network(self) -> EncoderSolverNet:
        return EncoderSolverNet(self.params(), self.channels)

    def state(self) -> dict:
        """Checkpoint: parameters, Adam moments and step count (flat float32 vectors)."""
        return {"params": self._read(WHICH_PARAMS), "m": self._read(WHICH_M), "v": self._read(WHICH_V),
                "step": self.steps, "lr": self.lr}

    def load_state(self, state: dict):
        self._write(WHICH_PARAMS, state["params"])
        self._write(WHICH_M, state["m"])
        self._write(WHICH_V, state["v"], step=int(state["step"]))
        self.steps = int(state["step"])


CHECKPOINT_FORMAT = "helmsolve-checkpoint v1"


def _arch_hash(channels) -> str:
    import hashlib

    spec = netparams.param_spec(tuple(channels))
    text = ";".join(f"{n}:{'x'.join(map(str, s))}:{k}" for n, s, k, _ in spec)
    return hashlib.sha256(text.encode()).hexdigest()[:16]


def save_checkpoint(path: str, state: dict, channels):
    """SPEC.md:384 checkpoint: a text manifest (key: value lines -- format, architecture hash, training
    metadata, then every tensor's name, shape, dtype and offset) plus ``<path>.bin``, one flat
    little-endian float32 blob in manifest order: the parameters (netparams.param_spec order, complex
    kernels as (re, im) pairs, running batch-norm statistics included), then Adam's m and v.
    Atomic (SPEC trainer concurrency model): both files are written to temporaries and renamed, the
    manifest last, so a reader never sees a manifest without its blob."""
    import os

    channels = tuple(int(c) for c in channels)
    params, m, v = (np.ascontiguousarray(state[k], dtype="<f4") for k in ("params", "m", "v"))
    lines = [f"format: {CHECKPOINT_FORMAT}", f"architecture: {_arch_hash(channels)}",
             f"channels: {','.join(map(str, channels))}", f"step: {int(state['step'])}", f"lr: {float(state['lr'])!r}",
             f"blob: {os.path.basename(path)}.bin", "blob_dtype: float32 little-endian",
             f"blob_floats: {params.size + m.size + v.size}"]
    off = 0
    for group, vec in (("param", params), ("adam_m", m), ("adam_v", v)):
        goff = 0
        for name, shape, kind, _ in netparams.param_spec(channels):
            n = int(np.prod(shape)) * (2 if kind == "implicit" else 1)
            dtype = "complex64 as (re, im) float32 pairs" if kind == "implicit" else "float32"
            lines.append(f"tensor: {group} {name} shape={'x'.join(map(str, shape))} dtype={dtype} offset={off + goff}")
            goff += n
        if goff != vec.size:
            raise DimensionError(f"{group}: {vec.size} floats, layout needs {goff}")
        off += goff
    for suffix, payload in ((".bin", np.concatenate([params, m, v]).tobytes()),
                            ("", ("\n".join(lines) + "\n").encode())):
        tmp = path + suffix + ".tmp"
        with open(tmp, "wb") as f:
            f.write(payload)
        os.replace(tmp, path + suffix)


def load_checkpoint(path: str) -> dict:
    """Read a SPEC manifest + blob checkpoint (``save_checkpoint``); round-1 ``.npz`` files still load."""
    import os

    with open(path, "rb") as f:
        head = f.read(len(CHECKPOINT_FORMAT) + 8)
    if not head.startswith(b"format:"):
        with np.load(path) as z:
            return {"params": z["params"], "m": z["m"], "v": z["v"], "step": int(z["step"]), "lr": float(z["lr"]),
                    "channels": tuple(int(c) for c in z["channels"])}
    meta = {}
    with open(path) as f:
        for line in f:
            k, _, val = line.rstrip("\n").partition(": ")
            if k != "tensor":
                meta[k] = val
    if meta.get("format") != CHECKPOINT_FORMAT:
        raise ConfigurationError(f"{path}: unknown checkpoint format {meta.get('format')!r}")
    channels = tuple(int(c) for c in meta["channels"].split(","))
    if meta["architecture"] != _arch_hash(channels):
        raise ConfigurationError(f"{path}: architecture hash does not match channels {channels}")
    blob = np.fromfile(os.path.join(os.path.dirname(path), meta["blob"]), dtype="<f4")
    if blob.size != int(meta["blob_floats"]) or blob.size % 3:
        raise DimensionError(f"{path}: blob holds {blob.size} floats, manifest says {meta['blob_floats']}")
    n = blob.size // 3
    return {"params": blob[:n].astype(np.float32), "m": blob[n : 2 * n].astype(np.float32),
            "v": blob[2 * n :].astype(np.float32), "step": int(meta["step"]), "lr": float(meta["lr"]),
            "channels": channels}


# ---------------------------------------------------------------- SPEC train schedule


@dataclass
class TrainConfig:
    """SPEC TrainConfig."""
    sizes: tuple = (129,)
    samples_per_epoch: tuple = (2000,)
    epochs_per_size_block: int = 20
    max_epochs: int = 250
    lr: float = 1e-3
    lr_decay_epochs: int = 100
    batch_size: int = 16
    seed: int = 0
    validation_fraction: float = 0.1

    def __post_init__(self):
        if list(self.sizes) != sorted(self.sizes):
            raise ConfigurationError("sizes must be sorted ascending")
        if len(self.samples_per_epoch) != len(self.sizes):
            raise ConfigurationError("one samples_per_epoch entry per size")
        if any(a < b for a, b in zip(self.samples_per_epoch, self.samples_per_epoch[1:])):
            raise ConfigurationError("samples_per_epoch must be non-increasing with size")


@dataclass
class History:
    rows: list = field(default_factory=list)  # (epoch, size, train_mse, val_mse, lr)
    state: dict | None = None  # final trainer state (checkpoint payload)

    def csv(self) -> str:
        lines = ["epoch,size,train_mse,val_mse,lr"]
        lines += [f"{e},{s},{t:.9e},{v:.9e},{lr:.3e}" for e, s, t, v, lr in self.rows]
        return "\n".join(lines) + "\n"


def _split(n, fraction, rng):
    idx = rng.permutation(n)
    nv = max(1, int(round(n * fraction))) if n > 1 else 0
    return idx[nv:], idx[:nv]


def train(net: EncoderSolverNet, config: TrainConfig, corpora: dict, checkpoint=None):
    """Multiscale training (SPEC ``train``): corpora[size] = (models, r, e, model_of) pair sets.

    Pairs come from datagen (``PairGenerator.pairs``); 10% of each size is held out for validation.
    Parameters and Adam state move between the per-size trainers at every size switch.
    Returns (trained EncoderSolverNet, History).
    """
    # data parallel (one process per GPU): every rank draws the same seeded epoch order and takes every
    # world-th batch of it; Trainer.step averages the gradients over ranks, so the parameters stay
    # identical and only the running batch-norm statistics (per rank, like PyTorch DDP) are averaged
    # at the end of every epoch before validation and checkpoints
    rank, world = 0, hdist.world_size()
    if world > 1:
        import torch.distributed as tdist

        rank = tdist.get_rank()
    rng = np.random.default_rng(config.seed)
    hist = History()
    trainers, splits, media = {}, {}, {}
    for size in config.sizes:
        if size not in corpora:
            raise ConfigurationError(f"no corpus for size {size}")
        models, r, e, owner = corpora[size]
        splits[size] = _split(len(r), config.validation_fraction, rng)
        media[size] = media_planes(models, len(net.channels))
        trainers[size] = Trainer(net, models[0].shape, models[0].h, config.batch_size, lr=config.lr)
    state = None
    active = None
    for epoch in range(config.max_epochs):
        size = config.sizes[(epoch // config.epochs_per_size_block) % len(config.sizes)]
        tr = trainers[size]
        if active is not size:
            if state is not None:
                tr.load_state(state)
            active = size
        tr.lr = config.lr * (0.1 ** (epoch // config.lr_decay_epochs))
        models, r, e, owner = corpora[size]
        train_idx, val_idx = splits[size]
        n_samples = config.samples_per_epoch[config.sizes.index(size)]
        order = rng.permutation(train_idx)
        order = np.resize(order, max(n_samples, config.batch_size))
        losses = []
        nb = (len(order) // config.batch_size) // world * world  # equal batch counts on every rank
        for bi in range(rank, nb, world):
            s = bi * config.batch_size
            b = order[s : s + config.batch_size]
            loss = tr.step(media[size], r[b], e[b], owner[b])
            if not np.isfinite(loss):
                raise NumericalError(f"non-finite loss at epoch {epoch}, batch {s // config.batch_size}")
            losses.append(loss)
        if world > 1:  # one running-statistics state for validation, checkpoints and the returned net
            import torch

            keep = torch.as_tensor(tr._read(WHICH_PARAMS)).cuda()
            hdist.allreduce_mean(keep)
            tr._write(WHICH_PARAMS, keep.cpu().numpy())
            losses = [hdist.reduce_scalar(float(np.mean(losses)), "sum") / world]
        # validation MSE (batch statistics, no update); the running statistics are restored after
        val = []
        vb = np.resize(val_idx, max(len(val_idx), config.batch_size)) if len(val_idx) else []
        if len(vb):
            keep = tr._read(WHICH_PARAMS)
            for s in range(0, len(vb) - config.batch_size + 1, config.batch_size):
                b = vb[s : s + config.batch_size]
                val.append(tr.step(media[size], r[b], e[b], owner[b], update=False))
            tr._write(WHICH_PARAMS, keep)
        hist.rows.append((epoch, size, float(np.mean(losses)), float(np.mean(val)) if val else float("nan"), tr.lr))
        state = tr.state()
        if checkpoint and (epoch + 1) % config.epochs_per_size_block == 0:
            save_checkpoint(checkpoint, state, net.channels)
    hist.state = state
    return EncoderSolverNet(unflatten(state["params"], net.channels), net.channels), hist
