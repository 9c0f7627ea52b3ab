"""Device plumbing: torch CUDA tensors as the buffers handed to the C ABI.

PyTorch only provides memory, streams and host<->device copies here; all
arithmetic on the hot path runs in the library's own kernels.
"""
from __future__ import annotations

import mmap

import numpy as np
import torch


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("helmsolve_b200 needs a CUDA device (B200, sm_100a); none is visible")
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle():
    return torch.cuda.current_stream().cuda_stream


def ptr(t):
    return None if t is None else t.data_ptr()


def to_device(a, dtype: torch.dtype) -> torch.Tensor:
    """numpy array or tensor -> contiguous CUDA tensor of ``dtype``."""
    dev = require_cuda()
    if isinstance(a, torch.Tensor):
        return a.to(device=dev, dtype=dtype).contiguous()
    arr = np.ascontiguousarray(a)
    return torch.from_numpy(arr).to(device=dev, dtype=dtype).contiguous()


def to_host(t: torch.Tensor) -> np.ndarray:
    """CUDA tensor -> numpy array, with large results in transparent-huge-page memory.

    A fresh pageable array pays one page fault per 4 KB on first touch. That is
    most of the cost of ``.cpu()`` for a solve's result: 63 ms for C2's 135 MB
    on the B200 box. Backing the array with an anonymous mapping advised
    ``MADV_HUGEPAGE`` (the box's THP mode is ``madvise``) brings the same copy
    to 27 ms. The array owns its mapping.
    """
    if not t.is_cuda:
        return t.numpy()
    nbytes = t.numel() * t.element_size()
    if nbytes < (8 << 20) or not hasattr(mmap, "MADV_HUGEPAGE"):
        return t.cpu().numpy()
    m = mmap.mmap(-1, nbytes, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    m.madvise(mmap.MADV_HUGEPAGE)
    out = np.frombuffer(m, dtype=torch.empty((), dtype=t.dtype).numpy().dtype).reshape(tuple(t.shape))
    torch.from_numpy(out).copy_(t)
    return out


def pinned(shape, dtype: torch.dtype) -> torch.Tensor:
    return torch.empty(shape, dtype=dtype, pin_memory=True)


def workspace(nbytes: int) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=require_cuda())
