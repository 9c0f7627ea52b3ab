"""The implicit layer: spectral inverse of a learnable 3x3 kernel (mirror of ``helmsolve.green``).

``green_function`` builds, once per kernel and size, the spectrum of the
kernel's regularised lattice inverse exactly as the reference does it
(``green.py:55-82``): corner-embed the kernel on a 6h x 6w grid, FFT,
``conj(S) / (S conj(S) + eps)`` against a centred point source, inverse FFT,
crop the centred 2h x 2w window, ifftshift, FFT -- with the reference's numpy-2
dtype flow (complex128 result).  ``implicit_apply`` is the per-channel
spectral convolution (``green.py:85-107``).  Both run on the GPU through the
C ABI (cuFFT for the transforms, own kernels for everything else).
"""
from __future__ import annotations

import numpy as np

from .errors import DimensionError

#: Regularisation added to |S|^2 (green.py:19).
SPECTRUM_EPS = 1e-5


def laplacian_plus_i_kernel(channels: int, dtype=np.complex64) -> np.ndarray:
    """Per-channel L + iI: the 5-point stencil with 4 + i at the centre (green.py:24-30)."""
    base = np.zeros((3, 3), dtype=dtype)
    base[1, 1] = 4 + 1j
    base[[0, 2, 1, 1], [1, 1, 0, 2]] = -1
    return np.tile(base, (channels, 1, 1))


def pad_kernel_corners(kernel, size: tuple[int, int]) -> np.ndarray:
    """Circulant embedding with the kernel centre at (0, 0) (green.py:33-41, autodiff.py:323-337)."""
    k = np.asarray(kernel)
    h, w = size
    if h < 3 or w < 3:
        raise DimensionError(f"target {size} too small for a 3x3 kernel")
    out = np.zeros(k.shape[:-2] + (h, w), dtype=k.dtype)
    rows, cols = (h - 1, 0, 1), (w - 1, 0, 1)
    for a in range(3):
        for b in range(3):
            out[..., rows[a], cols[b]] = k[..., a, b]
    return out


def green_function(kernel, coarse_size: tuple[int, int], eps: float = SPECTRUM_EPS):
    """(channels, 2h, 2w) complex128 spectrum of the regularised inverse (green.py:55-82), on the GPU."""
    import torch

    from . import _lib
    from .device import stream_handle, to_device

    h, w = coarse_size
    if h < 3 or w < 3:
        raise DimensionError(f"coarse size {coarse_size} too small")
    k = np.asarray(kernel.data if isinstance(kernel, KernelWeights) else kernel)
    if k.shape[-2:] != (3, 3):
        raise DimensionError(f"kernel must be 3x3 per channel, got {k.shape}")
    squeeze = k.ndim == 2
    kd = to_device(k.reshape(-1, 3, 3), torch.complex64)
    C = kd.shape[0]
    out = torch.empty((C, 2 * h, 2 * w), dtype=torch.complex128, device=kd.device)
    _lib.check(_lib.load().hs_green_spectrum_eps(kd.data_ptr(), C, h, w, float(eps), out.data_ptr(), stream_handle()),
               "green_function")
    res = out.cpu().numpy()
    return res[0] if squeeze else res


def implicit_apply(x, spectrum):
    """Per-channel spectral convolution: pad to (2h, 2w), FFT, multiply, IFFT, crop (green.py:85-107).

    x (batch, channels, h, w) complex, spectrum (channels, 2h, 2w); computed in
    complex64 on the GPU.  numpy in -> numpy out; CUDA tensors stay on device.
    """
    import torch

    from . import _lib
    from .device import stream_handle, to_device

    was_np = not isinstance(x, torch.Tensor)
    xs = np.shape(x)
    ss = np.shape(spectrum)
    n, c, h, w = xs
    if ss[0] != c:
        raise DimensionError(f"{c} input channels vs {ss[0]} kernel channels")
    if tuple(ss[-2:]) != (2 * h, 2 * w):
        raise DimensionError(f"spectrum {tuple(ss[-2:])} is not twice the input size {(h, w)}")
    xd = to_device(x, torch.complex64)
    sd = to_device(spectrum, torch.complex64)
    y = torch.empty_like(xd)
    _lib.check(_lib.load().hs_implicit_apply(xd.data_ptr(), sd.data_ptr(), y.data_ptr(), n, c, h, w,
                                             stream_handle()), "implicit_apply")
    return y.cpu().numpy() if was_np else y


def circular_conv(kernel, x):
    """Multiplication by the circulant of the corner-embedded kernel on x's grid (green.py:110-117)."""
    import torch

    from .device import to_device

    kp = to_device(pad_kernel_corners(np.asarray(kernel), np.shape(x)[-2:]), torch.complex128)
    xd = to_device(np.asarray(x), torch.complex128)
    out = torch.fft.ifft2(torch.fft.fft2(kp) * torch.fft.fft2(xd))
    return out.cpu().numpy()


class KernelWeights:
    """The implicit kernels as a versioned array: the part of the reference's autodiff ``Tensor``
    that ``ImplicitKernel`` relies on (``.data``, ``.version``, ``.bump_version()``; autodiff.py's
    Tensor, used at green.py:131, 139-146).  Change ``data`` in place, then ``bump_version()``."""

    def __init__(self, data):
        self.data = np.asarray(data)
        self.version = 0

    def bump_version(self):
        self.version += 1

    @property
    def shape(self):
        return self.data.shape

    @property
    def dtype(self):
        return self.data.dtype

    def __array__(self, dtype=None, copy=None):
        return self.data if dtype is None else self.data.astype(dtype)

    def __getitem__(self, idx):
        return self.data[idx]

    def __setitem__(self, idx, value):
        self.data[idx] = value


class ImplicitKernel:
    """Per-channel 3x3 complex kernels with a cached spectrum (green.py:120-149).

    The cache is keyed on (size, weights.version) like the reference's; call
    ``weights.bump_version()`` (or ``bump_version()`` here) after changing the weights in place.
    """

    def __init__(self, channels: int, dtype=np.complex64, weights=None):
        if weights is None:
            weights = laplacian_plus_i_kernel(channels, dtype)
        self.weights = KernelWeights(np.array(weights, dtype=dtype))
        self._cache = None
        self._cache_key = None

    @property
    def channels(self) -> int:
        return int(self.weights.shape[0])

    @property
    def version(self) -> int:
        return self.weights.version

    def bump_version(self):
        self.weights.bump_version()

    def spectrum(self, coarse_size: tuple[int, int]) -> np.ndarray:
        key = (tuple(coarse_size), self.weights.version)
        if self._cache_key != key:
            self._cache = green_function(self.weights.data, tuple(coarse_size))
            self._cache_key = key
        return self._cache

    def __call__(self, x):
        return implicit_apply(x, self.spectrum(np.shape(x)[-2:]))
