// Fused implicit (Green's-function) layer: pad, FFT2, spectrum, IFFT2, crop.
#pragma once
#include <cuda_runtime.h>

namespace hs {
// (h, w) = coarse grid; the padded transform is (2h, 2w).  Supported: h, w in {32, 64, 128} within the smem budget.
bool implicit_fused_supported(int h, int w);
// natural complex64 spectrum (C, 2h, 2w) -> the kernel's digit-reversed order (same size)
void implicit_permute_spectrum(const void* spec, void* spec_perm, int C, int h, int w, cudaStream_t st);
// y = crop(ifft2(fft2(pad(x)) * spec)) per (batch, channel); complex64 x / y addressed by strides (in
// complex elements) of batch, channel and pixel (p = row * w + col).  Items with active[b] == null are skipped.
int implicit_fused(const void* x, long long xb, long long xk, long long xp, void* y, long long yb, long long yk,
                   long long yp, const void* spec_perm, const void* const* active, int B, int C, int h, int w,
                   cudaStream_t st);
}  // namespace hs
