// Slowness-model preparation on the GPU (SPEC.md
// `[MODULE] datagen`, load_slowness_corpus / gaussian_smooth, reference
// SPEC.md:404-417,441): bilinear resize to (n+1)^2 nodes, separable truncated
// Gaussian smoothing (radius ceil(3 sigma), edge-replicated), affine
// normalisation onto [lo, hi] (a constant field maps to lo).  fp64 throughout,
// batched over fields; each pass is one coalesced sweep (HBM-bound).
#include <cmath>
#include <vector>

#include "common.cuh"

namespace hs {
namespace {

// corner-aligned bilinear: output node (i, j) samples input (i (hin-1)/(hout-1), j (win-1)/(wout-1))
__global__ void k_resize_bilinear(const double* __restrict__ in, double* __restrict__ out, int hin, int win,
                                  int hout, int wout) {
  const int b = blockIdx.y;
  const long long n = (long long)hout * wout;
  const double sy = hout > 1 ? (double)(hin - 1) / (hout - 1) : 0.0, sx = wout > 1 ? (double)(win - 1) / (wout - 1) : 0.0;
  const double* src = in + (long long)b * hin * win;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(p / wout), j = (int)(p - (long long)i * wout);
    const double y = __dmul_rn((double)i, sy), x = __dmul_rn((double)j, sx);
    const int y0 = min((int)floor(y), hin - 1), x0 = min((int)floor(x), win - 1);
    const int y1 = min(y0 + 1, hin - 1), x1 = min(x0 + 1, win - 1);
    const double fy = y - y0, fx = x - x0;
    // explicit rounding (no FMA contraction): the numpy oracle's evaluation order, bit for bit
    const double gx = __dsub_rn(1.0, fx), gy = __dsub_rn(1.0, fy);
    const double top = __dadd_rn(__dmul_rn(gx, src[(long long)y0 * win + x0]), __dmul_rn(fx, src[(long long)y0 * win + x1]));
    const double bot = __dadd_rn(__dmul_rn(gx, src[(long long)y1 * win + x0]), __dmul_rn(fx, src[(long long)y1 * win + x1]));
    out[(long long)b * n + p] = __dadd_rn(__dmul_rn(gy, top), __dmul_rn(fy, bot));
  }
}

// one separable pass along `axis` (0: rows i, 1: columns j) with edge replication;
// taps are accumulated in tap order (the oracle's order)
__global__ void k_smooth_axis(const double* __restrict__ in, double* __restrict__ out, int nx, int ny,
                              const double* __restrict__ taps, int r, int axis) {
  const int b = blockIdx.y;
  const long long n = (long long)nx * ny;
  const double* src = in + (long long)b * n;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(p / ny), j = (int)(p - (long long)i * ny);
    double acc = 0.0;
    for (int t = -r; t <= r; ++t) {
      const int ii = axis == 0 ? min(max(i + t, 0), nx - 1) : i;
      const int jj = axis == 1 ? min(max(j + t, 0), ny - 1) : j;
      acc = __dadd_rn(acc, __dmul_rn(taps[t + r], src[(long long)ii * ny + jj]));  // numpy's order
    }
    out[(long long)b * n + p] = acc;
  }
}

// per-field min / max (one block per field), then the affine map
__global__ void k_minmax(const double* __restrict__ in, long long n, double* __restrict__ mm) {
  const int b = blockIdx.x;
  const double* src = in + (long long)b * n;
  double lo = INFINITY, hi = -INFINITY;
  for (long long p = threadIdx.x; p < n; p += blockDim.x) {
    lo = fmin(lo, src[p]);
    hi = fmax(hi, src[p]);
  }
  for (int o = 16; o; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  __shared__ double s_lo[32], s_hi[32];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) {
    s_lo[w] = lo;
    s_hi[w] = hi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k) {
      lo = fmin(lo, s_lo[k]);
      hi = fmax(hi, s_hi[k]);
    }
    mm[2 * b] = lo;
    mm[2 * b + 1] = hi;
  }
}

__global__ void k_affine(const double* __restrict__ in, double* __restrict__ out, long long n,
                         const double* __restrict__ mm, double lo, double hi) {
  const int b = blockIdx.y;
  const double vmin = mm[2 * b], vmax = mm[2 * b + 1];
  const bool flat = !(vmax - vmin > 0.0);
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
    const long long q = (long long)b * n + p;
    out[q] = flat ? lo : __dadd_rn(lo, __ddiv_rn(__dmul_rn(hi - lo, __dsub_rn(in[q], vmin)), vmax - vmin));
  }
}

unsigned blocks_for(long long n) {
  const long long g = (n + 255) / 256;
  return (unsigned)(g > 2048 ? 2048 : (g < 1 ? 1 : g));
}

}  // namespace
}  // namespace hs

extern "C" {

HS_API int hs_resize_bilinear(const double* in, double* out, int B, int hin, int win, int hout, int wout,
                              void* stream) {
  if (B < 1 || hin < 1 || win < 1 || hout < 1 || wout < 1) return hs::set_error(HS_EDIMENSION, "resize shape");
  hs::k_resize_bilinear<<<dim3(hs::blocks_for((long long)hout * wout), B), 256, 0, (cudaStream_t)stream>>>(
      in, out, hin, win, hout, wout);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? HS_OK : hs::set_error(HS_ECUDA, cudaGetErrorString(e));
}

HS_API int hs_gaussian_smooth(const double* in, double* out, double* tmp, int B, int nx, int ny, double sigma,
                              void* stream) {
  if (B < 1 || nx < 1 || ny < 1) return hs::set_error(HS_EDIMENSION, "smooth shape");
  if (!(sigma >= 0.0)) return hs::set_error(HS_ECONFIG, "sigma must be >= 0");
  cudaStream_t st = (cudaStream_t)stream;
  const long long n = (long long)nx * ny;
  if (sigma == 0.0) {  // identity
    if (out != in) cudaMemcpyAsync(out, in, (size_t)B * n * sizeof(double), cudaMemcpyDeviceToDevice, st);
  } else {
    const int r = (int)std::ceil(3.0 * sigma);
    std::vector<double> t(2 * r + 1);
    double s = 0.0;
    for (int k = -r; k <= r; ++k) s += (t[k + r] = std::exp(-0.5 * (k / sigma) * (k / sigma)));
    for (double& v : t) v /= s;
    double* taps = nullptr;
    if (cudaMallocAsync(&taps, t.size() * sizeof(double), st) != cudaSuccess) return hs::set_error(HS_ECUDA, "taps");
    cudaMemcpyAsync(taps, t.data(), t.size() * sizeof(double), cudaMemcpyHostToDevice, st);
    const dim3 g(hs::blocks_for(n), B);
    hs::k_smooth_axis<<<g, 256, 0, st>>>(in, tmp, nx, ny, taps, r, 0);
    hs::k_smooth_axis<<<g, 256, 0, st>>>(tmp, out, nx, ny, taps, r, 1);
    cudaFreeAsync(taps, st);
    cudaStreamSynchronize(st);  // the host taps vector dies with this call
  }
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? HS_OK : hs::set_error(HS_ECUDA, cudaGetErrorString(e));
}

HS_API int hs_normalise_range(const double* in, double* out, double* minmax, int B, long long n, double lo,
                              double hi, void* stream) {
  if (B < 1 || n < 1) return hs::set_error(HS_EDIMENSION, "normalise shape");
  cudaStream_t st = (cudaStream_t)stream;
  hs::k_minmax<<<B, 512, 0, st>>>(in, n, minmax);
  hs::k_affine<<<dim3(hs::blocks_for(n), B), 256, 0, st>>>(in, out, n, minmax, lo, hi);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? HS_OK : hs::set_error(HS_ECUDA, cudaGetErrorString(e));
}

}  // extern "C"
