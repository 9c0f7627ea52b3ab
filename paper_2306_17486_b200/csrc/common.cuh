// Shared device helpers for the B200 Helmholtz FGMRES path.
//
// Layout conventions:
//   * a field is (nx, ny) row-major, iy fastest, exactly the reference's
//     ``data[ix, iy]`` C order (fields.py:5-12); a batch is (B, nx, ny);
//   * complex64 is interleaved float2, complex128 interleaved double2;
//   * outside the grid every field is zero (Dirichlet padding, fields.py:191-199).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define HS_DEV __device__ __forceinline__

// ------------------------------------------------------------------ complex

HS_DEV float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
HS_DEV float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
HS_DEV float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
HS_DEV float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// a / b for complex b (fp32; |b| is O(1/h^2) so no scaling is needed)
HS_DEV float2 cdiv(float2 a, float2 b) {
  float inv = __frcp_rn(b.x * b.x + b.y * b.y);  // correctly rounded, as 1.0f / x
  return make_float2((a.x * b.x + a.y * b.y) * inv, (a.y * b.x - a.x * b.y) * inv);
}

HS_DEV double2 zadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
HS_DEV double2 zsub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
HS_DEV double2 zscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
// exact numpy-style complex product (no FMA contraction): (ac - bd) + (ad + bc) i
HS_DEV double2 zmul(double2 a, double2 b) {
  return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                      __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}
// conj(a) * b
HS_DEV double2 zcmul(double2 a, double2 b) {
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
HS_DEV double2 f2d(float2 a) { return make_double2((double)a.x, (double)a.y); }
HS_DEV float2 d2f(double2 a) { return make_float2((float)a.x, (float)a.y); }

// ------------------------------------------------------------------ reductions

HS_DEV double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
// softplus(x) = max(x, 0) + log1p(e), e = exp(-|x|) in (0, 1], as
// max(x, 0) + ln2 * lg2(1 + e) with the MUFU ex2 / lg2 approximations: six
// instructions.  Absolute error ~1e-7 (the rounding of 1 + e dominates; for
// tiny e the result is exact to within e ulp-of-1), the fp32 class of the
// reference's np.logaddexp; the conv tests hold layers to 2e-6 relative.
// The .ftz MUFU forms skip the denormal range scaling the plain ones add around
// each MUFU op: the ex2 argument is <= 0 (a denormal result, x < -87, flushes to
// 0, an absolute error below 1e-38) and the lg2 argument lies in [1, 2].
HS_DEV float softplus_fast(float x) {
  float e, l;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(fabsf(x) * -1.4426950408889634f));
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l) : "f"(1.0f + e));
  return fmaf(l, 0.69314718055994531f, fmaxf(x, 0.f));
}

// 4x4 transpose of 16-byte chunks inside each group of four lanes: lane gi (= lane & 3) holds
// chunks ch[0..3] of its own pixel and ends with chunk gi of the group's pixels 0..3, so store j of a
// warp writes whole 64-byte pixels.  Two butterfly stages (partner gi ^ 1, then gi ^ 2): each swaps the
// chunks whose index bit differs from the lane's bit with the partner's mirrored chunk.
HS_DEV void group4_transpose(float4 (&ch)[4], int gi) {
  auto xchg = [](float4& keep_lo, float4& keep_hi, bool hi_lane, int mask) {
    const float4 send = hi_lane ? keep_lo : keep_hi;
    float4 got;
    got.x = __shfl_xor_sync(0xffffffffu, send.x, mask);
    got.y = __shfl_xor_sync(0xffffffffu, send.y, mask);
    got.z = __shfl_xor_sync(0xffffffffu, send.z, mask);
    got.w = __shfl_xor_sync(0xffffffffu, send.w, mask);
    if (hi_lane)
      keep_lo = got;
    else
      keep_hi = got;
  };
  xchg(ch[0], ch[1], gi & 1, 1);
  xchg(ch[2], ch[3], gi & 1, 1);
  xchg(ch[0], ch[2], gi & 2, 2);
  xchg(ch[1], ch[3], gi & 2, 2);
}

HS_DEV float warp_sumf(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum of NV doubles per thread; result valid in every thread.
// `scratch` must hold NV * (blockDim.x / 32) doubles.  Deterministic order.
template <int NV>
HS_DEV void block_sum(double (&v)[NV], double* scratch) {
  // scratch: NV * (nwarps + 1) doubles.  Warp sums, then thread i < NV folds
  // value i over the warps in warp order (deterministic), then a broadcast.
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i) v[i] = warp_sum(v[i]);
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) scratch[i * nw + warp] = v[i];
  }
  __syncthreads();
  double* total = scratch + NV * nw;
  for (int i = threadIdx.x; i < NV; i += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < nw; ++w) s += scratch[i * nw + w];
    total[i] = s;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < NV; ++i) v[i] = total[i];
  __syncthreads();
}

// Dynamic-count variant: n values per thread stored in v[0..n), n <= NMAX.
template <int NMAX>
HS_DEV void block_sum_n(double* v, int n, double* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = 0; i < n; ++i) v[i] = warp_sum(v[i]);
  __syncthreads();
  if (lane == 0)
    for (int i = 0; i < n; ++i) scratch[i * nw + warp] = v[i];
  __syncthreads();
  for (int i = 0; i < n; ++i) {
    double s = 0.0;
    for (int w = 0; w < nw; ++w) s += scratch[i * nw + w];
    v[i] = s;
  }
  __syncthreads();
}

// ------------------------------------------------------------------ errors

// status codes: HS_OK, HS_EDIMENSION, ... from the public header
#include "../../include/helmsolve_b200.h"


#include <string>
namespace hs {
int set_error(int code, const std::string& msg);
}

inline unsigned cdiv_u(long a, long b) { return (unsigned)((a + b - 1) / b); }
