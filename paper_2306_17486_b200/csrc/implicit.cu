// Fused implicit (Green's-function) layer: zero-pad, 2D FFT, spectrum
// multiply, inverse 2D FFT, crop, in one kernel (green.py:96-107,
// implicit_apply; autodiff.py:283-307 pad2d_to / crop2d).
//
// One CTA per (RHS, complex channel).  The padded grid is (H2, W2) = (2h, 2w)
// but only the top-left (h, w) quarter of the input is non-zero and only that
// quarter of the output is kept, so the transform runs as
//   1. h row FFTs of length W2 (half the inputs zero)        -> smem S[h][W2]
//   2. W2 column FFTs of length H2 (half the inputs zero), spectrum multiply,
//      inverse column FFTs keeping h outputs                   -> S in place
//   3. h inverse row FFTs keeping w outputs, 1/(H2 W2)         -> global
// so global memory sees the input and output once and the spectrum (L2
// resident, shared by all RHS) once per CTA.
//
// Each line is transformed by one warp in registers, N = 32 E points with
// E = N / 32 per lane (lane l holds n = l + 32 j):
//   forward: E-point DFT per lane, twiddle W_N^(l k1), radix-2 DIF across the
//            32 lanes (shuffles) -> lane l, register k1 holds X[k1 + E br5(l)]
//   inverse: the exact transpose (DIT across lanes from that digit-reversed
//            order, conjugate twiddles, inverse E-point DFT) -> natural order.
// The row transforms store their digit-reversed output as-is (column
// c = 32 k1 + l holds frequency k1 + E br5(l)); the spectrum is permuted into
// the same order once, at network setup.  Twiddles come from a per-CTA table
// built with sincospif (full fp32 accuracy).
#include "common.cuh"
#include "implicit.h"

namespace hs {
namespace {

constexpr int kImpThreads = 256;

HS_DEV int br5(int l) { return __brev(l) >> 27; }

// a * W_E^m, W_E = exp(-2 pi i / E), E in {2, 4, 8}, m a compile-time constant
// after unrolling: multiples of pi/2 are swaps / negations, odd multiples of
// pi/4 one scaled add (no multiplications by 0 or 1 survive)
template <int E>
HS_DEV float2 mul_wE(float2 a, int m) {
  constexpr float s = 0.70710678118654752f;
  switch ((m * (8 / E)) & 7) {  // in units of 2 pi / 8
    case 0: return a;
    case 1: return make_float2(s * (a.x + a.y), s * (a.y - a.x));    // (1 - i) / sqrt2
    case 2: return make_float2(a.y, -a.x);                          // -i
    case 3: return make_float2(s * (a.y - a.x), -s * (a.x + a.y));   // (-1 - i) / sqrt2
    case 4: return make_float2(-a.x, -a.y);                         // -1
    case 5: return make_float2(-s * (a.x + a.y), s * (a.x - a.y));   // (-1 + i) / sqrt2
    case 6: return make_float2(-a.y, a.x);                          // i
    default: return make_float2(s * (a.x - a.y), s * (a.x + a.y));  // (1 + i) / sqrt2
  }
}

HS_DEV float2 cmulc(float2 a, float2 b) {  // a * conj(b)
  return make_float2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}

HS_DEV float2 shfl_xor2(float2 v, int m) {
  return make_float2(__shfl_xor_sync(0xffffffffu, v.x, m), __shfl_xor_sync(0xffffffffu, v.y, m));
}

// forward: a[j] = x[l + 32 j] (zero for j >= NZ) -> a[k1] = X[k1 + E br5(l)]; tw[m] = W_N^m
template <int E, int NZ>
HS_DEV void fft_fwd(float2 (&a)[E], int lane, const float2* tw) {
  constexpr int N = 32 * E;
  float2 b[E];
#pragma unroll
  for (int k1 = 0; k1 < E; ++k1) {
    float2 s = a[0];
#pragma unroll
    for (int j = 1; j < NZ; ++j) s = cadd(s, mul_wE<E>(a[j], j * k1));
    b[k1] = k1 == 0 ? s : cmul(s, tw[lane * k1]);
  }
  // radix-2 DIF across lanes.  top lane: b + v; bottom lane: (v - b) w.  Written
  // branch-free as (v + sg b) * w' with sg = +-1 and w' = 1 on the top lane.
#pragma unroll
  for (int half = 16; half >= 1; half >>= 1) {
    const bool top = (lane & half) == 0;
    const float sg = top ? 1.f : -1.f;
    const float2 w = top ? make_float2(1.f, 0.f) : tw[(lane & (half - 1)) * (N / (2 * half))];
#pragma unroll
    for (int k1 = 0; k1 < E; ++k1) {
      const float2 v = shfl_xor2(b[k1], half);
      const float2 t = make_float2(fmaf(sg, b[k1].x, v.x), fmaf(sg, b[k1].y, v.y));
      b[k1] = cmul(t, w);
    }
  }
#pragma unroll
  for (int k1 = 0; k1 < E; ++k1) a[k1] = b[k1];
}

// inverse (unscaled, x N): a[k1] = X[k1 + E br5(l)] -> a[j] = N x[l + 32 j] for j < NOUT
template <int E, int NOUT>
HS_DEV void fft_inv(float2 (&a)[E], int lane, const float2* tw) {
  constexpr int N = 32 * E;
  // radix-2 DIT across lanes, the transpose of the DIF above: with s the top
  // lane's value and d the bottom's, top <- s + d conj(w), bottom <- s - d conj(w)
#pragma unroll
  for (int half = 1; half <= 16; half <<= 1) {
    const bool top = (lane & half) == 0;
    const float sg = top ? 1.f : -1.f;
    const float2 w = tw[(lane & (half - 1)) * (N / (2 * half))];
#pragma unroll
    for (int k1 = 0; k1 < E; ++k1) {
      const float2 v = shfl_xor2(a[k1], half);
      const float2 s = top ? a[k1] : v, d = top ? v : a[k1];
      const float2 dw = cmulc(d, w);
      a[k1] = make_float2(fmaf(sg, dw.x, s.x), fmaf(sg, dw.y, s.y));
    }
  }
#pragma unroll
  for (int k1 = 1; k1 < E; ++k1) a[k1] = cmulc(a[k1], tw[lane * k1]);
  float2 x[NOUT];
#pragma unroll
  for (int j = 0; j < NOUT; ++j) {
    float2 s = a[0];
#pragma unroll
    for (int k1 = 1; k1 < E; ++k1) s = cadd(s, mul_wE<E>(a[k1], (E - (j * k1) % E) % E));  // conj twiddle
    x[j] = s;
  }
#pragma unroll
  for (int j = 0; j < NOUT; ++j) a[j] = x[j];
}

struct ImpArgs {
  const float2* x;
  long long xb, xk, xp;  // strides (complex elements) of batch, channel, pixel (p = y w + x)
  float2* y;
  long long yb, yk, yp;
  const float2* spec;  // permuted spectrum [C][W2][EH][32]
  const void* const* active;
  int C;
};

template <int EW, int EH>
__global__ void __launch_bounds__(kImpThreads) k_implicit(ImpArgs a) {
  constexpr int W2 = 32 * EW, H2 = 32 * EH, h = H2 / 2, w = W2 / 2;
  constexpr int NZW = EW / 2, NZH = EH / 2, LD = W2 + 1;  // odd pitch: conflict-free column reads
  extern __shared__ float2 smem_imp[];
  float2* S = smem_imp;         // [h][LD]
  float2* twW = S + h * LD;     // W_W2^m
  float2* twH = twW + W2;       // W_H2^m
  const int b = blockIdx.y, k = blockIdx.x;
  if (a.active && a.active[b] == nullptr) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int m = threadIdx.x; m < W2; m += kImpThreads) {
    float s, c;
    sincospif(-2.f * m / W2, &s, &c);
    twW[m] = make_float2(c, s);
  }
  for (int m = threadIdx.x; m < H2; m += kImpThreads) {
    float s, c;
    sincospif(-2.f * m / H2, &s, &c);
    twH[m] = make_float2(c, s);
  }
  __syncthreads();
  const float2* xin = a.x + b * a.xb + k * a.xk;
  // 1. row transforms
  for (int r = warp; r < h; r += kImpThreads / 32) {
    float2 v[EW];
#pragma unroll
    for (int j = 0; j < EW; ++j) v[j] = j < NZW ? xin[(long long)(r * w + lane + 32 * j) * a.xp] : make_float2(0.f, 0.f);
    fft_fwd<EW, NZW>(v, lane, twW);
#pragma unroll
    for (int k1 = 0; k1 < EW; ++k1) S[r * LD + k1 * 32 + lane] = v[k1];
  }
  __syncthreads();
  // 2. column transforms, spectrum, inverse column transforms (rows < h kept)
  const float2* sp = a.spec + (long long)k * W2 * H2;
  for (int c = warp; c < W2; c += kImpThreads / 32) {
    float2 v[EH];
#pragma unroll
    for (int j = 0; j < EH; ++j) v[j] = j < NZH ? S[(lane + 32 * j) * LD + c] : make_float2(0.f, 0.f);
    fft_fwd<EH, NZH>(v, lane, twH);
#pragma unroll
    for (int k1 = 0; k1 < EH; ++k1) v[k1] = cmul(v[k1], __ldg(sp + (c * EH + k1) * 32 + lane));
    fft_inv<EH, NZH>(v, lane, twH);
#pragma unroll
    for (int j = 0; j < NZH; ++j) S[(lane + 32 * j) * LD + c] = v[j];
  }
  __syncthreads();
  // 3. inverse row transforms (columns < w kept), 1 / (H2 W2)
  float2* yout = a.y + b * a.yb + k * a.yk;
  const float inv = 1.f / (float)(H2 * W2);
  for (int r = warp; r < h; r += kImpThreads / 32) {
    float2 v[EW];
#pragma unroll
    for (int k1 = 0; k1 < EW; ++k1) v[k1] = S[r * LD + k1 * 32 + lane];
    fft_inv<EW, NZW>(v, lane, twW);
#pragma unroll
    for (int j = 0; j < NZW; ++j)
      yout[(long long)(r * w + lane + 32 * j) * a.yp] = make_float2(v[j].x * inv, v[j].y * inv);
  }
}

// natural spectrum [C][H2][W2] -> kernel order [C][c][k1'][l]: column c holds
// frequency f = c/32 + EW br5(c%32), entry (k1', l) row frequency u = k1' + EH br5(l)
__global__ void k_permute_spec(const float2* in, float2* out, int C, int H2, int W2) {
  const int EW = W2 / 32, EH = H2 / 32;
  const long long n = (long long)C * H2 * W2;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const int l = (int)(e % 32);
    const int k1 = (int)((e / 32) % EH);
    const int c = (int)((e / (32 * EH)) % W2);
    const int ch = (int)(e / ((long long)32 * EH * W2));
    const int f = c / 32 + EW * br5(c % 32), u = k1 + EH * br5(l);
    out[e] = in[((long long)ch * H2 + u) * W2 + f];
  }
}

size_t smem_bytes(int h, int w) { return ((size_t)h * (2 * w + 1) + 2 * w + 2 * h) * sizeof(float2); }

template <int EW, int EH>
void launch_imp(const ImpArgs& a, int B, cudaStream_t st) {
  constexpr int h = 16 * EH, w = 16 * EW;
  const size_t sm = smem_bytes(h, w);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_implicit<EW, EH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    attr = true;
  }
  k_implicit<EW, EH><<<dim3((unsigned)a.C, (unsigned)B), kImpThreads, sm, st>>>(a);
}

}  // namespace

bool implicit_fused_supported(int h, int w) {
  auto ok = [](int n) { return n == 32 || n == 64 || n == 128; };  // E = 2n / 32 in {2, 4, 8}
  return ok(h) && ok(w) && smem_bytes(h, w) <= 200 * 1024;
}

void implicit_permute_spectrum(const void* spec, void* spec_perm, int C, int h, int w, cudaStream_t st) {
  const long long n = (long long)C * 4 * h * w;
  const unsigned g = (unsigned)((n + 255) / 256 > 4096 ? 4096 : (n + 255) / 256);
  k_permute_spec<<<g, 256, 0, st>>>(static_cast<const float2*>(spec), static_cast<float2*>(spec_perm), C, 2 * h,
                                    2 * w);
}

int implicit_fused(const void* x, long long xb, long long xk, long long xp, void* y, long long yb, long long yk,
                   long long yp, const void* spec_perm, const void* const* active, int B, int C, int h, int w,
                   cudaStream_t st) {
  if (!implicit_fused_supported(h, w)) return HS_ECONFIG;
  ImpArgs a{static_cast<const float2*>(x), xb, xk, xp, static_cast<float2*>(y), yb, yk, yp,
            static_cast<const float2*>(spec_perm), active, C};
  const int EW = w / 16, EH = h / 16;
#define HS_IMP(A, Bq) \
  if (EW == A && EH == Bq) return launch_imp<A, Bq>(a, B, st), HS_OK;
  HS_IMP(2, 2)
  HS_IMP(4, 4)
  HS_IMP(8, 8)
  HS_IMP(4, 2)
  HS_IMP(2, 4)
  HS_IMP(8, 4)
  HS_IMP(4, 8)
  HS_IMP(8, 2)
  HS_IMP(2, 8)
#undef HS_IMP
  return HS_ECONFIG;
}

}  // namespace hs
