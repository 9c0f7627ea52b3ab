// Encoder-solver CNN (ARCH.md) and the implicit Green's-function layer.
//
// Activations are float32 NHWC [B][H][W][C]: one pixel's channels are
// contiguous, so a 3x3 tap of the implicit GEMM (M = pixels, N = cout,
// K = 9 cin) is a contiguous cin-vector.  Batch norm is folded into the
// convolution weights on the host; every convolution fuses its bias,
// softplus, encoder/skip addend and residual add into the epilogue.
//
// Reference semantics: conv2d / conv_transpose2d / batchnorm2d / softplus
// (autodiff.py:243-252, 472-607), pack/unpack_complex (:343-372),
// green_function / implicit_apply (green.py:55-107).
#include <cufft.h>

#include <cmath>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include <type_traits>
#include <algorithm>

#include "cnn.h"
#include "common.cuh"
#include "conv_tc.h"
#include "implicit.h"
#include "prof.h"

struct hs_net {
  hs_net_desc_t d;
  int hc, wc, cc;              // coarsest grid and complex channel count
  cufftComplex* spec = nullptr;       // (cc, 2hc, 2wc) complex64 Green spectrum
  cufftComplex* spec_perm = nullptr;  // the same in the fused kernel's order (implicit.cu), if supported
  const float* enc[8] = {nullptr};
  int n_models = 0;
  // host copies of the thin layers' weights ([tap][cin][cout], then the bias): passed to the
  // thin kernels by value (kernel-parameter constant bank) -- 0 encoder stem, 1 solver stem, 2 head
  std::vector<float> thin_w[3];
  mutable std::mutex plan_mu;
  mutable std::map<int, cufftHandle> plans;  // batch -> plan
  std::vector<const float*> wide_w;          // layers whose bf16x3 split is registered (conv_wide.cu)
  ~hs_net() {
    for (const float* w : wide_w) hs::conv_wide_unregister(w);
    for (auto& kv : plans) cufftDestroy(kv.second);
    if (spec) cudaFree(spec);
    if (spec_perm) cudaFree(spec_perm);
  }
};

namespace hs {
namespace {

constexpr int kConvThreads = 256;
constexpr int kCK = 8;  // input channels staged per smem pass

HS_DEV float softplusf(float x) { return fmaxf(x, 0.f) + log1pf(expf(-fabsf(x))); }

struct ConvArgs {
  const float* x;
  int H, W, cin;  // input
  float* y;
  int Ho, Wo, cout;  // output
  const float* w;    // [cout][9][cin]
  const float* bias;
  int softplus;
  const float* addend;  // NHWC like y, per model (model_of) or per batch item
  long long addend_bstride;
  const int* model_of;
  int addend_per_model;  // 1: addend indexed by model_of[b] (encodings), 0: by b (skips)
  const float* residual;  // NHWC like y
  const void* const* active;
  // thin kernels only: the stem may read the complex Krylov vector directly and
  // the head may write the complex preconditioner estimate directly
  // (gather / scatter fused away)
  VecIn cx;  // complex input (cin == 2) when cx_ld > 0: row r, column c at r * cx_ld + c, times scale[b]
  int cx_ld;
  float2* cy;  // complex output (cout == 2): value at (r, c) -> cy[b * cy_n + r * cy_ld + c]
  long long cy_n;
  int cy_ld, cy_h, cy_w;  // the output covers (cy_h, cy_w); outside (Ho, Wo) it is zero
  float cy_scale;
};

// optional complex I/O for the thin stem / head (see ConvArgs)
struct ThinIO {
  VecIn in;
  int in_ld;
  float2* out;
  long long out_n;
  int out_ld, out_h, out_w;
  float out_scale;
  const float* host_w = nullptr;  // [tap][cin][cout] + bias on the host: the by-value thin kernels
};

// Packed fp32x2 FMA (sm_100 FFMA2): acc.{lo,hi} = fma(x, {w0, w1}, acc.{lo,hi}),
// each half rounded exactly like fmaf, so results are bitwise those of two
// scalar FMAs; ptxas takes the broadcast x as a .F32 operand and the weight
// pair from uniform registers.
HS_DEV void ffma2(unsigned long long& acc, float x, float w0, float w1) {
  unsigned long long xx, ww;
  asm("mov.b64 %0, {%1, %1};" : "=l"(xx) : "f"(x));
  asm("mov.b64 %0, {%1, %2};" : "=l"(ww) : "f"(w0), "f"(w1));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(xx), "l"(ww));
}
HS_DEV float lo32(unsigned long long v) { return __uint_as_float((unsigned)(v & 0xffffffffull)); }
HS_DEV float hi32(unsigned long long v) { return __uint_as_float((unsigned)(v >> 32)); }
// channel q of a packed (PK) or scalar accumulator row
template <bool PK, typename A>
HS_DEV float acc_at(const A* row, int q) {
  if constexpr (PK) return (q & 1) ? hi32(row[q / 2]) : lo32(row[q / 2]);
  else return row[q];
}

template <int COUT>
struct Tile {
  static constexpr int CG = COUT < 16 ? COUT : 16;           // couts per thread
  static constexpr int PX = 4;                               // pixels per thread (along W)
  static constexpr int TPX = kConvThreads * PX * CG / COUT;  // pixels per block
  static constexpr int TW = 32;
  static constexpr int TH = TPX / TW;
};

// Direct 3x3 convolution, stride 1 or 2, SIMT fp32 (exact fp32 products).
template <int COUT, int STRIDE>
__global__ void __launch_bounds__(kConvThreads) k_conv(ConvArgs a) {
  using T = Tile<COUT>;
  constexpr int IH = (T::TH - 1) * STRIDE + 3, IW = (T::TW - 1) * STRIDE + 3;
  extern __shared__ float smem[];
  float* s_in = smem;                  // [kCK][IH][IW]
  float* s_w = smem + ((kCK * IH * IW + 3) & ~3);  // [kCK][9][COUT], 16-byte aligned (paired loads)
  const int b = blockIdx.z;
  if (a.active && a.active[b] == nullptr) return;
  const int tiles_x = (a.Wo + T::TW - 1) / T::TW;
  const int oy0 = (blockIdx.x / tiles_x) * T::TH, ox0 = (blockIdx.x % tiles_x) * T::TW;
  const int iy0 = oy0 * STRIDE - 1, ix0 = ox0 * STRIDE - 1;
  const int t = threadIdx.x;
  constexpr int PG = T::TPX / T::PX;  // pixel groups
  const int cg = t / PG, pg = t % PG;
  const int ly = pg / (T::TW / T::PX), lx = (pg % (T::TW / T::PX)) * T::PX;
  // output-channel pairs packed fp32x2 (FFMA2) when CG is even; scalar otherwise
  constexpr bool PK = T::CG % 2 == 0;
  constexpr int NQ = PK ? T::CG / 2 : T::CG;
  using AccT = typename std::conditional<PK, unsigned long long, float>::type;
  AccT acc[T::PX][NQ];
#pragma unroll
  for (int p = 0; p < T::PX; ++p)
#pragma unroll
    for (int q = 0; q < NQ; ++q) acc[p][q] = AccT(0);
  const float* xb = a.x + (long long)b * a.H * a.W * a.cin;
  for (int c0 = 0; c0 < a.cin; c0 += kCK) {
    const int ck = min(kCK, a.cin - c0);
    __syncthreads();
    for (int e = t; e < IH * IW * kCK; e += kConvThreads) {
      const int c = e % kCK, pix = e / kCK;
      const int r = pix / IW, col = pix % IW;
      const int gy = iy0 + r, gx = ix0 + col;
      float v = 0.f;
      if (c < ck && gy >= 0 && gy < a.H && gx >= 0 && gx < a.W) v = xb[((long long)gy * a.W + gx) * a.cin + c0 + c];
      s_in[(c * IH + r) * IW + col] = v;
    }
    for (int e = t; e < kCK * 9 * COUT; e += kConvThreads) {
      const int co = e % COUT, tap = (e / COUT) % 9, c = e / (9 * COUT);
      s_w[e] = c < ck ? a.w[((long long)co * 9 + tap) * a.cin + c0 + c] : 0.f;
    }
    __syncthreads();
    for (int c = 0; c < ck; ++c) {
#pragma unroll
      for (int ky = 0; ky < 3; ++ky)
#pragma unroll
        for (int kx = 0; kx < 3; ++kx) {
          float xv[T::PX];
#pragma unroll
          for (int p = 0; p < T::PX; ++p) xv[p] = s_in[(c * IH + ly * STRIDE + ky) * IW + (lx + p) * STRIDE + kx];
          const float* wr = s_w + (c * 9 + ky * 3 + kx) * COUT + cg * T::CG;
          if constexpr (PK) {
#pragma unroll
            for (int q = 0; q < T::CG; q += 2) {
              const float2 wv = *reinterpret_cast<const float2*>(wr + q);
#pragma unroll
              for (int p = 0; p < T::PX; ++p) ffma2(acc[p][q / 2], xv[p], wv.x, wv.y);
            }
          } else {
#pragma unroll
            for (int q = 0; q < T::CG; ++q) {
              const float wv = wr[q];
#pragma unroll
              for (int p = 0; p < T::PX; ++p) acc[p][q] = fmaf(xv[p], wv, acc[p][q]);
            }
          }
        }
    }
  }
  const int oy = oy0 + ly;
  if (oy >= a.Ho) return;
  const long long obase = (long long)b * a.Ho * a.Wo * COUT;
  const float* add = a.addend ? a.addend + (a.addend_per_model ? (a.model_of ? a.model_of[b] : 0) : b) * a.addend_bstride : nullptr;
#pragma unroll
  for (int p = 0; p < T::PX; ++p) {
    const int ox = ox0 + lx + p;
    if (ox >= a.Wo) continue;
    const long long o = obase + ((long long)oy * a.Wo + ox) * COUT + cg * T::CG;
    const long long oa = ((long long)oy * a.Wo + ox) * COUT + cg * T::CG;
#pragma unroll
    for (int q = 0; q < T::CG; ++q) {
      float v = acc_at<PK>(acc[p], q) + a.bias[cg * T::CG + q];
      if (a.softplus) v = softplusf(v);
      if (add) v += add[oa + q];
      if (a.residual) v += a.residual[o + q];
      a.y[o + q] = v;
    }
  }
}

// Transposed 3x3 convolution, stride 2, pad 1, out = 2 x in (autodiff.py:510-541).
// Output o along an axis receives x[q]*w[1] if o = 2q, and x[q+1]*w[0] +
// x[q]*w[2] if o = 2q+1.  Each thread handles 4 outputs of one parity class.
template <int COUT>
__global__ void __launch_bounds__(kConvThreads) k_tconv(ConvArgs a) {
  using T = Tile<COUT>;
  constexpr int QH = T::TH / 2, QW = T::TW / 2;  // per-class sub-tile
  constexpr int IH = QH + 1, IW = QW + 1;
  extern __shared__ float smem[];
  float* s_in = smem;
  float* s_w = smem + ((kCK * IH * IW + 3) & ~3);  // 16-byte aligned (paired weight loads)
  const int b = blockIdx.z;
  if (a.active && a.active[b] == nullptr) return;
  const int tiles_x = (a.Wo + T::TW - 1) / T::TW;
  const int oy0 = (blockIdx.x / tiles_x) * T::TH, ox0 = (blockIdx.x % tiles_x) * T::TW;
  const int qy0 = oy0 / 2, qx0 = ox0 / 2;
  const int t = threadIdx.x;
  constexpr int PG = T::TPX / T::PX;  // = 4 classes x (QH*QW/PX)
  constexpr int PGC = QH * QW / T::PX;
  const int cg = t / PG, pg = t % PG;
  const int cls = pg / PGC, pgc = pg % PGC;
  const int py = cls >> 1, px = cls & 1;
  const int qy = pgc / (QW / T::PX), qx = (pgc % (QW / T::PX)) * T::PX;
  // output-channel pairs packed fp32x2 (FFMA2) when CG is even; scalar otherwise
  constexpr bool PK = T::CG % 2 == 0;
  constexpr int NQ = PK ? T::CG / 2 : T::CG;
  using AccT = typename std::conditional<PK, unsigned long long, float>::type;
  AccT acc[T::PX][NQ];
#pragma unroll
  for (int p = 0; p < T::PX; ++p)
#pragma unroll
    for (int q = 0; q < NQ; ++q) acc[p][q] = AccT(0);
  const float* xb = a.x + (long long)b * a.H * a.W * a.cin;
  // taps per parity: even -> (k=1, d=0); odd -> (k=0, d=1), (k=2, d=0)
  const int nty = py ? 2 : 1, ntx = px ? 2 : 1;
  for (int c0 = 0; c0 < a.cin; c0 += kCK) {
    const int ck = min(kCK, a.cin - c0);
    __syncthreads();
    for (int e = t; e < IH * IW * kCK; e += kConvThreads) {
      const int c = e % kCK, pix = e / kCK;
      const int r = pix / IW, col = pix % IW;
      const int gy = qy0 + r, gx = qx0 + col;
      float v = 0.f;
      if (c < ck && gy < a.H && gx < a.W) v = xb[((long long)gy * a.W + gx) * a.cin + c0 + c];
      s_in[(c * IH + r) * IW + col] = v;
    }
    for (int e = t; e < kCK * 9 * COUT; e += kConvThreads) {
      const int co = e % COUT, tap = (e / COUT) % 9, c = e / (9 * COUT);
      s_w[e] = c < ck ? a.w[((long long)co * 9 + tap) * a.cin + c0 + c] : 0.f;
    }
    __syncthreads();
    for (int c = 0; c < ck; ++c) {
      for (int ty = 0; ty < nty; ++ty) {
        const int ky = py ? (ty ? 2 : 0) : 1, dy = (py && !ty) ? 1 : 0;
        for (int tx = 0; tx < ntx; ++tx) {
          const int kx = px ? (tx ? 2 : 0) : 1, dx = (px && !tx) ? 1 : 0;
          float xv[T::PX];
#pragma unroll
          for (int p = 0; p < T::PX; ++p) xv[p] = s_in[(c * IH + qy + dy) * IW + qx + p + dx];
          const float* wr = s_w + (c * 9 + ky * 3 + kx) * COUT + cg * T::CG;
          if constexpr (PK) {
#pragma unroll
            for (int q = 0; q < T::CG; q += 2) {
              const float2 wv = *reinterpret_cast<const float2*>(wr + q);
#pragma unroll
              for (int p = 0; p < T::PX; ++p) ffma2(acc[p][q / 2], xv[p], wv.x, wv.y);
            }
          } else {
#pragma unroll
            for (int q = 0; q < T::CG; ++q) {
              const float wv = wr[q];
#pragma unroll
              for (int p = 0; p < T::PX; ++p) acc[p][q] = fmaf(xv[p], wv, acc[p][q]);
            }
          }
        }
      }
    }
  }
  const int oy = oy0 + 2 * qy + py;
  if (oy >= a.Ho) return;
  const long long obase = (long long)b * a.Ho * a.Wo * COUT;
  const float* add = a.addend ? a.addend + (a.addend_per_model ? (a.model_of ? a.model_of[b] : 0) : b) * a.addend_bstride : nullptr;
#pragma unroll
  for (int p = 0; p < T::PX; ++p) {
    const int ox = ox0 + 2 * (qx + p) + px;
    if (ox >= a.Wo) continue;
    const long long oa = ((long long)oy * a.Wo + ox) * COUT + cg * T::CG;
    const long long o = obase + oa;
#pragma unroll
    for (int q = 0; q < T::CG; ++q) {
      float v = acc_at<PK>(acc[p], q) + a.bias[cg * T::CG + q];
      if (a.softplus) v = softplusf(v);
      if (add) v += add[oa + q];
      if (a.residual) v += a.residual[o + q];
      a.y[o + q] = v;
    }
  }
}

template <int COUT, int STRIDE>
size_t conv_smem() {
  using T = Tile<COUT>;
  constexpr int IH = (T::TH - 1) * STRIDE + 3, IW = (T::TW - 1) * STRIDE + 3;
  return sizeof(float) * (((kCK * IH * IW + 3) & ~3) + kCK * 9 * COUT);
}
template <int COUT>
size_t tconv_smem() {
  using T = Tile<COUT>;
  return sizeof(float) * (((kCK * (T::TH / 2 + 1) * (T::TW / 2 + 1) + 3) & ~3) + kCK * 9 * COUT);
}

template <int COUT, int STRIDE>
void launch_conv_t(const ConvArgs& a, int B, cudaStream_t st) {
  using T = Tile<COUT>;
  static bool attr = false;
  const size_t sm = conv_smem<COUT, STRIDE>();
  if (!attr) {
    cudaFuncSetAttribute(k_conv<COUT, STRIDE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    attr = true;
  }
  dim3 g(cdiv_u(a.Ho, T::TH) * cdiv_u(a.Wo, T::TW), 1, B);
  k_conv<COUT, STRIDE><<<g, kConvThreads, sm, st>>>(a);
}
template <int COUT>
void launch_tconv_t(const ConvArgs& a, int B, cudaStream_t st) {
  using T = Tile<COUT>;
  static bool attr = false;
  const size_t sm = tconv_smem<COUT>();
  if (!attr) {
    cudaFuncSetAttribute(k_tconv<COUT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    attr = true;
  }
  dim3 g(cdiv_u(a.Ho, T::TH) * cdiv_u(a.Wo, T::TW), 1, B);
  k_tconv<COUT><<<g, kConvThreads, sm, st>>>(a);
}

// Thin convolutions, stride 1: the 2-channel stems (cin = 2) and the
// 2-channel head (cout = 2).  Two lanes share an output pixel and split its
// wide side: stems give each lane cout / 2 output channels, heads give each
// lane cin / 2 input channels (partial sums reduced with a shuffle) -- the
// balance between per-lane work and registers (occupancy) that measured best.
// A thread walks a band of kThinRows rows top to bottom: each input row (pixels
// x-1, x, x+1) is read once and feeds the three output rows it touches, whose
// sums stay in registers (rolling window); an output row is stored when its
// last input row is in.  The next input row is loaded one iteration ahead and
// the row's addend / residual at the start of the iteration that stores it.
// Weights and bias sit in shared memory (broadcast reads).
constexpr int kThinRows = 32, kThinThreads = 128;
template <int CIN, int COUT>
__host__ __device__ constexpr int thin_lanes() { return 2; }

template <int N>
HS_DEV void load_vec(const float* p, float* v) {
  if constexpr (N % 4 == 0) {
#pragma unroll
    for (int i = 0; i < N; i += 4) {
      const float4 t = __ldg(reinterpret_cast<const float4*>(p + i));
      v[i] = t.x, v[i + 1] = t.y, v[i + 2] = t.z, v[i + 3] = t.w;
    }
  } else if constexpr (N == 2) {
    const float2 t = __ldg(reinterpret_cast<const float2*>(p));
    v[0] = t.x, v[1] = t.y;
  } else {
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = __ldg(p + i);
  }
}

template <int N>
HS_DEV void store_vec(float* p, const float* v) {
  if constexpr (N % 4 == 0) {
#pragma unroll
    for (int i = 0; i < N; i += 4) *reinterpret_cast<float4*>(p + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
  } else if constexpr (N == 2) {
    *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
  } else {
#pragma unroll
    for (int i = 0; i < N; ++i) p[i] = v[i];
  }
}

template <int CIN, int COUT>
__global__ void __launch_bounds__(kThinThreads) k_conv_thin(ConvArgs a) {
  constexpr bool kSplitIn = CIN > COUT;              // head: lanes split cin; stem: lanes split cout
  constexpr int L = thin_lanes<CIN, COUT>();
  constexpr int GI = kSplitIn ? CIN / L : CIN;       // input channels per lane
  constexpr int GO = kSplitIn ? COUT : COUT / L;     // output channels per lane
  static_assert(GI * L == CIN || !kSplitIn, "lane split");
  static_assert(GO * L == COUT || kSplitIn, "lane split");
  __shared__ __align__(16) float s_w[9 * CIN * COUT + COUT];  // [tap][cin][cout], then the bias
  for (int e = threadIdx.x; e < 9 * CIN * COUT; e += blockDim.x) {
    const int n = e % COUT, c = (e / COUT) % CIN, t = e / (COUT * CIN);
    s_w[e] = a.w[(n * 9 + t) * CIN + c];
  }
  __syncthreads();
  const int b = blockIdx.z;
  if (a.active && a.active[b] == nullptr) return;
  const int q = threadIdx.x % L;
  const int x = blockIdx.x * (kThinThreads / L) + threadIdx.x / L;
  const bool cout_c = COUT == 2 && a.cy != nullptr;     // complex output (head -> u0)
  const int Hl = cout_c ? a.cy_h : a.Ho, Wl = cout_c ? a.cy_w : a.Wo;  // extents walked
  const bool x_ok = x < Wl;  // whole lane groups agree: shuffles stay within live lanes
  const int ci0 = kSplitIn ? GI * q : 0, co0 = kSplitIn ? 0 : GO * q;
  const int oy0 = blockIdx.y * kThinRows, oy1 = min(Hl, oy0 + kThinRows);
  const float* xb = a.x ? a.x + (long long)b * a.H * a.W * CIN : nullptr;
  const bool cin_c = CIN == 2 && a.cx_ld > 0;  // complex input (Krylov vector -> stem)
  const float2* xc = cin_c ? (a.cx.tab ? a.cx.tab[b] : a.cx.base + (long long)b * a.cx.bstride) : nullptr;
  const float xcs = cin_c && a.cx.scale ? a.cx.scale[b] : 1.f;
  const float* add = a.addend ? a.addend + (a.addend_per_model ? (a.model_of ? a.model_of[b] : 0) : b) * a.addend_bstride
                              : nullptr;
  // acc[0]: output row iy - 1 (its ky = 2 tap), acc[1]: row iy (ky = 1), acc[2]: row iy + 1 (ky = 0);
  // bias is added once, at the store (after the cin reduction for heads)
  float acc[3][GO];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int n = 0; n < GO; ++n) acc[r][n] = 0.f;
  // the next input row's three pixel vectors are loaded one iteration ahead
  auto load_row = [&](int iy, float(&xv)[3][GI]) {
#pragma unroll
    for (int kx = 0; kx < 3; ++kx) {
      const int ix = x + kx - 1;
      if (x_ok && iy >= 0 && iy < a.H && ix >= 0 && ix < a.W) {
        if (cin_c) {
          const float2 v = xc[(long long)iy * a.cx_ld + ix];
          xv[kx][0] = v.x * xcs;
          xv[kx][GI > 1 ? 1 : 0] = v.y * xcs;
        } else {
          load_vec<GI>(xb + ((long long)iy * a.W + ix) * CIN + ci0, xv[kx]);
        }
      } else
#pragma unroll
        for (int c = 0; c < GI; ++c) xv[kx][c] = 0.f;
    }
  };
  // addend + residual of an output row, summed, fetched one row ahead as well
  const bool store_lane = x_ok && (!kSplitIn || q == 0);
  // (a single side input is a plain load into sd: nothing waits on it until the store)
  auto load_side = [&](int oy, float(&sd)[GO]) {
#pragma unroll
    for (int n = 0; n < GO; ++n) sd[n] = 0.f;
    if (!store_lane || oy < oy0 || oy >= oy1) return;
    const long long p = (long long)oy * a.Wo + x;
    const float* res = a.residual ? a.residual + (long long)b * a.Ho * a.Wo * COUT + p * COUT + co0 : nullptr;
    if (add && !res) {
      load_vec<GO>(add + p * COUT + co0, sd);
    } else if (res && !add) {
      load_vec<GO>(res, sd);
    } else if (add && res) {
      float t[GO], u[GO];
      load_vec<GO>(add + p * COUT + co0, t);
      load_vec<GO>(res, u);
#pragma unroll
      for (int n = 0; n < GO; ++n) sd[n] = t[n] + u[n];
    }
  };
  // bias from shared memory (broadcast) rather than GO more registers
  float* s_bias = s_w + 9 * CIN * COUT;
  for (int n = threadIdx.x; n < COUT; n += blockDim.x) s_bias[n] = a.bias[n];
  __syncthreads();
  float nx[3][GI];
  load_row(oy0 - 1, nx);
  for (int iy = oy0 - 1; iy <= oy1; ++iy) {
    float xv[3][GI], sd[GO];
#pragma unroll
    for (int kx = 0; kx < 3; ++kx)
#pragma unroll
      for (int c = 0; c < GI; ++c) xv[kx][c] = nx[kx][c];
    if (iy < oy1) load_row(iy + 1, nx);
    load_side(iy - 1, sd);  // consumed by this iteration's store, after the row's FMAs
#pragma unroll
    for (int kx = 0; kx < 3; ++kx)
#pragma unroll
      for (int ky = 0; ky < 3; ++ky) {
        float* ac = acc[2 - ky];
#pragma unroll
        for (int c = 0; c < GI; ++c)
#pragma unroll
          for (int n = 0; n < GO; ++n) ac[n] = fmaf(xv[kx][c], s_w[((ky * 3 + kx) * CIN + ci0 + c) * COUT + co0 + n], ac[n]);
      }
    const int oy = iy - 1;  // complete: rows oy - 1, oy, oy + 1 are in
    if (oy >= oy0 && oy < oy1) {
      float v[GO];
#pragma unroll
      for (int n = 0; n < GO; ++n) {
        v[n] = acc[0][n];
        if (kSplitIn)
#pragma unroll
          for (int sh = 1; sh < L; sh <<= 1) v[n] += __shfl_xor_sync(0xffffffffu, v[n], sh);
      }
      if (store_lane) {
        const long long o = (long long)b * a.Ho * a.Wo * COUT + ((long long)oy * a.Wo + x) * COUT + co0;
#pragma unroll
        for (int n = 0; n < GO; ++n) {
          float t = v[n] + s_bias[co0 + n];
          if (a.softplus) t = softplus_fast(t);
          v[n] = t + sd[n];
        }
        if (cout_c) {
          const bool valid = oy < a.Ho && x < a.Wo;
          a.cy[(long long)b * a.cy_n + (long long)oy * a.cy_ld + x] =
              valid ? make_float2(a.cy_scale * v[0], a.cy_scale * v[GO > 1 ? 1 : 0]) : make_float2(0.f, 0.f);
        } else {
          store_vec<GO>(a.y + o, v);
        }
      }
    }
#pragma unroll
    for (int n = 0; n < GO; ++n) {
      acc[0][n] = acc[1][n];
      acc[1][n] = acc[2][n];
      acc[2][n] = 0.f;
    }
  }
}

template <int CIN, int COUT>
void launch_thin(const ConvArgs& a, int B, cudaStream_t st) {
  constexpr int pix = kThinThreads / thin_lanes<CIN, COUT>();
  const int Hl = a.cy ? a.cy_h : a.Ho, Wl = a.cy ? a.cy_w : a.Wo;
  const dim3 grid((unsigned)((Wl + pix - 1) / pix), (unsigned)((Hl + kThinRows - 1) / kThinRows),
                  (unsigned)B);
  k_conv_thin<CIN, COUT><<<grid, kThinThreads, 0, st>>>(a);
}

// Thin convolutions with the weights in the kernel-parameter constant bank: one thread per output
// column walks kThinRows rows (rolling window as k_conv_thin) and owns every channel of its pixel,
// so all weight indices are compile-time constants and each FFMA takes its weight straight from
// the constant bank -- no shared-memory weight reads, no lane split, no shuffles.

template <int CIN, int COUT>
struct ThinW {
  float w[9 * CIN * COUT];  // [tap][cin][cout]
  float b[COUT];
};

template <int CIN, int COUT>
__global__ void __launch_bounds__(kThinThreads) k_conv_thin1(ConvArgs a, const __grid_constant__ ThinW<CIN, COUT> wt) {
  const int b = blockIdx.z;
  if (a.active && a.active[b] == nullptr) return;
  const int x = blockIdx.x * kThinThreads + threadIdx.x;
  const bool cout_c = COUT == 2 && a.cy != nullptr;
  const int Hl = cout_c ? a.cy_h : a.Ho, Wl = cout_c ? a.cy_w : a.Wo;
  if (x >= Wl) return;
  const int oy0 = blockIdx.y * kThinRows, oy1 = min(Hl, oy0 + kThinRows);
  const float* xb = a.x ? a.x + (long long)b * a.H * a.W * CIN : nullptr;
  const bool cin_c = CIN == 2 && a.cx_ld > 0;
  const float2* xc = cin_c ? (a.cx.tab ? a.cx.tab[b] : a.cx.base + (long long)b * a.cx.bstride) : nullptr;
  const float xcs = cin_c && a.cx.scale ? a.cx.scale[b] : 1.f;
  const float* add = a.addend ? a.addend + (a.addend_per_model ? (a.model_of ? a.model_of[b] : 0) : b) * a.addend_bstride
                              : nullptr;
  static_assert(COUT % 2 == 0, "packed accumulators");
  unsigned long long acc[3][COUT / 2];  // output channel pairs, packed fp32x2
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int n = 0; n < COUT / 2; ++n) acc[r][n] = 0ull;
  auto load_row = [&](int iy, float(&xv)[3][CIN]) {
#pragma unroll
    for (int kx = 0; kx < 3; ++kx) {
      const int ix = x + kx - 1;
      if (iy >= 0 && iy < a.H && ix >= 0 && ix < a.W) {
        if (cin_c) {
          const float2 v = xc[(long long)iy * a.cx_ld + ix];
          xv[kx][0] = v.x * xcs;
          xv[kx][CIN > 1 ? 1 : 0] = v.y * xcs;
        } else {
          load_vec<CIN>(xb + ((long long)iy * a.W + ix) * CIN, xv[kx]);
        }
      } else {
#pragma unroll
        for (int c = 0; c < CIN; ++c) xv[kx][c] = 0.f;
      }
    }
  };
  auto load_side = [&](int oy, float(&sd)[COUT]) {
#pragma unroll
    for (int n = 0; n < COUT; ++n) sd[n] = 0.f;
    if (oy < oy0 || oy >= oy1 || oy >= a.Ho || x >= a.Wo) return;
    const long long p = (long long)oy * a.Wo + x;
    if (add) load_vec<COUT>(add + p * COUT, sd);
    if (a.residual) {
      float u[COUT];
      load_vec<COUT>(a.residual + (long long)b * a.Ho * a.Wo * COUT + p * COUT, u);
#pragma unroll
      for (int n = 0; n < COUT; ++n) sd[n] += u[n];
    }
  };
  float nx[3][CIN];
  load_row(oy0 - 1, nx);
  for (int iy = oy0 - 1; iy <= oy1; ++iy) {
    float xv[3][CIN], sd[COUT];
#pragma unroll
    for (int kx = 0; kx < 3; ++kx)
#pragma unroll
      for (int c = 0; c < CIN; ++c) xv[kx][c] = nx[kx][c];
    if (iy < oy1) load_row(iy + 1, nx);
    load_side(iy - 1, sd);
#pragma unroll
    for (int ky = 0; ky < 3; ++ky)
#pragma unroll
      for (int kx = 0; kx < 3; ++kx)
#pragma unroll
        for (int c = 0; c < CIN; ++c)
#pragma unroll
          for (int n = 0; n < COUT / 2; ++n)
            ffma2(acc[2 - ky][n], xv[kx][c], wt.w[((ky * 3 + kx) * CIN + c) * COUT + 2 * n],
                  wt.w[((ky * 3 + kx) * CIN + c) * COUT + 2 * n + 1]);
    const int oy = iy - 1;
    if (oy >= oy0 && oy < oy1) {
      float v[COUT];
#pragma unroll
      for (int n = 0; n < COUT; ++n) {
        float t = ((n & 1) ? hi32(acc[0][n / 2]) : lo32(acc[0][n / 2])) + wt.b[n];
        if (a.softplus) t = softplus_fast(t);
        v[n] = t + sd[n];
      }
      if (cout_c) {
        const bool valid = oy < a.Ho && x < a.Wo;
        a.cy[(long long)b * a.cy_n + (long long)oy * a.cy_ld + x] =
            valid ? make_float2(a.cy_scale * v[0], a.cy_scale * v[COUT > 1 ? 1 : 0]) : make_float2(0.f, 0.f);
      } else if (oy < a.Ho) {
        store_vec<COUT>(a.y + (long long)b * a.Ho * a.Wo * COUT + ((long long)oy * a.Wo + x) * COUT, v);
      }
    }
#pragma unroll
    for (int n = 0; n < COUT / 2; ++n) {
      acc[0][n] = acc[1][n];
      acc[1][n] = acc[2][n];
      acc[2][n] = 0ull;
    }
  }
}

// The stem (2 -> 16) as one thread per output pixel: the nine complex inputs come from L1 (neighbouring
// threads and rows share them), so no rolling three-row window of accumulators is kept and the kernel
// runs at full occupancy; the weights are in the kernel-parameter constant bank as in k_conv_thin1.
#ifndef HS_STEM_TR
#define HS_STEM_TR 0  // measured: the group-of-four transposed stores are slower here (1.17 vs 0.94 ms at C3)
#endif
#ifndef HS_STEM_PX
#define HS_STEM_PX 1
#endif
template <int COUT>
__global__ void __launch_bounds__(256) k_conv_stem_px(ConvArgs a, const __grid_constant__ ThinW<2, COUT> wt) {
  const int b = blockIdx.z;
  if (a.active && a.active[b] == nullptr) return;
  const int x = blockIdx.x * 256 + threadIdx.x, oy = blockIdx.y;
  // TR: each group of four lanes transposes its pixels' 16-byte chunks so every store / side load
  // moves whole 64-byte pixels (all lanes stay for the shuffles)
  constexpr bool TR = HS_STEM_TR && COUT == 16;
  if (!TR && x >= a.Wo) return;
  const int gi = threadIdx.x & 3, xg = x - gi;
  const bool cin_c = a.cx_ld > 0;
  const float* xb = a.x ? a.x + (long long)b * a.H * a.W * 2 : nullptr;
  const float2* xc = cin_c ? (a.cx.tab ? a.cx.tab[b] : a.cx.base + (long long)b * a.cx.bstride) : nullptr;
  const float xcs = cin_c && a.cx.scale ? a.cx.scale[b] : 1.f;
  const float* add = a.addend ? a.addend + (a.addend_per_model ? (a.model_of ? a.model_of[b] : 0) : b) * a.addend_bstride
                              : nullptr;
  const long long p = (long long)oy * a.Wo + x;
  float sd[COUT];
#pragma unroll
  for (int n = 0; n < COUT; ++n) sd[n] = 0.f;
  if (TR) {  // chunk gi of pixels xg .. xg + 3
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (xg + j >= a.Wo) continue;
      const long long pj = ((long long)oy * a.Wo + xg + j) * COUT + 4 * gi;
      if (add) load_vec<4>(add + pj, &sd[4 * j]);
      if (a.residual) {
        float u[4];
        load_vec<4>(a.residual + (long long)b * a.Ho * a.Wo * COUT + pj, u);
#pragma unroll
        for (int n = 0; n < 4; ++n) sd[4 * j + n] += u[n];
      }
    }
  } else if (add) {
    load_vec<COUT>(add + p * COUT, sd);
  }
  if (!TR && a.residual) {
    float u[COUT];
    load_vec<COUT>(a.residual + (long long)b * a.Ho * a.Wo * COUT + p * COUT, u);
#pragma unroll
    for (int n = 0; n < COUT; ++n) sd[n] += u[n];
  }
  float2 xv[3][3];
#pragma unroll
  for (int ky = 0; ky < 3; ++ky)
#pragma unroll
    for (int kx = 0; kx < 3; ++kx) {
      const int iy = oy + ky - 1, ix = x + kx - 1;
      float2 v = make_float2(0.f, 0.f);
      if (iy >= 0 && iy < a.H && ix >= 0 && ix < a.W) {
        if (cin_c) {
          const float2 c = xc[(long long)iy * a.cx_ld + ix];
          v = make_float2(c.x * xcs, c.y * xcs);
        } else {
          v = *reinterpret_cast<const float2*>(xb + ((long long)iy * a.W + ix) * 2);
        }
      }
      xv[ky][kx] = v;
    }
  unsigned long long acc[COUT / 2];
#pragma unroll
  for (int n = 0; n < COUT / 2; ++n) acc[n] = 0ull;
#pragma unroll
  for (int ky = 0; ky < 3; ++ky)
#pragma unroll
    for (int kx = 0; kx < 3; ++kx)
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int n = 0; n < COUT / 2; ++n)
          ffma2(acc[n], c ? xv[ky][kx].y : xv[ky][kx].x, wt.w[((ky * 3 + kx) * 2 + c) * COUT + 2 * n],
                wt.w[((ky * 3 + kx) * 2 + c) * COUT + 2 * n + 1]);
  float v[COUT];
#pragma unroll
  for (int n = 0; n < COUT; ++n) {
    float t = ((n & 1) ? hi32(acc[n / 2]) : lo32(acc[n / 2])) + wt.b[n];
    if (a.softplus) t = softplus_fast(t);
    v[n] = TR ? t : t + sd[n];
  }
  if constexpr (TR) {
    float4 ch[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) ch[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    group4_transpose(ch, gi);
    float* yrow = a.y + (long long)b * a.Ho * a.Wo * COUT + (long long)oy * a.Wo * COUT;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (xg + j < a.Wo)
        *reinterpret_cast<float4*>(yrow + (long long)(xg + j) * COUT + 4 * gi) =
            make_float4(ch[j].x + sd[4 * j], ch[j].y + sd[4 * j + 1], ch[j].z + sd[4 * j + 2], ch[j].w + sd[4 * j + 3]);
  } else {
    store_vec<COUT>(a.y + (long long)b * a.Ho * a.Wo * COUT + p * COUT, v);
  }
}

template <int CIN, int COUT>
void launch_thin1(const ConvArgs& a, const float* host_w, int B, cudaStream_t st) {
  ThinW<CIN, COUT> wt;
  for (int i = 0; i < 9 * CIN * COUT; ++i) wt.w[i] = host_w[i];
  for (int n = 0; n < COUT; ++n) wt.b[n] = host_w[9 * CIN * COUT + n];
  const int Hl = a.cy ? a.cy_h : a.Ho, Wl = a.cy ? a.cy_w : a.Wo;
  if constexpr (CIN == 2 && COUT == 16 && HS_STEM_PX) {
    if (!a.cy) {
      k_conv_stem_px<COUT><<<dim3((unsigned)((a.Wo + 255) / 256), (unsigned)a.Ho, (unsigned)B), 256, 0, st>>>(a, wt);
      return;
    }
  }
  const dim3 grid((unsigned)((Wl + kThinThreads - 1) / kThinThreads), (unsigned)((Hl + kThinRows - 1) / kThinRows),
                  (unsigned)B);
  k_conv_thin1<CIN, COUT><<<grid, kThinThreads, 0, st>>>(a, wt);
}

template <int CIN, int COUT>
__global__ void __launch_bounds__(kThinThreads) k_conv_thin1w(ConvArgs a, const __grid_constant__ ThinW<CIN, COUT> wt) {
  // warp = a 32-column strip of one band of kThinRows rows; every lane loads
  // only its own pixel and takes its left / right neighbours from the adjacent
  // lanes (lanes 0 and 31 also load the one pixel outside the strip)
  const int b = blockIdx.z;
  if (a.active && a.active[b] == nullptr) return;
  const int lane = threadIdx.x & 31;
  const int x = blockIdx.x * 32 + lane;
  const bool cout_c = COUT == 2 && a.cy != nullptr;
  const int Hl = cout_c ? a.cy_h : a.Ho, Wl = cout_c ? a.cy_w : a.Wo;
  const int oy0 = (blockIdx.y * (kThinThreads / 32) + (threadIdx.x >> 5)) * kThinRows, oy1 = min(Hl, oy0 + kThinRows);
  if (oy0 >= Hl) return;  // whole warp
  const bool xin = x < Wl;
  const float* xb = a.x ? a.x + (long long)b * a.H * a.W * CIN : nullptr;
  const bool cin_c = CIN == 2 && a.cx_ld > 0;
  const float2* xc = cin_c ? (a.cx.tab ? a.cx.tab[b] : a.cx.base + (long long)b * a.cx.bstride) : nullptr;
  const float xcs = cin_c && a.cx.scale ? a.cx.scale[b] : 1.f;
  const float* add = a.addend ? a.addend + (a.addend_per_model ? (a.model_of ? a.model_of[b] : 0) : b) * a.addend_bstride
                              : nullptr;
  static_assert(COUT % 2 == 0, "packed accumulators");
  unsigned long long acc[3][COUT / 2];  // output channel pairs, packed fp32x2
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int n = 0; n < COUT / 2; ++n) acc[r][n] = 0ull;
  auto load_px = [&](int iy, int ix, float(&v)[CIN]) {
    if (iy >= 0 && iy < a.H && ix >= 0 && ix < a.W) {
      if (cin_c) {
        const float2 t = xc[(long long)iy * a.cx_ld + ix];
        v[0] = t.x * xcs;
        v[CIN > 1 ? 1 : 0] = t.y * xcs;
      } else {
        load_vec<CIN>(xb + ((long long)iy * a.W + ix) * CIN, v);
      }
    } else {
#pragma unroll
      for (int c = 0; c < CIN; ++c) v[c] = 0.f;
    }
  };
  // own pixel and (edge lanes) the outside neighbour of a row
  auto load_row = [&](int iy, float(&own)[CIN], float(&edge)[CIN]) {
    load_px(iy, x, own);
    if (lane == 0) load_px(iy, x - 1, edge);
    if (lane == 31) load_px(iy, x + 1, edge);
  };
  auto load_side = [&](int oy, float(&sd)[COUT]) {
#pragma unroll
    for (int n = 0; n < COUT; ++n) sd[n] = 0.f;
    if (oy < oy0 || oy >= oy1 || oy >= a.Ho || x >= a.Wo) return;
    const long long p = (long long)oy * a.Wo + x;
    if (add) load_vec<COUT>(add + p * COUT, sd);
    if (a.residual) {
      float u[COUT];
      load_vec<COUT>(a.residual + (long long)b * a.Ho * a.Wo * COUT + p * COUT, u);
#pragma unroll
      for (int n = 0; n < COUT; ++n) sd[n] += u[n];
    }
  };
  float nown[CIN], nedge[CIN];
#pragma unroll
  for (int c = 0; c < CIN; ++c) nedge[c] = 0.f;
  load_row(oy0 - 1, nown, nedge);
  for (int iy = oy0 - 1; iy <= oy1; ++iy) {
    float xv[3][CIN], sd[COUT];
#pragma unroll
    for (int c = 0; c < CIN; ++c) {
      const float up = __shfl_up_sync(0xffffffffu, nown[c], 1), dn = __shfl_down_sync(0xffffffffu, nown[c], 1);
      xv[0][c] = lane == 0 ? nedge[c] : up;
      xv[1][c] = nown[c];
      xv[2][c] = lane == 31 ? nedge[c] : dn;
    }
    if (iy < oy1) load_row(iy + 1, nown, nedge);
    load_side(iy - 1, sd);
#pragma unroll
    for (int ky = 0; ky < 3; ++ky)
#pragma unroll
      for (int kx = 0; kx < 3; ++kx)
#pragma unroll
        for (int c = 0; c < CIN; ++c)
#pragma unroll
          for (int n = 0; n < COUT / 2; ++n)
            ffma2(acc[2 - ky][n], xv[kx][c], wt.w[((ky * 3 + kx) * CIN + c) * COUT + 2 * n],
                  wt.w[((ky * 3 + kx) * CIN + c) * COUT + 2 * n + 1]);
    const int oy = iy - 1;
    if (oy >= oy0 && oy < oy1 && xin) {
      float v[COUT];
#pragma unroll
      for (int n = 0; n < COUT; ++n) {
        float t = ((n & 1) ? hi32(acc[0][n / 2]) : lo32(acc[0][n / 2])) + wt.b[n];
        if (a.softplus) t = softplus_fast(t);
        v[n] = t + sd[n];
      }
      if (cout_c) {
        const bool valid = oy < a.Ho && x < a.Wo;
        a.cy[(long long)b * a.cy_n + (long long)oy * a.cy_ld + x] =
            valid ? make_float2(a.cy_scale * v[0], a.cy_scale * v[COUT > 1 ? 1 : 0]) : make_float2(0.f, 0.f);
      } else if (oy < a.Ho) {
        store_vec<COUT>(a.y + (long long)b * a.Ho * a.Wo * COUT + ((long long)oy * a.Wo + x) * COUT, v);
      }
    }
#pragma unroll
    for (int n = 0; n < COUT / 2; ++n) {
      acc[0][n] = acc[1][n];
      acc[1][n] = acc[2][n];
      acc[2][n] = 0ull;
    }
  }
}

template <int CIN, int COUT>
void launch_thin1w(const ConvArgs& a, const float* host_w, int B, cudaStream_t st) {
  ThinW<CIN, COUT> wt;
  for (int i = 0; i < 9 * CIN * COUT; ++i) wt.w[i] = host_w[i];
  for (int n = 0; n < COUT; ++n) wt.b[n] = host_w[9 * CIN * COUT + n];
  const int Hl = a.cy ? a.cy_h : a.Ho, Wl = a.cy ? a.cy_w : a.Wo;
  const int bands = (Hl + kThinRows - 1) / kThinRows, wpb = kThinThreads / 32;
  const dim3 grid((unsigned)((Wl + 31) / 32), (unsigned)((bands + wpb - 1) / wpb), (unsigned)B);
  k_conv_thin1w<CIN, COUT><<<grid, kThinThreads, 0, st>>>(a, wt);
}

int launch_conv(const hs_conv_t& c, const float* x, int B, int H, int W, float* y, const float* addend,
                long long addend_bstride, const int* model_of, const float* residual, const void* const* active,
                cudaStream_t st, bool model_of_addend = false, const ThinIO* io = nullptr, bool planar_out = false) {
  ConvArgs a{};
  if (io) {  // complex Krylov-vector input (stem) and / or complex u0 output (head): thin kernels only
    if (io->in_ld > 0 && c.cin == 2) {
      a.cx = io->in;
      a.cx_ld = io->in_ld;
    }
    if (io->out && c.cout == 2) {
      a.cy = io->out;
      a.cy_n = io->out_n;
      a.cy_ld = io->out_ld;
      a.cy_h = io->out_h;
      a.cy_w = io->out_w;
      a.cy_scale = io->out_scale;
    }
  }
  a.x = x;
  a.H = H;
  a.W = W;
  a.cin = c.cin;
  a.y = y;
  a.cout = c.cout;
  if (c.transposed) {
    a.Ho = 2 * H;
    a.Wo = 2 * W;
  } else {
    a.Ho = (H - 1) / c.stride + 1;
    a.Wo = (W - 1) / c.stride + 1;
  }
  a.w = c.w;
  a.bias = c.b;
  a.softplus = c.softplus;
  a.addend = addend;
  a.addend_bstride = addend_bstride;
  a.model_of = model_of;
  a.addend_per_model = addend && model_of_addend;
  prof::count(1);
  const double flops =
      2.0 * 9.0 * c.cin * c.cout * (c.transposed ? (double)H * W : (double)a.Ho * a.Wo) * prof::active_hint(B);
  const bool l0 = c.cin == 16 && c.cout == 16 && c.stride == 1 && !c.transposed;
  // CONV_L0 records algorithmic HBM bytes: input + output (+ per-RHS addend) (+ residual), once each; an
  // addend shared by a model's RHS (the encoder features) is read from DRAM once per model, not per RHS,
  // and is not counted
  const double l0_bytes = 4.0 * 16 * (double)H * W * (2 + (addend && !model_of_addend ? 1 : 0) + (residual ? 1 : 0)) *
                          prof::active_hint(B);
  const bool wide = (c.cin >= 64 || c.cout >= 64) && c.cin > 2 && c.cout > 2;
  struct Scope2 {
    int s1, s2;
    cudaStream_t st;
    double w1, w2;
    ~Scope2() {
      prof::stop(s2, st, w2);
      prof::stop(s1, st, w1);
    }
  };
  prof::set_label(c.cin * 100000 + c.cout * 100 + (c.transposed ? 2 : c.stride - 1));
  Scope2 scope{prof::start(prof::CONV, st),
               l0 ? prof::start(prof::CONV_L0, st) : (wide ? prof::start(prof::CONV_WIDE, st) : -1), st, flops,
               l0 ? l0_bytes : flops};
  a.residual = residual;
  a.active = active;
  if ((a.cx_ld > 0 || a.cy) && !(!c.transposed && c.stride == 1 && (c.cin == 2 || c.cout == 2)))
    return HS_ECONFIG;  // complex I/O is fused into the thin stem / head only
  if (!c.transposed && c.stride == 1 && io && io->host_w) {
    if (c.cin == 2 && c.cout == 16) return launch_thin1<2, 16>(a, io->host_w, B, st), HS_OK;
    if (c.cin == 16 && c.cout == 2) return launch_thin1w<16, 2>(a, io->host_w, B, st), HS_OK;
    if (c.cin == 2 && c.cout == 8) return launch_thin1<2, 8>(a, io->host_w, B, st), HS_OK;
    if (c.cin == 8 && c.cout == 2) return launch_thin1w<8, 2>(a, io->host_w, B, st), HS_OK;
  }
  if (!c.transposed && c.stride == 1) {
    if (c.cin == 2 && c.cout == 16) return launch_thin<2, 16>(a, B, st), HS_OK;
    if (c.cin == 2 && c.cout == 8) return launch_thin<2, 8>(a, B, st), HS_OK;
    if (c.cin == 16 && c.cout == 2) return launch_thin<16, 2>(a, B, st), HS_OK;
    if (c.cin == 8 && c.cout == 2) return launch_thin<8, 2>(a, B, st), HS_OK;
  }
  if (conv_wide_launch(a.x, a.H, a.W, a.cin, a.y, a.Ho, a.Wo, a.cout, c.stride, c.transposed, a.w, a.bias,
                       a.softplus, a.addend, a.addend_bstride, a.addend_per_model, a.model_of, a.residual, a.active, B,
                       st, planar_out ? 1 : 0))
    return HS_OK;
  if (conv_tc_supported(c.cin, c.cout, c.stride, c.transposed, H, W, a.Wo, planar_out ? 1 : 0) &&
      conv_tc_launch(a.x, a.H, a.W, a.cin, a.y, a.Ho, a.Wo, a.cout, c.stride, c.transposed, a.w, a.bias, a.softplus,
                     a.addend, a.addend_bstride, a.addend_per_model, a.model_of, a.residual, a.active, B, st,
                     planar_out ? 1 : 0))
    return HS_OK;
  if (planar_out) return HS_ECONFIG;  // only the tcgen05 epilogue writes the planar layout
#define HS_CONV_CASE(CO)                          \
  case CO:                                        \
    if (c.transposed)                             \
      launch_tconv_t<CO>(a, B, st);               \
    else if (c.stride == 2)                       \
      launch_conv_t<CO, 2>(a, B, st);             \
    else                                          \
      launch_conv_t<CO, 1>(a, B, st);             \
    return HS_OK;
  switch (c.cout) {
    HS_CONV_CASE(2)
    HS_CONV_CASE(4)
    HS_CONV_CASE(5)
    HS_CONV_CASE(8)
    HS_CONV_CASE(16)
    HS_CONV_CASE(32)
    HS_CONV_CASE(64)
    HS_CONV_CASE(128)
    default:
      return HS_ECONFIG;
  }
#undef HS_CONV_CASE
}

// ------------------------------------------------------- input / output glue

// NHWC real (C = 2 cc) at (h, w) -> complex NCHW (cc, 2h, 2w) zero-padded at the high end
__global__ void k_pack_pad(const float* x, const void* const* active, cufftComplex* z, int h, int w, int cc) {
  const int b = blockIdx.y;
  if (active && active[b] == nullptr) return;
  const int H2 = 2 * h, W2 = 2 * w;
  const long long n = (long long)cc * H2 * W2;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(e / ((long long)H2 * W2));
    const int rem = (int)(e - (long long)k * H2 * W2);
    const int y = rem / W2, xx = rem % W2;
    cufftComplex v = make_float2(0.f, 0.f);
    if (y < h && xx < w) {
      const float* px = x + (((long long)b * h + y) * w + xx) * (2 * cc);
      v = make_float2(px[2 * k], px[2 * k + 1]);
    }
    z[(long long)b * n + e] = v;
  }
}

__global__ void k_spec_mul(cufftComplex* z, const void* const* active, const cufftComplex* spec, long long per_b) {
  const int b = blockIdx.y;
  if (active && active[b] == nullptr) return;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < per_b; e += (long long)gridDim.x * blockDim.x)
    z[(long long)b * per_b + e] = cmul(z[(long long)b * per_b + e], spec[e]);
}

// (B, C, h, w) complex -> (B, C, 2h, 2w) zero-padded at the high end (pad2d_to, autodiff.py:283-294)
__global__ void k_pad_nchw(const cufftComplex* x, cufftComplex* z, int C, int h, int w) {
  const int b = blockIdx.y;
  const long long per_b = (long long)C * 4 * h * w;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < per_b; e += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(e / (4LL * h * w));
    const int rem = (int)(e - (long long)k * 4 * h * w);
    const int r = rem / (2 * w), c = rem % (2 * w);
    z[b * per_b + e] = (r < h && c < w) ? x[(((long long)b * C + k) * h + r) * w + c] : make_float2(0.f, 0.f);
  }
}

// (B, C, 2h, 2w) -> crop [:h, :w] with the inverse FFT's 1/N (ifft2 + crop2d)
__global__ void k_crop_nchw(const cufftComplex* z, cufftComplex* y, int C, int h, int w) {
  const int b = blockIdx.y;
  const long long per_b = (long long)C * h * w;
  const float inv = 1.f / (4.f * h * w);
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < per_b; e += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(e / ((long long)h * w));
    const int rem = (int)(e - (long long)k * h * w);
    const int r = rem / w, c = rem % w;
    cufftComplex v = z[(((long long)b * C + k) * 2 * h + r) * 2 * w + c];
    y[b * per_b + e] = make_float2(v.x * inv, v.y * inv);
  }
}

// complex NCHW (cc, 2h, 2w) -> crop [:h, :w], / (4hw), unpack to NHWC real (2cc)
__global__ void k_crop_unpack(const cufftComplex* z, const void* const* active, float* x, int h, int w, int cc) {
  const int b = blockIdx.y;
  if (active && active[b] == nullptr) return;
  const int H2 = 2 * h, W2 = 2 * w;
  const float inv = 1.f / (float)(H2 * W2);
  const long long n = (long long)h * w * cc;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(e % cc);
    const long long pix = e / cc;
    const int y = (int)(pix / w), xx = (int)(pix % w);
    cufftComplex v = z[(long long)b * cc * H2 * W2 + ((long long)k * H2 + y) * W2 + xx];
    float* px = x + (((long long)b * h + y) * w + xx) * (2 * cc);
    px[2 * k] = v.x * inv;
    px[2 * k + 1] = v.y * inv;
  }
}

// ------------------------------------------------------- Green spectrum (setup)

__global__ void k_green_embed(const float2* kern, cufftDoubleComplex* kp, int C, int bh, int bw) {
  const long long n = (long long)C * bh * bw;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(e / ((long long)bh * bw));
    const int rem = (int)(e - (long long)c * bh * bw);
    const int r = rem / bw, col = rem % bw;
    // place_kernel_corners (autodiff.py:323-337): rows (bh-1, 0, 1), cols (bw-1, 0, 1)
    int a = r == bh - 1 ? 0 : (r == 0 ? 1 : (r == 1 ? 2 : -1));
    int q = col == bw - 1 ? 0 : (col == 0 ? 1 : (col == 1 ? 2 : -1));
    cufftDoubleComplex v = make_double2(0.0, 0.0);
    if (a >= 0 && q >= 0) {
      float2 k = kern[c * 9 + a * 3 + q];
      v = make_double2(k.x, k.y);
    }
    kp[e] = v;
  }
}

// resp_hat = conj(S)/(S conj(S) + eps) * delta_hat with the reference's dtype flow
__global__ void k_green_divide(cufftDoubleComplex* s, long long n, int bh, int bw, double eps) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const int rem = (int)(e % ((long long)bh * bw));
    const int u = rem / bw, v = rem % bw;
    // S rounded to complex64 (ad.fft2 casts to the input's complex dtype)
    const float sr = (float)s[e].x, si = (float)s[e].y;
    // S * conj(S) in complex64 arithmetic, then + eps promotes to complex128
    const float pr = sr * sr - si * (-si);
    const float pi = sr * (-si) + si * sr;
    const double dr = (double)pr + eps, di = (double)pi;
    // conj(S) / denom in complex128
    const double cr = sr, ci = -(double)si;
    const double den = dr * dr + di * di;
    const double qr = (cr * dr + ci * di) / den, qi = (ci * dr - cr * di) / den;
    // delta at (bh/2, bw/2): spectrum (-1)^(u+v) for even sizes, rounded to complex64
    const double ph = -2.0 * M_PI * ((double)u * (bh / 2) / bh + (double)v * (bw / 2) / bw);
    const double er = (double)(float)cos(ph), ei = (double)(float)sin(ph);
    s[e] = make_double2(qr * er - qi * ei, qr * ei + qi * er);
  }
}

// crop the centred (gh, gw) window, ifftshift, scale the inverse FFT by 1/N
__global__ void k_green_crop_shift(const cufftDoubleComplex* resp, cufftDoubleComplex* out, int C, int bh, int bw,
                                   int gh, int gw) {
  const long long n = (long long)C * gh * gw;
  const double inv = 1.0 / ((double)bh * bw);
  const int oy = bh / 2 - gh / 2, ox = bw / 2 - gw / 2;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(e / ((long long)gh * gw));
    const int rem = (int)(e - (long long)c * gh * gw);
    const int r = rem / gw, col = rem % gw;
    // ifftshift: out[r] = in[(r + g/2) mod g] (numpy, any parity: shift by -(g//2))
    const int sr = (r + gh / 2) % gh, sc = (col + gw / 2) % gw;
    cufftDoubleComplex v = resp[((long long)c * bh + oy + sr) * bw + ox + sc];
    out[e] = make_double2(v.x * inv, v.y * inv);
  }
}

__global__ void k_c128_to_c64(const cufftDoubleComplex* in, cufftComplex* out, long long n) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x)
    out[e] = make_float2((float)in[e].x, (float)in[e].y);
}

unsigned grid1(long long n) {
  long long g = (n + 255) / 256;
  return (unsigned)(g > 4096 ? 4096 : (g < 1 ? 1 : g));
}

size_t align_up(size_t v) { return (v + 255) & ~size_t(255); }

// per-level activation buffers of the forward pass
struct FwdLayout {
  size_t lvl_x[8], lvl_t[8], lvl_s[8], fftz, total;
};

FwdLayout fwd_layout(const hs_net_desc_t& d, int B, bool fused_implicit) {
  FwdLayout L{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += align_up(bytes);
    return o;
  };
  for (int l = 0; l < d.levels; ++l) {
    size_t n = (size_t)B * (d.ix >> l) * (d.iy >> l) * d.channels[l] * sizeof(float);
    L.lvl_x[l] = take(n);
    L.lvl_t[l] = take(n);
    L.lvl_s[l] = take(n);
  }
  const int L1 = d.levels - 1;
  const int hc = d.ix >> L1, wc = d.iy >> L1, cc = d.channels[L1] / 2;
  // cuFFT fallback planes only where the fused implicit kernel does not apply
  L.fftz = take(fused_implicit ? 0 : (size_t)B * cc * 4 * hc * wc * sizeof(cufftComplex));
  L.total = off;
  return L;
}

}  // namespace

size_t cnn_workspace_bytes(const hs_net_t* net, int B) {
  return fwd_layout(net->d, B, net->spec_perm != nullptr).total;
}

static int green_spectrum_c128(const float2* kern, int C, int h, int w, cufftDoubleComplex* out, cudaStream_t st,
                               double eps = 1e-5) {
  const int gh = 2 * h, gw = 2 * w, bh = 3 * gh, bw = 3 * gw;
  cufftDoubleComplex* big = nullptr;
  const long long nb = (long long)C * bh * bw;
  if (cudaMalloc(&big, nb * sizeof(cufftDoubleComplex)) != cudaSuccess) return HS_ECUDA;
  cufftHandle p1, p2;
  int n1[2] = {bh, bw}, n2[2] = {gh, gw};
  int rc = HS_OK;
  if (cufftPlanMany(&p1, 2, n1, nullptr, 1, bh * bw, nullptr, 1, bh * bw, CUFFT_Z2Z, C) != CUFFT_SUCCESS) rc = HS_ECUDA;
  if (rc == HS_OK &&
      cufftPlanMany(&p2, 2, n2, nullptr, 1, gh * gw, nullptr, 1, gh * gw, CUFFT_Z2Z, C) != CUFFT_SUCCESS)
    rc = HS_ECUDA;
  if (rc == HS_OK) {
    cufftSetStream(p1, st);
    cufftSetStream(p2, st);
    k_green_embed<<<grid1(nb), 256, 0, st>>>(kern, big, C, bh, bw);
    cufftExecZ2Z(p1, big, big, CUFFT_FORWARD);
    k_green_divide<<<grid1(nb), 256, 0, st>>>(big, nb, bh, bw, eps);
    cufftExecZ2Z(p1, big, big, CUFFT_INVERSE);
    k_green_crop_shift<<<grid1((long long)C * gh * gw), 256, 0, st>>>(big, out, C, bh, bw, gh, gw);
    cufftExecZ2Z(p2, out, out, CUFFT_FORWARD);
    cudaStreamSynchronize(st);
    cufftDestroy(p1);
    cufftDestroy(p2);
  }
  cudaFree(big);
  return rc;
}

static int implicit_apply_dev(const hs_net_t* net, const float* x_nhwc, float* y_nhwc, cufftComplex* z,
                              const void* const* active, int B, cudaStream_t st, bool x_planar = false) {
  const int hc = net->hc, wc = net->wc, cc = net->cc;
  if (net->spec_perm) {
    const long long pix = (long long)hc * wc;
    prof::count(1);
    // input NHWC (channel pairs at pixel stride cc) or complex-planar (pixel stride 1)
    return implicit_fused(x_nhwc, pix * cc, x_planar ? pix : 1, x_planar ? 1 : cc, y_nhwc, pix * cc, 1, cc,
                          net->spec_perm, active, B, cc, hc, wc, st);
  }
  if (x_planar) return HS_ECONFIG;
  cufftHandle plan;
  {
    std::lock_guard<std::mutex> g(net->plan_mu);
    auto it = net->plans.find(B);
    if (it == net->plans.end()) {
      int n[2] = {2 * hc, 2 * wc};
      if (cufftPlanMany(&plan, 2, n, nullptr, 1, 4 * hc * wc, nullptr, 1, 4 * hc * wc, CUFFT_C2C, B * cc) !=
          CUFFT_SUCCESS)
        return HS_ECUDA;
      net->plans[B] = plan;
    } else {
      plan = it->second;
    }
  }
  cufftSetStream(plan, st);
  const long long per_b = (long long)cc * 4 * hc * wc;
  dim3 g(grid1(per_b), B);
  prof::count(3);  // pack, spectral multiply, crop (cuFFT kernels not counted)
  k_pack_pad<<<g, 256, 0, st>>>(x_nhwc, active, z, hc, wc, cc);
  if (cufftExecC2C(plan, z, z, CUFFT_FORWARD) != CUFFT_SUCCESS) return HS_ECUDA;
  k_spec_mul<<<g, 256, 0, st>>>(z, active, net->spec, per_b);
  if (cufftExecC2C(plan, z, z, CUFFT_INVERSE) != CUFFT_SUCCESS) return HS_ECUDA;
  k_crop_unpack<<<dim3(grid1((long long)hc * wc * cc), B), 256, 0, st>>>(z, active, y_nhwc, hc, wc, cc);
  return HS_OK;
}

// The solver U-Net (ARCH.md) on NHWC buffers; input 2-channel `in`, output
// 2-channel `head`.  RHS with active[b] == null are skipped.
// whether the coarsest residual block writes the implicit layer's input complex-planar
static bool coarse_planar(const hs_net_t* net, int h, int w) {
  const hs_conv_t& c = net->d.sol_res_b[net->d.levels - 1];
  return net->spec_perm != nullptr && !c.transposed && c.stride == 1 &&
         (conv_wide_supported(c.cin, c.cout, c.stride, c.transposed, h, w, w) ||
          conv_tc_supported(c.cin, c.cout, c.stride, c.transposed, h, w, w, 1));
}

static int solver_forward(const hs_net_t* net, const float* in, float* head, const ThinIO* io, char* ws,
                          const FwdLayout& L,
                          const int* model_of, const void* const* active, int B, cudaStream_t st) {
  const hs_net_desc_t& d = net->d;
  float* X[8];
  float* Tm[8];
  float* S[8];
  for (int l = 0; l < d.levels; ++l) {
    X[l] = reinterpret_cast<float*>(ws + L.lvl_x[l]);
    Tm[l] = reinterpret_cast<float*>(ws + L.lvl_t[l]);
    S[l] = reinterpret_cast<float*>(ws + L.lvl_s[l]);
  }
  auto lvl_bstride = [&](int l) { return (long long)(d.ix >> l) * (d.iy >> l) * d.channels[l]; };
  int rc;
  // level 0: stem (+ encoding 0), residual block -> skip 0
  ThinIO io_stem = io ? *io : ThinIO{}, io_head = io ? *io : ThinIO{};
  io_stem.host_w = net->thin_w[1].empty() ? nullptr : net->thin_w[1].data();
  io_head.host_w = net->thin_w[2].empty() ? nullptr : net->thin_w[2].data();
  if ((rc = launch_conv(d.sol_stem, in, B, d.ix, d.iy, X[0], net->enc[0], lvl_bstride(0), model_of, nullptr, active,
                        st, true, &io_stem)))
    return rc;
  if ((rc = launch_conv(d.sol_res_a[0], X[0], B, d.ix, d.iy, Tm[0], nullptr, 0, nullptr, nullptr, active, st)))
    return rc;
  if ((rc = launch_conv(d.sol_res_b[0], Tm[0], B, d.ix, d.iy, S[0], nullptr, 0, nullptr, X[0], active, st))) return rc;
  for (int l = 1; l < d.levels; ++l) {
    const int H = d.ix >> (l - 1), W = d.iy >> (l - 1), h = d.ix >> l, w = d.iy >> l;
    if ((rc = launch_conv(d.sol_down[l], S[l - 1], B, H, W, X[l], net->enc[l], lvl_bstride(l), model_of, nullptr,
                          active, st, true)))
      return rc;
    if ((rc = launch_conv(d.sol_res_a[l], X[l], B, h, w, Tm[l], nullptr, 0, nullptr, nullptr, active, st))) return rc;
    // the coarsest level's S feeds only the implicit layer: stored complex-planar
    // there (coalesced FFT-line reads) when the fused kernel and the tcgen05 conv run
    const bool planar = l == d.levels - 1 && coarse_planar(net, h, w);
    if ((rc = launch_conv(d.sol_res_b[l], Tm[l], B, h, w, S[l], nullptr, 0, nullptr, X[l], active, st, false, nullptr,
                          planar)))
      return rc;
  }
  // coarsest: implicit layer S[L-1] -> X[L-1]
  const int L1 = d.levels - 1;
  const int islot = prof::start(prof::IMPLICIT, st);
  rc = implicit_apply_dev(net, S[L1], X[L1], reinterpret_cast<cufftComplex*>(ws + L.fftz), active, B, st,
                          L1 > 0 && coarse_planar(net, d.ix >> L1, d.iy >> L1));
  // algorithmic bytes: complex64 input + output of every (RHS, complex channel) (the spectrum is L2-resident)
  prof::stop(islot, st,
             2.0 * 8.0 * (d.channels[L1] / 2) * (double)(d.ix >> L1) * (double)(d.iy >> L1) * prof::active_hint(B));
  if (rc) return rc;
  // up path: X[l] -> (tconv + skip) X[l-1] -> residual block
  for (int l = L1; l >= 1; --l) {
    const int h = d.ix >> l, w = d.iy >> l, H = d.ix >> (l - 1), W = d.iy >> (l - 1);
    (void)H;
    (void)W;
    float* src = X[l];
    if ((rc = launch_conv(d.sol_up[l], src, B, h, w, Tm[l - 1], S[l - 1], lvl_bstride(l - 1), nullptr, nullptr,
                          active, st)))
      return rc;
    // Tm[l-1] holds x = softplus(BN(tconv)) + skip; residual block into X[l-1]
    if ((rc = launch_conv(d.sol_ures_a[l - 1], Tm[l - 1], B, d.ix >> (l - 1), d.iy >> (l - 1), S[l - 1], nullptr, 0,
                          nullptr, nullptr, active, st)))
      return rc;
    if ((rc = launch_conv(d.sol_ures_b[l - 1], S[l - 1], B, d.ix >> (l - 1), d.iy >> (l - 1), X[l - 1], nullptr, 0,
                          nullptr, Tm[l - 1], active, st)))
      return rc;
  }
  return launch_conv(d.sol_head, X[0], B, d.ix, d.iy, head, nullptr, 0, nullptr, nullptr, active, st, false, &io_head);
}

int cnn_preconditioner_estimate(const hs_net_t* net, VecIn vin, const float2* const* active, float2* u0,
                                const int* model_of, int B, void* ws, cudaStream_t st) {
  const hs_net_desc_t& d = net->d;
  FwdLayout L = fwd_layout(d, B, net->spec_perm != nullptr);
  char* w = static_cast<char*>(ws);
  const void* const* act = reinterpret_cast<const void* const*>(active);
  const int slot = prof::start(prof::CNN, st);
  // the stem reads r[:ix, :iy] straight from the Krylov vector and the head writes
  // u0 = (h^2/64) net(.) zero-padded to (nx, ny) (ARCH.md), so no gather / scatter pass
  ThinIO io{vin, d.ny, u0, (long long)d.nx * d.ny, d.ny, d.nx, d.ny, d.out_scale};
  const int rc = solver_forward(net, nullptr, nullptr, &io, w, L, model_of, act, B, st);
  prof::stop(slot, st, 0.0);
  return rc;
}

}  // namespace hs

// ------------------------------------------------------------------ C ABI

namespace {
int cfail(int code, const char* m) { return hs::set_error(code, m); }
int ccheck(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return hs::set_error(HS_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return HS_OK;
}
}  // namespace

HS_API int hs_net_create(hs_net_t** out, const hs_net_desc_t* desc, void* stream) {
  if (!out || !desc) return cfail(HS_ECONFIG, "null argument");
  if (desc->levels < 2 || desc->levels > 8) return cfail(HS_ECONFIG, "levels must lie in [2, 8]");
  const int L1 = desc->levels - 1;
  if ((desc->ix >> L1) << L1 != desc->ix || (desc->iy >> L1) << L1 != desc->iy)
    return cfail(HS_EDIMENSION, "network grid not divisible by 2^(levels-1)");
  auto* n = new hs_net();
  n->d = *desc;
  n->hc = desc->ix >> L1;
  n->wc = desc->iy >> L1;
  n->cc = desc->channels[L1] / 2;
  if (n->hc < 3 || n->wc < 3) {
    delete n;
    return cfail(HS_EDIMENSION, "coarse size too small for the implicit layer");
  }
  cudaStream_t st = (cudaStream_t)stream;
  // host copies of the thin layers ([cout][9][cin] on the device -> [tap][cin][cout] + bias)
  const hs_conv_t* thin[3] = {&desc->enc_stem, &desc->sol_stem, &desc->sol_head};
  for (int k = 0; k < 3; ++k) {
    const hs_conv_t& c = *thin[k];
    if (!c.w || !c.b || c.stride != 1 || c.transposed) continue;
    const int ci = c.cin, co = c.cout, nw = 9 * ci * co;
    std::vector<float> w(nw), b(co);
    if (cudaMemcpy(w.data(), c.w, nw * sizeof(float), cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(b.data(), c.b, co * sizeof(float), cudaMemcpyDeviceToHost) != cudaSuccess) {
      delete n;
      return cfail(HS_ECUDA, "thin weights");
    }
    auto& h = n->thin_w[k];
    h.assign(nw + co, 0.f);
    for (int o = 0; o < co; ++o)
      for (int t = 0; t < 9; ++t)
        for (int i = 0; i < ci; ++i) h[(t * ci + i) * co + o] = w[(o * 9 + t) * ci + i];
    for (int o = 0; o < co; ++o) h[nw + o] = b[o];
  }
  // the >= 64-channel layers: bf16x3 weight pieces for the K-streamed tcgen05 kernel, split once here
  {
    const hs_conv_t* all[] = {&desc->enc_stem, &desc->sol_stem, &desc->sol_head};
    std::vector<const hs_conv_t*> convs(all, all + 3);
    for (int l = 0; l < desc->levels; ++l)
      for (const hs_conv_t* c : {&desc->enc_res_a[l], &desc->enc_res_b[l], &desc->enc_down[l], &desc->sol_res_a[l],
                                 &desc->sol_res_b[l], &desc->sol_down[l], &desc->sol_up[l], &desc->sol_ures_a[l],
                                 &desc->sol_ures_b[l]})
        convs.push_back(c);
    for (const hs_conv_t* c : convs) {
      if (!c->w || std::find(n->wide_w.begin(), n->wide_w.end(), c->w) != n->wide_w.end()) continue;
      if (!hs::conv_wide_eligible(c->cin, c->cout)) continue;
      if (hs::conv_wide_register(c->w, c->cin, c->cout, st)) {
        delete n;
        return cfail(HS_ECUDA, "wide-layer weight split");
      }
      n->wide_w.push_back(c->w);
    }
  }
  const long long ns = (long long)n->cc * 4 * n->hc * n->wc;
  cufftDoubleComplex* s128 = nullptr;
  if (cudaMalloc(&s128, ns * sizeof(cufftDoubleComplex)) != cudaSuccess ||
      cudaMalloc(&n->spec, ns * sizeof(cufftComplex)) != cudaSuccess) {
    delete n;
    return cfail(HS_ECUDA, "cudaMalloc spectrum");
  }
  int rc = hs::green_spectrum_c128(static_cast<const float2*>(desc->implicit_w), n->cc, n->hc, n->wc, s128, st);
  if (rc == HS_OK) {
    hs::k_c128_to_c64<<<hs::grid1(ns), 256, 0, st>>>(s128, n->spec, ns);
    if (hs::implicit_fused_supported(n->hc, n->wc)) {
      if (cudaMalloc(&n->spec_perm, ns * sizeof(cufftComplex)) != cudaSuccess) rc = HS_ECUDA;
      else hs::implicit_permute_spectrum(n->spec, n->spec_perm, n->cc, n->hc, n->wc, st);
    }
    cudaStreamSynchronize(st);
  }
  cudaFree(s128);
  if (rc != HS_OK || ccheck("hs_net_create") != HS_OK) {
    delete n;
    return cfail(HS_ECUDA, "green spectrum");
  }
  *out = n;
  return HS_OK;
}

HS_API void hs_net_destroy(hs_net_t* net) { delete net; }

static size_t enc_level_bytes(const hs_net_desc_t& d, int n_models) {
  size_t m = 0;
  for (int l = 0; l < d.levels; ++l) {
    size_t b = (size_t)n_models * (d.ix >> l) * (d.iy >> l) * d.channels[l] * sizeof(float);
    m = b > m ? b : m;
  }
  return hs::align_up(m);
}

HS_API size_t hs_net_encode_workspace_bytes(const hs_net_t* net, int n_models) {
  return 2 * enc_level_bytes(net->d, n_models);
}

HS_API int hs_net_encode(hs_net_t* net, const float* media, int n_models, float* const* enc, void* ws,
                         size_t ws_bytes, void* stream) {
  const hs_net_desc_t& d = net->d;
  if (ws_bytes < hs_net_encode_workspace_bytes(net, n_models)) return cfail(HS_ECONFIG, "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  char* w = static_cast<char*>(ws);
  const size_t big = enc_level_bytes(d, n_models);
  float* t0 = reinterpret_cast<float*>(w);
  float* t1 = reinterpret_cast<float*>(w + big);
  int rc;
  // e0 = res0(cbs(stem(media))), e_l = res_l(cbs(down_l(e_{l-1})))
  hs::ThinIO io_enc{};
  io_enc.host_w = net->thin_w[0].empty() ? nullptr : net->thin_w[0].data();
  if ((rc = hs::launch_conv(d.enc_stem, media, n_models, d.ix, d.iy, t0, nullptr, 0, nullptr, nullptr, nullptr, st,
                            false, &io_enc)))
    return cfail(rc, "encoder stem");
  for (int l = 0; l < d.levels; ++l) {
    const int h = d.ix >> l, ww = d.iy >> l;
    if (l > 0) {
      if ((rc = hs::launch_conv(d.enc_down[l], enc[l - 1], n_models, d.ix >> (l - 1), d.iy >> (l - 1), t0, nullptr, 0,
                                nullptr, nullptr, nullptr, st)))
        return cfail(rc, "encoder down");
    }
    if ((rc = hs::launch_conv(d.enc_res_a[l], t0, n_models, h, ww, t1, nullptr, 0, nullptr, nullptr, nullptr, st)))
      return cfail(rc, "encoder res a");
    if ((rc = hs::launch_conv(d.enc_res_b[l], t1, n_models, h, ww, enc[l], nullptr, 0, nullptr, t0, nullptr, st)))
      return cfail(rc, "encoder res b");
    net->enc[l] = enc[l];
  }
  net->n_models = n_models;
  return ccheck("hs_net_encode");
}

HS_API size_t hs_net_workspace_bytes(const hs_net_t* net, int B) { return hs::cnn_workspace_bytes(net, B); }

HS_API int hs_net_forward(const hs_net_t* net, const void* r, void* u0, const int* model_of, int B, void* ws,
                          size_t ws_bytes, void* stream) {
  if (!net->enc[0]) return cfail(HS_ECONFIG, "encodings not computed (hs_net_encode)");
  if (ws_bytes < hs::cnn_workspace_bytes(net, B)) return cfail(HS_ECONFIG, "workspace too small");
  const hs_net_desc_t& d = net->d;
  hs::VecIn vin{nullptr, static_cast<const float2*>(r), (long long)d.nx * d.ny, nullptr};
  const int rc = hs::cnn_preconditioner_estimate(net, vin, nullptr, static_cast<float2*>(u0), model_of, B, ws,
                                                 (cudaStream_t)stream);
  if (rc) return cfail(rc, "network forward");
  return ccheck("hs_net_forward");
}

HS_API int hs_green_spectrum(const void* kernel, int C, int h, int w, void* spectrum, void* stream) {
  return hs_green_spectrum_eps(kernel, C, h, w, 1e-5, spectrum, stream);
}

HS_API int hs_green_spectrum_eps(const void* kernel, int C, int h, int w, double eps, void* spectrum, void* stream) {
  if (h < 3 || w < 3) return cfail(HS_EDIMENSION, "coarse size too small");
  if (!(eps >= 0.0)) return cfail(HS_ECONFIG, "eps must be >= 0");
  int rc = hs::green_spectrum_c128(static_cast<const float2*>(kernel), C, h, w,
                                   static_cast<cufftDoubleComplex*>(spectrum), (cudaStream_t)stream, eps);
  return rc == HS_OK ? ccheck("hs_green_spectrum") : cfail(rc, "cufft");
}

HS_API int hs_implicit_apply(const void* x, const void* spectrum, void* y, int B, int C, int h, int w, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const long long per_b = (long long)C * 4 * h * w;
  if (hs::implicit_fused_supported(h, w)) {
    void* sp = nullptr;
    if (cudaMalloc(&sp, (size_t)per_b * sizeof(cufftComplex)) != cudaSuccess) return cfail(HS_ECUDA, "cudaMalloc");
    hs::implicit_permute_spectrum(spectrum, sp, C, h, w, st);
    const long long hw = (long long)h * w;
    const int rc = hs::implicit_fused(x, C * hw, hw, 1, y, C * hw, hw, 1, sp, nullptr, B, C, h, w, st);
    cudaStreamSynchronize(st);
    cudaFree(sp);
    if (rc) return cfail(rc, "implicit layer");
    return ccheck("hs_implicit_apply");
  }
  cufftHandle plan;
  int n[2] = {2 * h, 2 * w};
  if (cufftPlanMany(&plan, 2, n, nullptr, 1, 4 * h * w, nullptr, 1, 4 * h * w, CUFFT_C2C, B * C) != CUFFT_SUCCESS)
    return cfail(HS_ECUDA, "cufft plan");
  cufftSetStream(plan, st);
  cufftComplex* z = nullptr;
  if (cudaMalloc(&z, (size_t)B * per_b * sizeof(cufftComplex)) != cudaSuccess) {
    cufftDestroy(plan);
    return cfail(HS_ECUDA, "cudaMalloc");
  }
  dim3 g(hs::grid1(per_b), B);
  hs::k_pad_nchw<<<g, 256, 0, st>>>(static_cast<const cufftComplex*>(x), z, C, h, w);
  cufftExecC2C(plan, z, z, CUFFT_FORWARD);
  hs::k_spec_mul<<<g, 256, 0, st>>>(z, nullptr, static_cast<const cufftComplex*>(spectrum), per_b);
  cufftExecC2C(plan, z, z, CUFFT_INVERSE);
  hs::k_crop_nchw<<<g, 256, 0, st>>>(z, static_cast<cufftComplex*>(y), C, h, w);
  cudaStreamSynchronize(st);
  cudaFree(z);
  cufftDestroy(plan);
  return ccheck("hs_implicit_apply");
}

HS_API int hs_conv2d(const float* x, const hs_conv_t* conv, const float* addend, const float* residual, float* y,
                     int B, int H, int W, void* stream) {
  const int Ho = conv->transposed ? 2 * H : (H - 1) / conv->stride + 1;
  const int Wo = conv->transposed ? 2 * W : (W - 1) / conv->stride + 1;
  int rc = hs::launch_conv(*conv, x, B, H, W, y, addend, (long long)Ho * Wo * conv->cout, nullptr, residual, nullptr,
                           (cudaStream_t)stream);
  if (rc) return cfail(rc, "unsupported channel count");
  return ccheck("hs_conv2d");
}

HS_API int hs_net_set_encodings(hs_net_t* net, int levels, const float* const* enc) {
  if (levels != net->d.levels) return cfail(HS_EDIMENSION, "encodings for every level are needed");
  for (int l = 0; l < levels; ++l) net->enc[l] = enc[l];
  return HS_OK;
}
