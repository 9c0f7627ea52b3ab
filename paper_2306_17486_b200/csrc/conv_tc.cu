// tcgen05 implicit-GEMM 3x3 convolution with 3xTF32 (fp32-class) accuracy.
//
// GEMM view of one output tile: D[m][n] = sum_k A[m][k] B[n][k] with m = 128
// consecutive output pixels of one row, n = cout, k = (tap, cin).  Input rows
// are staged in shared memory in the UMMA K-major "interleaved" canonical
// layout (core matrix = 8 pixels x 16 bytes, pixels consecutive at a 16-byte
// pitch, 4-channel chunks LBO apart).  Because pixels sit at a 16-byte pitch,
// the A operand of tap (ky, kx) is just the staged row with the descriptor
// start address moved by kx * 16 bytes: no im2col copies.  Stride-2
// convolutions stage each input row de-interleaved (even columns, then odd
// columns) so every tap is again a unit-pitch window; the transposed
// convolution is split into its two column-parity classes (1 and 2 taps)
// with two TMEM accumulators.
//
// Streaming: a CTA owns a band of output rows of one 128-pixel column block
// and walks it top to bottom.  Input rows live in a ring of shared-memory
// slots, so each input row is loaded and split once per band (one new row per
// output row at stride 1).  The MMAs of row t run while the CTA prefetches the
// rows of t+1 and drains row t-1's accumulator (two TMEM accumulators).
//
// Precision: every fp32 operand x is split into tf32 hi = rna(x) and
// lo = rna(x - hi); the MMA accumulates hi*hi + hi*lo + lo*hi in fp32 TMEM
// (relative error ~1e-6, fp32 class; SURVEY.md §0.5 rules out 1xTF32/BF16).
#include <cstdio>

#include "common.cuh"
#include "conv_tc.h"

namespace hs {
namespace {

constexpr int kNT = 256;  // threads per CTA (8 warps)
constexpr int kM = 128;   // pixels per tile (UMMA M)
constexpr int kBand = 32; // output rows per work unit

HS_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// UMMA shared-memory descriptor, K-major, SWIZZLE_NONE (version 1 = sm_100)
HS_DEV uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}

// instruction descriptor: D f32, A/B tf32, both K-major, M x N
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

HS_DEV void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

HS_DEV void mma_commit(uint32_t mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mbar)
               : "memory");
}

HS_DEV void mbar_init(uint32_t mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mbar), "r"(count));
}

HS_DEV void mbar_wait(uint32_t mbar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tLAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE;\n\tbra LAB_WAIT;\n\tDONE:\n\t}\n" ::"r"(mbar),
      "r"(phase));
}

HS_DEV void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
HS_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
HS_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

HS_DEV uint32_t tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

// split x into tf32 hi + tf32 lo
HS_DEV void split3(float4 v, uint4& hi, uint4& lo) {
  hi.x = tf32_rna(v.x);
  hi.y = tf32_rna(v.y);
  hi.z = tf32_rna(v.z);
  hi.w = tf32_rna(v.w);
  lo.x = tf32_rna(v.x - __uint_as_float(hi.x));
  lo.y = tf32_rna(v.y - __uint_as_float(hi.y));
  lo.z = tf32_rna(v.z - __uint_as_float(hi.z));
  lo.w = tf32_rna(v.w - __uint_as_float(hi.w));
}

HS_DEV void tmem_ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

HS_DEV float softplus_f(float x) { return fmaxf(x, 0.f) + log1pf(expf(-fabsf(x))); }

struct TcArgs {
  const float* x;
  int H, W;
  float* y;
  int Ho, Wo;
  const float* w;  // [cout][9][cin]
  const float* bias;
  int softplus;
  const float* addend;
  long long addend_bstride;
  int addend_per_model;
  const int* model_of;
  const float* residual;
  const void* const* active;
  int B;
};

// MODE 0: stride 1; MODE 1: stride 2; MODE 2: transposed stride 2 (out = 2 x in)
template <int MODE>
struct Geo {
  static constexpr int RW = MODE == 0 ? kM + 2 : (MODE == 1 ? 2 * kM + 1 : kM + 1);  // pixels per staged row
  static constexpr int NS = MODE == 0 ? 4 : (MODE == 1 ? 5 : 3);                     // ring slots
  static constexpr int NACC = MODE == 2 ? 2 : 1;  // accumulators per tile (column-parity classes)
};

template <int CIN, int COUT, int MODE>
struct Cfg {
  static constexpr int KCH = CIN / 4;                                    // 16-byte channel chunks
  static constexpr int XPL = Geo<MODE>::NS * Geo<MODE>::RW;              // pixels per chunk plane
  static constexpr size_t W_BYTES = (size_t)9 * KCH * COUT * 16;
  static constexpr size_t X_BYTES = (size_t)KCH * XPL * 16;
  static constexpr size_t TOTAL = 2 * W_BYTES + 2 * X_BYTES + 64;
  static constexpr int EPT = (Geo<MODE>::RW * KCH + kNT - 1) / kNT;     // row elements per thread
  static constexpr int ACOLS = COUT * Geo<MODE>::NACC;                   // TMEM columns per accumulator
  static constexpr int NCOLS_RAW = 2 * ACOLS;
  static constexpr int NCOLS = NCOLS_RAW <= 32 ? 32 : (NCOLS_RAW <= 64 ? 64 : (NCOLS_RAW <= 128 ? 128 : 256));
};

// input column of staged pixel p in a row of column block xb
template <int MODE>
HS_DEV int stage_col(int xb, int p) {
  if (MODE == 0) return xb * kM - 1 + p;
  if (MODE == 1) return p < kM ? 2 * (xb * kM + p) : 2 * (xb * kM + (p - kM)) - 1;
  return xb * kM + p;
}

template <int CIN, int COUT, int MODE>
struct RowPrefetch {
  float4 v[Cfg<CIN, COUT, MODE>::EPT];
  int gy;
};

template <int CIN, int COUT, int MODE>
HS_DEV void row_load(RowPrefetch<CIN, COUT, MODE>& pf, const float* xb_ptr, int H, int W, int xb, int gy) {
  using C = Cfg<CIN, COUT, MODE>;
  constexpr int RW = Geo<MODE>::RW;
  pf.gy = gy;
#pragma unroll
  for (int i = 0; i < C::EPT; ++i) {
    const int e = threadIdx.x + i * kNT;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (e < RW * C::KCH) {
      const int c = e / RW, p = e - c * RW;
      const int gx = stage_col<MODE>(xb, p);
      if (gy >= 0 && gy < H && gx >= 0 && gx < W)
        v = __ldg(reinterpret_cast<const float4*>(xb_ptr + ((size_t)gy * W + gx) * CIN + 4 * c));
    }
    pf.v[i] = v;
  }
}

template <int CIN, int COUT, int MODE>
HS_DEV void row_store(const RowPrefetch<CIN, COUT, MODE>& pf, unsigned char* x_hi, unsigned char* x_lo) {
  using C = Cfg<CIN, COUT, MODE>;
  constexpr int RW = Geo<MODE>::RW, NS = Geo<MODE>::NS;
  const int slot = ((pf.gy % NS) + NS) % NS;
#pragma unroll
  for (int i = 0; i < C::EPT; ++i) {
    const int e = threadIdx.x + i * kNT;
    if (e < RW * C::KCH) {
      const int c = e / RW, p = e - c * RW;
      uint4 hi, lo;
      split3(pf.v[i], hi, lo);
      const size_t off = ((size_t)c * C::XPL + slot * RW + p) * 16;
      *reinterpret_cast<uint4*>(x_hi + off) = hi;
      *reinterpret_cast<uint4*>(x_lo + off) = lo;
    }
  }
}

// input rows a tile needs: [lo, hi]
template <int MODE>
HS_DEV void tile_rows(int oy, int& lo, int& hi) {
  if (MODE == 0) {
    lo = oy - 1;
    hi = oy + 1;
  } else if (MODE == 1) {
    lo = 2 * oy - 1;
    hi = 2 * oy + 1;
  } else {
    lo = oy >> 1;
    hi = (oy >> 1) + 1;
  }
}

template <int CIN, int COUT, int MODE>
HS_DEV void issue_mmas(int oy, uint32_t d0, uint32_t xh, uint32_t xl, uint32_t wh, uint32_t wl) {
  using C = Cfg<CIN, COUT, MODE>;
  constexpr int RW = Geo<MODE>::RW, NS = Geo<MODE>::NS;
  constexpr uint32_t X_LBO = C::XPL * 16, W_LBO = COUT * 16;
  constexpr uint32_t IDESC = idesc_tf32(kM, COUT);
  auto slot_of = [](int gy) { return ((gy % NS) + NS) % NS; };
  for (int acc = 0; acc < Geo<MODE>::NACC; ++acc) {
    const uint32_t d = d0 + acc * COUT;
    uint32_t first = 1;
    for (int ky = 0; ky < 3; ++ky) {
      for (int kx = 0; kx < 3; ++kx) {
        int gy, px;  // staged input row and pixel offset feeding this tap
        if (MODE == 0) {
          gy = oy - 1 + ky;
          px = kx;
        } else if (MODE == 1) {
          gy = 2 * oy - 1 + ky;
          px = kx == 1 ? 0 : (kx == 0 ? kM : kM + 1);
        } else {
          // out row 2q: ky = 1 at row q; out row 2q+1: ky = 0 at q+1, ky = 2 at q
          // out col 2q (acc 0): kx = 1 at q; out col 2q+1 (acc 1): kx = 0 at q+1, kx = 2 at q
          const int py = oy & 1, q = oy >> 1;
          if (py == 0 && ky != 1) continue;
          if (py == 1 && ky == 1) continue;
          if (acc == 0 && kx != 1) continue;
          if (acc == 1 && kx == 1) continue;
          gy = (py && ky == 0) ? q + 1 : q;
          px = (acc && kx == 0) ? 1 : 0;
        }
        const uint32_t xo = (uint32_t)(slot_of(gy) * RW + px) * 16;
        const uint32_t wo = (uint32_t)((ky * 3 + kx) * C::KCH * COUT * 16);
#pragma unroll
        for (int kk = 0; kk < C::KCH / 2; ++kk) {
          const uint32_t xk = xo + kk * 2 * X_LBO, wk = wo + kk * 2 * W_LBO;
          const uint64_t ah = umma_desc(xh + xk, X_LBO, 128), al = umma_desc(xl + xk, X_LBO, 128);
          const uint64_t bh = umma_desc(wh + wk, W_LBO, 128), bl = umma_desc(wl + wk, W_LBO, 128);
          mma_tf32(d, ah, bh, IDESC, first ? 0u : 1u);
          first = 0;
          mma_tf32(d, ah, bl, IDESC, 1u);
          mma_tf32(d, al, bh, IDESC, 1u);
        }
      }
    }
  }
}

// warp w drains TMEM lane quarter (w % 4) (= tile pixels 32(w%4) + lane), column half (w / 4)
template <int CIN, int COUT, int MODE>
HS_DEV void epilogue(const TcArgs& a, uint32_t d0, int b, int oy, int xb) {
  constexpr int HALF = COUT / 2;  // 8, 16, 32 or 64 columns per warp
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int quarter = warp & 3, half = warp >> 2;
  const int m = quarter * 32 + lane;
  const float* add =
      a.addend ? a.addend + (a.addend_per_model ? (a.model_of ? a.model_of[b] : 0) : b) * a.addend_bstride : nullptr;
  for (int acc = 0; acc < Geo<MODE>::NACC; ++acc) {
    const int ox = MODE == 2 ? 2 * (xb * kM + m) + acc : xb * kM + m;
    const size_t pix = (size_t)oy * a.Wo + ox;
    const size_t obase = (size_t)b * a.Ho * a.Wo * COUT + pix * COUT;
#pragma unroll
    for (int n0 = half * HALF; n0 < (half + 1) * HALF; n0 += 8) {
      float4 ad[2], rs[2];
      if (add) {
        ad[0] = __ldg(reinterpret_cast<const float4*>(add + pix * COUT + n0));
        ad[1] = __ldg(reinterpret_cast<const float4*>(add + pix * COUT + n0 + 4));
      }
      if (a.residual) {
        rs[0] = __ldg(reinterpret_cast<const float4*>(a.residual + obase + n0));
        rs[1] = __ldg(reinterpret_cast<const float4*>(a.residual + obase + n0 + 4));
      }
      float v[8];
      tmem_ld8(d0 + ((uint32_t)(quarter * 32) << 16) + acc * COUT + n0, v);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        float t = v[u] + __ldg(a.bias + n0 + u);
        if (a.softplus) t = softplus_f(t);
        if (add) t += (&ad[u >> 2].x)[u & 3];
        if (a.residual) t += (&rs[u >> 2].x)[u & 3];
        v[u] = t;
      }
      *reinterpret_cast<float4*>(a.y + obase + n0) = make_float4(v[0], v[1], v[2], v[3]);
      *reinterpret_cast<float4*>(a.y + obase + n0 + 4) = make_float4(v[4], v[5], v[6], v[7]);
    }
  }
}

template <int CIN, int COUT, int MODE>
__global__ void __launch_bounds__(kNT) k_conv_tc(TcArgs a) {
  using C = Cfg<CIN, COUT, MODE>;
  constexpr int KCH = C::KCH;
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* w_hi = smem;
  unsigned char* w_lo = smem + C::W_BYTES;
  unsigned char* x_hi = smem + 2 * C::W_BYTES;
  unsigned char* x_lo = x_hi + C::X_BYTES;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(x_lo + C::X_BYTES);  // [2]
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(mbar + 2);
  const int tid = threadIdx.x, warp = tid >> 5;

  // ---- weights: [cout][tap][cin] fp32 -> hi/lo tf32, layout (tap, chunk, n) x 16 B
  for (int e = tid; e < 9 * KCH * COUT; e += kNT) {
    const int n = e % COUT, c = (e / COUT) % KCH, t = e / (COUT * KCH);
    const float4 v = __ldg(reinterpret_cast<const float4*>(a.w + ((size_t)n * 9 + t) * CIN + 4 * c));
    uint4 hi, lo;
    split3(v, hi, lo);
    const size_t off = ((size_t)(t * KCH + c) * COUT + n) * 16;
    *reinterpret_cast<uint4*>(w_hi + off) = hi;
    *reinterpret_cast<uint4*>(w_lo + off) = lo;
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s_tmem)),
                 "r"(C::NCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(smem_u32(&mbar[0]), 1);
    mbar_init(smem_u32(&mbar[1]), 1);
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;
  const uint32_t xh = smem_u32(x_hi), xl = smem_u32(x_lo), wh = smem_u32(w_hi), wl = smem_u32(w_lo);
  uint32_t phase[2] = {0u, 0u};

  const int xblocks = MODE == 2 ? a.W / kM : a.Wo / kM;
  const int nbands = (a.Ho + kBand - 1) / kBand;
  const long long nunits = (long long)a.B * xblocks * nbands;
  for (long long unit = blockIdx.x; unit < nunits; unit += gridDim.x) {
    const int xb = (int)(unit % xblocks);
    const int band = (int)((unit / xblocks) % nbands);
    const int b = (int)(unit / ((long long)xblocks * nbands));
    if (a.active && a.active[b] == nullptr) continue;  // uniform per CTA
    const float* xb_ptr = a.x + (size_t)b * a.H * a.W * CIN;
    const int oy0 = band * kBand, oy1 = min(a.Ho, oy0 + kBand);
    // prologue: stage every input row of the first tile
    int lo, hi;
    tile_rows<MODE>(oy0, lo, hi);
    for (int gy = lo; gy <= hi; ++gy) {
      RowPrefetch<CIN, COUT, MODE> pf;
      row_load<CIN, COUT, MODE>(pf, xb_ptr, a.H, a.W, xb, gy);
      row_store<CIN, COUT, MODE>(pf, x_hi, x_lo);
    }
    int staged_hi = hi;
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    for (int oy = oy0; oy < oy1; ++oy) {
      const int t = oy - oy0, s = t & 1;
      // (A) MMAs of row oy into accumulator s
      if (tid == 0) {
        tc_fence_after();
        issue_mmas<CIN, COUT, MODE>(oy, tmem + s * C::ACOLS, xh, xl, wh, wl);
        mma_commit(smem_u32(&mbar[s]));
      }
      // (B) prefetch the new input rows of row oy+1 (at most two)
      RowPrefetch<CIN, COUT, MODE> pf0, pf1;
      int nnew = 0;
      if (oy + 1 < oy1) {
        tile_rows<MODE>(oy + 1, lo, hi);
        if (hi > staged_hi) {
          row_load<CIN, COUT, MODE>(pf0, xb_ptr, a.H, a.W, xb, staged_hi + 1);
          nnew = 1;
          if (hi > staged_hi + 1) {
            row_load<CIN, COUT, MODE>(pf1, xb_ptr, a.H, a.W, xb, staged_hi + 2);
            nnew = 2;
          }
        }
      }
      // (C) drain row oy-1 (its MMAs overlapped with (A)/(B))
      if (t > 0) {
        mbar_wait(smem_u32(&mbar[s ^ 1]), phase[s ^ 1]);
        phase[s ^ 1] ^= 1u;
        tc_fence_after();
        epilogue<CIN, COUT, MODE>(a, tmem + (s ^ 1) * C::ACOLS, b, oy - 1, xb);
      }
      // (D) rows for oy+1 overwrite slots only rows <= oy-1's inputs used (their MMAs are complete)
      if (nnew >= 1) row_store<CIN, COUT, MODE>(pf0, x_hi, x_lo);
      if (nnew >= 2) row_store<CIN, COUT, MODE>(pf1, x_hi, x_lo);
      staged_hi += nnew;
      fence_async_smem();
      tc_fence_before();
      __syncthreads();
    }
    // drain the last row
    const int tl = oy1 - 1 - oy0, sl = tl & 1;
    mbar_wait(smem_u32(&mbar[sl]), phase[sl]);
    phase[sl] ^= 1u;
    tc_fence_after();
    epilogue<CIN, COUT, MODE>(a, tmem + sl * C::ACOLS, b, oy1 - 1, xb);
    tc_fence_before();
    __syncthreads();
  }
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::NCOLS));
  }
}

template <int CIN, int COUT, int MODE>
void launch_tc(const TcArgs& a, cudaStream_t st) {
  using C = Cfg<CIN, COUT, MODE>;
  static int grid_cap = 0;
  if (!grid_cap) {
    cudaFuncSetAttribute(k_conv_tc<CIN, COUT, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::TOTAL);
    int per_sm = 0, sms = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_conv_tc<CIN, COUT, MODE>, kNT, C::TOTAL);
    grid_cap = sms * (per_sm > 0 ? per_sm : 1);
  }
  const long long xblocks = MODE == 2 ? a.W / kM : a.Wo / kM;
  const long long nunits = (long long)a.B * xblocks * ((a.Ho + kBand - 1) / kBand);
  const int grid = (int)(nunits < grid_cap ? nunits : grid_cap);
  k_conv_tc<CIN, COUT, MODE><<<grid, kNT, C::TOTAL, st>>>(a);
}

}  // namespace

bool conv_tc_enabled = true;

bool conv_tc_supported(int cin, int cout, int stride, int transposed, int H, int W, int Wo) {
  (void)H;
  if (!conv_tc_enabled) return false;
  const int mode = transposed ? 2 : (stride == 2 ? 1 : 0);
  const int width = mode == 2 ? W : Wo;
  if (width % kM) return false;
  if (mode == 0) return (cin == 16 && cout == 16) || (cin == 32 && cout == 32);
  if (mode == 1) return cin == 16 && cout == 32;
  return cin == 32 && cout == 16;
}

void conv_tc_launch(const float* x, int H, int W, int cin, float* y, int Ho, int Wo, int cout, int stride,
                    int transposed, const float* w, const float* bias, int softplus, const float* addend,
                    long long addend_bstride, int addend_per_model, const int* model_of, const float* residual,
                    const void* const* active, int B, cudaStream_t st) {
  TcArgs a{x, H, W, y, Ho, Wo, w, bias, softplus, addend, addend_bstride, addend_per_model, model_of, residual,
           active, B};
  const int mode = transposed ? 2 : (stride == 2 ? 1 : 0);
  if (mode == 0 && cin == 16 && cout == 16) launch_tc<16, 16, 0>(a, st);
  else if (mode == 0 && cin == 32 && cout == 32) launch_tc<32, 32, 0>(a, st);
  else if (mode == 1 && cin == 16 && cout == 32) launch_tc<16, 32, 1>(a, st);
  else if (mode == 2 && cin == 32 && cout == 16) launch_tc<32, 16, 2>(a, st);
}

}  // namespace hs
