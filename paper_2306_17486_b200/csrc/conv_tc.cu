// tcgen05 implicit-GEMM 3x3 convolution with 3xTF32 (fp32-class) accuracy.
//
// GEMM view of one output tile: D[m][n] = sum_k A[m][k] B[n][k] with m = 128
// consecutive output pixels of one row, n = cout, k = (tap, cin).  The input
// rows the tile needs are staged ONCE in shared memory in the UMMA K-major
// "interleaved" canonical layout (core matrix = 8 pixels x 16 bytes, pixels
// consecutive at 16-byte pitch, channel chunks LBO apart).  Because pixels
// sit at a 16-byte pitch, the A operand of tap (ky, kx) is the same buffer
// with the descriptor start address moved by (ky * row_pixels + kx) * 16
// bytes: no im2col copies.  Stride-2 convolutions store each input row
// de-interleaved (even columns, then odd columns) so every tap is again a
// unit-pitch window; the transposed convolution is split into its two
// column-parity classes (1 and 2 taps) with two TMEM accumulators.
//
// Precision: every fp32 operand x is split into tf32 hi = rna(x) and
// lo = rna(x - hi); the MMA accumulates hi*hi + hi*lo + lo*hi in fp32 TMEM
// (relative error ~1e-6, fp32 class; SURVEY.md §0.5 rules out 1xTF32/BF16).
//
// Roles: all 128 threads fill shared memory; thread 0 issues the MMAs and
// commits them to an mbarrier; the 4 warps then read their 32 TMEM lanes
// (tcgen05.ld) and run the fused epilogue (bias, softplus, encoder/skip
// addend, residual).  CTAs are persistent over tiles; weights stay resident.
#include <cstdio>

#include "common.cuh"
#include "conv_tc.h"

namespace hs {
namespace {

constexpr int kTcThreads = 128;
constexpr int kM = 128;  // pixels per tile (UMMA M)

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

HS_DEV void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
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
  static constexpr int NR = MODE == 2 ? 2 : 3;                 // staged input rows
  static constexpr int RW = MODE == 0 ? kM + 2 : (MODE == 1 ? 2 * kM + 1 : kM + 1);  // pixels per row
  static constexpr int XPL = NR * RW;                          // pixels per channel-chunk plane
  static constexpr int NACC = MODE == 2 ? 2 : 1;               // accumulators (column-parity classes)
};

template <int CIN, int COUT, int MODE>
struct Smem {
  static constexpr int KCH = CIN / 4;
  static constexpr size_t W_BYTES = (size_t)9 * KCH * COUT * 16;
  static constexpr size_t X_BYTES = (size_t)KCH * Geo<MODE>::XPL * 16;
  static constexpr size_t TOTAL = 2 * W_BYTES + 2 * X_BYTES + 64;
};

template <int CIN, int COUT, int MODE>
__global__ void __launch_bounds__(kTcThreads) k_conv_tc(TcArgs a) {
  using G = Geo<MODE>;
  using S = Smem<CIN, COUT, MODE>;
  constexpr int KCH = S::KCH;
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* w_hi = smem;
  unsigned char* w_lo = smem + S::W_BYTES;
  unsigned char* x_hi = smem + 2 * S::W_BYTES;
  unsigned char* x_lo = x_hi + S::X_BYTES;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(x_lo + S::X_BYTES);
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(mbar + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // ---- weights: [cout][tap][cin] fp32 -> hi/lo tf32, layout (tap, chunk, n) x 16 B
  for (int e = tid; e < 9 * KCH * COUT; e += kTcThreads) {
    const int n = e % COUT, c = (e / COUT) % KCH, t = e / (COUT * KCH);
    const float4 v = *reinterpret_cast<const float4*>(a.w + ((size_t)n * 9 + t) * CIN + 4 * c);
    uint4 hi, lo;
    split3(v, hi, lo);
    const size_t off = ((size_t)(t * KCH + c) * COUT + n) * 16;
    *reinterpret_cast<uint4*>(w_hi + off) = hi;
    *reinterpret_cast<uint4*>(w_lo + off) = lo;
  }
  constexpr int NCOLS_RAW = COUT * G::NACC;
  constexpr int NCOLS = NCOLS_RAW <= 32 ? 32 : (NCOLS_RAW <= 64 ? 64 : (NCOLS_RAW <= 128 ? 128 : 256));
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s_tmem)),
                 "r"(NCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) mbar_init(smem_u32(mbar), 1);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;
  constexpr uint32_t IDESC = idesc_tf32(kM, COUT);
  uint32_t phase = 0;

  // tiles: MODE 0/1 -> (b, oy, x-block of kM outputs); MODE 2 -> (b, oy, q-block of kM inputs)
  const int xblocks = MODE == 2 ? a.W / kM : a.Wo / kM;
  const long long ntiles = (long long)a.B * a.Ho * xblocks;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int xb = (int)(tile % xblocks);
    const int oy = (int)((tile / xblocks) % a.Ho);
    const int b = (int)(tile / ((long long)xblocks * a.Ho));
    if (a.active && a.active[b] == nullptr) continue;  // uniform per CTA
    const float* xb_ptr = a.x + (size_t)b * a.H * a.W * CIN;
    // ---- stage input rows (hi/lo) in the interleaved layout
    for (int e = tid; e < KCH * G::XPL; e += kTcThreads) {
      const int P = e % G::XPL, c = e / G::XPL;
      const int r = P / G::RW, p = P % G::RW;
      int gy, gx;
      if (MODE == 0) {
        gy = oy - 1 + r;
        gx = xb * kM - 1 + p;
      } else if (MODE == 1) {
        gy = 2 * oy - 1 + r;
        gx = p < kM ? 2 * (xb * kM + p) : 2 * (xb * kM + (p - kM)) - 1;
      } else {
        gy = (oy >> 1) + r;
        gx = xb * kM + p;
      }
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (gy >= 0 && gy < a.H && gx >= 0 && gx < a.W)
        v = *reinterpret_cast<const float4*>(xb_ptr + ((size_t)gy * a.W + gx) * CIN + 4 * c);
      uint4 hi, lo;
      split3(v, hi, lo);
      const size_t off = ((size_t)c * G::XPL + P) * 16;
      *reinterpret_cast<uint4*>(x_hi + off) = hi;
      *reinterpret_cast<uint4*>(x_lo + off) = lo;
    }
    fence_async_smem();
    __syncthreads();
    // ---- MMAs (one thread)
    if (tid == 0) {
      tc_fence_after();
      const uint32_t xh = smem_u32(x_hi), xl = smem_u32(x_lo), wh = smem_u32(w_hi), wl = smem_u32(w_lo);
      constexpr uint32_t X_LBO = G::XPL * 16, W_LBO = COUT * 16;
      for (int acc = 0; acc < G::NACC; ++acc) {
        uint32_t first = 1;
        const int py = oy & 1;
        // tap list of this accumulator: (ky, kx, input pixel offset in the staged rows)
        int nt = 0, tky[9], tkx[9], toff[9];
        if (MODE == 0) {
          for (int ky = 0; ky < 3; ++ky)
            for (int kx = 0; kx < 3; ++kx) {
              tky[nt] = ky;
              tkx[nt] = kx;
              toff[nt++] = ky * G::RW + kx;
            }
        } else if (MODE == 1) {
          for (int ky = 0; ky < 3; ++ky)
            for (int kx = 0; kx < 3; ++kx) {
              tky[nt] = ky;
              tkx[nt] = kx;
              toff[nt++] = ky * G::RW + (kx == 1 ? 0 : (kx == 0 ? kM : kM + 1));
            }
        } else {
          // rows: py = 0 -> ky = 1 at row qy (r = 0); py = 1 -> ky = 0 at qy+1 (r = 1), ky = 2 at qy (r = 0)
          // cols: px = 0 -> kx = 1 at q; px = 1 -> kx = 0 at q+1, kx = 2 at q
          const int nky = py ? 2 : 1, nkx = acc ? 2 : 1;
          for (int i = 0; i < nky; ++i)
            for (int j = 0; j < nkx; ++j) {
              const int ky = py ? (i ? 2 : 0) : 1, r = (py && !i) ? 1 : 0;
              const int kx = acc ? (j ? 2 : 0) : 1, dx = (acc && !j) ? 1 : 0;
              tky[nt] = ky;
              tkx[nt] = kx;
              toff[nt++] = r * G::RW + dx;
            }
        }
        const uint32_t d = tmem + acc * COUT;
        for (int t = 0; t < nt; ++t) {
          const int tap = tky[t] * 3 + tkx[t];
          const uint32_t xo = toff[t] * 16, wo = tap * KCH * COUT * 16;
#pragma unroll
          for (int kk = 0; kk < KCH / 2; ++kk) {
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
      mma_commit(smem_u32(mbar));
    }
    mbar_wait(smem_u32(mbar), phase);
    phase ^= 1u;
    tc_fence_after();
    // ---- epilogue: warp w owns TMEM lanes / tile pixels [32w, 32w + 32)
    const int m = warp * 32 + lane;
    const float* add = a.addend
                           ? a.addend + (a.addend_per_model ? (a.model_of ? a.model_of[b] : 0) : b) * a.addend_bstride
                           : nullptr;
    for (int acc = 0; acc < G::NACC; ++acc) {
      const int ox = MODE == 2 ? 2 * (xb * kM + m) + acc : xb * kM + m;
      const size_t pix = (size_t)oy * a.Wo + ox;
      const size_t obase = (size_t)b * a.Ho * a.Wo * COUT + pix * COUT;
#pragma unroll
      for (int n0 = 0; n0 < COUT; n0 += 16) {
        float v[16];
        tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + acc * COUT + n0, v);
#pragma unroll
        for (int q = 0; q < 16; q += 4) {
          float4 o;
          float* po = &o.x;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            float t = v[q + u] + a.bias[n0 + q + u];
            if (a.softplus) t = softplus_f(t);
            po[u] = t;
          }
          if (add) {
            const float4 ad = *reinterpret_cast<const float4*>(add + pix * COUT + n0 + q);
            o.x += ad.x;
            o.y += ad.y;
            o.z += ad.z;
            o.w += ad.w;
          }
          if (a.residual) {
            const float4 rs = *reinterpret_cast<const float4*>(a.residual + obase + n0 + q);
            o.x += rs.x;
            o.y += rs.y;
            o.z += rs.z;
            o.w += rs.w;
          }
          *reinterpret_cast<float4*>(a.y + obase + n0 + q) = o;
        }
      }
    }
    tc_fence_before();
    __syncthreads();  // TMEM and staged rows are free for the next tile
  }
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(NCOLS));
  }
}

template <int CIN, int COUT, int MODE>
void launch_tc(const TcArgs& a, cudaStream_t st) {
  using S = Smem<CIN, COUT, MODE>;
  static int grid_cap = 0;
  if (!grid_cap) {
    cudaFuncSetAttribute(k_conv_tc<CIN, COUT, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::TOTAL);
    int per_sm = 0, sms = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_conv_tc<CIN, COUT, MODE>, kTcThreads, S::TOTAL);
    grid_cap = sms * (per_sm > 0 ? per_sm : 1);
  }
  const long long xblocks = MODE == 2 ? a.W / kM : a.Wo / kM;
  const long long ntiles = (long long)a.B * a.Ho * xblocks;
  const int grid = (int)(ntiles < grid_cap ? ntiles : grid_cap);
  k_conv_tc<CIN, COUT, MODE><<<grid, kTcThreads, S::TOTAL, st>>>(a);
}

}  // namespace

bool conv_tc_enabled = true;

bool conv_tc_supported(int cin, int cout, int stride, int transposed, int H, int W, int Wo) {
  if (!conv_tc_enabled) return false;
  const int mode = transposed ? 2 : (stride == 2 ? 1 : 0);
  const int width = mode == 2 ? W : Wo;
  if (width % kM) return false;
  if (mode == 0) return (cin == 16 && cout == 16) || (cin == 32 && cout == 32);
  if (mode == 1) return cin == 16 && cout == 32;
  return cin == 32 && cout == 16;
  (void)H;
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
