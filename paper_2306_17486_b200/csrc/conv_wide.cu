// tcgen05 implicit-GEMM 3x3 convolution for the wide (>= 64-channel) layers, K-streamed.
//
// Serves the reference conv2d / conv_transpose2d (autodiff.py:472-541, _corr :407-421, _corr_t
// :442-469) with batch norm folded (autodiff.py:595-607), softplus (:243-252) and the skip /
// encoder / residual adds of the ARCH.md network, at the channel counts whose bf16x3 weights do
// not fit in shared memory (9 x 128 x 128 x 3 parts x 2 B = 884 KB for a 128 -> 128 layer):
// 64 -> 64 and 128 -> 128 (stride 1), 64 -> 128 and 128 -> 128 (stride 2), 128 -> 64 (transposed).
//
// GEMM view.  One tile = M = 128 output pixels of one row (transposed: 128 input columns, two
// accumulators for the even / odd output columns) x N = cout, K = 9 taps x cin.  A pass covers R
// tiles (consecutive output rows of one 128-column block of one RHS) and streams K in chunks of
// 16 input channels:
//   for chunk c:  for tap row ky:  for tap kx:  B piece (c, ky, kx) = 16 x cout weights x 3 parts
//                                               for every tile using the tap: 3 (G = 3) or 5 MMAs
// Precision (BF16x3, x = x0 + x1 + x2 exactly; the dropped products are below 2^-16).
// The weight parts are stacked along N in every B piece ([W0 | W1 | W2], 3 cout rows per K plane),
// and each tile keeps G fp32 TMEM column groups so that the leading products a0 w0 are the ONLY
// terms of group 0: the tensor core's accumulation adds one rounding per K step to the large
// partial sums, exactly like a plain fp32 dot product, and every correction term goes to a group
// 2^8 smaller (measured: putting all six products in one accumulator made these layers 10x less
// accurate than fp32 SIMT).  The epilogue sums g0 + (g1 [+ g2]).
//   G = 3 (cout 64):  A0 x [W0 W1 W2] -> g0 g1 g2;  A1 x [W0 W1] -> g1 g2;  A2 x W0 -> g2
//   G = 2 (cout 128, transposed): A0 x [W0 W1] -> g0 g1;  A0 x W2, A1 x W0, A1 x W1, A2 x W0 -> g1
// (one UMMA has N <= 256, hence two groups for cout 128).
//
// Warp roles (one persistent CTA per SM):
//   warps 0-7    epilogue: tcgen05.ld of lane quarter (warp % 4) x column half (warp / 4), bias,
//                softplus, encoder / skip addend, residual, NHWC (or complex-planar) stores
//   warps 8-15   A converters: raw fp32 row chunks (RW pixels x 16 channels) -> exact bf16x3 split
//                -> A ring (UMMA K-major interleaved layout, 16 B pixel pitch, so the A operand of tap
//                kx is the staged row with its start address moved by kx)
//   warp 16      B producer: one cp.async.bulk per weight piece into the B ring (mbarrier tx-count)
//   warp 17      A producer: one TMA tensor load (cp.async.bulk.tensor.4d, box 16 ch x 130 px of the
//                NHWC activation, zero-filled outside the image) per row chunk into a raw ring
//   warp 18      MMA issuer (one elected lane issues tcgen05.mma; commits release ring slots and
//                hand the accumulators to the epilogue)
// The weights are split once into bf16x3 pieces laid out exactly like a B ring slot
// (k_wide_split: at network creation for the network's layers, conv_wide_register; otherwise a
// stream-ordered temporary per launch).  Every activation element is read from HBM once (the first
// channel chunk of a pass pulls the pass's input rows into L2 with bulk prefetches, the other chunks
// hit L2).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <map>
#include <mutex>

#include "common.cuh"
#include "conv_tc.h"
#include "prof.h"
#include "tc_util.cuh"

namespace hs {
namespace {
using namespace tc;

// measurement-variant switches (tools/_variants only; the product build uses the defaults):
// HS_WIDE_PROBE bit 1 skips the epilogue's side loads / math / stores, bit 2 the MMAs, bit 4 the
// A conversion, bit 8 the B pipeline (no weight copies, no B waits); HS_WIDE_G64 = column groups for cout 64 (3, or 2 to double-buffer the accumulators)
#ifndef HS_WIDE_PROBE
#define HS_WIDE_PROBE 0
#endif
#ifndef HS_WIDE_G64
#define HS_WIDE_G64 3
#endif
#ifndef HS_WIDE_EXTRA
#define HS_WIDE_EXTRA 0  // also 64 -> 32 transposed (measurement variant: 1.40 vs 1.09 ms on the resident-weight kernel)
#endif
#ifndef HS_WIDE_S2_32
#define HS_WIDE_S2_32 1  // 32 -> 64 stride 2 on this kernel (measured at C3: 0.85 vs 1.14 ms on the resident-weight kernel)
#endif
#ifndef HS_WIDE_RD_MAX
#define HS_WIDE_RD_MAX 8
#endif
#ifndef HS_WIDE_NAS_EXTRA
#define HS_WIDE_NAS_EXTRA 4
#endif
#ifndef HS_WIDE_ACV
#define HS_WIDE_ACV 8
#endif
constexpr int kWEpi = 8, kWAcv = HS_WIDE_ACV;
constexpr int kWarpA0 = kWEpi, kWarpB = kWEpi + kWAcv, kWarpAP = kWarpB + 1, kWarpMma = kWarpAP + 1;
constexpr int kWThreads = 32 * (kWarpMma + 1);
constexpr size_t kWSmemMax = 232448;

template <int CIN, int COUT, int MODE>
struct WCfg {
  static constexpr int MT = 128;                     // tile pixels (UMMA M)
  static constexpr int NACC = MODE == 2 ? 2 : 1;     // accumulators per tile (transposed: column parity)
  static constexpr int G = COUT <= 64 && NACC == 1 ? HS_WIDE_G64 : 2;  // column groups per accumulator (see above)
  static constexpr int ACC_COLS = G * COUT;
  // output rows (tiles) per pass: as many as TMEM holds, 4 at most (transposed: an even number)
  static constexpr int R = NACC * ACC_COLS * 4 <= 512 ? 4 : 2;
  static constexpr int SET_COLS = R * NACC * ACC_COLS;  // TMEM columns of one pass
  static constexpr int NSETS = 2 * SET_COLS <= 512 ? 2 : 1;  // double-buffered when it fits
  static constexpr int NCH = CIN / 16;               // K chunks
  static constexpr int RW = MODE == 0 ? MT + 2 : (MODE == 1 ? 2 * MT + 1 : MT + 1);  // staged pixels per row
  static constexpr int NROWS = MODE == 0 ? R + 2 : (MODE == 1 ? 2 * R + 1 : R / 2 + 1);  // input rows per pass
  static constexpr uint32_t A_PLANE = (uint32_t)RW * 16;   // one (part, 8-channel half) plane
  static constexpr uint32_t A_SLOT = 6 * A_PLANE;          // 3 parts x 2 halves
  static constexpr uint32_t B_PLANE = (uint32_t)3 * COUT * 16;  // one 8-channel half: rows [W0 | W1 | W2]
  static constexpr uint32_t B_SLOT = 2 * B_PLANE;
  static constexpr int IPT = (2 * RW + 32 * kWAcv - 1) / (32 * kWAcv);  // A items per converter thread
  // B ring: the bulk copies of the weight pieces are latency-bound (a few KB each from L2), so the
  // ring is made as deep as shared memory allows once the A ring has NROWS + 3 slots (16 at most)
  // raw fp32 ring filled by the A producer's TMA loads: one slot = NLOAD boxes of 130 pixels x 16
  // channels (64 B per pixel; stride 2 needs 257 pixels, two boxes)
  static constexpr int BOXW = 130, NLOAD = MODE == 1 ? 2 : 1;
  static constexpr size_t RAW_SLOT = (size_t)NLOAD * BOXW * 64;  // a multiple of 128 (TMA destination)
  // B ring slots (measured: a deeper ring is slower, the weight copies are not the limiter); the
  // stride-2 layers' 257-pixel rows need the space
#ifndef HS_WIDE_NBS
#define HS_WIDE_NBS 6
#endif
  static constexpr int NBS = MODE == 1 ? 4 : HS_WIDE_NBS;
  // staged drain: with one accumulator set, the epilogue copies the pass's group-summed accumulators
  // into shared memory and releases TMEM before its math and stores, so the next pass's MMAs overlap
  // them (cout 64 stride 1 only: the staging is R x 128 pixels x (cout + 4) floats, 70 KB)
  static constexpr int STG_PITCH = COUT + 4;  // floats per staged pixel (16-byte skew: conflict-free)
  static constexpr bool STG = NSETS == 1 && MODE == 0 && COUT == 64;
  static constexpr size_t STG_BYTES = STG ? (size_t)R * NACC * 128 * STG_PITCH * 4 : 0;
  static constexpr int pick_rd() {
    for (int n = HS_WIDE_RD_MAX; n > 2; --n)
      if (1024 + STG_BYTES + (size_t)n * RAW_SLOT + (size_t)NBS * B_SLOT + (size_t)(NROWS + 2) * A_SLOT <= kWSmemMax)
        return n;
    return 2;
  }
  static constexpr int RD = pick_rd();
  static constexpr size_t BASE = 1024 + STG_BYTES + RD * RAW_SLOT;  // staging, raw ring, barriers, bias
  static constexpr size_t FIXED = BASE + (size_t)NBS * B_SLOT;
  static constexpr int pick_nas() {
    for (int n = NROWS + HS_WIDE_NAS_EXTRA; n > NROWS; --n)
      if (FIXED + (size_t)n * A_SLOT <= kWSmemMax) return n;
    // (stride 2: the 257-pixel rows leave room for NROWS + 1 slots at most)
    return NROWS;
  }
  static constexpr int NAS = pick_nas();                   // A ring slots (>= rows of one chunk)
  static constexpr size_t TOTAL = FIXED + (size_t)NAS * A_SLOT;
  static constexpr int NCOLS = NSETS * SET_COLS <= 128 ? 128 : (NSETS * SET_COLS <= 256 ? 256 : 512);
  static_assert(NSETS * SET_COLS <= 512, "TMEM");
  static_assert(TOTAL <= kWSmemMax, "shared memory");
  static_assert(CIN % 16 == 0 && COUT % 32 == 0 && COUT <= 256, "shapes");
  static_assert(RAW_SLOT % 128 == 0 && RW <= NLOAD * BOXW, "raw ring");
};

struct WArgs {
  const unsigned char* wsplit;  // bf16x3 weight pieces [chunk][tap] x B_SLOT bytes (k_wide_split)
  const float* x;
  int H, W;
  float* y;
  int Ho, Wo;
  const float* w;  // [cout][ky][kx][cin] (transposed layers in the same order, see cnn.h)
  const float* bias;
  int softplus;
  const float* addend;
  long long addend_bstride;
  int addend_per_model;
  const int* model_of;
  const float* residual;
  const void* const* active;
  int B;
  int planar;
  int ldc;   // channels per pixel of y / addend / residual (COUT, or the full width for a cout slice)
  int coff;  // first channel of this launch's slice (bias is already offset)
};

struct Pass {
  int b, xb, oy0;
};

template <int MODE, typename C>
__host__ __device__ inline long long num_passes(const WArgs& a) {
  const int xblocks = (MODE == 2 ? a.W : a.Wo) / C::MT;
  return (long long)a.B * xblocks * ((a.Ho + C::R - 1) / C::R);
}

// pass u -> (b, column block, first output row); RHS slowest so neighbouring CTAs share input rows in L2
template <int MODE, typename C>
HS_DEV bool pass_at(const WArgs& a, long long u, Pass& P) {
  const int xblocks = (MODE == 2 ? a.W : a.Wo) / C::MT;
  const int bands = (a.Ho + C::R - 1) / C::R;
  P.xb = (int)(u % xblocks);
  P.oy0 = (int)((u / xblocks) % bands) * C::R;
  P.b = (int)(u / ((long long)xblocks * bands));
  return !(a.active && a.active[P.b] == nullptr);
}

// first input row of the pass and first input column of the staged segment
template <int MODE>
HS_DEV int first_row(int oy0) { return MODE == 0 ? oy0 - 1 : (MODE == 1 ? 2 * oy0 - 1 : oy0 >> 1); }
template <int MODE>
HS_DEV int first_col(int xb) { return MODE == 0 ? 128 * xb - 1 : (MODE == 1 ? 256 * xb - 1 : 128 * xb); }
// raw pixel p of the segment -> staged pixel (stride 2 de-interleaves: even columns, then odd)
template <int MODE>
HS_DEV int staged(int p) {
  if (MODE != 1) return p;
  return (p & 1) ? (p - 1) >> 1 : 128 + (p >> 1);
}

// Tap usage.  For output row r of the pass (0..R-1) and tap (ky, kx): the input row (relative to
// first_row), the staged start pixel of the A window and the accumulator parity, or -1 if unused.
template <int MODE>
HS_DEV int tap_row(int r, int ky) {
  if (MODE == 0) return r + ky;
  if (MODE == 1) return 2 * r + ky;
  // transposed: out row 2q <- (ky 1, in row q); out row 2q+1 <- (ky 0, row q+1), (ky 2, row q)
  if ((r & 1) == 0) return ky == 1 ? (r >> 1) : -1;
  return ky == 0 ? (r >> 1) + 1 : (ky == 2 ? (r >> 1) : -1);
}
template <int MODE>
HS_DEV int tap_px(int kx) {
  if (MODE == 0) return kx;
  if (MODE == 1) return kx == 0 ? 128 : (kx == 1 ? 0 : 129);
  // transposed: out col 2q (acc 0) <- (kx 1, in col q); out col 2q+1 (acc 1) <- (kx 0, q+1), (kx 2, q)
  return kx == 0 ? 1 : 0;
}
template <int MODE>
HS_DEV int tap_acc(int kx) { return MODE == 2 ? (kx == 1 ? 0 : 1) : 0; }
// the last tap row that reads input row i of a pass (its A slot is released after it)
template <int MODE, int R>
HS_DEV int last_ky(int i) {
  int m = -1;
  for (int r = 0; r < R; ++r)
    for (int ky = 0; ky < 3; ++ky)
      if (tap_row<MODE>(r, ky) == i) m = ky > m ? ky : m;
  return m;
}

template <int CIN, int COUT, int MODE>
__global__ void __launch_bounds__(kWThreads, 1) k_conv_wide(const __grid_constant__ WArgs a,
                                                             const __grid_constant__ CUtensorMap tmx) {
  using C = WCfg<CIN, COUT, MODE>;
  constexpr int R = C::R, NCH = C::NCH, NAS = C::NAS, NBS = C::NBS, NROWS = C::NROWS, RD = C::RD;
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* araw = smem;  // TMA destinations first: 128-byte aligned
  float* stg = reinterpret_cast<float*>(araw + (size_t)RD * C::RAW_SLOT);  // staged drain (C::STG)
  unsigned char* bring = araw + (size_t)RD * C::RAW_SLOT + C::STG_BYTES;
  unsigned char* aring = bring + (size_t)NBS * C::B_SLOT;
  uint64_t* bars = reinterpret_cast<uint64_t*>(aring + (size_t)NAS * C::A_SLOT);
  uint64_t* a_full = bars;
  uint64_t* a_empty = a_full + NAS;
  uint64_t* b_full = a_empty + NAS;
  uint64_t* b_empty = b_full + NBS;
  uint64_t* acc_full = b_empty + NBS;
  uint64_t* acc_empty = acc_full + 2;
  uint64_t* raw_full = acc_empty + 2;
  uint64_t* raw_empty = raw_full + RD;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(raw_empty + RD);
  float* s_bias = reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(bars) + 512);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long npass = num_passes<MODE, C>(a);

  for (int n = tid; n < COUT; n += kWThreads) s_bias[n] = a.bias[n];
  if (tid == 0) {
    for (int i = 0; i < NAS; ++i) {
      mbar_init(smem_u32(&a_full[i]), kWAcv);
      mbar_init(smem_u32(&a_empty[i]), 1);
    }
    for (int i = 0; i < NBS; ++i) {
      mbar_init(smem_u32(&b_full[i]), 1);
      mbar_init(smem_u32(&b_empty[i]), 1);
    }
    for (int i = 0; i < RD; ++i) {
      mbar_init(smem_u32(&raw_full[i]), 1);
      mbar_init(smem_u32(&raw_empty[i]), kWAcv);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(&acc_full[i]), 1);
      mbar_init(smem_u32(&acc_empty[i]), kWEpi);
    }
    fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s_tmem)),
                 "r"(C::NCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;
  // programmatic dependent launch: set-up above overlaps the previous kernel's tail (persistent grid)
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");

  auto pass_of = [&](long long& u, Pass& P) {  // first active pass at or after u
    while (u < npass && !pass_at<MODE, C>(a, u, P)) u += gridDim.x;
    return u < npass;
  };
  if (warp == kWarpAP) {
    // ================= A producer: TMA row-chunk loads (pass, chunk, row) into the raw ring
    if (lane == 0) {
      uint32_t seq = 0;
      Pass P;
      for (long long u = blockIdx.x; pass_of(u, P); u += gridDim.x) {
        const int g0 = first_row<MODE>(P.oy0), x0 = first_col<MODE>(P.xb);
        {  // all channels of the pass's input rows and its side-input rows into L2: later chunks hit L2
          const int clo = max(x0, 0), chi = min(x0 + C::RW, a.W);
          const float* img = a.x + (size_t)P.b * a.H * a.W * CIN;
          for (int r = 0; r < NROWS; ++r) {
            const int g = g0 + r;
            if (g >= 0 && g < a.H && chi > clo)
              prefetch_l2(img + ((size_t)g * a.W + clo) * CIN, (uint32_t)(chi - clo) * CIN * 4);
          }
          const float* add = a.addend ? a.addend + (a.addend_per_model ? (a.model_of ? a.model_of[P.b] : 0) : P.b) *
                                                       a.addend_bstride
                                      : nullptr;
          constexpr int OXN = MODE == 2 ? 256 : 128;  // output columns of a tile
          for (int r = 0; r < R && P.oy0 + r < a.Ho; ++r) {
            const size_t pix = (size_t)(P.oy0 + r) * a.Wo + (size_t)OXN * P.xb;
            if (add) prefetch_l2(add + pix * COUT, OXN * COUT * 4);
            if (a.residual) prefetch_l2(a.residual + ((size_t)P.b * a.Ho * a.Wo + pix) * COUT, OXN * COUT * 4);
          }
        }
        for (int c = 0; c < NCH; ++c)
          for (int i = 0; i < NROWS; ++i, ++seq) {
            const uint32_t s = seq % RD, use = seq / RD;
            if (use > 0) mbar_wait(smem_u32(&raw_empty[s]), (use - 1) & 1);
            const uint32_t bar = smem_u32(&raw_full[s]);
            mbar_arrive_tx(bar, (uint32_t)C::RAW_SLOT);
#pragma unroll
            for (int l = 0; l < C::NLOAD; ++l)  // coordinates (channel, column, row, RHS); outside -> zeros
              asm volatile(
                  "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
                  "%4, %5}], [%6];" ::"r"(smem_u32(araw + (size_t)s * C::RAW_SLOT + (size_t)l * C::BOXW * 64)),
                  "l"(reinterpret_cast<uint64_t>(&tmx)), "r"(16 * c), "r"(x0 + l * C::BOXW), "r"(g0 + i), "r"(P.b),
                  "r"(bar)
                  : "memory");
          }
      }
    }
  } else if (warp >= kWarpA0 && warp < kWarpA0 + kWAcv) {
    // ================= A converters: raw row chunks -> bf16x3 A ring.  Item e of a row is (pixel
    // e % RW, channel half e / RW): pixel fastest, so the 16-byte smem stores of a warp are contiguous.
    const int t = tid - 32 * kWarpA0;
    constexpr int NT = 32 * kWAcv, IPT = C::IPT;
    uint32_t seq = 0;
    Pass P;
    for (long long u = blockIdx.x; pass_of(u, P); u += gridDim.x)
      for (int c = 0; c < NCH; ++c)
        for (int i = 0; i < NROWS; ++i, ++seq) {
          const uint32_t rs = seq % RD;
          mbar_wait(smem_u32(&raw_full[rs]), (seq / RD) & 1);
          const uint32_t s = seq % NAS, use = seq / NAS;
          if (use > 0) mbar_wait(smem_u32(&a_empty[s]), (use - 1) & 1);
          unsigned char* slot = aring + (size_t)s * C::A_SLOT;
          const unsigned char* raw = araw + (size_t)rs * C::RAW_SLOT;
          // every item's raw loads first, then the conversions and stores (the compiler cannot hoist
          // the loads of a later item over the earlier item's stores to the A ring)
          constexpr int NI = (HS_WIDE_PROBE & 4) ? 0 : IPT;
          float4 va[NI > 0 ? NI : 1][2];
#pragma unroll
          for (int k = 0; k < NI; ++k) {
            const int e = t + k * NT;
            const int p = e % C::RW, h = e / C::RW;
            if (e < 2 * C::RW) {
              va[k][0] = *reinterpret_cast<const float4*>(raw + (size_t)p * 64 + h * 32);
              va[k][1] = *reinterpret_cast<const float4*>(raw + (size_t)p * 64 + h * 32 + 16);
            }
          }
#pragma unroll
          for (int k = 0; k < NI; ++k) {
            const int e = t + k * NT;
            if (e >= 2 * C::RW) break;
            const int p = e % C::RW, h = e / C::RW;
            const float v[8] = {va[k][0].x, va[k][0].y, va[k][0].z, va[k][0].w,
                                va[k][1].x, va[k][1].y, va[k][1].z, va[k][1].w};
            uint4 q0, q1, q2;
            split_bf16x3(v, q0, q1, q2);
            const size_t off = (size_t)h * C::A_PLANE + (size_t)staged<MODE>(p) * 16;
            *reinterpret_cast<uint4*>(slot + off) = q0;
            *reinterpret_cast<uint4*>(slot + 2 * C::A_PLANE + off) = q1;
            *reinterpret_cast<uint4*>(slot + 4 * C::A_PLANE + off) = q2;
          }
          fence_async_smem();
          __syncwarp();
          if (lane == 0) {
            mbar_arrive(smem_u32(&a_full[s]));
            mbar_arrive(smem_u32(&raw_empty[rs]));
          }
        }
  } else if (warp == kWarpB) {
    // ================= B producer: pre-split weight pieces (c, ky, kx), one bulk copy each, in MMA order
    if (lane == 0 && !(HS_WIDE_PROBE & 8)) {
      uint32_t seq = 0;
      for (long long u = blockIdx.x; u < npass; u += gridDim.x) {
        Pass P;
        if (!pass_at<MODE, C>(a, u, P)) continue;
        for (int pc = 0; pc < NCH * 9; ++pc, ++seq) {
          const uint32_t s = seq % NBS, use = seq / NBS;
          if (use > 0) mbar_wait(smem_u32(&b_empty[s]), (use - 1) & 1);
          const uint32_t bar = smem_u32(&b_full[s]);
          mbar_arrive_tx(bar, C::B_SLOT);
          bulk_g2s(smem_u32(bring + (size_t)s * C::B_SLOT), a.wsplit + (size_t)pc * C::B_SLOT, C::B_SLOT, bar);
        }
      }
    }
  } else if (warp == kWarpMma) {
    // ================= MMA issuer
    // The per-row bookkeeping is hoisted out of the tap loops: the A descriptors of a chunk's rows are
    // formed once, the staged-row waits happen once per tap row, and the taps (fully unrolled) issue
    // each tile's three (G = 3) or five (G = 2) MMAs from one asm block with one elect.
    constexpr uint32_t I1 = idesc_bf16(128, COUT), I2 = idesc_bf16(128, 2 * COUT), I3 = idesc_bf16(128, 3 * COUT);
    constexpr uint32_t WROW = (uint32_t)COUT * 16;  // byte offset of weight part p: p * WROW
    const uint32_t a_base = smem_u32(aring), b_base = smem_u32(bring);
    uint32_t aseq = 0, bseq = 0, pass = 0;
    for (long long u = blockIdx.x; u < npass; u += gridDim.x) {
      Pass P;
      if (!pass_at<MODE, C>(a, u, P)) continue;
      const uint32_t set = pass % C::NSETS, suse = pass / C::NSETS;
      if (suse > 0) mbar_wait(smem_u32(&acc_empty[set]), (suse - 1) & 1);
      tc_fence_after();
      const uint32_t dset = tmem + set * C::SET_COLS;
      uint32_t started = 0;  // bit (r * NACC + k): accumulator written
      for (int c = 0; c < NCH; ++c) {
        uint32_t arow[NROWS];  // descriptor low word of each row's part 0, pixel 0
#pragma unroll
        for (int i = 0; i < NROWS; ++i) arow[i] = desc_lo(a_base + ((aseq + (uint32_t)i) % NAS) * C::A_SLOT, C::A_PLANE);
        int have = -1;  // highest input row of this chunk known to be staged
#pragma unroll
        for (int ky = 0; ky < 3; ++ky) {
          int need = -1;
#pragma unroll
          for (int r = 0; r < R; ++r) need = tap_row<MODE>(r, ky) > need ? tap_row<MODE>(r, ky) : need;
          for (; have < need; ++have) {
            const uint32_t sq = aseq + (uint32_t)(have + 1);
            mbar_wait(smem_u32(&a_full[sq % NAS]), (sq / NAS) & 1);
          }
          tc_fence_after();
#pragma unroll
          for (int kx = 0; kx < 3; ++kx, ++bseq) {
            const uint32_t bs = bseq % NBS;
            if (!(HS_WIDE_PROBE & 8)) mbar_wait(smem_u32(&b_full[bs]), (bseq / NBS) & 1);
            const uint32_t w0 = desc_lo(b_base + bs * C::B_SLOT, C::B_PLANE);
#pragma unroll
            for (int r = 0; r < R; ++r) {
              const int i = tap_row<MODE>(r, ky);
              if (i < 0) continue;
              const int k = tap_acc<MODE>(kx);
              const uint32_t bit = 1u << (r * C::NACC + k);
              const uint32_t d = dset + (uint32_t)((r * C::NACC + k) * C::ACC_COLS);
              const uint32_t a0 = arow[i] + (uint32_t)tap_px<MODE>(kx);  // 16-byte pixel steps
              const uint32_t acc = (started & bit) ? 1u : 0u;
              if constexpr ((HS_WIDE_PROBE & 2) != 0) {
              } else if constexpr (C::G == 3) {
                // g0 g1 g2 += a0 [w0 w1 w2];  g1 g2 += a1 [w0 w1];  g2 += a2 w0
                asm volatile(
                    "{\n\t.reg .pred p, t, e;\n\t.reg .b64 da, db;\n\t.reg .b32 al, dd;\n\t"
                    "setp.ne.b32 p, %3, 0;\n\tsetp.eq.b32 t, %3, %3;\n\telect.sync _|e, 0xffffffff;\n\t"
                    "mov.b64 db, {%2, %4};\n\tmov.b64 da, {%1, %4};\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %5, p;\n\t"
                    "add.u32 al, %1, %8;\n\tmov.b64 da, {al, %4};\n\tadd.u32 dd, %0, %10;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [dd], da, db, %6, t;\n\t"
                    "add.u32 al, %1, %9;\n\tmov.b64 da, {al, %4};\n\tadd.u32 dd, %0, %11;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [dd], da, db, %7, t;\n\t}\n" ::"r"(d),
                    "r"(a0), "r"(w0), "r"(acc), "n"(kDescHi), "n"(I3), "n"(I2), "n"(I1),
                    "n"((2 * C::A_PLANE) >> 4), "n"((4 * C::A_PLANE) >> 4), "n"(COUT), "n"(2 * COUT));
              } else {
                // g0 g1 += a0 [w0 w1];  g1 += a0 w2, a1 w0, a1 w1, a2 w0
                asm volatile(
                    "{\n\t.reg .pred p, t, e;\n\t.reg .b64 da, db;\n\t.reg .b32 al, bl, dd;\n\t"
                    "setp.ne.b32 p, %3, 0;\n\tsetp.eq.b32 t, %3, %3;\n\telect.sync _|e, 0xffffffff;\n\t"
                    "mov.b64 db, {%2, %4};\n\tmov.b64 da, {%1, %4};\n\tadd.u32 dd, %0, %10;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %5, p;\n\t"
                    "add.u32 bl, %2, %9;\n\tmov.b64 db, {bl, %4};\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [dd], da, db, %6, t;\n\t"
                    "add.u32 al, %1, %7;\n\tmov.b64 da, {al, %4};\n\tmov.b64 db, {%2, %4};\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [dd], da, db, %6, t;\n\t"
                    "add.u32 bl, %2, %11;\n\tmov.b64 db, {bl, %4};\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [dd], da, db, %6, t;\n\t"
                    "add.u32 al, %1, %8;\n\tmov.b64 da, {al, %4};\n\tmov.b64 db, {%2, %4};\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [dd], da, db, %6, t;\n\t}\n" ::"r"(d),
                    "r"(a0), "r"(w0), "r"(acc), "n"(kDescHi), "n"(I2), "n"(I1),
                    "n"((2 * C::A_PLANE) >> 4), "n"((4 * C::A_PLANE) >> 4), "n"((2 * WROW) >> 4), "n"(COUT),
                    "n"(WROW >> 4));
              }
              started |= bit;
            }
            if (!(HS_WIDE_PROBE & 8)) mma_commit(smem_u32(&b_empty[bs]));  // the piece is free once its MMAs completed
          }
          // input rows whose last reader was this tap row go back to the converters
#pragma unroll
          for (int i = 0; i < NROWS; ++i)
            if (last_ky<MODE, R>(i) == ky) mma_commit(smem_u32(&a_empty[(aseq + (uint32_t)i) % NAS]));
        }
        aseq += NROWS;
      }
      mma_commit(smem_u32(&acc_full[set]));
      ++pass;
    }
  } else if (warp < kWEpi) {
    // ================= epilogue: lane quarter q (tile pixel m = 32 q + lane), column half hc
    constexpr int EH = COUT / 2;
    const int q4 = warp & 3, hc = warp >> 2;
    const int m = 32 * q4 + lane;
    uint32_t pass = 0;
    for (long long u = blockIdx.x; u < npass; u += gridDim.x) {
      Pass P;
      if (!pass_at<MODE, C>(a, u, P)) continue;
      const uint32_t set = pass % C::NSETS;
      mbar_wait(smem_u32(&acc_full[set]), (pass / C::NSETS) & 1);
      tc_fence_after();
      if constexpr (C::STG) {
        // drain: group-summed accumulators of every tile into this thread's staging rows, then TMEM is free
#pragma unroll 1
        for (int rk = 0; rk < R * C::NACC; ++rk)
#pragma unroll
          for (int n0 = 0; n0 < EH; n0 += 8) {
            uint32_t v[8], v1[8], v2[8];
            const uint32_t col = tmem + ((uint32_t)(32 * q4) << 16) + set * C::SET_COLS +
                                 (uint32_t)(rk * C::ACC_COLS) + hc * EH + n0;
            tmem_ld8(col, v);
            tmem_ld8(col + COUT, v1);
            if constexpr (C::G == 3) tmem_ld8(col + 2 * COUT, v2);
            tmem_wait_ld();
            float gs[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float corr = C::G == 3 ? __uint_as_float(v1[j]) + __uint_as_float(v2[j]) : __uint_as_float(v1[j]);
              gs[j] = __uint_as_float(v[j]) + corr;
            }
            float4* dp = reinterpret_cast<float4*>(stg + ((size_t)rk * 128 + m) * C::STG_PITCH + hc * EH + n0);
            dp[0] = make_float4(gs[0], gs[1], gs[2], gs[3]);
            dp[1] = make_float4(gs[4], gs[5], gs[6], gs[7]);
          }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&acc_empty[set]));
      }
      const float* add = a.addend ? a.addend + (a.addend_per_model ? (a.model_of ? a.model_of[P.b] : 0) : P.b) *
                                                   a.addend_bstride
                                  : nullptr;
      // side input (encoder / skip addend or residual) of one 16-channel segment: loaded a segment
      // ahead of its use (the converters pulled the pass's side rows into L2 when the pass started)
      constexpr int SEG = 16, NSEG = EH / SEG;
      const float* side = add ? add : a.residual;
      const bool side_res = !add;  // addend rows are indexed by pixel, residual rows by (b, pixel)
      // NHWC stores: the four lanes of a group transpose their pixels' 16-byte chunks (group4_transpose),
      // so every store / side load instruction moves whole 64-byte segments; lane gi then owns chunk gi
      // of the group's pixels j = 0..3 (tile pixel m - gi + j)
      const bool tr = !a.planar;
      const int gi = lane & 3;
      auto ox_of = [&](int mm, int k) { return MODE == 2 ? 2 * (128 * P.xb + mm) + k : 128 * P.xb + mm; };
      auto side_ptr = [&](int r, int k, int sg, int mm) -> const float4* {
        const size_t pix = (size_t)(P.oy0 + r) * a.Wo + ox_of(mm, k);
        const size_t base = side_res ? ((size_t)P.b * a.Ho * a.Wo + pix) * a.ldc : pix * a.ldc;
        return reinterpret_cast<const float4*>(side + base + a.coff + hc * EH + sg * SEG);
      };
      float4 sd[SEG / 4], sn[SEG / 4];
      auto load_side = [&](int r, int k, int sg, float4 (&dst)[SEG / 4]) {
#pragma unroll
        for (int q = 0; q < SEG / 4; ++q) dst[q] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (side && P.oy0 + r < a.Ho) {
          if (tr) {
#pragma unroll
            for (int j = 0; j < SEG / 4; ++j) dst[j] = __ldg(side_ptr(r, k, sg, m - gi + j) + gi);
          } else {
            const float4* sp = side_ptr(r, k, sg, m);
#pragma unroll
            for (int q = 0; q < SEG / 4; ++q) dst[q] = __ldg(sp + q);
          }
        }
      };
      if (HS_WIDE_PROBE & 1) side = nullptr;  // probe build only
      load_side(0, 0, 0, sn);
      for (int step = 0; step < R * C::NACC * NSEG; ++step) {
        const int sg = step % NSEG, k = (step / NSEG) % C::NACC, r = step / (NSEG * C::NACC);
#pragma unroll
        for (int q = 0; q < SEG / 4; ++q) sd[q] = sn[q];
        if (step + 1 < R * C::NACC * NSEG) {
          const int s1 = step + 1;
          load_side(s1 / (NSEG * C::NACC), (s1 / NSEG) % C::NACC, s1 % NSEG, sn);
        }
        const int oy = P.oy0 + r;
        const int ox = MODE == 2 ? 2 * (128 * P.xb + m) + k : 128 * P.xb + m;
        const size_t pix = (size_t)oy * a.Wo + ox;
        const size_t obase = ((size_t)P.b * a.Ho * a.Wo + pix) * a.ldc + a.coff + hc * EH + sg * SEG;
        float o[SEG];
#pragma unroll
        for (int n0 = 0; n0 < SEG; n0 += 8) {
          float gs[8];  // g0 + (g1 [+ g2]): the corrections are summed first
          if constexpr (C::STG) {
            const float4* sp4 = reinterpret_cast<const float4*>(
                stg + ((size_t)(r * C::NACC + k) * 128 + m) * C::STG_PITCH + hc * EH + sg * SEG + n0);
            const float4 g0 = sp4[0], g1 = sp4[1];
            gs[0] = g0.x, gs[1] = g0.y, gs[2] = g0.z, gs[3] = g0.w, gs[4] = g1.x, gs[5] = g1.y, gs[6] = g1.z,
            gs[7] = g1.w;
          } else {
            uint32_t v[8], v1[8], v2[8];
            const uint32_t col = tmem + ((uint32_t)(32 * q4) << 16) + set * C::SET_COLS +
                                 (uint32_t)((r * C::NACC + k) * C::ACC_COLS) + hc * EH + sg * SEG + n0;
            tmem_ld8(col, v);
            tmem_ld8(col + COUT, v1);
            if constexpr (C::G == 3) tmem_ld8(col + 2 * COUT, v2);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float corr = C::G == 3 ? __uint_as_float(v1[j]) + __uint_as_float(v2[j]) : __uint_as_float(v1[j]);
              gs[j] = __uint_as_float(v[j]) + corr;
            }
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            float x = gs[j] + s_bias[hc * EH + sg * SEG + n0 + j];
            if (a.softplus) x = softplus_fast(x);
            o[n0 + j] = x;
          }
        }
        if (oy >= a.Ho || (HS_WIDE_PROBE & 1)) continue;  // (warp-uniform: every lane has the same row)
        if (tr) {
          float4 ch[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) ch[q] = make_float4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
          group4_transpose(ch, gi);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            ch[j].x += sd[j].x, ch[j].y += sd[j].y, ch[j].z += sd[j].z, ch[j].w += sd[j].w;
            const size_t pj = (size_t)oy * a.Wo + ox_of(m - gi + j, k);
            const size_t oj = ((size_t)P.b * a.Ho * a.Wo + pj) * a.ldc + a.coff + hc * EH + sg * SEG + 4 * gi;
            if (add && a.residual) {
              const float4 rv = __ldg(reinterpret_cast<const float4*>(a.residual + oj));
              ch[j].x += rv.x, ch[j].y += rv.y, ch[j].z += rv.z, ch[j].w += rv.w;
            }
            *reinterpret_cast<float4*>(a.y + oj) = ch[j];
          }
          continue;
        }
#pragma unroll
        for (int q = 0; q < SEG / 4; ++q) {
          o[4 * q] += sd[q].x, o[4 * q + 1] += sd[q].y, o[4 * q + 2] += sd[q].z, o[4 * q + 3] += sd[q].w;
        }
        if (add && a.residual) {  // both side inputs (not used by the ARCH.md network): the residual directly
          const float4* rp = reinterpret_cast<const float4*>(a.residual + obase);
#pragma unroll
          for (int q = 0; q < SEG / 4; ++q) {
            const float4 rv = __ldg(rp + q);
            o[4 * q] += rv.x, o[4 * q + 1] += rv.y, o[4 * q + 2] += rv.z, o[4 * q + 3] += rv.w;
          }
        }
        if (a.planar) {  // channel pairs (2c, 2c+1) -> complex plane c (the implicit layer's input)
          float2* yp = reinterpret_cast<float2*>(a.y) +
                       ((size_t)P.b * (COUT / 2) + (hc * EH + sg * SEG) / 2) * ((size_t)a.Ho * a.Wo) + pix;
#pragma unroll
          for (int j = 0; j < SEG / 2; ++j) yp[(size_t)j * a.Ho * a.Wo] = make_float2(o[2 * j], o[2 * j + 1]);
        } else {
          float4* yp = reinterpret_cast<float4*>(a.y + obase);
#pragma unroll
          for (int q = 0; q < SEG / 4; ++q) yp[q] = make_float4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
        }
      }
      if constexpr (!C::STG) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&acc_empty[set]));
      }
      ++pass;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::NCOLS));
  }
}

// bf16x3 weight pieces in B-slot layout: piece (c, tap) = [half h][row = part * cout + n] x 16 B, the
// 8 channels 16 c + 8 h .. + 7 of part `part` of w[n][tap][:]
template <int CIN, int COUT>
__global__ void k_wide_split(const float* __restrict__ w, uint4* __restrict__ out) {
  constexpr int NCH = CIN / 16, ROWS = 3 * COUT;
  const long long total = (long long)NCH * 9 * 2 * COUT;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const int n = (int)(e % COUT), h = (int)((e / COUT) % 2), pc = (int)(e / (2 * COUT));
    const int c = pc / 9, tap = pc % 9;
    const float4* s4 = reinterpret_cast<const float4*>(w + ((size_t)n * 9 + tap) * CIN + 16 * c + 8 * h);
    const float4 v0 = __ldg(s4), v1 = __ldg(s4 + 1);
    const float v[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
    uint4 q[3];
    split_bf16x3(v, q[0], q[1], q[2]);
    uint4* piece = out + (size_t)pc * 2 * ROWS;
#pragma unroll
    for (int part = 0; part < 3; ++part) piece[(size_t)h * ROWS + part * COUT + n] = q[part];
  }
}

size_t split_bytes(int cin, int cout) { return (size_t)(cin / 16) * 9 * 2 * 3 * cout * 16; }

cudaError_t run_split(const float* w, int cin, int cout, void* out, cudaStream_t st) {
  const int blocks = (int)((split_bytes(cin, cout) / 16 / 3 + 255) / 256);
  if (cin == 64 && cout == 64) k_wide_split<64, 64><<<blocks, 256, 0, st>>>(w, static_cast<uint4*>(out));
  else if (cin == 128 && cout == 128) k_wide_split<128, 128><<<blocks, 256, 0, st>>>(w, static_cast<uint4*>(out));
  else if (cin == 64 && cout == 128) k_wide_split<64, 128><<<blocks, 256, 0, st>>>(w, static_cast<uint4*>(out));
  else if (cin == 128 && cout == 64) k_wide_split<128, 64><<<blocks, 256, 0, st>>>(w, static_cast<uint4*>(out));
#if HS_WIDE_S2_32
  else if (cin == 32 && cout == 64) k_wide_split<32, 64><<<blocks, 256, 0, st>>>(w, static_cast<uint4*>(out));
#endif
#if HS_WIDE_EXTRA
  else if (cin == 64 && cout == 32) k_wide_split<64, 32><<<blocks, 256, 0, st>>>(w, static_cast<uint4*>(out));
#endif
  else return cudaErrorInvalidValue;
  prof::count(1);
  return cudaGetLastError();
}

// weights registered by hs_net_create: device weight pointer -> its split pieces
std::mutex reg_mu;
std::map<const float*, void*> reg;
// 128 -> 128 layers also keep the bf16x3 split of each 64-output-channel slice: a transposed 128 -> 128
// layer runs as two 128 -> 64 launches (its two parity accumulators of 256 columns do not fit TMEM)
std::map<std::pair<const float*, int>, void*> reg_slice;
constexpr size_t kSlice128 = (size_t)64 * 9 * 128;  // floats of one 64-channel weight slice

// TMA descriptor of the NHWC activation x: 4-D (channel, column, row, RHS), box 16 channels x 130
// columns x 1 x 1, fp32, zero fill outside the tensor (the convolution's padding and halo)
bool make_tmap(CUtensorMap* tm, const float* x, int cin, int H, int W, int B) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return false;
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint64_t dims[4] = {(cuuint64_t)cin, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)B};
  const cuuint64_t strides[3] = {(cuuint64_t)cin * 4, (cuuint64_t)W * cin * 4, (cuuint64_t)H * W * cin * 4};
  const cuuint32_t box[4] = {16, 130, 1, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  return encode(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(x), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int CIN, int COUT, int MODE>
void launch_wide(const WArgs& a, const CUtensorMap& tm, cudaStream_t st) {
  using C = WCfg<CIN, COUT, MODE>;
  static int sms = 0;
  if (!sms) {
    cudaFuncSetAttribute(k_conv_wide<CIN, COUT, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::TOTAL);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  long long grid = sms;
  const long long np = num_passes<MODE, C>(a);
  if (np < grid) grid = np;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kWThreads);
  cfg.dynamicSmemBytes = C::TOTAL;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k_conv_wide<CIN, COUT, MODE>, a, tm);
}

}  // namespace

bool conv_wide_supported(int cin, int cout, int stride, int transposed, int H, int W, int Wo) {
  (void)H;
  if (!conv_tc_enabled) return false;
  const int mode = transposed ? 2 : (stride == 2 ? 1 : 0);
  if ((mode == 2 ? W : Wo) % 128) return false;
  return (mode == 0 && ((cin == 64 && cout == 64) || (cin == 128 && cout == 128))) ||
         (mode == 1 && ((cin == 64 && cout == 128) || (cin == 128 && cout == 128) ||
                        (HS_WIDE_S2_32 && cin == 32 && cout == 64))) ||
         (mode == 2 && ((cin == 128 && cout == 64) || (cin == 128 && cout == 128) ||
                        (HS_WIDE_EXTRA && cin == 64 && cout == 32)));
}

bool conv_wide_eligible(int cin, int cout) {
  return (cin == 64 && cout == 64) || (cin == 128 && cout == 128) || (cin == 64 && cout == 128) ||
         (cin == 128 && cout == 64) || (HS_WIDE_S2_32 && cin == 32 && cout == 64) ||
         (HS_WIDE_EXTRA && cin == 64 && cout == 32);
}

int conv_wide_register(const float* w, int cin, int cout, cudaStream_t st) {
  if (!conv_wide_eligible(cin, cout)) return 0;
  void* buf = nullptr;
  if (cudaMalloc(&buf, split_bytes(cin, cout)) != cudaSuccess) return 1;
  if (run_split(w, cin, cout, buf, st) != cudaSuccess) {
    cudaFree(buf);
    return 1;
  }
  void* half[2] = {nullptr, nullptr};
  if (cin == 128 && cout == 128)
    for (int h = 0; h < 2; ++h)
      if (cudaMalloc(&half[h], split_bytes(128, 64)) != cudaSuccess ||
          run_split(w + h * kSlice128, 128, 64, half[h], st) != cudaSuccess)
        return 1;
  std::lock_guard<std::mutex> g(reg_mu);
  auto it = reg.find(w);
  if (it != reg.end()) cudaFree(it->second);
  reg[w] = buf;
  for (int h = 0; h < 2; ++h)
    if (half[h]) {
      auto is = reg_slice.find({w, h});
      if (is != reg_slice.end()) cudaFree(is->second);
      reg_slice[{w, h}] = half[h];
    }
  return 0;
}

void conv_wide_unregister(const float* w) {
  std::lock_guard<std::mutex> g(reg_mu);
  for (int h = 0; h < 2; ++h) {
    auto is = reg_slice.find({w, h});
    if (is != reg_slice.end()) {
      cudaFree(is->second);
      reg_slice.erase(is);
    }
  }
  auto it = reg.find(w);
  if (it == reg.end()) return;
  cudaFree(it->second);  // synchronises the device: only at network destruction
  reg.erase(it);
}

bool conv_wide_launch(const float* x, int H, int W, int cin, float* y, int Ho, int Wo, int cout, int stride,
                      int transposed, const float* w, const float* bias, int softplus, const float* addend,
                      long long addend_bstride, int addend_per_model, const int* model_of, const float* residual,
                      const void* const* active, int B, cudaStream_t st, int planar) {
  if (!conv_wide_supported(cin, cout, stride, transposed, H, W, Wo)) return false;
  if (transposed && cin == 128 && cout == 128) {
    // two 64-channel output slices, each a 128 -> 64 transposed launch writing its half of every pixel
    if (planar) return false;
    CUtensorMap tm;
    if (!make_tmap(&tm, x, cin, H, W, B)) return false;
    for (int h = 0; h < 2; ++h) {
      const void* split = nullptr;
      {
        std::lock_guard<std::mutex> g(reg_mu);
        auto it = reg_slice.find({w, h});
        if (it != reg_slice.end()) split = it->second;
      }
      void* tmp = nullptr;
      if (!split) {
        if (cudaMallocAsync(&tmp, split_bytes(128, 64), st) != cudaSuccess) return false;
        if (run_split(w + h * kSlice128, 128, 64, tmp, st) != cudaSuccess) return false;
        split = tmp;
      }
      WArgs a{static_cast<const unsigned char*>(split), x, H, W, y, Ho, Wo, w + h * kSlice128, bias + 64 * h, softplus,
              addend, addend_bstride, addend_per_model, model_of, residual, active, B, 0, 128, 64 * h};
      launch_wide<128, 64, 2>(a, tm, st);
      if (tmp) cudaFreeAsync(tmp, st);
    }
    return true;
  }
  const void* split = nullptr;
  {
    std::lock_guard<std::mutex> g(reg_mu);
    auto it = reg.find(w);
    if (it != reg.end()) split = it->second;
  }
  void* tmp = nullptr;
  if (!split) {  // unregistered weights (hs_conv2d): a stream-ordered temporary split
    if (cudaMallocAsync(&tmp, split_bytes(cin, cout), st) != cudaSuccess) return false;
    if (run_split(w, cin, cout, tmp, st) != cudaSuccess) return false;
    split = tmp;
  }
  WArgs a{static_cast<const unsigned char*>(split), x, H, W, y, Ho, Wo, w, bias, softplus, addend, addend_bstride,
          addend_per_model, model_of, residual, active, B, planar, cout, 0};
  CUtensorMap tm;
  if (!make_tmap(&tm, x, cin, H, W, B)) {
    if (tmp) cudaFreeAsync(tmp, st);
    return false;
  }
  const int mode = transposed ? 2 : (stride == 2 ? 1 : 0);
  if (mode == 0 && cin == 64) launch_wide<64, 64, 0>(a, tm, st);
  else if (mode == 0 && cin == 128) launch_wide<128, 128, 0>(a, tm, st);
  else if (mode == 1 && cin == 64) launch_wide<64, 128, 1>(a, tm, st);
  else if (mode == 1 && cin == 128) launch_wide<128, 128, 1>(a, tm, st);
  else if (mode == 2 && cout == 64) launch_wide<128, 64, 2>(a, tm, st);
#if HS_WIDE_S2_32
  else if (mode == 1 && cin == 32) launch_wide<32, 64, 1>(a, tm, st);
#endif
#if HS_WIDE_EXTRA
  else if (mode == 2 && cout == 32) launch_wide<64, 32, 2>(a, tm, st);
#endif
  if (tmp) cudaFreeAsync(tmp, st);
  return true;
}

}  // namespace hs
