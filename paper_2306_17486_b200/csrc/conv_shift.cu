// 16 -> 16 stride-1 3x3 convolution (the level-0 residual blocks) on tcgen05 with the A operand in
// TMEM and the horizontal taps made by tcgen05.shift -- no im2col, no tap views, no staged copy.
//
// Replaces the A-in-TMEM variant of conv_tc.cu (Cfg::ATM) for this layer shape.  There the converters
// wrote every input row into TMEM three times (tap views kx = 0, 1, 2 of pixel m + kx, 72 columns),
// which needed a staged bf16x3 copy of the row in shared memory (store, group barrier, 18 16-byte
// loads per thread): 37 KB of the 93 KB of shared-memory traffic per 128-pixel tile, and the
// converter warps set the pace of the whole pipeline (ncu, profiles/r02_summary.md).
//
// Here a TMEM lane holds ONE pixel of an input row (three bf16 parts, 24 columns, written straight
// from the raw fp32 row), and the MMA warp moves the row sideways between taps:
//   tcgen05.shift.down moves a 32-byte column block one lane down inside every 32-lane quarter
//   (lane m <- lane m + 1; the last lane of a quarter keeps its value), and MMA / shift / MMA issued
//   by one thread run in issue order (tools/shift_probe.cu, measured on B200).
// A quarter of 32 lanes therefore serves 30 output pixels: lane j starts with input pixel P0 + j
// (tap kx = 0 of output pixel P0 + j + 1), holds P0 + j + 1 after one shift and P0 + j + 2 after two;
// lanes 30 and 31 end up stale and are never stored.  A tile is four such segments of one row (120
// output pixels, 122 input pixels).
//
// The schedule is input-row stationary: input row g (one TMEM slot) feeds output rows g + 1 (ky = 0),
// g (ky = 1) and g - 1 (ky = 2) while it is shifted twice, so three accumulators are open at a time and
// output row g - 1 is complete when row g retires.  TMEM: six 48-column accumulators ([W0|W1|W2]
// column groups, as in conv_tc.cu) + nine 24-column A slots.
//
// Warp roles (one persistent CTA per SM): warps 0-7 epilogue (two groups of four alternate output rows,
// one warp per lane quarter), warps 8-11 converters (one per lane quarter: raw fp32 pixel -> exact
// bf16x3 split -> tcgen05.st), warp 12 producer (one bulk copy per input row into a 12-deep raw ring),
// warp 13 MMA issuer.  Precision and results follow conv_tc.cu: six bf16 products per fp32 product,
// the three column groups summed in the epilogue, bias, softplus, addend / residual, NHWC stores as whole
// 64-byte pixels (group-of-four transpose).
// Reference: helmsolve.autodiff.conv2d (/root/reference/pkg/src/helmsolve/autodiff.py:472-507).
#include <cuda_bf16.h>

#include "common.cuh"
#include "conv_tc.h"
#include "prof.h"
#include "tc_util.cuh"

namespace hs {
namespace {
using namespace tc;

#ifndef HS_SH_BAND_MAX
#define HS_SH_BAND_MAX 32
#endif
#ifndef HS_SH_X
#define HS_SH_X 1  // 1: a raw slot is released after its row is in TMEM (see the converter); other bits: measurement builds
#endif
#ifndef HS_SH_NR
#define HS_SH_NR 12
#endif

// Stage-removal probes for a separate measurement build only (`make variant DEFS=-DHS_SH_PROBE=<mask>`): 1 no shifts,
// 2 no MMAs, 4 no split / TMEM writes, 8 no epilogue math and stores, 16 one accumulator for a row's three output rows,
// 32 no TMEM drain, 64 MMA-warp cycle counts into y[0..3] (waiting for A slots, issuing, rows, waiting for accumulators).  The product build compiles with 0.
#ifndef HS_SH_PROBE
#define HS_SH_PROBE 0
#endif
constexpr int kShProbe = HS_SH_PROBE;
constexpr int CIN = 16, COUT = 16;
constexpr int SEG = 30;                 // output pixels per lane quarter
constexpr int TPX = 4 * SEG;            // output pixels per tile
constexpr int RAWPX = TPX + 2;          // input pixels per raw row
constexpr int RAW_BYTES = RAWPX * CIN * 4;
constexpr int NW = 48, KC = 2;          // stacked weight rows [W0; W1; W2], 16-byte chunks per part
constexpr uint32_t WT = KC * NW;        // weight units (16 B) per tap
constexpr int W_BYTES = 9 * KC * NW * 16;
constexpr int NR = HS_SH_NR;            // raw ring depth (rows in flight per SM)
constexpr int NACC = 6, ACOLS = 48;     // TMEM accumulators
constexpr int AOFF = NACC * ACOLS;      // first A slot column
constexpr int SLOT_COLS = 24;           // three parts x 8 columns
constexpr int NSA = (512 - AOFF) / SLOT_COLS;
constexpr int kEpi = 8, kCvt0 = 8, kProd = 12, kMma = 13, NT = 32 * 14;
constexpr size_t SMEM = W_BYTES + (size_t)NR * RAW_BYTES + 8 * (2 * NR + 2 * NSA + 2 * NACC) + 16 + 4 * COUT;
static_assert(NSA >= 4, "A slots");
static_assert(RAW_BYTES % 128 == 0, "raw slots stay 128-byte aligned");

struct ShArgs {
  const float* x;
  int H, W;
  float* y;
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
  int band, ntile, nbands;
};

struct Unit {
  int b, t, oy0, oy1;
};

HS_DEV bool unit_at(const ShArgs& a, long long u, Unit& U) {
  U.t = (int)(u % a.ntile);
  const int band = (int)((u / a.ntile) % a.nbands);
  U.b = (int)(u / ((long long)a.ntile * a.nbands));
  U.oy0 = band * a.band;
  U.oy1 = min(a.H, U.oy0 + a.band);
  return !(a.active && a.active[U.b] == nullptr);
}

// All tcgen05 work of one input row: for kx = 0, 1, 2 the taps (ky, kx) into the accumulators of output
// rows g + 1 (ky 0, d0; its very first MMA overwrites), g (ky 1, d1) and g - 1 (ky 2, d2), each tap as
// parts a0 [W0|W1|W2] (N 48), a1 [W0|W1] (N 32), a2 [W0] (N 16); the A slot is shifted one lane down
// after kx = 0 and kx = 1.  One asm block, one elect: the issuing warp is the pipeline's pace-setter once
// the converters and the epilogue are out of the way (every instruction between two MMAs costs).
// E0 / E1 / E2: the predicates of the MMAs of output rows g + 1 / g / g - 1.
#define HS_SH_TAP(D, E, P0, WOFF)                                                   \
  "add.u32 bl, %4, " WOFF ";\n\tmov.b64 db, {bl, hi};\n\t"                         \
  "@" E " tcgen05.mma.cta_group::1.kind::f16 [" D "], [%3], db, i0, " P0 ";\n\t"    \
  "@" E " tcgen05.mma.cta_group::1.kind::f16 [" D "], [ta1], db, i1, pt;\n\t"       \
  "@" E " tcgen05.mma.cta_group::1.kind::f16 [" D "], [ta2], db, i2, pt;\n\t"
#define HS_SH_SHIFT                                                                 \
  "@es tcgen05.shift.cta_group::1.down [%3];\n\t"                                   \
  "@es tcgen05.shift.cta_group::1.down [ta1];\n\t"                                  \
  "@es tcgen05.shift.cta_group::1.down [ta2];\n\t"
#define HS_SH_KX(E0, E1, E2, P0, W0, W1, W2, SH) \
  HS_SH_TAP("%0", E0, P0, W0) HS_SH_TAP("%1", E1, "pt", W1) HS_SH_TAP("%2", E2, "pt", W2) SH
#define HS_SH_ROW(E0, E1, E2)                                                       \
  HS_SH_KX(E0, E1, E2, "pz", "%10", "%13", "%16", HS_SH_SHIFT)                      \
  HS_SH_KX(E0, E1, E2, "pt", "%11", "%14", "%17", HS_SH_SHIFT)                      \
  HS_SH_KX(E0, E1, E2, "pt", "%12", "%15", "%18", "")
#define HS_SH_OPERANDS                                                                                          \
  "r"(d0), "r"(d1), "r"(d2), "r"(abase), "r"(wlo), "r"(valid), "n"(kDescHi), "n"(I0), "n"(I1), "n"(I2), "n"(0 * WT), \
      "n"(1 * WT), "n"(2 * WT), "n"(3 * WT), "n"(4 * WT), "n"(5 * WT), "n"(6 * WT), "n"(7 * WT), "n"(8 * WT)
#define HS_SH_HEAD                                                                                              \
  "{\n\t.reg .pred e, es, e0, e1, e2, pz, pt;\n\t.reg .b64 db;\n\t.reg .b32 hi, i0, i1, i2, ta1, ta2, bl, m;\n\t" \
  "mov.b32 hi, %6;\n\tmov.b32 i0, %7;\n\tmov.b32 i1, %8;\n\tmov.b32 i2, %9;\n\t"                                  \
  "elect.sync _|e, 0xffffffff;\n\t"                                                                             \
  "setp.ne.b32 pz, %5, %5;\n\tsetp.eq.b32 pt, %5, %5;\n\t"                                                       \
  "add.u32 ta1, %3, 8;\n\tadd.u32 ta2, %3, 16;\n\t"

// interior rows: all three output rows lie inside the band.  The elected lane branches into an
// unpredicated block (predicated tcgen05 instructions made ptxas re-materialise the uniform operands of
// every MMA: two R2UR, a VOTEU and three UMOV each).
HS_DEV void row_mmas_all(uint32_t d0, uint32_t d1, uint32_t d2, uint32_t abase, uint32_t wlo) {
  constexpr uint32_t I0 = idesc_bf16(128, 48), I1 = idesc_bf16(128, 32), I2 = idesc_bf16(128, 16);
  const uint32_t valid = (kShProbe & 1) ? 0u : 1u;
  if (kShProbe & 2) return;
  asm volatile(HS_SH_HEAD
               "@!e bra SH_SKIP_%=;\n\t"
               "setp.ne.b32 es, %5, 0;\n\t" HS_SH_ROW("pt", "pt", "pt") "SH_SKIP_%=:\n\t}\n" ::HS_SH_OPERANDS
               : "memory");
  __syncwarp();
}

// band edges: valid bit 0 / 1 / 2 = output row g + 1 / g / g - 1 lies inside the band
HS_DEV void row_mmas_edge(uint32_t d0, uint32_t d1, uint32_t d2, uint32_t abase, uint32_t wlo, uint32_t valid) {
  constexpr uint32_t I0 = idesc_bf16(128, 48), I1 = idesc_bf16(128, 32), I2 = idesc_bf16(128, 16);
  if (kShProbe & 2) return;
  asm volatile(HS_SH_HEAD
               "and.b32 m, %5, 1;\n\tsetp.ne.b32 e0, m, 0;\n\tand.pred e0, e0, e;\n\t"
               "and.b32 m, %5, 2;\n\tsetp.ne.b32 e1, m, 0;\n\tand.pred e1, e1, e;\n\t"
               "and.b32 m, %5, 4;\n\tsetp.ne.b32 e2, m, 0;\n\tand.pred e2, e2, e;\n\t"
               "and.pred es, e, e;\n\t" HS_SH_ROW("e0", "e1", "e2") "}\n" ::HS_SH_OPERANDS
               : "memory");
}
#undef HS_SH_TAP
#undef HS_SH_SHIFT
#undef HS_SH_KX
#undef HS_SH_ROW
#undef HS_SH_OPERANDS
#undef HS_SH_HEAD

HS_DEV void tmem_st8(uint32_t taddr, const uint4& lo, const uint4& hi) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(lo.x),
               "r"(lo.y), "r"(lo.z), "r"(lo.w), "r"(hi.x), "r"(hi.y), "r"(hi.z), "r"(hi.w));
}

__global__ void __launch_bounds__(NT, 1) k_conv16_shift(ShArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* wst = smem;
  unsigned char* raw = smem + W_BYTES;
  uint64_t* raw_full = reinterpret_cast<uint64_t*>(raw + (size_t)NR * RAW_BYTES);
  uint64_t* raw_empty = raw_full + NR;
  uint64_t* a_full = raw_empty + NR;
  uint64_t* a_empty = a_full + NSA;
  uint64_t* acc_full = a_empty + NSA;
  uint64_t* acc_empty = acc_full + NACC;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(acc_empty + NACC);
  float* s_bias = reinterpret_cast<float*>(s_tmem + 4);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long nunits = (long long)a.B * a.ntile * a.nbands;

  // ---- setup: resident weight stack [W0; W1; W2], layout (tap, chunk, row) x 16 B (as conv_tc.cu)
  for (int e = tid; e < 9 * KC * COUT; e += NT) {
    const int n = e % COUT, c = (e / COUT) % KC, t = e / (COUT * KC);
    const float* src = a.w + ((size_t)n * 9 + t) * CIN + 8 * c;
    const float4 v0 = __ldg(reinterpret_cast<const float4*>(src)), v1 = __ldg(reinterpret_cast<const float4*>(src + 4));
    const float v[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
    uint4 p[3];
    split_bf16x3(v, p[0], p[1], p[2]);
#pragma unroll
    for (int part = 0; part < 3; ++part)
      *reinterpret_cast<uint4*>(wst + ((size_t)(t * KC + c) * NW + part * COUT + n) * 16) = p[part];
  }
  if (tid < COUT) s_bias[tid] = a.bias[tid];
  if (tid == 0) {
    for (int i = 0; i < NR; ++i) {
      mbar_init(smem_u32(&raw_full[i]), 1);
      mbar_init(smem_u32(&raw_empty[i]), 4);  // one arrival per converter warp
    }
    for (int i = 0; i < NSA; ++i) {
      mbar_init(smem_u32(&a_full[i]), 4);
      mbar_init(smem_u32(&a_empty[i]), 1);
    }
    for (int i = 0; i < NACC; ++i) {
      mbar_init(smem_u32(&acc_full[i]), 1);
      mbar_init(smem_u32(&acc_empty[i]), 4);  // the four warps of the draining group
    }
    fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s_tmem)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;
  // programmatic dependent launch, as conv_tc.cu: nothing above touches the previous kernel's data
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");

  if (warp == kProd) {
    // ================= producer: one bulk copy per input row (122 pixels x 64 B, clipped to the image)
    if (lane == 0) {
      uint32_t seq = 0;
      for (long long u = blockIdx.x; u < nunits; u += gridDim.x) {
        Unit U;
        if (!unit_at(a, u, U)) continue;
        const int x0 = TPX * U.t - 1;
        const int clo = max(x0, 0), chi = min(x0 + RAWPX, a.W);
        const float* img = a.x + (size_t)U.b * a.H * a.W * CIN;
        for (int g = U.oy0 - 1; g <= U.oy1; ++g, ++seq) {
          const uint32_t s = seq % NR, use = seq / NR;
          if (use > 0) mbar_wait(smem_u32(&raw_empty[s]), (use - 1) & 1);
          const uint32_t bar = smem_u32(&raw_full[s]);
          if (g >= 0 && g < a.H && chi > clo) {
            const uint32_t bytes = (uint32_t)(chi - clo) * CIN * 4;
            mbar_arrive_tx(bar, bytes);
            bulk_g2s(smem_u32(raw + (size_t)s * RAW_BYTES + (size_t)(clo - x0) * CIN * 4),
                     img + ((size_t)g * a.W + clo) * CIN, bytes, bar);
          } else {
            mbar_arrive(bar);
          }
        }
      }
    }
  } else if (warp >= kCvt0 && warp < kCvt0 + 4) {
    // ================= converters: warp q owns TMEM lane quarter q; lane j holds input pixel x0 + 30 q + j
    const int q = warp - kCvt0;
    uint32_t seq = 0;
    for (long long u = blockIdx.x; u < nunits; u += gridDim.x) {
      Unit U;
      if (!unit_at(a, u, U)) continue;
      const int prel = SEG * q + lane;              // pixel within the raw row
      const int xin = TPX * U.t - 1 + prel;
      const bool xok = xin >= 0 && xin < a.W;
      for (int g = U.oy0 - 1; g <= U.oy1; ++g, ++seq) {
        const uint32_t s = seq % NR;
        mbar_wait(smem_u32(&raw_full[s]), (seq / NR) & 1);
        float4 v[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) v[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (xok && g >= 0 && g < a.H) {
          const float4* src = reinterpret_cast<const float4*>(raw + (size_t)s * RAW_BYTES + (size_t)prel * CIN * 4);
#pragma unroll
          for (int i = 0; i < 4; ++i) v[i] = src[i];
        }
        uint4 lo[3] = {}, hi[3] = {};
        if (!(kShProbe & 4)) {
          const float f0[8] = {v[0].x, v[0].y, v[0].z, v[0].w, v[1].x, v[1].y, v[1].z, v[1].w};
          const float f1[8] = {v[2].x, v[2].y, v[2].z, v[2].w, v[3].x, v[3].y, v[3].z, v[3].w};
          split_bf16x3(f0, lo[0], lo[1], lo[2]);
          split_bf16x3(f1, hi[0], hi[1], hi[2]);
        }
#if !(HS_SH_X & 1)
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&raw_empty[s]));
#endif
        const uint32_t as = seq % NSA, ause = seq / NSA;
        if (ause > 0) mbar_wait(smem_u32(&a_empty[as]), (ause - 1) & 1);
        tc_fence_after();
        const uint32_t tcol = tmem + ((uint32_t)(32 * q) << 16) + AOFF + as * SLOT_COLS;
#pragma unroll
        for (int part = 0; part < 3; ++part)
          if (!(kShProbe & 4)) tmem_st8(tcol + 8 * part, lo[part], hi[part]);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&a_full[as]));
#if HS_SH_X & 1
        fence_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&raw_empty[s]));
#endif
      }
    }
  } else if (warp == kMma) {
    // ================= MMA issuer: input-row stationary, two shifts per row.  The whole warp walks the
    // schedule with warp-uniform incremental bookkeeping (no divisions); one asm block per input row
    // issues its 27 MMAs and 6 shifts from the elected lane.
    const uint32_t wlo = desc_lo(smem_u32(wst), NW * 16);
    const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
    uint32_t as = 0, a_par = 0;        // A slot of the next input row and the parity of its a_full phase
    uint32_t s_next = 0, epoch = 0;    // accumulator slot of the next output row to open, completed wraps
    long long dbg_wait = 0, dbg_wait2 = 0, dbg_issue = 0, dbg_rows = 0;  // kShProbe & 64: cycles per row waiting / issuing
    for (long long u = blockIdx.x; u < nunits; u += gridDim.x) {
      Unit U;
      if (!unit_at(a, u, U)) continue;
      uint32_t s_new = 0, s_cur = 0, s_old = 0;
      for (int g = U.oy0 - 1; g <= U.oy1; ++g) {
        const long long tq0 = (kShProbe & 64) ? clock64() : 0;
        mbar_wait(smem_u32(&a_full[as]), a_par);
        const bool v_new = g + 1 < U.oy1, v_cur = g >= U.oy0 && g < U.oy1, v_old = g - 1 >= U.oy0;
        s_old = s_cur;
        s_cur = s_new;
        const long long tq01 = (kShProbe & 64) ? clock64() : 0;
        if (v_new) {  // output row g + 1 opens its accumulator: the previous user must have drained it
          s_new = s_next;
          if (epoch > 0) mbar_wait(smem_u32(&acc_empty[s_new]), (epoch - 1) & 1);
          if (++s_next == (uint32_t)NACC) {
            s_next = 0;
            ++epoch;
          }
        }
        tc_fence_after();
        const long long tq1 = (kShProbe & 64) ? clock64() : 0;
        const uint32_t abase = tm + AOFF + as * SLOT_COLS;
        if ((kShProbe & 16) && v_new && v_cur && v_old)  // timing probe: one accumulator for all three output rows
          row_mmas_all(tm + s_new * ACOLS, tm + s_new * ACOLS, tm + s_new * ACOLS, abase, wlo);
        else if (v_new && v_cur && v_old)
          row_mmas_all(tm + s_new * ACOLS, tm + s_cur * ACOLS, tm + s_old * ACOLS, abase, wlo);
        else
          row_mmas_edge(tm + s_new * ACOLS, tm + s_cur * ACOLS, tm + s_old * ACOLS, abase, wlo,
                        (v_new ? 1u : 0u) | (v_cur ? 2u : 0u) | (v_old ? 4u : 0u));
        mma_commit(smem_u32(&a_empty[as]));
        if (v_old) mma_commit(smem_u32(&acc_full[s_old]));
        if (++as == (uint32_t)NSA) {
          as = 0;
          a_par ^= 1;
        }
        if (kShProbe & 64) {
          const long long tq2 = clock64();
          dbg_wait += tq01 - tq0;
          dbg_wait2 += tq1 - tq01;
          dbg_issue += tq2 - tq1;
          ++dbg_rows;
        }
      }
    }
    if ((kShProbe & 64) && blockIdx.x == 0 && lane == 0) {
      a.y[0] = (float)dbg_wait / (float)dbg_rows;
      a.y[1] = (float)dbg_issue / (float)dbg_rows;
      a.y[2] = (float)dbg_rows;
      a.y[3] = (float)dbg_wait2 / (float)dbg_rows;
    }
  } else {
    // ================= epilogue: group hg drains the output rows with tile % 2 == hg; warp q4 its lane quarter
    const int q4 = warp & 3, hg = warp >> 2;
    const int gi = lane & 3, gb = lane & ~3;
    uint32_t tile = 0;
    for (long long u = blockIdx.x; u < nunits; u += gridDim.x) {
      Unit U;
      if (!unit_at(a, u, U)) continue;
      const float* add = a.addend ? a.addend + (a.addend_per_model ? (a.model_of ? a.model_of[U.b] : 0) : U.b) *
                                                   a.addend_bstride
                                  : nullptr;
      const float* res = a.residual ? a.residual + (size_t)U.b * a.H * a.W * COUT : nullptr;
      float* yimg = a.y + (size_t)U.b * a.H * a.W * COUT;
      const int xg0 = SEG * (4 * U.t + q4) + gb;  // output pixel of this lane group's first lane
      bool ok[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) ok[j] = gb + j < SEG && xg0 + j < a.W;
      // side inputs (addend, residual) in the post-transpose layout (chunk gi of the group's four pixels).
      // A row's side inputs are requested as soon as the group's previous row has used its own (two output
      // rows ahead) and are only touched at the store, so their DRAM latency runs under the next accumulator
      // wait, drain and softplus.  (Requested right before the accumulator wait, their first use held 28% of
      // all stall samples in ncu; summing addend and residual at load time stalls on the loads just the same.)
      float4 sa[4], sr[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) sa[j] = sr[j] = make_float4(0.f, 0.f, 0.f, 0.f);
      auto issue_side = [&](int oy) {
        const size_t gp = (size_t)oy * a.W + xg0;
        if (add) {
          const float4* ap = reinterpret_cast<const float4*>(add + gp * COUT);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (ok[j]) sa[j] = __ldg(ap + j * 4 + gi);
        }
        if (res) {
          const float4* rp = reinterpret_cast<const float4*>(res + gp * COUT);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (ok[j]) sr[j] = __ldg(rp + j * 4 + gi);
        }
      };
      {
        const int first = U.oy0 + (int)((tile ^ (uint32_t)hg) & 1);  // this group's first row of the unit
        if (first < U.oy1) issue_side(first);
      }
      for (int oy = U.oy0; oy < U.oy1; ++oy, ++tile) {
        if ((int)(tile & 1) != hg) continue;
        const uint32_t acc = tile % NACC;
        const size_t gpix = (size_t)oy * a.W + xg0;
        mbar_wait(smem_u32(&acc_full[acc]), (tile / NACC) & 1);
        tc_fence_after();
        float o[16] = {};
#pragma unroll
        for (int n0 = 0; n0 < 16; n0 += 8) {
          if (kShProbe & 32) break;
          uint32_t r0[8], r1[8], r2[8];
          const uint32_t col = tmem + ((uint32_t)(q4 * 32) << 16) + acc * ACOLS + n0;
          tmem_ld8(col, r0);
          tmem_ld8(col + COUT, r1);
          tmem_ld8(col + 2 * COUT, r2);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 8; j += 2) {  // (x0 + x1) + x2 partial sums, channel pairs packed (FADD2)
            const uint64_t sm = add2(add2(pk2(r0[j], r0[j + 1]), pk2(r1[j], r1[j + 1])), pk2(r2[j], r2[j + 1]));
            o[n0 + j] = __uint_as_float((uint32_t)sm);
            o[n0 + j + 1] = __uint_as_float((uint32_t)(sm >> 32));
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&acc_empty[acc]));  // TMEM free; finish from registers
        if (kShProbe & 8) {
          if (oy + 2 < U.oy1) issue_side(oy + 2);
          continue;
        }
        float4 ch[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4 bs = *reinterpret_cast<const float4*>(s_bias + 4 * q);
          const uint64_t o01 = add2(pkf(o[4 * q], o[4 * q + 1]), pkf(bs.x, bs.y));
          const uint64_t o23 = add2(pkf(o[4 * q + 2], o[4 * q + 3]), pkf(bs.z, bs.w));
          float4 v = make_float4(lo_f(o01), hi_f(o01), lo_f(o23), hi_f(o23));
          if (a.softplus) {
            v.x = softplus_fast(v.x);
            v.y = softplus_fast(v.y);
            v.z = softplus_fast(v.z);
            v.w = softplus_fast(v.w);
          }
          ch[q] = v;
        }
        group4_transpose(ch, gi);  // lane gi: chunk gi of the group's four pixels
        float4* yb = reinterpret_cast<float4*>(yimg + gpix * COUT);
#pragma unroll
        for (int j = 0; j < 4; ++j) {  // o + (addend + residual), as conv_tc.cu
          const uint64_t s01 = add2(pkf(sa[j].x, sa[j].y), pkf(sr[j].x, sr[j].y));
          const uint64_t s23 = add2(pkf(sa[j].z, sa[j].w), pkf(sr[j].z, sr[j].w));
          const uint64_t q01 = add2(pkf(ch[j].x, ch[j].y), s01), q23 = add2(pkf(ch[j].z, ch[j].w), s23);
          if (ok[j]) yb[j * 4 + gi] = make_float4(lo_f(q01), hi_f(q01), lo_f(q23), hi_f(q23));
        }
        if (oy + 2 < U.oy1) issue_side(oy + 2);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

}  // namespace

bool conv_shift_launch(const float* x, int H, int W, float* y, const float* w, const float* bias, int softplus,
                       const float* addend, long long addend_bstride, int addend_per_model, const int* model_of,
                       const float* residual, const void* const* active, int B, cudaStream_t st) {
  static int sms = 0;
  if (!sms) {
    cudaFuncSetAttribute(k_conv16_shift, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  ShArgs a{x, H, W, y, w, bias, softplus, addend, addend_bstride, addend_per_model, model_of, residual, active, B,
           HS_SH_BAND_MAX, (W + TPX - 1) / TPX, 0};
  // band height as conv_tc.cu: halve it until the RHS still iterating give every CTA >= 6 units
  const double act = prof::active_hint(B);
  long long grid = sms;
  while (a.band > 8 && act * a.ntile * ((H + a.band - 1) / a.band) < 6.0 * grid) a.band /= 2;
  a.nbands = (H + a.band - 1) / a.band;
  const long long nunits = (long long)B * a.ntile * a.nbands;
  if (nunits < grid) grid = nunits;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_conv16_shift, a) == cudaSuccess;
}

}  // namespace hs
