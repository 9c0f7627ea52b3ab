// 16 -> 16 and 32 -> 32 stride-1 3x3 convolutions (the level-0 and level-1 residual blocks) on tcgen05 with the A operand in
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
// lanes 30 and 31 end up stale and are never stored.  A tile is four such segments, taken in order from
// the segments of a group of 1, 2 or 4 bands of rows (so few lane quarters stay empty whatever the width);
// its quarters walk their bands' rows in lockstep.
//
// The schedule is input-row stationary: input row g (one TMEM slot) feeds output rows g + 1 (ky = 0),
// g (ky = 1) and g - 1 (ky = 2) while it is shifted twice, so three accumulators are open at a time and
// output row g - 1 is complete when row g retires.  TMEM: six 48-column accumulators ([W0|W1|W2]
// column groups, as in conv_tc.cu) + nine 24-column A slots.
//
// Warp roles (one persistent CTA per SM): warps 0-7 epilogue (two groups of four alternate output rows,
// one warp per lane quarter), warps 8-11 converters (one per lane quarter: raw fp32 pixel -> exact
// bf16x3 split -> tcgen05.st), warp 12 producer (per input row one bulk copy per lane quarter into a 12-deep raw ring),
// warp 13 MMA issuer.  Precision and results follow conv_tc.cu: six bf16 products per fp32 product,
// the three column groups summed in the epilogue, bias, softplus, addend / residual, NHWC stores as whole
// 64-byte pixels (group-of-four transpose).
// 32 channels (template C = 32): a slot is 48 columns (three parts x two K steps), an accumulator 96, so TMEM
// holds four accumulators and two A slots (the converters keep the next row split in registers while they
// wait for a slot); the two epilogue groups take the two 16-channel halves of every output row instead of
// alternate rows; the converters read their 128-byte pixels in rotated order (no bank conflicts).  With A in
// shared memory this layer was bound by the MMAs' operand reads (36 KB per tile and tap).
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
#ifndef HS_SH_ROT
#define HS_SH_ROT 0  // 16 channels: converters read their pixel's four 16-byte pieces in rotated order (measured equal)
#endif
#ifndef HS_SH_FRAG
#define HS_SH_FRAG 0  // stride-1 epilogue drains TMEM as 16x256b fragments (no transposes; 8-byte stores, full sectors): measured equal, in isolation and in the network
#endif
#ifndef HS_SH_NOROT
#define HS_SH_NOROT 0  // 1: plain piece order in the 128-byte-pixel converters (8-way bank conflicts, no select stages)
#endif
#ifndef HS_SH_NR
#define HS_SH_NR 12
#endif

// Stage-removal probes for a separate measurement build only (`make variant DEFS=-DHS_SH_PROBE=<mask>`): 1 no shifts,
// 2 no MMAs, 4 no split / TMEM writes, 8 no epilogue math and stores, 32 no TMEM drain, 64 MMA-warp cycle counts into
// y[0..3] (waiting for A slots, issuing, rows, waiting for accumulators).  The product build compiles with 0.
#ifndef HS_SH_PROBE
#define HS_SH_PROBE 0
#endif
constexpr int kShProbe = HS_SH_PROBE;
constexpr int SEG = 30;                 // output pixels per lane quarter
constexpr int RAWPX = 128;              // input pixels per raw row: 32 per lane quarter (30 + the two halo columns)
constexpr int kCvt0 = 8, kProd = 12, kMma = 13, NT = 32 * 14;

template <int C>
struct Cfg {
  static constexpr int KC = C / 8;                 // 16-byte chunks per part
  static constexpr int KSTEPS = C / 16;            // MMA K steps per tap
  static constexpr int NW = 3 * C;                 // stacked weight rows [W0; W1; W2]
  static constexpr uint32_t WT = KC * NW;          // weight units (16 B) per tap
  static constexpr int W_BYTES = 9 * KC * NW * 16;
  static constexpr int RAW_BYTES = RAWPX * C * 4;
  static constexpr int NR = C == 16 ? HS_SH_NR : 8;        // raw ring depth (rows in flight per SM)
  static constexpr int NACC = C == 16 ? 6 : 4, ACOLS = 3 * C;  // TMEM accumulators
  static constexpr int AOFF = NACC * ACOLS;        // first A slot column
  static constexpr int SLOT_COLS = 3 * (C / 2);    // three parts x C bf16
  static constexpr int NSA = (512 - AOFF) / SLOT_COLS;
  static constexpr bool HALVES = C == 32;          // epilogue groups: channel halves of every row (else alternate rows)
  static constexpr size_t SMEM = W_BYTES + (size_t)NR * RAW_BYTES + 8 * (2 * NR + 2 * NSA + 2 * NACC) + 16 + 4 * C;
  static_assert(NSA >= 2, "A slots");
  static_assert(RAW_BYTES % 128 == 0, "raw slots stay 128-byte aligned");
  static_assert(SMEM <= 232448, "shared memory budget");
};

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
  int Ho, Wo;  // output size (stride 1: H, W)
  int rows;    // the banded dimension: output rows, or input rows for the transposed kernel
  // Work units.  A row of the image is nseg segments of 30 output pixels; a unit is one tile (four segments, one per
  // lane quarter) of a group of nb bands of one image, the group's nb * nseg segments taken in order.  The four
  // quarters of a tile may therefore sit in different bands; they walk their bands' rows in lockstep.  nb is
  // chosen by the launcher so that few quarters stay empty (W = 512: 18 segments per row, nb = 2 fills 9 tiles).
  int band, nseg, nb, ntile, ngroups;
};

struct Unit {
  int b, t, grp, bh;  // image, tile of the band group, band group, rows per band
};

HS_DEV bool unit_at(const ShArgs& a, long long u, Unit& U) {
  U.t = (int)(u % a.ntile);
  U.grp = (int)((u / a.ntile) % a.ngroups);
  U.b = (int)(u / ((long long)a.ntile * a.ngroups));
  U.bh = min(a.rows - U.grp * a.nb * a.band, a.band);  // nb > 1 only when the band height divides the row count
  return !(a.active && a.active[U.b] == nullptr);
}

// lane quarter q of unit U: first output row and segment, or false if the quarter is empty
HS_DEV bool quarter_at(const ShArgs& a, const Unit& U, int q, int& oy0, int& seg) {
  const int s = 4 * U.t + q;
  const int bl = s / a.nseg;
  seg = s - bl * a.nseg;
  oy0 = (U.grp * a.nb + bl) * a.band;
  return s < a.nb * a.nseg;
}

// All tcgen05 work of one input row: for kx = 0, 1, 2 the taps (ky, kx) into the accumulators of output
// rows g + 1 (ky 0, d0; its very first MMA overwrites), g (ky 1, d1) and g - 1 (ky 2, d2), each tap and K
// step as parts a0 [W0|W1|W2] (N 3C), a1 [W0|W1] (N 2C), a2 [W0] (N C); the A slot is shifted one lane down
// after kx = 0 and kx = 1.  One asm block, one elect: the issuing warp is the pipeline's pace-setter once
// the converters and the epilogue are out of the way (every instruction between two MMAs costs).
// E0 / E1 / E2: the predicates of the MMAs of output rows g + 1 / g / g - 1.  A slot columns: part p, K step
// k at 8 (KSTEPS p + k), registers %3, ta1 .. ta5.
#define HS_SH_MMA3(D, E, P0, A0, A1, A2)                                            \
  "@" E " tcgen05.mma.cta_group::1.kind::f16 [" D "], [" A0 "], db, i0, " P0 ";\n\t" \
  "@" E " tcgen05.mma.cta_group::1.kind::f16 [" D "], [" A1 "], db, i1, pt;\n\t"     \
  "@" E " tcgen05.mma.cta_group::1.kind::f16 [" D "], [" A2 "], db, i2, pt;\n\t"
#define HS_SH_TAP16(D, E, P0, WOFF) \
  "add.u32 bl, %4, " WOFF ";\n\tmov.b64 db, {bl, hi};\n\t" HS_SH_MMA3(D, E, P0, "%3", "ta1", "ta2")
#define HS_SH_TAP32(D, E, P0, WOFF)                                                                   \
  "add.u32 bl, %4, " WOFF ";\n\tmov.b64 db, {bl, hi};\n\t" HS_SH_MMA3(D, E, P0, "%3", "ta2", "ta4")  \
  "add.u32 bl, bl, %19;\n\tmov.b64 db, {bl, hi};\n\t" HS_SH_MMA3(D, E, "pt", "ta1", "ta3", "ta5")
#define HS_SH_S(A) "@es tcgen05.shift.cta_group::1.down [" A "];\n\t"
#define HS_SH_SHIFT16 HS_SH_S("%3") HS_SH_S("ta1") HS_SH_S("ta2")
#define HS_SH_SHIFT32 HS_SH_S("%3") HS_SH_S("ta1") HS_SH_S("ta2") HS_SH_S("ta3") HS_SH_S("ta4") HS_SH_S("ta5")
#define HS_SH_KX(TAP, E0, E1, E2, P0, W0, W1, W2, SH) TAP("%0", E0, P0, W0) TAP("%1", E1, "pt", W1) TAP("%2", E2, "pt", W2) SH
#define HS_SH_ROW(TAP, SH, E0, E1, E2)                                              \
  HS_SH_KX(TAP, E0, E1, E2, "pz", "%10", "%13", "%16", SH)                          \
  HS_SH_KX(TAP, E0, E1, E2, "pt", "%11", "%14", "%17", SH)                          \
  HS_SH_KX(TAP, E0, E1, E2, "pt", "%12", "%15", "%18", "")
#define HS_SH_OPERANDS                                                                                          \
  "r"(d0), "r"(d1), "r"(d2), "r"(abase), "r"(wlo), "r"(valid), "n"(kDescHi), "n"(I0), "n"(I1), "n"(I2), "n"(0 * WT), \
      "n"(1 * WT), "n"(2 * WT), "n"(3 * WT), "n"(4 * WT), "n"(5 * WT), "n"(6 * WT), "n"(7 * WT), "n"(8 * WT), "n"(KK)
#define HS_SH_HEAD                                                                                              \
  "{\n\t.reg .pred e, es, e0, e1, e2, pz, pt;\n\t.reg .b64 db;\n\t.reg .b32 hi, i0, i1, i2, ta1, ta2, ta3, ta4, ta5, bl, m;\n\t" \
  "mov.b32 hi, %6;\n\tmov.b32 i0, %7;\n\tmov.b32 i1, %8;\n\tmov.b32 i2, %9;\n\t"                                  \
  "elect.sync _|e, 0xffffffff;\n\t"                                                                             \
  "setp.ne.b32 pz, %5, %5;\n\tsetp.eq.b32 pt, %5, %5;\n\t"                                                       \
  "add.u32 ta1, %3, 8;\n\tadd.u32 ta2, %3, 16;\n\tadd.u32 ta3, %3, 24;\n\tadd.u32 ta4, %3, 32;\n\tadd.u32 ta5, %3, 40;\n\t"

// interior rows: all three output rows lie inside the band.  The elected lane branches into an
// unpredicated block (predicated tcgen05 instructions made ptxas re-materialise the uniform operands of
// every MMA: two R2UR, a VOTEU and three UMOV each).
template <int C>
HS_DEV void row_mmas_all(uint32_t d0, uint32_t d1, uint32_t d2, uint32_t abase, uint32_t wlo) {
  constexpr uint32_t I0 = idesc_bf16(128, 3 * C), I1 = idesc_bf16(128, 2 * C), I2 = idesc_bf16(128, C);
  constexpr uint32_t WT = Cfg<C>::WT, KK = 2 * Cfg<C>::NW;  // KK: weight units between K steps (two chunks)
  const uint32_t valid = (kShProbe & 1) ? 0u : 1u;
  if (kShProbe & 2) return;
  if constexpr (C == 16)
    asm volatile(HS_SH_HEAD "@!e bra SH_SKIP_%=;\n\tsetp.ne.b32 es, %5, 0;\n\t"
                 HS_SH_ROW(HS_SH_TAP16, HS_SH_SHIFT16, "pt", "pt", "pt") "SH_SKIP_%=:\n\t}\n" ::HS_SH_OPERANDS
                 : "memory");
  else
    asm volatile(HS_SH_HEAD "@!e bra SH_SKIP_%=;\n\tsetp.ne.b32 es, %5, 0;\n\t"
                 HS_SH_ROW(HS_SH_TAP32, HS_SH_SHIFT32, "pt", "pt", "pt") "SH_SKIP_%=:\n\t}\n" ::HS_SH_OPERANDS
                 : "memory");
  __syncwarp();
}

// band edges: valid bit 0 / 1 / 2 = output row g + 1 / g / g - 1 lies inside the band
// (the elected lane branches in, as in row_mmas_all; the row predicates come from `valid` alone, so they are
// warp-uniform and cost no per-MMA operand re-materialisation)
#define HS_SH_EDGE_PREDS                                                              \
  "@!e bra SH_SKIPE_%=;\n\t"                                                           \
  "and.b32 m, %5, 1;\n\tsetp.ne.b32 e0, m, 0;\n\t"                                     \
  "and.b32 m, %5, 2;\n\tsetp.ne.b32 e1, m, 0;\n\t"                                     \
  "and.b32 m, %5, 4;\n\tsetp.ne.b32 e2, m, 0;\n\t"                                     \
  "setp.eq.b32 es, %5, %5;\n\t"
template <int C>
HS_DEV void row_mmas_edge(uint32_t d0, uint32_t d1, uint32_t d2, uint32_t abase, uint32_t wlo, uint32_t valid) {
  constexpr uint32_t I0 = idesc_bf16(128, 3 * C), I1 = idesc_bf16(128, 2 * C), I2 = idesc_bf16(128, C);
  constexpr uint32_t WT = Cfg<C>::WT, KK = 2 * Cfg<C>::NW;
  if (kShProbe & 2) return;
  if constexpr (C == 16)
    asm volatile(HS_SH_HEAD HS_SH_EDGE_PREDS HS_SH_ROW(HS_SH_TAP16, HS_SH_SHIFT16, "e0", "e1", "e2") "SH_SKIPE_%=:\n\t}\n" ::HS_SH_OPERANDS
                 : "memory");
  else
    asm volatile(HS_SH_HEAD HS_SH_EDGE_PREDS HS_SH_ROW(HS_SH_TAP32, HS_SH_SHIFT32, "e0", "e1", "e2") "SH_SKIPE_%=:\n\t}\n" ::HS_SH_OPERANDS
                 : "memory");
  __syncwarp();
}
#undef HS_SH_MMA3
#undef HS_SH_TAP16
#undef HS_SH_TAP32
#undef HS_SH_S
#undef HS_SH_SHIFT16
#undef HS_SH_SHIFT32
#undef HS_SH_KX
#undef HS_SH_ROW
#undef HS_SH_OPERANDS
#undef HS_SH_HEAD
#undef HS_SH_EDGE_PREDS

HS_DEV void tmem_st8(uint32_t taddr, const uint4& lo, const uint4& hi) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(lo.x),
               "r"(lo.y), "r"(lo.z), "r"(lo.w), "r"(hi.x), "r"(hi.y), "r"(hi.z), "r"(hi.w));
}

// tcgen05.ld 16x256b.x2: 16 TMEM lanes x 16 columns as an MMA-style fragment.  Measured (tools/ld_probe.cu): register
// j of lane l holds TMEM lane (lane base) + l / 4 + 8 ((j / 2) % 2), column (column base) + 8 (j / 4) + 2 (l % 4) + j % 2.
HS_DEV void tmem_ld_frag16(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}

template <int C>
__global__ void __launch_bounds__(NT, 1) k_conv_shift(ShArgs a) {
  using F = Cfg<C>;
  constexpr int KC = F::KC, NW = F::NW, NR = F::NR, NACC = F::NACC, NSA = F::NSA, ACOLS = F::ACOLS;
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* wst = smem;
  unsigned char* raw = smem + F::W_BYTES;
  uint64_t* raw_full = reinterpret_cast<uint64_t*>(raw + (size_t)NR * F::RAW_BYTES);
  uint64_t* raw_empty = raw_full + NR;
  uint64_t* a_full = raw_empty + NR;
  uint64_t* a_empty = a_full + NSA;
  uint64_t* acc_full = a_empty + NSA;
  uint64_t* acc_empty = acc_full + NACC;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(acc_empty + NACC);
  float* s_bias = reinterpret_cast<float*>(s_tmem + 4);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long nunits = (long long)a.B * a.ntile * a.ngroups;

  // ---- setup: resident weight stack [W0; W1; W2], layout (tap, chunk, row) x 16 B (as conv_tc.cu)
  for (int e = tid; e < 9 * KC * C; e += NT) {
    const int n = e % C, c = (e / C) % KC, t = e / (C * KC);
    const float* src = a.w + ((size_t)n * 9 + t) * C + 8 * c;
    const float4 v0 = __ldg(reinterpret_cast<const float4*>(src)), v1 = __ldg(reinterpret_cast<const float4*>(src + 4));
    const float v[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
    uint4 p[3];
    split_bf16x3(v, p[0], p[1], p[2]);
#pragma unroll
    for (int part = 0; part < 3; ++part)
      *reinterpret_cast<uint4*>(wst + ((size_t)(t * KC + c) * NW + part * C + n) * 16) = p[part];
  }
  if (tid < C) s_bias[tid] = a.bias[tid];
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
      mbar_init(smem_u32(&acc_empty[i]), F::HALVES ? 8 : 4);  // the warps that drain one output row
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
    // ================= producer: per input row one bulk copy per lane quarter (32 pixels, clipped to the image)
    if (lane == 0) {
      uint32_t seq = 0;
      for (long long u = blockIdx.x; u < nunits; u += gridDim.x) {
        Unit U;
        if (!unit_at(a, u, U)) continue;
        const float* img = a.x + (size_t)U.b * a.H * a.W * C;
        int qy0[4], qx0[4];
        bool qv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          int seg;
          qv[q] = quarter_at(a, U, q, qy0[q], seg);
          qx0[q] = SEG * seg - 1;
        }
        for (int i = -1; i <= U.bh; ++i, ++seq) {
          const uint32_t s = seq % NR, use = seq / NR;
          if (use > 0) mbar_wait(smem_u32(&raw_empty[s]), (use - 1) & 1);
          const uint32_t bar = smem_u32(&raw_full[s]);
          uint32_t total = 0;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int g = qy0[q] + i, clo = max(qx0[q], 0), chi = min(qx0[q] + 32, a.W);
            if (qv[q] && g >= 0 && g < a.H && chi > clo) total += (uint32_t)(chi - clo) * C * 4;
          }
          if (total) {
            mbar_arrive_tx(bar, total);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int g = qy0[q] + i, clo = max(qx0[q], 0), chi = min(qx0[q] + 32, a.W);
              if (qv[q] && g >= 0 && g < a.H && chi > clo)
                bulk_g2s(smem_u32(raw + (size_t)s * F::RAW_BYTES + (size_t)(32 * q + clo - qx0[q]) * C * 4),
                         img + ((size_t)g * a.W + clo) * C, (uint32_t)(chi - clo) * C * 4, bar);
            }
          } else {
            mbar_arrive(bar);
          }
        }
      }
    }
  } else if (warp >= kCvt0 && warp < kCvt0 + 4) {
    // ================= converters: warp q owns TMEM lane quarter q; lane j holds input pixel 30 seg - 1 + j of its segment
    const int q = warp - kCvt0;
    uint32_t seq = 0;
    for (long long u = blockIdx.x; u < nunits; u += gridDim.x) {
      Unit U;
      if (!unit_at(a, u, U)) continue;
      const int prel = 32 * q + lane;               // pixel within the raw row
      int qy0, seg;
      const bool qv = quarter_at(a, U, q, qy0, seg);
      const int xin = SEG * seg - 1 + lane;
      const bool xok = qv && xin >= 0 && xin < a.W;
      for (int i = -1; i <= U.bh; ++i, ++seq) {
        const int g = qy0 + i;
        const uint32_t s = seq % NR;
        mbar_wait(smem_u32(&raw_full[s]), (seq / NR) & 1);
        constexpr int NP = C / 4;  // 16-byte pieces of a pixel
        float4 v[NP];
#pragma unroll
        for (int i = 0; i < NP; ++i) v[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (xok && g >= 0 && g < a.H) {
          const float4* src = reinterpret_cast<const float4*>(raw + (size_t)s * F::RAW_BYTES + (size_t)prel * C * 4);
          if constexpr (C == 32 || HS_SH_ROT) {
            // a lane's pixel is 4 C bytes, so eight lanes reading piece i of their pixels would hit one or two
            // bank groups; lane L reads its pieces rotated by r instead -- eight distinct bank groups per
            // wavefront -- and rotates them back in registers (log2(NP) select stages)
            const int r = HS_SH_NOROT ? 0 : (C == 32 ? (lane & 7) : ((lane >> 1) & 3));
            float4 w4[NP];
#pragma unroll
            for (int i = 0; i < NP; ++i) w4[i] = src[(i + r) & (NP - 1)];
#pragma unroll
            for (int st = 1; st < NP; st <<= 1) {
              float4 t4[NP];
#pragma unroll
              for (int i = 0; i < NP; ++i) t4[i] = (r & st) ? w4[(i + NP - st) & (NP - 1)] : w4[i];
#pragma unroll
              for (int i = 0; i < NP; ++i) w4[i] = t4[i];
            }
#pragma unroll
            for (int i = 0; i < NP; ++i) v[i] = w4[i];
          } else {
#pragma unroll
            for (int i = 0; i < NP; ++i) v[i] = src[i];
          }
        }
        // part p of the row: chunk c (8 channels) at words 4 c .. 4 c + 3
        uint4 pw[3][KC] = {};
        if (!(kShProbe & 4)) {
#pragma unroll
          for (int c = 0; c < KC; ++c) {
            const float f[8] = {v[2 * c].x, v[2 * c].y, v[2 * c].z, v[2 * c].w,
                                v[2 * c + 1].x, v[2 * c + 1].y, v[2 * c + 1].z, v[2 * c + 1].w};
            split_bf16x3(f, pw[0][c], pw[1][c], pw[2][c]);
          }
        }
        const uint32_t as = seq % NSA, ause = seq / NSA;
        if (ause > 0) mbar_wait(smem_u32(&a_empty[as]), (ause - 1) & 1);
        tc_fence_after();
        const uint32_t tcol = tmem + ((uint32_t)(32 * q) << 16) + F::AOFF + as * F::SLOT_COLS;
        if (!(kShProbe & 4)) {
#pragma unroll
          for (int part = 0; part < 3; ++part)
#pragma unroll
            for (int c = 0; c < KC; c += 2) tmem_st8(tcol + (C / 2) * part + 4 * c, pw[part][c], pw[part][c + 1]);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&a_full[as]));
        // The raw slot is released only now: released right after the loads (before the split), the producer's
        // next bulk copy overwrote pixels of rows whose bank-conflicted loads were still replaying (rare wrong
        // pixels, caught by tests/test_gpu_determinism.py); here the TMEM writes depend on the loaded values.
        fence_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&raw_empty[s]));
      }
    }
  } else if (warp == kMma) {
    // ================= MMA issuer: input-row stationary, two shifts per row.  The whole warp walks the
    // schedule with warp-uniform incremental bookkeeping (no divisions); one asm block per input row
    // issues its MMAs and shifts from the elected lane.
    const uint32_t wlo = desc_lo(smem_u32(wst), NW * 16);
    const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
    uint32_t as = 0, a_par = 0;        // A slot of the next input row and the parity of its a_full phase
    uint32_t s_next = 0, epoch = 0;    // accumulator slot of the next output row to open, completed wraps
    long long dbg_wait = 0, dbg_wait2 = 0, dbg_issue = 0, dbg_rows = 0;  // kShProbe & 64: cycles per row waiting / issuing
    for (long long u = blockIdx.x; u < nunits; u += gridDim.x) {
      Unit U;
      if (!unit_at(a, u, U)) continue;
      uint32_t s_new = 0, s_cur = 0, s_old = 0;
      for (int g = -1; g <= U.bh; ++g) {  // g: input row relative to the quarters' bands
        const long long tq0 = (kShProbe & 64) ? clock64() : 0;
        mbar_wait(smem_u32(&a_full[as]), a_par);
        const bool v_new = g + 1 < U.bh, v_cur = g >= 0 && g < U.bh, v_old = g - 1 >= 0;
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
        const uint32_t abase = tm + F::AOFF + as * F::SLOT_COLS;
        if (v_new && v_cur && v_old)
          row_mmas_all<C>(tm + s_new * ACOLS, tm + s_cur * ACOLS, tm + s_old * ACOLS, abase, wlo);
        else
          row_mmas_edge<C>(tm + s_new * ACOLS, tm + s_cur * ACOLS, tm + s_old * ACOLS, abase, wlo,
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
    // ================= epilogue: warp q4 drains its lane quarter.  16 channels: group hg takes the output rows
    // with tile % 2 == hg; 32 channels: group hg takes channels 16 hg .. 16 hg + 15 of every output row.
#if HS_SH_FRAG
    // The accumulator is read as 16x256b fragments (tmem_ld_frag16): a thread holds, of each 16-lane half hh, the
    // rows l / 4 and l / 4 + 8 and the channel pairs 2 (l % 4) + {0, 1} of both 8-channel blocks, so four lanes
    // cover 32 contiguous bytes of a pixel and every 8-byte store (and side-input load) instruction moves whole
    // sectors -- without the 4x4 transposes the lane-per-pixel layout needed (64 shuffles and selects per row).
    const int q4 = warp & 3, hg = warp >> 2;
    const int l4 = lane >> 2, c2 = 2 * (lane & 3);
    const int ch0 = (F::HALVES ? 16 * hg : 0) + c2;  // this thread's first channel (block 0); block 1 at + 8
    constexpr int STEP = F::HALVES ? 1 : 2;          // output rows between two rows of this group
    uint32_t tile = 0;
    for (long long u = blockIdx.x; u < nunits; u += gridDim.x) {
      Unit U;
      if (!unit_at(a, u, U)) continue;
      const float* add = a.addend ? a.addend + (a.addend_per_model ? (a.model_of ? a.model_of[U.b] : 0) : U.b) *
                                                   a.addend_bstride
                                  : nullptr;
      const float* res = a.residual ? a.residual + (size_t)U.b * a.H * a.W * C : nullptr;
      float* yimg = a.y + (size_t)U.b * a.H * a.W * C;
      int qy0, seg;
      const bool qv = quarter_at(a, U, q4, qy0, seg);
      const int oy_end = qy0 + U.bh;
      // this thread's four pixels: row (hh, rh) = 16 hh + 8 rh + l4 of the segment
      int px[4];
      bool ok[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int row = 16 * (k >> 1) + 8 * (k & 1) + l4;
        px[k] = SEG * seg + row;
        ok[k] = qv && row < SEG && px[k] < a.W;
      }
      const float2 bs0 = *reinterpret_cast<const float2*>(s_bias + ch0), bs1 = *reinterpret_cast<const float2*>(s_bias + ch0 + 8);
      // side inputs: requested when the group's previous row has stored, first touched at the store
      float2 sa[4][2], sr[4][2];
#pragma unroll
      for (int k = 0; k < 4; ++k) sa[k][0] = sa[k][1] = sr[k][0] = sr[k][1] = make_float2(0.f, 0.f);
      auto issue_side = [&](int oy) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (!ok[k]) continue;
          const size_t gp = ((size_t)oy * a.W + px[k]) * C + ch0;
          if (add) {
            sa[k][0] = __ldg(reinterpret_cast<const float2*>(add + gp));
            sa[k][1] = __ldg(reinterpret_cast<const float2*>(add + gp + 8));
          }
          if (res) {
            sr[k][0] = __ldg(reinterpret_cast<const float2*>(res + gp));
            sr[k][1] = __ldg(reinterpret_cast<const float2*>(res + gp + 8));
          }
        }
      };
      {
        const int first = F::HALVES ? qy0 : qy0 + (int)((tile ^ (uint32_t)hg) & 1);  // this group's first row
        if (first < oy_end) issue_side(first);
      }
      for (int oy = qy0; oy < oy_end; ++oy, ++tile) {
        if (!F::HALVES && (int)(tile & 1) != hg) continue;
        const uint32_t acc = tile % NACC;
        mbar_wait(smem_u32(&acc_full[acc]), (tile / NACC) & 1);
        tc_fence_after();
        uint64_t o[2][4];  // [hh][j / 2]: (rh, block) = (0, 0), (1, 0), (0, 1), (1, 1), channel pairs packed
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          uint32_t r0[8], r1[8], r2[8];
          const uint32_t col = tmem + ((uint32_t)(q4 * 32 + 16 * hh) << 16) + acc * ACOLS + (F::HALVES ? 16 * hg : 0);
          if (!(kShProbe & 32)) {
            tmem_ld_frag16(col, r0);
            tmem_ld_frag16(col + C, r1);
            tmem_ld_frag16(col + 2 * C, r2);
            tmem_wait_ld();
          }
#pragma unroll
          for (int j = 0; j < 8; j += 2)  // (x0 + x1) + x2 partial sums (FADD2)
            o[hh][j / 2] = add2(add2(pk2(r0[j], r0[j + 1]), pk2(r1[j], r1[j + 1])), pk2(r2[j], r2[j + 1]));
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&acc_empty[acc]));  // TMEM free; finish from registers
        if (!(kShProbe & 8)) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {  // pixel (hh, rh) = (k >> 1, k & 1)
#pragma unroll
            for (int blk = 0; blk < 2; ++blk) {
              const float2 bs = blk ? bs1 : bs0;
              const uint64_t v = add2(o[k >> 1][2 * blk + (k & 1)], pkf(bs.x, bs.y));
              float vx = lo_f(v), vy = hi_f(v);
              if (a.softplus) {
                vx = softplus_fast(vx);
                vy = softplus_fast(vy);
              }
              const uint64_t sd = add2(pkf(sa[k][blk].x, sa[k][blk].y), pkf(sr[k][blk].x, sr[k][blk].y));
              const uint64_t q = add2(pkf(vx, vy), sd);  // o + (addend + residual), as conv_tc.cu
              if (ok[k])
                *reinterpret_cast<float2*>(yimg + ((size_t)oy * a.W + px[k]) * C + ch0 + 8 * blk) = make_float2(lo_f(q), hi_f(q));
            }
          }
        }
        if (oy + STEP < oy_end) issue_side(oy + STEP);
      }
    }
  }
#else
    const int q4 = warp & 3, hg = warp >> 2;
    const int gi = lane & 3, gb = lane & ~3;
    const int ch0 = F::HALVES ? 16 * hg : 0;  // first channel of this warp
    constexpr int STEP = F::HALVES ? 1 : 2;   // output rows between two rows of this group
    uint32_t tile = 0;
    for (long long u = blockIdx.x; u < nunits; u += gridDim.x) {
      Unit U;
      if (!unit_at(a, u, U)) continue;
      const float* add = a.addend ? a.addend + (a.addend_per_model ? (a.model_of ? a.model_of[U.b] : 0) : U.b) *
                                                   a.addend_bstride
                                  : nullptr;
      const float* res = a.residual ? a.residual + (size_t)U.b * a.H * a.W * C : nullptr;
      float* yimg = a.y + (size_t)U.b * a.H * a.W * C;
      int qy0, seg;
      const bool qv = quarter_at(a, U, q4, qy0, seg);
      const int xg0 = SEG * seg + gb;  // output pixel of this lane group's first lane
      const int oy_end = qy0 + U.bh;
      bool ok[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) ok[j] = qv && gb + j < SEG && xg0 + j < a.W;
      // side inputs (addend, residual) in the post-transpose layout (chunk gi of the group's four pixels).
      // A row's side inputs are requested as soon as the group's previous row has used its own and are only
      // touched at the store, so their DRAM latency runs under the next accumulator wait, drain and softplus.
      // (Requested right before the accumulator wait, their first use held 28% of all stall samples in ncu;
      // summing addend and residual at load time stalls on the loads just the same.)
      float4 sa[4], sr[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) sa[j] = sr[j] = make_float4(0.f, 0.f, 0.f, 0.f);
      auto issue_side = [&](int oy) {
        const size_t gp = ((size_t)oy * a.W + xg0) * C + ch0;
        if (add) {
          const float4* ap = reinterpret_cast<const float4*>(add + gp);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (ok[j]) sa[j] = __ldg(ap + j * (C / 4) + gi);
        }
        if (res) {
          const float4* rp = reinterpret_cast<const float4*>(res + gp);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (ok[j]) sr[j] = __ldg(rp + j * (C / 4) + gi);
        }
      };
      {
        const int first = F::HALVES ? qy0 : qy0 + (int)((tile ^ (uint32_t)hg) & 1);  // this group's first row
        if (first < oy_end) issue_side(first);
      }
      for (int oy = qy0; oy < oy_end; ++oy, ++tile) {
        if (!F::HALVES && (int)(tile & 1) != hg) continue;
        const uint32_t acc = tile % NACC;
        const size_t gpix = ((size_t)oy * a.W + xg0) * C + ch0;
        mbar_wait(smem_u32(&acc_full[acc]), (tile / NACC) & 1);
        tc_fence_after();
        float o[16] = {};
#pragma unroll
        for (int n0 = 0; n0 < 16; n0 += 8) {
          if (kShProbe & 32) break;
          uint32_t r0[8], r1[8], r2[8];
          const uint32_t col = tmem + ((uint32_t)(q4 * 32) << 16) + acc * ACOLS + ch0 + n0;
          tmem_ld8(col, r0);
          tmem_ld8(col + C, r1);
          tmem_ld8(col + 2 * C, r2);
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
          if (oy + STEP < oy_end) issue_side(oy + STEP);
          continue;
        }
        float4 ch[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4 bs = *reinterpret_cast<const float4*>(s_bias + ch0 + 4 * q);
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
        float4* yb = reinterpret_cast<float4*>(yimg + gpix);
#pragma unroll
        for (int j = 0; j < 4; ++j) {  // o + (addend + residual), as conv_tc.cu
          const uint64_t s01 = add2(pkf(sa[j].x, sa[j].y), pkf(sr[j].x, sr[j].y));
          const uint64_t s23 = add2(pkf(sa[j].z, sa[j].w), pkf(sr[j].z, sr[j].w));
          const uint64_t q01 = add2(pkf(ch[j].x, ch[j].y), s01), q23 = add2(pkf(ch[j].z, ch[j].w), s23);
          if (ok[j]) yb[j * (C / 4) + gi] = make_float4(lo_f(q01), hi_f(q01), lo_f(q23), hi_f(q23));
        }
        if (oy + STEP < oy_end) issue_side(oy + STEP);
      }
    }
  }
#endif
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// ---------------------------------------------------------------------------------------------------------------
// 16 -> 32 stride-2 layer on the same scheme.  A TMEM lane holds the PAIR of input pixels (2 ox, 2 ox + 1) of its
// output pixel ox: 32 floats, split and written exactly like a 32-channel pixel (part p: even pixel at columns
// 16 p, odd pixel at 16 p + 8).  Taps kx = 1 / 2 read the even / odd columns; tap kx = 0 needs the odd pixel of
// output ox - 1, so the lanes of a quarter hold DESCENDING ox (lane j: ox = 31 seg + 30 - j) and one shift of the
// odd columns brings it in (lane 31 goes stale: 31 output pixels per quarter, 64 input pixels per raw segment).
// Rows: input row 2 oy - 1 + i of a band: even i closes output row i / 2 - 1 (ky 2) and opens i / 2 (ky 0), odd i
// adds ky 1 to output row (i - 1) / 2.  TMEM: four 96-column accumulators, two 48-column A slots.  The two
// epilogue groups take the two 16-channel halves of every output row.
constexpr int SEG2 = 31;
struct S2 {
  static constexpr int CIN = 16, COUT = 32, KC = 2, NW = 3 * COUT;
  static constexpr uint32_t WT = KC * NW;
  static constexpr int W_BYTES = 9 * KC * NW * 16;
  static constexpr int QBYTES = 64 * CIN * 4;          // raw bytes of one lane quarter's 64 input pixels
  static constexpr int RAW_BYTES = 4 * QBYTES;
  static constexpr int NR = 8, NACC = 4, ACOLS = 3 * COUT, AOFF = NACC * ACOLS, SLOT_COLS = 48;
  static constexpr int NSA = (512 - AOFF) / SLOT_COLS;
  static constexpr size_t SMEM = W_BYTES + (size_t)NR * RAW_BYTES + 8 * (2 * NR + 2 * NSA + 2 * NACC) + 16 + 4 * COUT;
  static_assert(SMEM <= 232448, "shared memory budget");
};

// the tcgen05 work of one input row: target X (accumulator dx, weight taps of its ky at wx, all accumulating)
// and target Y (dy, wy; its first MMA overwrites); valid bit 0 / 1 enables X / Y
HS_DEV void s2_row_mmas(uint32_t dx, uint32_t dy, uint32_t abase, uint32_t wx, uint32_t wy, uint32_t valid) {
  constexpr uint32_t I0 = idesc_bf16(128, 96), I1 = idesc_bf16(128, 64), I2 = idesc_bf16(128, 32);
  if (kShProbe & 2) return;
#define HS_S2_MMA3(D, E, P0, A0, A1, A2)                                            \
  "@" E " tcgen05.mma.cta_group::1.kind::f16 [" D "], [" A0 "], db, i0, " P0 ";\n\t" \
  "@" E " tcgen05.mma.cta_group::1.kind::f16 [" D "], [" A1 "], db, i1, pt;\n\t"     \
  "@" E " tcgen05.mma.cta_group::1.kind::f16 [" D "], [" A2 "], db, i2, pt;\n\t"
#define HS_S2_TAP(WR, KOFF, D, E, P0, A0, A1, A2) \
  "add.u32 bl, " WR ", " KOFF ";\n\tmov.b64 db, {bl, hi};\n\t" HS_S2_MMA3(D, E, P0, A0, A1, A2)
  asm volatile(
      "{\n\t.reg .pred e, ex, ey, pz, pt;\n\t.reg .b64 db;\n\t.reg .b32 hi, i0, i1, i2, e1, e2, o0, o1, o2, bl, m;\n\t"
      "mov.b32 hi, %6;\n\tmov.b32 i0, %7;\n\tmov.b32 i1, %8;\n\tmov.b32 i2, %9;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t@!e bra S2_SKIP_%=;\n\t"  // the elected lane branches in: uniform predicates below
      "and.b32 m, %5, 1;\n\tsetp.ne.b32 ex, m, 0;\n\t"
      "and.b32 m, %5, 2;\n\tsetp.ne.b32 ey, m, 0;\n\t"
      "setp.ne.b32 pz, %5, %5;\n\tsetp.eq.b32 pt, %5, %5;\n\t"
      "add.u32 e1, %2, 16;\n\tadd.u32 e2, %2, 32;\n\tadd.u32 o0, %2, 8;\n\tadd.u32 o1, %2, 24;\n\tadd.u32 o2, %2, 40;\n\t"
      HS_S2_TAP("%3", "%10", "%0", "ex", "pt", "%2", "e1", "e2") HS_S2_TAP("%4", "%10", "%1", "ey", "pz", "%2", "e1", "e2")
      HS_S2_TAP("%3", "%11", "%0", "ex", "pt", "o0", "o1", "o2") HS_S2_TAP("%4", "%11", "%1", "ey", "pt", "o0", "o1", "o2")
      "tcgen05.shift.cta_group::1.down [o0];\n\ttcgen05.shift.cta_group::1.down [o1];\n\t"
      "tcgen05.shift.cta_group::1.down [o2];\n\t"
      HS_S2_TAP("%3", "0", "%0", "ex", "pt", "o0", "o1", "o2") HS_S2_TAP("%4", "0", "%1", "ey", "pt", "o0", "o1", "o2")
      "S2_SKIP_%=:\n\t}\n" ::"r"(dx), "r"(dy), "r"(abase), "r"(wx), "r"(wy), "r"(valid), "n"(kDescHi), "n"(I0), "n"(I1), "n"(I2),
      "n"(1 * S2::WT), "n"(2 * S2::WT)
      : "memory");
#undef HS_S2_MMA3
#undef HS_S2_TAP
  __syncwarp();
}

__global__ void __launch_bounds__(NT, 1) k_conv_shift_s2(ShArgs a) {
  using F = S2;
  constexpr int C = F::CIN, CO = F::COUT, KC = F::KC, NW = F::NW, NR = F::NR, NACC = F::NACC, NSA = F::NSA,
                ACOLS = F::ACOLS;
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* wst = smem;
  unsigned char* raw = smem + F::W_BYTES;
  uint64_t* raw_full = reinterpret_cast<uint64_t*>(raw + (size_t)NR * F::RAW_BYTES);
  uint64_t* raw_empty = raw_full + NR;
  uint64_t* a_full = raw_empty + NR;
  uint64_t* a_empty = a_full + NSA;
  uint64_t* acc_full = a_empty + NSA;
  uint64_t* acc_empty = acc_full + NACC;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(acc_empty + NACC);
  float* s_bias = reinterpret_cast<float*>(s_tmem + 4);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long nunits = (long long)a.B * a.ntile * a.ngroups;

  for (int e = tid; e < 9 * KC * CO; e += NT) {  // resident weight stack, layout (tap, chunk, row) x 16 B
    const int n = e % CO, c = (e / CO) % KC, t = e / (CO * KC);
    const float* src = a.w + ((size_t)n * 9 + t) * C + 8 * c;
    const float4 v0 = __ldg(reinterpret_cast<const float4*>(src)), v1 = __ldg(reinterpret_cast<const float4*>(src + 4));
    const float v[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
    uint4 p[3];
    split_bf16x3(v, p[0], p[1], p[2]);
#pragma unroll
    for (int part = 0; part < 3; ++part)
      *reinterpret_cast<uint4*>(wst + ((size_t)(t * KC + c) * NW + part * CO + n) * 16) = p[part];
  }
  if (tid < CO) s_bias[tid] = a.bias[tid];
  if (tid == 0) {
    for (int i = 0; i < NR; ++i) {
      mbar_init(smem_u32(&raw_full[i]), 1);
      mbar_init(smem_u32(&raw_empty[i]), 4);
    }
    for (int i = 0; i < NSA; ++i) {
      mbar_init(smem_u32(&a_full[i]), 4);
      mbar_init(smem_u32(&a_empty[i]), 1);
    }
    for (int i = 0; i < NACC; ++i) {
      mbar_init(smem_u32(&acc_full[i]), 1);
      mbar_init(smem_u32(&acc_empty[i]), 8);
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
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");

  if (warp == kProd) {
    if (lane == 0) {
      uint32_t seq = 0;
      for (long long u = blockIdx.x; u < nunits; u += gridDim.x) {
        Unit U;
        if (!unit_at(a, u, U)) continue;
        const float* img = a.x + (size_t)U.b * a.H * a.W * C;
        int qy0[4], qx0[4];
        bool qv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          int seg;
          qv[q] = quarter_at(a, U, q, qy0[q], seg);
          qx0[q] = 2 * SEG2 * seg - 2;  // first input pixel of the quarter's raw segment
        }
        for (int i = 0; i <= 2 * U.bh; ++i, ++seq) {
          const uint32_t s = seq % NR, use = seq / NR;
          if (use > 0) mbar_wait(smem_u32(&raw_empty[s]), (use - 1) & 1);
          const uint32_t bar = smem_u32(&raw_full[s]);
          uint32_t total = 0;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int g = 2 * qy0[q] - 1 + i, clo = max(qx0[q], 0), chi = min(qx0[q] + 64, a.W);
            if (qv[q] && g >= 0 && g < a.H && chi > clo) total += (uint32_t)(chi - clo) * C * 4;
          }
          if (total) {
            mbar_arrive_tx(bar, total);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int g = 2 * qy0[q] - 1 + i, clo = max(qx0[q], 0), chi = min(qx0[q] + 64, a.W);
              if (qv[q] && g >= 0 && g < a.H && chi > clo)
                bulk_g2s(smem_u32(raw + (size_t)s * F::RAW_BYTES + (size_t)q * F::QBYTES + (size_t)(clo - qx0[q]) * C * 4),
                         img + ((size_t)g * a.W + clo) * C, (uint32_t)(chi - clo) * C * 4, bar);
            }
          } else {
            mbar_arrive(bar);
          }
        }
      }
    }
  } else if (warp >= kCvt0 && warp < kCvt0 + 4) {
    const int q = warp - kCvt0;
    uint32_t seq = 0;
    for (long long u = blockIdx.x; u < nunits; u += gridDim.x) {
      Unit U;
      if (!unit_at(a, u, U)) continue;
      int qy0, seg;
      const bool qv = quarter_at(a, U, q, qy0, seg);
      const int xe = 2 * (SEG2 * seg + 30 - lane);  // even input pixel of this lane's pair
      const bool oke = qv && xe >= 0 && xe < a.W, oko = qv && xe + 1 >= 0 && xe + 1 < a.W;
      for (int i = 0; i <= 2 * U.bh; ++i, ++seq) {
        const int g = 2 * qy0 - 1 + i;
        const uint32_t s = seq % NR;
        mbar_wait(smem_u32(&raw_full[s]), (seq / NR) & 1);
        float4 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        if ((oke || oko) && g >= 0 && g < a.H) {
          const float4* src = reinterpret_cast<const float4*>(raw + (size_t)s * F::RAW_BYTES + (size_t)q * F::QBYTES +
                                                              (size_t)(31 - lane) * 128);
          const int r = HS_SH_NOROT ? 0 : (lane & 7);  // rotated piece order: eight bank groups per quarter-warp wavefront
          float4 w4[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) w4[k] = src[(k + r) & 7];
#pragma unroll
          for (int st = 1; st < 8; st <<= 1) {
            float4 t4[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) t4[k] = (r & st) ? w4[(k + 8 - st) & 7] : w4[k];
#pragma unroll
            for (int k = 0; k < 8; ++k) w4[k] = t4[k];
          }
#pragma unroll
          for (int k = 0; k < 8; ++k)
            if (k < 4 ? oke : oko) v[k] = w4[k];
        }
        uint4 pw[3][4] = {};
        if (!(kShProbe & 4)) {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const float f[8] = {v[2 * c].x, v[2 * c].y, v[2 * c].z, v[2 * c].w,
                                v[2 * c + 1].x, v[2 * c + 1].y, v[2 * c + 1].z, v[2 * c + 1].w};
            split_bf16x3(f, pw[0][c], pw[1][c], pw[2][c]);
          }
        }
        const uint32_t as = seq % NSA, ause = seq / NSA;
        if (ause > 0) mbar_wait(smem_u32(&a_empty[as]), (ause - 1) & 1);
        tc_fence_after();
        const uint32_t tcol = tmem + ((uint32_t)(32 * q) << 16) + F::AOFF + as * F::SLOT_COLS;
        if (!(kShProbe & 4)) {
#pragma unroll
          for (int part = 0; part < 3; ++part) {
            tmem_st8(tcol + 16 * part, pw[part][0], pw[part][1]);      // even pixel
            tmem_st8(tcol + 16 * part + 8, pw[part][2], pw[part][3]);  // odd pixel
          }
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&a_full[as]));
        fence_async_smem();  // the raw slot is released after the row is in TMEM (see k_conv_shift)
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&raw_empty[s]));
      }
    }
  } else if (warp == kMma) {
    const uint32_t wlo = desc_lo(smem_u32(wst), NW * 16);
    const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
    uint32_t as = 0, a_par = 0, s_next = 0, epoch = 0;
    for (long long u = blockIdx.x; u < nunits; u += gridDim.x) {
      Unit U;
      if (!unit_at(a, u, U)) continue;
      uint32_t s_new = 0, s_old = 0;  // accumulator of the newest open output row and of the one before it
      for (int i = 0; i <= 2 * U.bh; ++i) {
        mbar_wait(smem_u32(&a_full[as]), a_par);
        const uint32_t abase = tm + F::AOFF + as * F::SLOT_COLS;
        if ((i & 1) == 0) {
          // input row 2 r - 1 (r = i / 2): ky 2 of output row r - 1 (closes it), ky 0 of output row r (opens it)
          const bool v_old = i > 0, v_new = i < 2 * U.bh;
          s_old = s_new;
          if (v_new) {
            s_new = s_next;
            if (epoch > 0) mbar_wait(smem_u32(&acc_empty[s_new]), (epoch - 1) & 1);
            if (++s_next == (uint32_t)NACC) {
              s_next = 0;
              ++epoch;
            }
          }
          tc_fence_after();
          s2_row_mmas(tm + s_old * ACOLS, tm + s_new * ACOLS, abase, wlo + 6 * F::WT, wlo,
                      (v_old ? 1u : 0u) | (v_new ? 2u : 0u));
          mma_commit(smem_u32(&a_empty[as]));
          if (v_old) mma_commit(smem_u32(&acc_full[s_old]));
        } else {
          // input row 2 r: ky 1 of output row r = (i - 1) / 2
          tc_fence_after();
          s2_row_mmas(tm + s_new * ACOLS, tm + s_new * ACOLS, abase, wlo + 3 * F::WT, wlo, 1u);
          mma_commit(smem_u32(&a_empty[as]));
        }
        if (++as == (uint32_t)NSA) {
          as = 0;
          a_par ^= 1;
        }
      }
    }
  } else {
    // epilogue: warp q4 drains its lane quarter; group hg takes channels 16 hg .. 16 hg + 15 of every output row
    const int q4 = warp & 3, hg = warp >> 2;
    const int gi = lane & 3, gb = lane & ~3;
    const int ch0 = 16 * hg;
    uint32_t tile = 0;
    for (long long u = blockIdx.x; u < nunits; u += gridDim.x) {
      Unit U;
      if (!unit_at(a, u, U)) continue;
      const float* add = a.addend ? a.addend + (a.addend_per_model ? (a.model_of ? a.model_of[U.b] : 0) : U.b) *
                                                   a.addend_bstride
                                  : nullptr;
      const float* res = a.residual ? a.residual + (size_t)U.b * a.Ho * a.Wo * CO : nullptr;
      float* yimg = a.y + (size_t)U.b * a.Ho * a.Wo * CO;
      int qy0, seg;
      const bool qv = quarter_at(a, U, q4, qy0, seg);
      const int xg0 = SEG2 * seg + 30 - gb;  // output pixel of this lane group's first lane; the group's pixel j is xg0 - j
      const int oy_end = qy0 + U.bh;
      bool ok[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) ok[j] = qv && gb + j < SEG2 && xg0 - j >= 0 && xg0 - j < a.Wo;
      float4 sa[4], sr[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) sa[j] = sr[j] = make_float4(0.f, 0.f, 0.f, 0.f);
      auto issue_side = [&](int oy) {
        const long long gp = ((long long)oy * a.Wo + xg0) * CO + ch0;
        if (add) {
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (ok[j]) sa[j] = __ldg(reinterpret_cast<const float4*>(add + gp - (long long)j * CO) + gi);
        }
        if (res) {
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (ok[j]) sr[j] = __ldg(reinterpret_cast<const float4*>(res + gp - (long long)j * CO) + gi);
        }
      };
      if (qy0 < oy_end) issue_side(qy0);
      for (int oy = qy0; oy < oy_end; ++oy, ++tile) {
        const uint32_t acc = tile % NACC;
        const long long gpix = ((long long)oy * a.Wo + xg0) * CO + ch0;
        mbar_wait(smem_u32(&acc_full[acc]), (tile / NACC) & 1);
        tc_fence_after();
        float o[16] = {};
#pragma unroll
        for (int n0 = 0; n0 < 16; n0 += 8) {
          uint32_t r0[8], r1[8], r2[8];
          const uint32_t col = tmem + ((uint32_t)(q4 * 32) << 16) + acc * ACOLS + ch0 + n0;
          tmem_ld8(col, r0);
          tmem_ld8(col + CO, r1);
          tmem_ld8(col + 2 * CO, r2);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 8; j += 2) {
            const uint64_t sm = add2(add2(pk2(r0[j], r0[j + 1]), pk2(r1[j], r1[j + 1])), pk2(r2[j], r2[j + 1]));
            o[n0 + j] = __uint_as_float((uint32_t)sm);
            o[n0 + j + 1] = __uint_as_float((uint32_t)(sm >> 32));
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&acc_empty[acc]));
        float4 ch[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4 bs = *reinterpret_cast<const float4*>(s_bias + ch0 + 4 * q);
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
        group4_transpose(ch, gi);  // lane gi: chunk gi of the group's four pixels (pixel j at xg0 - j)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint64_t s01 = add2(pkf(sa[j].x, sa[j].y), pkf(sr[j].x, sr[j].y));
          const uint64_t s23 = add2(pkf(sa[j].z, sa[j].w), pkf(sr[j].z, sr[j].w));
          const uint64_t q01 = add2(pkf(ch[j].x, ch[j].y), s01), q23 = add2(pkf(ch[j].z, ch[j].w), s23);
          if (ok[j])
            reinterpret_cast<float4*>(yimg + gpix - (long long)j * CO)[gi] = make_float4(lo_f(q01), hi_f(q01), lo_f(q23), hi_f(q23));
        }
        if (oy + 1 < oy_end) issue_side(oy + 1);
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

// ---------------------------------------------------------------------------------------------------------------
// 32 -> 16 transposed (stride-2) layer on the same scheme.  Lanes hold INPUT pixels p (ascending, 31 valid per
// quarter); output (2 q + a, 2 p + b) takes, as conv_tc.cu's transposed tiles,
//   rows:  a = 0: (ky 1, input row q);  a = 1: (ky 0, row q + 1), (ky 2, row q)
//   cols:  b = 0: (kx 1, pixel p);      b = 1: (kx 0, pixel p + 1), (kx 2, pixel p)
// so input row r feeds output rows 2 r - 1 (ky 0, closes it), 2 r (ky 1, opens and closes it) and 2 r + 1 (ky 2,
// opens it), each with two column-parity accumulators of 48 columns (96 per output row); the taps kx 1 and kx 2
// read the row as written, kx 0 after one shift.  Bands run over input rows; a band reads one input row past its
// end (ky 0 of its last odd output row).  TMEM: four 96-column accumulators, two 48-column A slots.  The two
// epilogue groups take the even and the odd output columns of every output row: a lane's 16 channels are one
// 64-byte pixel, and the group-of-four transpose makes every store write whole pixels.
// 64 -> 32 (template CIN = 64): a CTA computes one 16-channel half of the output (units of the two halves run
// side by side, so the input rows are shared in L2) and takes a row's 64 input channels as two 32-channel halves
// through the two A slots in turn: the second half accumulates onto the first, and the converters refill one slot
// while the MMAs read the other.
template <int CIN_>
struct ST {
  static constexpr int CIN = CIN_, COUT = 16, COUT_T = CIN / 2, NSPLIT = COUT_T / COUT, KH = CIN / 32;
  static constexpr int KC = CIN / 8, NW = 3 * COUT;
  static constexpr uint32_t WT = KC * NW, KK = 2 * NW, WH = 4 * NW;  // weight units per tap / K step / K half
  static constexpr int W_BYTES = 9 * KC * NW * 16;
  static constexpr int QBYTES = 32 * CIN * 4;          // raw bytes of one lane quarter's 32 input pixels
  static constexpr int RAW_BYTES = 4 * QBYTES;
  static constexpr int NR = CIN == 32 ? 8 : 4, NACC = 4, ACOLS = 6 * COUT, AOFF = NACC * ACOLS, SLOT_COLS = 48;
  static constexpr int NSA = (512 - AOFF) / SLOT_COLS;
  static constexpr size_t SMEM = W_BYTES + (size_t)NR * RAW_BYTES + 8 * (2 * NR + 2 * NSA + 2 * NACC) + 16 + 4 * COUT;
  static_assert(SMEM <= 232448, "shared memory budget");
};

// the tcgen05 work of one input row: targets a (output row 2 r - 1, ky 0, accumulating), b (2 r, ky 1) and
// c (2 r + 1, ky 2), both opened here (their first MMA per column parity overwrites unless valid bit 3 says
// this is a later K half); valid bits 0 / 1 / 2 enable a / b / c
template <typename F>
HS_DEV void t_row_mmas(uint32_t da, uint32_t db_, uint32_t dc, uint32_t abase, uint32_t wlo, uint32_t valid) {
  constexpr uint32_t I0 = idesc_bf16(128, 48), I1 = idesc_bf16(128, 32), I2 = idesc_bf16(128, 16);
  if (kShProbe & 2) return;
#define HS_T_MMA3(D, E, P0, A0, A1, A2)                                             \
  "@" E " tcgen05.mma.cta_group::1.kind::f16 [" D "], [" A0 "], db, i0, " P0 ";\n\t" \
  "@" E " tcgen05.mma.cta_group::1.kind::f16 [" D "], [" A1 "], db, i1, pt;\n\t"     \
  "@" E " tcgen05.mma.cta_group::1.kind::f16 [" D "], [" A2 "], db, i2, pt;\n\t"
#define HS_T_TAP(WOFF, D, E, P0)                                                                          \
  "add.u32 bl, %4, " WOFF ";\n\tmov.b64 db, {bl, hi};\n\t" HS_T_MMA3(D, E, P0, "%3", "a10", "a20")        \
  "add.u32 bl, bl, %19;\n\tmov.b64 db, {bl, hi};\n\t" HS_T_MMA3(D, E, "pt", "a01", "a11", "a21")
  asm volatile(
      "{\n\t.reg .pred e, ea, eb, ec, pz, pt;\n\t.reg .b64 db;\n\t"
      ".reg .b32 hi, i0, i1, i2, a01, a10, a11, a20, a21, da1, db1, dc1, bl, m;\n\t"
      "mov.b32 hi, %6;\n\tmov.b32 i0, %7;\n\tmov.b32 i1, %8;\n\tmov.b32 i2, %9;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t@!e bra T_SKIP_%=;\n\t"  // the elected lane branches in: uniform predicates below
      "and.b32 m, %5, 1;\n\tsetp.ne.b32 ea, m, 0;\n\t"
      "and.b32 m, %5, 2;\n\tsetp.ne.b32 eb, m, 0;\n\t"
      "and.b32 m, %5, 4;\n\tsetp.ne.b32 ec, m, 0;\n\t"
      "and.b32 m, %5, 8;\n\tsetp.ne.b32 pz, m, 0;\n\tsetp.eq.b32 pt, %5, %5;\n\t"
      "add.u32 a01, %3, 8;\n\tadd.u32 a10, %3, 16;\n\tadd.u32 a11, %3, 24;\n\tadd.u32 a20, %3, 32;\n\tadd.u32 a21, %3, 40;\n\t"
      "add.u32 da1, %0, 48;\n\tadd.u32 db1, %1, 48;\n\tadd.u32 dc1, %2, 48;\n\t"
      // row as written: kx 1 -> even output columns, kx 2 -> odd output columns
      HS_T_TAP("%11", "%0", "ea", "pt") HS_T_TAP("%14", "%1", "eb", "pz") HS_T_TAP("%17", "%2", "ec", "pz")
      HS_T_TAP("%12", "da1", "ea", "pt") HS_T_TAP("%15", "db1", "eb", "pz") HS_T_TAP("%18", "dc1", "ec", "pz")
      "tcgen05.shift.cta_group::1.down [%3];\n\ttcgen05.shift.cta_group::1.down [a01];\n\t"
      "tcgen05.shift.cta_group::1.down [a10];\n\ttcgen05.shift.cta_group::1.down [a11];\n\t"
      "tcgen05.shift.cta_group::1.down [a20];\n\ttcgen05.shift.cta_group::1.down [a21];\n\t"
      // shifted row (pixel p + 1): kx 0 -> odd output columns
      HS_T_TAP("%10", "da1", "ea", "pt") HS_T_TAP("%13", "db1", "eb", "pt") HS_T_TAP("%16", "dc1", "ec", "pt")
      "T_SKIP_%=:\n\t}\n" ::"r"(da), "r"(db_), "r"(dc), "r"(abase), "r"(wlo), "r"(valid), "n"(kDescHi), "n"(I0), "n"(I1), "n"(I2),
      "n"(0 * F::WT), "n"(1 * F::WT), "n"(2 * F::WT), "n"(3 * F::WT), "n"(4 * F::WT), "n"(5 * F::WT),
      "n"(6 * F::WT), "n"(7 * F::WT), "n"(8 * F::WT), "n"(F::KK)
      : "memory");
#undef HS_T_MMA3
#undef HS_T_TAP
  __syncwarp();
}

template <int CIN_>
__global__ void __launch_bounds__(NT, 1) k_conv_shift_t(ShArgs a) {
  using F = ST<CIN_>;
  constexpr int C = F::CIN, CO = F::COUT, CT = F::COUT_T, KH = F::KH, NSPLIT = F::NSPLIT, KC = F::KC, NW = F::NW, NR = F::NR, NACC = F::NACC, NSA = F::NSA,
                ACOLS = F::ACOLS;
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* wst = smem;
  unsigned char* raw = smem + F::W_BYTES;
  uint64_t* raw_full = reinterpret_cast<uint64_t*>(raw + (size_t)NR * F::RAW_BYTES);
  uint64_t* raw_empty = raw_full + NR;
  uint64_t* a_full = raw_empty + NR;
  uint64_t* a_empty = a_full + NSA;
  uint64_t* acc_full = a_empty + NSA;
  uint64_t* acc_empty = acc_full + NACC;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(acc_empty + NACC);
  float* s_bias = reinterpret_cast<float*>(s_tmem + 4);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // units: the cout halves of one tile run side by side; a persistent CTA keeps one half (grid is a multiple of NSPLIT)
  const long long nunits = (long long)a.B * a.ntile * a.ngroups * NSPLIT;
  const int split = (int)(blockIdx.x % NSPLIT);

  for (int e = tid; e < 9 * KC * CO; e += NT) {  // resident weight stack of this half, layout (tap, chunk, row) x 16 B
    const int n = e % CO, c = (e / CO) % KC, t = e / (CO * KC);
    const float* src = a.w + ((size_t)(split * CO + n) * 9 + t) * C + 8 * c;
    const float4 v0 = __ldg(reinterpret_cast<const float4*>(src)), v1 = __ldg(reinterpret_cast<const float4*>(src + 4));
    const float v[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
    uint4 p[3];
    split_bf16x3(v, p[0], p[1], p[2]);
#pragma unroll
    for (int part = 0; part < 3; ++part)
      *reinterpret_cast<uint4*>(wst + ((size_t)(t * KC + c) * NW + part * CO + n) * 16) = p[part];
  }
  if (tid < CO) s_bias[tid] = a.bias[split * CO + tid];
  if (tid == 0) {
    for (int i = 0; i < NR; ++i) {
      mbar_init(smem_u32(&raw_full[i]), 1);
      mbar_init(smem_u32(&raw_empty[i]), 4);
    }
    for (int i = 0; i < NSA; ++i) {
      mbar_init(smem_u32(&a_full[i]), 4);
      mbar_init(smem_u32(&a_empty[i]), 1);
    }
    for (int i = 0; i < NACC; ++i) {
      mbar_init(smem_u32(&acc_full[i]), 1);
      mbar_init(smem_u32(&acc_empty[i]), 8);
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
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");

  if (warp == kProd) {
    if (lane == 0) {
      uint32_t seq = 0;
      for (long long u = blockIdx.x; u < nunits; u += gridDim.x) {
        Unit U;
        if (!unit_at(a, u / NSPLIT, U)) continue;
        const float* img = a.x + (size_t)U.b * a.H * a.W * C;
        int qy0[4], qx0[4];
        bool qv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          int seg;
          qv[q] = quarter_at(a, U, q, qy0[q], seg);
          qx0[q] = SEG2 * seg;  // first input pixel of the quarter
        }
        for (int i = 0; i <= U.bh; ++i, ++seq) {
          const uint32_t s = seq % NR, use = seq / NR;
          if (use > 0) mbar_wait(smem_u32(&raw_empty[s]), (use - 1) & 1);
          const uint32_t bar = smem_u32(&raw_full[s]);
          uint32_t total = 0;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int g = qy0[q] + i, chi = min(qx0[q] + 32, a.W);
            if (qv[q] && g < a.H && chi > qx0[q]) total += (uint32_t)(chi - qx0[q]) * C * 4;
          }
          if (total) {
            mbar_arrive_tx(bar, total);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int g = qy0[q] + i, chi = min(qx0[q] + 32, a.W);
              if (qv[q] && g < a.H && chi > qx0[q])
                bulk_g2s(smem_u32(raw + (size_t)s * F::RAW_BYTES + (size_t)q * F::QBYTES),
                         img + ((size_t)g * a.W + qx0[q]) * C, (uint32_t)(chi - qx0[q]) * C * 4, bar);
            }
          } else {
            mbar_arrive(bar);
          }
        }
      }
    }
  } else if (warp >= kCvt0 && warp < kCvt0 + 4) {
    const int q = warp - kCvt0;
    uint32_t seq = 0;
    for (long long u = blockIdx.x; u < nunits; u += gridDim.x) {
      Unit U;
      if (!unit_at(a, u / NSPLIT, U)) continue;
      int qy0, seg;
      const bool qv = quarter_at(a, U, q, qy0, seg);
      const bool xok = qv && SEG2 * seg + lane < a.W;
      for (int i = 0; i <= U.bh; ++i, ++seq) {
        const int g = qy0 + i;
        const uint32_t s = seq % NR;
        mbar_wait(smem_u32(&raw_full[s]), (seq / NR) & 1);
#pragma unroll 1
        for (int h = 0; h < KH; ++h) {  // 32 input channels at a time, one A slot each
          float4 v[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) v[k] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (xok && g < a.H) {
            const float4* src = reinterpret_cast<const float4*>(raw + (size_t)s * F::RAW_BYTES + (size_t)q * F::QBYTES +
                                                                (size_t)lane * (C * 4) + (size_t)h * 128);
            const int r = HS_SH_NOROT ? 0 : (lane & 7);  // rotated piece order: eight bank groups per quarter-warp wavefront
            float4 w4[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) w4[k] = src[(k + r) & 7];
#pragma unroll
            for (int st = 1; st < 8; st <<= 1) {
              float4 t4[8];
#pragma unroll
              for (int k = 0; k < 8; ++k) t4[k] = (r & st) ? w4[(k + 8 - st) & 7] : w4[k];
#pragma unroll
              for (int k = 0; k < 8; ++k) w4[k] = t4[k];
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = w4[k];
          }
          uint4 pw[3][4] = {};
          if (!(kShProbe & 4)) {
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const float f[8] = {v[2 * c].x, v[2 * c].y, v[2 * c].z, v[2 * c].w,
                                  v[2 * c + 1].x, v[2 * c + 1].y, v[2 * c + 1].z, v[2 * c + 1].w};
              split_bf16x3(f, pw[0][c], pw[1][c], pw[2][c]);
            }
          }
          const uint32_t aseq = seq * KH + h, as = aseq % NSA, ause = aseq / NSA;
          if (ause > 0) mbar_wait(smem_u32(&a_empty[as]), (ause - 1) & 1);
          tc_fence_after();
          const uint32_t tcol = tmem + ((uint32_t)(32 * q) << 16) + F::AOFF + as * F::SLOT_COLS;
          if (!(kShProbe & 4)) {
#pragma unroll
            for (int part = 0; part < 3; ++part) {
              tmem_st8(tcol + 16 * part, pw[part][0], pw[part][1]);      // channels 0-15 of the half (K step 0)
              tmem_st8(tcol + 16 * part + 8, pw[part][2], pw[part][3]);  // channels 16-31 (K step 1)
            }
          }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(&a_full[as]));
        }
        fence_async_smem();  // the raw slot is released after the row is in TMEM (see k_conv_shift)
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&raw_empty[s]));
      }
    }
  } else if (warp == kMma) {
    const uint32_t wlo = desc_lo(smem_u32(wst), NW * 16);
    const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
    uint32_t as = 0, a_par = 0, s_next = 0, epoch = 0;
    auto open_acc = [&]() {  // next output row's accumulator: its previous user must have drained it
      const uint32_t sl = s_next;
      if (epoch > 0) mbar_wait(smem_u32(&acc_empty[sl]), (epoch - 1) & 1);
      if (++s_next == (uint32_t)NACC) {
        s_next = 0;
        ++epoch;
      }
      return sl;
    };
    for (long long u = blockIdx.x; u < nunits; u += gridDim.x) {
      Unit U;
      if (!unit_at(a, u / NSPLIT, U)) continue;
      uint32_t s_a = 0, s_b = 0, s_c = 0;
      for (int i = 0; i <= U.bh; ++i) {
        const bool v_a = i > 0, v_bc = i < U.bh;
#pragma unroll 1
        for (int h = 0; h < KH; ++h) {
          mbar_wait(smem_u32(&a_full[as]), a_par);
          if (h == 0) {
            s_a = s_c;  // output row 2 r - 1 was opened as the previous input row's target c
            if (v_bc) {
              s_b = open_acc();
              s_c = open_acc();
            }
          }
          tc_fence_after();
          t_row_mmas<F>(tm + s_a * ACOLS, tm + s_b * ACOLS, tm + s_c * ACOLS, tm + F::AOFF + as * F::SLOT_COLS,
                        wlo + (uint32_t)h * F::WH, (v_a ? 1u : 0u) | (v_bc ? 6u : 0u) | (h ? 8u : 0u));
          mma_commit(smem_u32(&a_empty[as]));
          if (++as == (uint32_t)NSA) {
            as = 0;
            a_par ^= 1;
          }
        }
        if (v_a) mma_commit(smem_u32(&acc_full[s_a]));
        if (v_bc) mma_commit(smem_u32(&acc_full[s_b]));
      }
    }
  } else {
    // epilogue: warp q4 drains its lane quarter; group hg takes the output columns 2 p + hg of every output row
    const int q4 = warp & 3, hg = warp >> 2;
    const int gi = lane & 3, gb = lane & ~3;
    uint32_t tile = 0;
    for (long long u = blockIdx.x; u < nunits; u += gridDim.x) {
      Unit U;
      if (!unit_at(a, u / NSPLIT, U)) continue;
      const float* add = a.addend ? a.addend + (a.addend_per_model ? (a.model_of ? a.model_of[U.b] : 0) : U.b) *
                                                   a.addend_bstride
                                  : nullptr;
      const float* res = a.residual ? a.residual + (size_t)U.b * a.Ho * a.Wo * CT : nullptr;
      float* yimg = a.y + (size_t)U.b * a.Ho * a.Wo * CT;
      int qy0, seg;
      const bool qv = quarter_at(a, U, q4, qy0, seg);
      const int pg0 = SEG2 * seg + gb;  // input pixel of this lane group's first lane; the group's pixel j is pg0 + j
      bool ok[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) ok[j] = qv && gb + j < SEG2 && pg0 + j < a.W;
      const int oy_first = 2 * qy0, oy_end = 2 * (qy0 + U.bh);
      float4 sa[4], sr[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) sa[j] = sr[j] = make_float4(0.f, 0.f, 0.f, 0.f);
      auto issue_side = [&](int oy) {
        const size_t gp = ((size_t)oy * a.Wo + 2 * pg0 + hg) * CT + split * CO;
        if (add) {
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (ok[j]) sa[j] = __ldg(reinterpret_cast<const float4*>(add + gp + (size_t)j * 2 * CT) + gi);
        }
        if (res) {
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (ok[j]) sr[j] = __ldg(reinterpret_cast<const float4*>(res + gp + (size_t)j * 2 * CT) + gi);
        }
      };
      if (oy_first < oy_end) issue_side(oy_first);
      for (int oy = oy_first; oy < oy_end; ++oy, ++tile) {
        const uint32_t acc = tile % NACC;
        const size_t gpix = ((size_t)oy * a.Wo + 2 * pg0 + hg) * CT + split * CO;
        mbar_wait(smem_u32(&acc_full[acc]), (tile / NACC) & 1);
        tc_fence_after();
        float o[16] = {};
#pragma unroll
        for (int n0 = 0; n0 < 16; n0 += 8) {
          uint32_t r0[8], r1[8], r2[8];
          const uint32_t col = tmem + ((uint32_t)(q4 * 32) << 16) + acc * ACOLS + 48 * hg + n0;
          tmem_ld8(col, r0);
          tmem_ld8(col + CO, r1);
          tmem_ld8(col + 2 * CO, r2);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 8; j += 2) {
            const uint64_t sm = add2(add2(pk2(r0[j], r0[j + 1]), pk2(r1[j], r1[j + 1])), pk2(r2[j], r2[j + 1]));
            o[n0 + j] = __uint_as_float((uint32_t)sm);
            o[n0 + j + 1] = __uint_as_float((uint32_t)(sm >> 32));
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&acc_empty[acc]));
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
        group4_transpose(ch, gi);  // lane gi: chunk gi of the group's four pixels (output pixel 2 (pg0 + j) + hg)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint64_t s01 = add2(pkf(sa[j].x, sa[j].y), pkf(sr[j].x, sr[j].y));
          const uint64_t s23 = add2(pkf(sa[j].z, sa[j].w), pkf(sr[j].z, sr[j].w));
          const uint64_t q01 = add2(pkf(ch[j].x, ch[j].y), s01), q23 = add2(pkf(ch[j].z, ch[j].w), s23);
          if (ok[j])
            reinterpret_cast<float4*>(yimg + gpix + (size_t)j * 2 * CT)[gi] = make_float4(lo_f(q01), hi_f(q01), lo_f(q23), hi_f(q23));
        }
        if (oy + 1 < oy_end) issue_side(oy + 1);
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

// band height and band groups for a layer with Ho output rows of nseg segments (both kernels)
void plan_units(ShArgs& a, int Ho, int nseg, int sms, long long& grid) {
  a.band = HS_SH_BAND_MAX;
  a.nseg = nseg;
  // band height as conv_tc.cu: halve it until the RHS still iterating give every CTA >= 6 units
  const double act = prof::active_hint(a.B);
  grid = sms;
  while (a.band > 8 && act * ((a.nseg + 3) / 4) * ((Ho + a.band - 1) / a.band) < 6.0 * grid) a.band /= 2;
  const int nbands = (Ho + a.band - 1) / a.band;
  // bands per unit group: the smallest of 1, 2, 4 that leaves the fewest empty lane quarters
  a.nb = 1;
  if (Ho % a.band == 0) {
    double best = (double)a.nseg / (4 * ((a.nseg + 3) / 4));
    for (int nb = 2; nb <= 4; nb *= 2) {
      if (nbands % nb) break;
      const double eff = (double)(nb * a.nseg) / (4 * ((nb * a.nseg + 3) / 4));
      if (eff > best + 1e-9) {
        best = eff;
        a.nb = nb;
      }
    }
  }
  a.ntile = (a.nb * a.nseg + 3) / 4;
  a.ngroups = nbands / a.nb;
  const long long nunits = (long long)a.B * a.ntile * a.ngroups;
  if (nunits < grid) grid = nunits;
}

template <typename K>
bool launch_pdl(K kernel, const ShArgs& a, long long grid, size_t smem_bytes, cudaStream_t st) {
  if (grid <= 0) return true;  // empty batch or image: nothing to do
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem_bytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, a) == cudaSuccess;
}

template <int C>
bool launch_shift(ShArgs a, cudaStream_t st) {
  using F = Cfg<C>;
  static int sms = 0;
  if (!sms) {
    cudaFuncSetAttribute(k_conv_shift<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)F::SMEM);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  long long grid;
  plan_units(a, a.H, (a.W + SEG - 1) / SEG, sms, grid);
  return launch_pdl(k_conv_shift<C>, a, grid, F::SMEM, st);
}

}  // namespace

bool conv_shift_launch(int channels, const float* x, int H, int W, float* y, const float* w, const float* bias,
                       int softplus, const float* addend, long long addend_bstride, int addend_per_model,
                       const int* model_of, const float* residual, const void* const* active, int B,
                       cudaStream_t st) {
  ShArgs a{x, H, W, y, w, bias, softplus, addend, addend_bstride, addend_per_model, model_of, residual, active, B,
           H, W, H, 0, 0, 0, 0, 0};
  if (channels == 16) return launch_shift<16>(a, st);
  if (channels == 32) return launch_shift<32>(a, st);
  return false;
}

bool conv_shift_s2_launch(const float* x, int H, int W, float* y, int Ho, int Wo, const float* w, const float* bias,
                          int softplus, const float* addend, long long addend_bstride, int addend_per_model,
                          const int* model_of, const float* residual, const void* const* active, int B,
                          cudaStream_t st) {
  static int sms = 0;
  if (!sms) {
    cudaFuncSetAttribute(k_conv_shift_s2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S2::SMEM);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  ShArgs a{x, H, W, y, w, bias, softplus, addend, addend_bstride, addend_per_model, model_of, residual, active, B,
           Ho, Wo, Ho, 0, 0, 0, 0, 0};
  long long grid;
  plan_units(a, Ho, (Wo + SEG2 - 1) / SEG2, sms, grid);
  return launch_pdl(k_conv_shift_s2, a, grid, S2::SMEM, st);
}

template <int CIN_>
static bool launch_shift_t(ShArgs a, cudaStream_t st) {
  using F = ST<CIN_>;
  static int sms = 0;
  if (!sms) {
    cudaFuncSetAttribute(k_conv_shift_t<CIN_>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)F::SMEM);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  long long grid;
  plan_units(a, a.H, (a.W + SEG2 - 1) / SEG2, sms / F::NSPLIT, grid);  // grid: tiles; each has NSPLIT cout halves
  return launch_pdl(k_conv_shift_t<CIN_>, a, grid * F::NSPLIT, F::SMEM, st);
}

bool conv_shift_t_launch(int cin, const float* x, int H, int W, float* y, const float* w, const float* bias,
                         int softplus, const float* addend, long long addend_bstride, int addend_per_model,
                         const int* model_of, const float* residual, const void* const* active, int B,
                         cudaStream_t st) {
  ShArgs a{x, H, W, y, w, bias, softplus, addend, addend_bstride, addend_per_model, model_of, residual, active, B,
           2 * H, 2 * W, H, 0, 0, 0, 0, 0};
  if (cin == 32) return launch_shift_t<32>(a, st);
  if (cin == 64) return launch_shift_t<64>(a, st);
  return false;
}

}  // namespace hs
