// tcgen05 implicit-GEMM 3x3 convolution with fp32-class accuracy (BF16x3).
//
// GEMM view of one output tile: D[m][n] = sum_k A[m][k] B[n][k] with m = MT
// (128 or 64) consecutive output pixels of one row, n = output channels of
// this CTA's cout slice, k = (tap, cin).  Input rows are staged in shared
// memory in the UMMA K-major "interleaved" canonical layout (core matrix =
// 8 pixels x 16 bytes, pixels consecutive at a 16-byte pitch, 8-channel chunks
// LBO apart).  Because pixels sit at a 16-byte pitch, the A operand of tap
// (ky, kx) is just the staged row with the descriptor start address moved by
// kx * 16 bytes: no im2col copies.  Stride-2 convolutions stage each input
// row de-interleaved (even columns, then odd columns) so every tap is again a
// unit-pitch window; the transposed convolution is split into its two
// column-parity classes (1 and 2 taps) with two TMEM accumulators.
//
// Precision (SURVEY.md §0.5 rules out plain TF32/BF16): every fp32 operand is
// split exactly into three bf16 parts x = x0 + x1 + x2 (8+8+8 mantissa bits)
// and the six products with weight >= 2^-16 are accumulated in fp32 TMEM:
//   A0 [W0 | W1 | W2]  (N = 3 cs),  A1 [W0 | W1]  (N = 2 cs),  A2 W0  (N = cs)
// The weight parts are stacked along N, so each activation part is read from
// shared memory once per K step (thin cout makes these MMAs operand-bound,
// not math-bound); the epilogue sums the three column groups.
//
// Warp-specialised pipeline (one persistent CTA per SM, weights resident):
//   warp 10 (1 lane) producer  : cp.async.bulk of raw NHWC input rows into a
//                                ring of raw slots (mbarrier tx-count)
//   warps 8-9        converters: raw fp32 -> bf16x3 split, re-laid out into
//                                the staged ring (smem -> smem)
//   warp 11          MMA issuer: tcgen05.mma per tile into one of four TMEM
//                                accumulators; commits release staged rows
//                                and hand accumulators to the epilogue
//   warps 0-7        epilogue  : tcgen05.ld of their TMEM lane quarter and
//                                channel half, then
//                                bias, softplus, encoder/skip addend,
//                                residual, NHWC stores
// A CTA walks a band of output rows of one MT-pixel column block top to
// bottom, so every input row is fetched and split once per band.  Wide
// layers split cout across CTAs (CS channels each) so the resident bf16x3
// weights fit in shared memory.  M = 64 tiles use the half-lane TMEM layout
// (tile row m -> lane 32*(m/16) + m%16).
#include <cuda_bf16.h>

#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "conv_tc.h"
#include "prof.h"
#include "tc_util.cuh"

namespace hs {
namespace {
using namespace tc;

#ifndef HS_TC_PREFETCH
#define HS_TC_PREFETCH 4
#endif
constexpr int kPrefetch = HS_TC_PREFETCH;  // rows pulled into L2 ahead of the bulk copies / epilogue loads
#ifndef HS_TC_PREF_OUT
#define HS_TC_PREF_OUT 0  // bulk L2 prefetch of the epilogue's side rows (measured: off is faster, 32->16 t 1.37 -> 1.25 ms at C3)
#endif
#ifndef HS_TC_PREF_IN
#define HS_TC_PREF_IN 1  // bulk L2 prefetch of the input rows
#endif
constexpr int kNA = 4;    // TMEM accumulators in flight
constexpr int kEpiWarps = 8, kCvtWarp0 = 8;  // epilogue warps 0-7, converters from warp 8
constexpr size_t kSmemMax = 232448;
// Stage-removal probes for a separate measurement build only (tools/; `make PROBE=<mask>`): 1 skip
// conversion, 2 skip MMAs, 4 skip epilogue math, 32 force M = 64, 64 skip stores, 128 skip input loads,
// 256 skip addend loads.  The product build compiles with 0, so nothing read at run time can change
// what a launch computes.
#ifndef HS_TC_PROBE
#define HS_TC_PROBE 0
#endif
constexpr int kProbe = HS_TC_PROBE;
// programmatic dependent launch between chained convolutions (0 only in an A/B probe build)
#ifndef HS_TC_PDL
#define HS_TC_PDL 1
#endif
#ifndef HS_TC_BAND_MAX
#define HS_TC_BAND_MAX 32  // output rows per work unit before the launcher halves it for load balance
#endif
#ifndef HS_TC_ATM_NA
#define HS_TC_ATM_NA 2
#endif
#ifndef HS_TC_S2_CVT
#define HS_TC_S2_CVT 6
#endif
#ifndef HS_TC_PAIR
#define HS_TC_PAIR 1  // 16-channel stride-1 layers: the converter group takes input rows two at a time
#endif
#ifndef HS_TC_T_CVT
#define HS_TC_T_CVT 2  // converter warps of the wide transposed tiles (64 -> 32 t at M = 64)
#endif
#ifndef HS_TC_XPL_SKEW
#define HS_TC_XPL_SKEW 1  // staged chunk-plane pitch chosen per KC (see Cfg::XPL)
#endif
#ifndef HS_TC_RAW_SWZ
#define HS_TC_RAW_SWZ 1  // converters' raw-row loads: halves in swizzled order (no 2-way bank conflict)
#endif
#ifndef HS_TC_SHIFT
#define HS_TC_SHIFT 1  // 16 -> 16 stride-1 layers on the tcgen05.shift kernel (conv_shift.cu); 0 keeps the tap-view kernel below
#endif
#ifndef HS_TC_SHIFT_T64
#define HS_TC_SHIFT_T64 1  // 64 -> 32 transposed layer on the tcgen05.shift kernel (cout halves per CTA, two K halves)
#endif
#ifndef HS_TC_SHIFT_T
#define HS_TC_SHIFT_T 1  // 32 -> 16 transposed layer on the tcgen05.shift kernel
#endif
#ifndef HS_TC_SHIFT_S2
#define HS_TC_SHIFT_S2 1  // 16 -> 32 stride-2 layer on the tcgen05.shift kernel
#endif
#ifndef HS_TC_SHIFT32
#define HS_TC_SHIFT32 1  // 32 -> 32 stride-1 layers on the tcgen05.shift kernel as well
#endif
#ifndef HS_TC_CVT_GROUPS
#define HS_TC_CVT_GROUPS 1  // measured round 2 (C3 and C2 level-0 shapes): one group of four converter warps is 9-10% faster than two
#endif

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
  int band;  // output rows per work unit (a CTA walks a band of one column block top to bottom)
  int planar;  // complex-planar output (conv_tc.h)
};

// MODE 0: stride 1; MODE 1: stride 2; MODE 2: transposed stride 2 (out = 2 x in).
// MT: pixels per tile (UMMA M, 128 or 64); CS: output channels per CTA.
template <int CIN, int COUT, int MODE, int MT, int CS>
struct Cfg {
  static constexpr int NSPLIT = COUT / CS;
  static constexpr int KC = CIN / 8;                                                // 16-byte chunks per part
  static constexpr int KSTEPS = CIN / 16;                                           // MMA K steps per tap
  static constexpr int RW = MODE == 0 ? MT + 2 : (MODE == 1 ? 2 * MT + 1 : MT + 1); // pixels per staged row
  static constexpr int NACC = MODE == 2 ? 2 : 1;  // accumulators per tile (column-parity classes)
  static constexpr int RAW_BYTES = RW * CIN * 4;
  static constexpr int NW = 3 * CS;                            // stacked weight rows [W0; W1; W2]
  static constexpr size_t W_BYTES = (size_t)9 * KC * NW * 16;
  // A operand in TMEM (see below) for 16-channel stride-1 layers at M = 128
  static constexpr bool ATM = KSTEPS == 1 && MODE == 0 && MT == 128;
  static constexpr int NCG_ = ATM ? HS_TC_CVT_GROUPS : 1;  // converter groups (see NCG)
  // warp roles: epilogue 0-7, converters (four when they also write the TMEM A
  // slots: a warp may only touch its own TMEM lane quarter), producer, MMA issuer
  // four converter warps (measured best), except for the wide transposed tiles whose epilogue
  // needs the registers a 14-warp CTA cannot give
  // stride-2 layers convert two input rows per output row: six converter warps at M = 128
  // (measured; the M = 64 ones with two MMA warps would spill)
  static constexpr int NCVT_BASE = (MODE == 2 && CS * NACC > 32) ? HS_TC_T_CVT : (MODE == 1 && MT == 128 ? HS_TC_S2_CVT : 4);
  // ATM: two groups of four converter warps (one per TMEM lane quarter each)
  // take alternate input rows, so two rows' convert -> stage -> TMEM chains
  // overlap instead of running back to back
  static constexpr int NCG = NCG_;
  static constexpr int NCVT = NCVT_BASE * NCG, CVT_THREADS = 32 * NCVT;
  static constexpr int GCVT_THREADS = 32 * NCVT_BASE;  // threads of one converter group
  // MMA issuer warps: one warp issues a tcgen05.mma every ~45 cycles; the M = 64
  // layers (twice the MMAs per pixel) give alternate tiles to two issuers
  static constexpr int NMW = (MT == 64 && MODE != 2) ? 2 : 1;  // measured: helps only the M = 64 layers
  static constexpr int PROD = kCvtWarp0 + NCVT, MMAW = PROD + 1, NT = 32 * (MMAW + NMW);
  // staged ring: ATM converters consume their own staged rows at once; each
  // converter group alternates between two slots, so a thread may convert the
  // group's next row while a slower one still reads the previous (the group
  // barrier of the next row orders the reuse)
  // PAIR (one converter group): rows are converted two at a time into four staged slots
  static constexpr bool PAIR = ATM && NCG_ == 1 && HS_TC_PAIR;
  static constexpr int NS_MIN = ATM ? (PAIR ? 4 : 2 * NCG_) : 3,
                       NS_MAX = ATM ? (PAIR ? 4 : 2 * NCG_) : (MODE == 0 ? 10 : (MODE == 1 ? 8 : 6));
  static constexpr int XP_RES = (HS_TC_XPL_SKEW && MODE != 1 && KC < 8) ? 8 / KC : 1;
  static constexpr int pitch(int ns) { return ns * RW + ((8 + XP_RES - ((ns * RW) & 7)) & 7); }
  static constexpr size_t row_stage_bytes(int ns) { return (size_t)3 * KC * 16 * pitch(ns); }
  static constexpr size_t total(int ns, int nr) {
    return W_BYTES + row_stage_bytes(ns) + (size_t)nr * RAW_BYTES + 8 * (2 * nr + 2 * ns + 2 * kNA + 12) + 16 +
           4 * CS;
  }
  // deepest rings that fit: raw ring 6..2, staged ring NS_MAX..3
  static constexpr int pick_nr() {
    for (int nr = ATM ? 8 : 6; nr >= 2; --nr)
      if (total(NS_MIN, nr) <= kSmemMax && total(NS_MAX < 4 ? NS_MAX : 4, nr) <= kSmemMax) return nr;
    return 2;
  }
  static constexpr int NR = pick_nr();
  static constexpr int pick_ns() {
    for (int ns = NS_MAX; ns > NS_MIN; --ns)
      if (total(ns, NR) <= kSmemMax) return ns;
    return NS_MIN;
  }
  static constexpr int NS = pick_ns();
  // chunk-plane pitch mod 8 (16-byte bank groups): the converters' staged stores put the KC chunks of
  // 8 / KC consecutive pixels in one quarter-warp wavefront, so a pitch == 8 / KC (mod 8) lands them in
  // eight distinct bank groups (ncu at the C3 level-0 shape: == 1 gave every 16-channel store a 2-way
  // conflict).  Stride 2 de-interleaves the pixels, where no pitch removes the conflict: it keeps 1.
  static constexpr int XPL = pitch(NS);
  static constexpr size_t XP_BYTES = (size_t)KC * XPL * 16;   // one activation part
  static constexpr size_t R_BYTES = (size_t)NR * RAW_BYTES;
  static constexpr size_t TOTAL = total(NS, NR);
  static constexpr int ACOLS = NW * NACC;  // TMEM columns per accumulator
  // A operand in TMEM (16-channel stride-1 layers): the converters write every
  // input row once into a TMEM slot as its three tap views x three parts
  // (9 x 8 columns, tcgen05.st), and the 27 MMAs of a tile read only B from
  // shared memory.  With A in shared memory each MMA is bound by its 4 KB A
  // read (~40 cycles at 128 B/clk, measured); from TMEM an N = 48 MMA issues
  // at its math rate (24 cycles).
  static constexpr int SLOT_COLS = 9 * 8;
  // accumulators in flight; ATM keeps two and gives TMEM to five A slots (a tile
  // reads three rows, so the converters run two rows ahead of the MMAs)
  // ATM: two barrier pairs (the two epilogue groups alternate tiles) over NTA TMEM accumulators; with
  // one accumulator TMEM holds six A slots instead of five (the converters run three rows ahead)
  static constexpr int NA = ATM ? 2 : (4 * ACOLS <= 512 ? 4 : 2);
  static constexpr int NTA = ATM ? HS_TC_ATM_NA : NA;                             // TMEM accumulators
  // more accumulators than barrier pairs would let the MMA warp complete a pair's phase twice ahead of
  // the epilogue's parity wait (a deadlock)
  static_assert(NTA <= NA, "one acc_full / acc_empty pair per TMEM accumulator at most");
  static constexpr int AOFF = NTA * ACOLS;                                        // first A slot column
  static constexpr int NSA = ATM ? (512 - AOFF) / SLOT_COLS : 0;                  // TMEM A slots
  static_assert(!ATM || (NSA >= 4 && NSA <= 6), "a tile reads three rows; spare slots keep writes ahead");
  static constexpr int NCOLS_RAW = ATM ? 512 : NA * ACOLS;
  static constexpr int NCOLS = NCOLS_RAW <= 32    ? 32
                               : NCOLS_RAW <= 64  ? 64
                               : NCOLS_RAW <= 128 ? 128
                               : NCOLS_RAW <= 256 ? 256
                                                  : 512;
};

// input rows a tile (output row oy) needs: [lo, hi]
template <int MODE>
__host__ __device__ inline void tile_rows(int oy, int& lo, int& hi) {
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

// first input column of the raw row segment of column block xb
template <int MODE, int MT>
HS_DEV int raw_x0(int xb) {
  return MODE == 0 ? xb * MT - 1 : (MODE == 1 ? 2 * xb * MT - 1 : xb * MT);
}

// raw pixel p -> staged pixel (stride 2 de-interleaves even / odd columns)
template <int MODE, int MT>
HS_DEV int staged_px(int p) {
  if (MODE != 1) return p;
  return (p & 1) ? (p - 1) >> 1 : MT + (p >> 1);  // column 2x0-1+p: odd p is an even column
}

// One 8-channel chunk (32 bytes) of a raw fp32 row, element e = pixel * KC + chunk.  Consecutive
// elements sit 32 bytes apart, so loading every lane's first half and then its second half puts lanes e
// and e + 4 of a quarter warp on the same banks; lanes with bit 2 of e set load their halves in the
// other order, so each wavefront covers 128 distinct bytes.  Measured at C3: stride 2 / transposed
// 1-3.5% faster; the 16-channel stride-1 (A-in-TMEM) converters 8-16% SLOWER, so they keep the plain order.
template <bool SWZ>
HS_DEV void load_chunk(const unsigned char* p, int e, float4& lo, float4& hi) {
  const float4* s4 = reinterpret_cast<const float4*>(p);
  if (SWZ) {
    const int sw = (e >> 2) & 1;
    const float4 a = s4[sw], b = s4[sw ^ 1];
    lo = sw ? b : a;
    hi = sw ? a : b;
  } else {
    lo = s4[0];
    hi = s4[1];
  }
}

struct Unit {
  int split, b, xb, oy0, oy1, glo, ghi;  // cout slice, rows [oy0, oy1), input rows [glo, ghi]
};

template <int MODE, int MT>
__host__ __device__ inline long long num_units(const TcArgs& a, int nsplit) {
  const int xblocks = MODE == 2 ? a.W / MT : a.Wo / MT;
  return (long long)nsplit * a.B * xblocks * ((a.Ho + a.band - 1) / a.band);
}

template <int MODE, int MT>
HS_DEV bool unit_at(const TcArgs& a, int nsplit, long long u, Unit& U) {
  const int xblocks = MODE == 2 ? a.W / MT : a.Wo / MT;
  const int nbands = (a.Ho + a.band - 1) / a.band;
  U.split = (int)(u % nsplit);  // slices of one band run side by side: the input rows are reused from L2
  u /= nsplit;
  U.xb = (int)(u % xblocks);
  const int band = (int)((u / xblocks) % nbands);
  U.b = (int)(u / ((long long)xblocks * nbands));
  U.oy0 = band * a.band;
  U.oy1 = min(a.Ho, U.oy0 + a.band);
  int lo, hi;
  tile_rows<MODE>(U.oy0, lo, hi);
  U.glo = lo;
  tile_rows<MODE>(U.oy1 - 1, lo, hi);
  U.ghi = hi;
  return !(a.active && a.active[U.b] == nullptr);
}

// Descriptor bases: moving a window is a 32-bit add of offset >> 4 to the
// low word (smem addresses < 256 KB never carry out of the 14-bit field).
struct DescBase {
  uint32_t x[3], w;
};

// The three MMAs of one (tap, K step): activation parts x0, x1, x2 against
// the stacked weights [W0|W1|W2] (N = 3 cs, 2 cs, cs).  One asm block, one
// elect, immediates for the instruction descriptors and the descriptors'
// high word: the per-MMA cost is a 64-bit move and the issue itself.
template <uint32_t I0, uint32_t I1, uint32_t I2>
HS_DEV void mma_parts3(uint32_t d, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t b, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, t, e;\n\t.reg .b64 da, db;\n\t.reg .b32 hi, i0, i1, i2;\n\t"
      "mov.b32 hi, %6;\n\tmov.b32 i0, %7;\n\tmov.b32 i1, %8;\n\tmov.b32 i2, %9;\n\t"
      "setp.ne.b32 p, %5, 0;\n\tsetp.eq.b32 t, %5, %5;\n\telect.sync _|e, 0xffffffff;\n\t"
      "mov.b64 db, {%4, hi};\n\t"
      "mov.b64 da, {%1, hi};\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, i0, p;\n\t"
      "mov.b64 da, {%2, hi};\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, i1, t;\n\t"
      "mov.b64 da, {%3, hi};\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, i2, t;\n\t}\n" ::"r"(d),
      "r"(a0), "r"(a1), "r"(a2), "r"(b), "r"(accumulate), "n"(kDescHi), "n"(I0), "n"(I1), "n"(I2));
}

// The nine MMAs of one filter row (taps kx = 0, 1, 2 of row ky, one K step):
// one asm block whose descriptor arithmetic is all immediate adds, so ptxas
// moves three values into uniform registers per nine MMAs.
template <uint32_t I0, uint32_t I1, uint32_t I2, uint32_t PX0, uint32_t PX1, uint32_t PX2, uint32_t WT, uint32_t PS>
HS_DEV void mma_row9(uint32_t d, uint32_t xbase, uint32_t wbase, uint32_t accumulate) {
#define HS_MMA_PARTS(PX, P0)                                             \
  "add.u32 al, %1, " PX ";\n\tmov.b64 da, {al, hi};\n\t"              \
  "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, i0, " P0 ";\n\t" \
  "add.u32 al, al, %12;\n\tmov.b64 da, {al, hi};\n\t"                 \
  "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, i1, t;\n\t"      \
  "add.u32 al, al, %12;\n\tmov.b64 da, {al, hi};\n\t"                 \
  "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, i2, t;\n\t"
  asm volatile(
      "{\n\t.reg .pred p, t, e;\n\t.reg .b64 da, db;\n\t.reg .b32 hi, i0, i1, i2, al, bl;\n\t"
      "mov.b32 hi, %4;\n\tmov.b32 i0, %5;\n\tmov.b32 i1, %6;\n\tmov.b32 i2, %7;\n\t"
      "setp.ne.b32 p, %3, 0;\n\tsetp.eq.b32 t, %3, %3;\n\telect.sync _|e, 0xffffffff;\n\t"
      "mov.b64 db, {%2, hi};\n\t" HS_MMA_PARTS("%8", "p")
      "add.u32 bl, %2, %11;\n\tmov.b64 db, {bl, hi};\n\t" HS_MMA_PARTS("%9", "t")
      "add.u32 bl, %2, %13;\n\tmov.b64 db, {bl, hi};\n\t" HS_MMA_PARTS("%10", "t") "}\n" ::"r"(d),
      "r"(xbase), "r"(wbase), "r"(accumulate), "n"(kDescHi), "n"(I0), "n"(I1), "n"(I2), "n"(PX0), "n"(PX1),
      "n"(PX2), "n"(WT), "n"(PS), "n"(2 * WT));
#undef HS_MMA_PARTS
}

// A-in-TMEM variants (Cfg::ATM).  cp_row9: copy one staged row into a TMEM
// slot as tap views kx = 0, 1, 2 (start pixel PXkx) x parts 0, 1, 2, each a
// 128-lane x 256-bit block (8 columns).  mma_row9_tm: the nine MMAs of filter
// row ky reading those blocks; B (weights) stays in shared memory.
template <uint32_t PX0, uint32_t PX1, uint32_t PX2, uint32_t PS>
HS_DEV void cp_row9(uint32_t tbase, uint32_t sbase) {
#define HS_CP_PARTS(PX, T0)                                                    \
  "add.u32 sl, %1, " PX ";\n\tmov.b64 ds, {sl, hi};\n\t"                    \
  "add.u32 ta, %0, " T0 ";\n\t@e tcgen05.cp.cta_group::1.128x256b [ta], ds;\n\t" \
  "add.u32 sl, sl, %6;\n\tmov.b64 ds, {sl, hi};\n\t"                         \
  "add.u32 ta, ta, 8;\n\t@e tcgen05.cp.cta_group::1.128x256b [ta], ds;\n\t"   \
  "add.u32 sl, sl, %6;\n\tmov.b64 ds, {sl, hi};\n\t"                         \
  "add.u32 ta, ta, 8;\n\t@e tcgen05.cp.cta_group::1.128x256b [ta], ds;\n\t"
  asm volatile(
      "{\n\t.reg .pred e;\n\t.reg .b64 ds;\n\t.reg .b32 hi, sl, ta;\n\t"
      "mov.b32 hi, %2;\n\telect.sync _|e, 0xffffffff;\n\t"
      HS_CP_PARTS("%3", "0") HS_CP_PARTS("%4", "24") HS_CP_PARTS("%5", "48") "}\n" ::"r"(tbase),
      "r"(sbase), "n"(kDescHi), "n"(PX0), "n"(PX1), "n"(PX2), "n"(PS)
      : "memory");
#undef HS_CP_PARTS
}

template <uint32_t I0, uint32_t I1, uint32_t I2, uint32_t WT>
HS_DEV void mma_row9_tm(uint32_t d, uint32_t abase, uint32_t wbase, uint32_t accumulate) {
#define HS_MMA_TM(B0, P0)                                                           \
  "add.u32 bl, %2, " B0 ";\n\tmov.b64 db, {bl, hi};\n\t"                          \
  "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], db, i0, " P0 ";\n\tadd.u32 ta, ta, 8;\n\t" \
  "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], db, i1, t;\n\tadd.u32 ta, ta, 8;\n\t"      \
  "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], db, i2, t;\n\tadd.u32 ta, ta, 8;\n\t"
  asm volatile(
      "{\n\t.reg .pred p, t, e;\n\t.reg .b64 db;\n\t.reg .b32 hi, i0, i1, i2, bl, ta;\n\t"
      "mov.b32 hi, %4;\n\tmov.b32 i0, %5;\n\tmov.b32 i1, %6;\n\tmov.b32 i2, %7;\n\t"
      "setp.ne.b32 p, %3, 0;\n\tsetp.eq.b32 t, %3, %3;\n\telect.sync _|e, 0xffffffff;\n\t"
      "mov.b32 ta, %1;\n\t"
      HS_MMA_TM("0", "p") HS_MMA_TM("%8", "t") HS_MMA_TM("%9", "t") "}\n" ::"r"(d), "r"(abase), "r"(wbase),
      "r"(accumulate), "n"(kDescHi), "n"(I0), "n"(I1), "n"(I2), "n"(WT), "n"(2 * WT));
#undef HS_MMA_TM
}

template <typename C, int MT>
HS_DEV void tap_mmas(uint32_t d, const DescBase& db, uint32_t x_units, uint32_t w_units, uint32_t& first) {
  constexpr uint32_t X_STEP = 2 * C::XPL, W_STEP = 2 * C::NW;  // two 16-byte chunks per K step
  constexpr int CS = C::NW / 3;
  constexpr uint32_t I0 = idesc_bf16(MT, 3 * CS), I1 = idesc_bf16(MT, 2 * CS), I2 = idesc_bf16(MT, CS);
#pragma unroll
  for (int kk = 0; kk < C::KSTEPS; ++kk) {
    const uint32_t xo = x_units + kk * X_STEP, wo = db.w + w_units + kk * W_STEP;
    mma_parts3<I0, I1, I2>(d, db.x[0] + xo, db.x[1] + xo, db.x[2] + xo, wo, first ? 0u : 1u);
    first = 0;
  }
}

// all MMAs of output row oy; slot(g) = staged slot holding input row g
template <typename C, int MODE, int MT, typename SlotOf>
HS_DEV void issue_mmas(int oy, uint32_t d0, const DescBase& db, SlotOf slot) {
  constexpr uint32_t WT = C::KC * C::NW;  // weight units per tap
  auto row_units = [&](int g) { return (uint32_t)(slot(g) * C::RW); };
  uint32_t first = 1;
  if (MODE == 0 || MODE == 1) {
    const int g0 = MODE == 0 ? oy - 1 : 2 * oy - 1;
    constexpr int CS = C::NW / 3;
    constexpr uint32_t I0 = idesc_bf16(MT, 3 * CS), I1 = idesc_bf16(MT, 2 * CS), I2 = idesc_bf16(MT, CS);
    constexpr uint32_t PX0 = MODE == 0 ? 0 : MT, PX1 = MODE == 0 ? 1 : 0, PX2 = MODE == 0 ? 2 : MT + 1;
    constexpr uint32_t PS = (uint32_t)(C::XP_BYTES / 16);  // activation part planes, 16-byte units
    constexpr uint32_t X_STEP = 2 * C::XPL, W_STEP = 2 * C::NW;
#pragma unroll
    for (int ky = 0; ky < 3; ++ky) {
      const uint32_t r = row_units(g0 + ky);
#pragma unroll
      for (int kk = 0; kk < C::KSTEPS; ++kk)
        mma_row9<I0, I1, I2, PX0, PX1, PX2, WT, PS>(d0, db.x[0] + r + kk * X_STEP, db.w + ky * 3 * WT + kk * W_STEP,
                                                    (ky | kk) ? 1u : 0u);
    }
    (void)first;
    return;
  }
  // transposed: out row 2q <- (ky 1, row q); out row 2q+1 <- (ky 0, row q+1), (ky 2, row q)
  //             out col 2q (acc 0) <- (kx 1, q); out col 2q+1 (acc 1) <- (kx 0, q+1), (kx 2, q)
  const int q = oy >> 1;
  const uint32_t rq = row_units(q), rq1 = row_units(q + 1);
  const uint32_t d1 = d0 + C::NW;
  if ((oy & 1) == 0) {
    tap_mmas<C, MT>(d0, db, rq, (1 * 3 + 1) * WT, first);
    first = 1;
    tap_mmas<C, MT>(d1, db, rq + 1, (1 * 3 + 0) * WT, first);
    tap_mmas<C, MT>(d1, db, rq, (1 * 3 + 2) * WT, first);
  } else {
    tap_mmas<C, MT>(d0, db, rq1, (0 * 3 + 1) * WT, first);
    tap_mmas<C, MT>(d0, db, rq, (2 * 3 + 1) * WT, first);
    first = 1;
    tap_mmas<C, MT>(d1, db, rq1 + 1, (0 * 3 + 0) * WT, first);
    tap_mmas<C, MT>(d1, db, rq1, (0 * 3 + 2) * WT, first);
    tap_mmas<C, MT>(d1, db, rq + 1, (2 * 3 + 0) * WT, first);
    tap_mmas<C, MT>(d1, db, rq, (2 * 3 + 2) * WT, first);
  }
}

template <int CIN, int COUT, int MODE, int MT, int CS>
__global__ void __launch_bounds__(Cfg<CIN, COUT, MODE, MT, CS>::NT, 1) k_conv_tc(TcArgs a) {
  using C = Cfg<CIN, COUT, MODE, MT, CS>;
  constexpr int KC = C::KC, NS = C::NS, NR = C::NR, NW = C::NW, NSPLIT = C::NSPLIT;
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* wst = smem;
  unsigned char* xp[3] = {smem + C::W_BYTES, smem + C::W_BYTES + C::XP_BYTES, smem + C::W_BYTES + 2 * C::XP_BYTES};
  unsigned char* raw = smem + C::W_BYTES + 3 * C::XP_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(raw + C::R_BYTES);
  uint64_t* raw_full = bars;
  uint64_t* raw_empty = raw_full + NR;
  uint64_t* stg_full = raw_empty + NR;
  uint64_t* stg_empty = stg_full + NS;
  uint64_t* acc_full = stg_empty + NS;
  uint64_t* acc_empty = acc_full + C::NA;
  uint64_t* a_full = acc_empty + C::NA;  // TMEM A slots (C::ATM)
  uint64_t* a_empty = a_full + 6;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(a_empty + 6);
  float* s_bias = reinterpret_cast<float*>(s_tmem + 4);  // this CTA's cout slice
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long nunits = num_units<MODE, MT>(a, NSPLIT);
  // a persistent CTA keeps one cout slice: its units are u = blockIdx.x + k gridDim.x
  // with gridDim.x a multiple of NSPLIT, so u % NSPLIT is fixed per CTA
  const int my_split = (int)(blockIdx.x % NSPLIT);

  // ---- setup: resident weight stack [W0; W1; W2] of this slice, layout (tap, chunk, row) x 16 B
  for (int e = tid; e < 9 * KC * CS; e += C::NT) {
    const int n = e % CS, c = (e / CS) % KC, t = e / (CS * KC);
    const float* src = a.w + ((size_t)(my_split * CS + n) * 9 + t) * CIN + 8 * c;
    const float4 v0 = __ldg(reinterpret_cast<const float4*>(src)), v1 = __ldg(reinterpret_cast<const float4*>(src + 4));
    const float v[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
    uint4 p[3];
    split_bf16x3(v, p[0], p[1], p[2]);
#pragma unroll
    for (int part = 0; part < 3; ++part)
      *reinterpret_cast<uint4*>(wst + ((size_t)(t * KC + c) * NW + part * CS + n) * 16) = p[part];
  }
  for (int n = tid; n < CS; n += C::NT) s_bias[n] = a.bias[my_split * CS + n];
  if (tid == 0) {
    for (int i = 0; i < NR; ++i) {
      mbar_init(smem_u32(&raw_full[i]), 1);
      mbar_init(smem_u32(&raw_empty[i]), C::NCVT_BASE);  // one arrival per converter warp
    }
    for (int i = 0; i < NS; ++i) {
      mbar_init(smem_u32(&stg_full[i]), C::NCVT);
      mbar_init(smem_u32(&stg_empty[i]), C::NMW);  // every MMA warp releases every staged row
    }
    for (int i = 0; i < C::NA; ++i) {
      mbar_init(smem_u32(&acc_full[i]), 1);
      mbar_init(smem_u32(&acc_empty[i]), C::ATM ? kEpiWarps / 2 : kEpiWarps);  // one arrival per draining warp
    }
    for (int i = 0; i < C::NSA; ++i) {
      mbar_init(smem_u32(&a_full[i]), C::NCVT_BASE);
      mbar_init(smem_u32(&a_empty[i]), 1);
    }
    fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s_tmem)),
                 "r"(C::NCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;
  // Programmatic dependent launch: the set-up above (weights, barriers, TMEM)
  // does not touch the previous kernel's data, so it overlaps that kernel's
  // tail; every global read or write of activations comes after the wait.
  // Triggering at once is safe because this grid is persistent (one CTA per
  // SM, all resident): the next conv's CTAs only take SMs this grid leaves.
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");

  if (warp == C::PROD) {
    // ================= producer: raw row segments, global -> smem (bulk copies)
    if (lane == 0) {
      uint32_t seq = 0;  // 32-bit ring bookkeeping: divisions by the ring depths stay cheap
      for (long long u = blockIdx.x; u < nunits; u += gridDim.x) {
        Unit U;
        if (!unit_at<MODE, MT>(a, NSPLIT, u, U)) continue;
        const int x0 = raw_x0<MODE, MT>(U.xb);
        const int clo = max(x0, 0), chi = min(x0 + C::RW, a.W);
        const float* img = a.x + (size_t)U.b * a.H * a.W * CIN;
        // The raw ring holds only a few rows, too few bytes in flight to cover
        // DRAM latency: rows kPrefetch ahead (input rows and the epilogue's
        // addend / residual rows) are pulled into L2 with bulk prefetches.
        const float* add = a.addend ? a.addend + (a.addend_per_model ? (a.model_of ? a.model_of[U.b] : 0) : U.b) *
                                                     a.addend_bstride
                                    : nullptr;
        const float* res = a.residual ? a.residual + (size_t)U.b * a.Ho * a.Wo * COUT : nullptr;
        const int ox0 = MODE == 2 ? 2 * U.xb * MT : U.xb * MT;
        const uint32_t out_bytes = (uint32_t)(MODE == 2 ? 2 * MT : MT) * COUT * 4;
        auto prefetch_in = [&](int g) {
          if (HS_TC_PREF_IN && g <= U.ghi && g >= 0 && g < a.H && chi > clo)
            prefetch_l2(img + ((size_t)g * a.W + clo) * CIN, (uint32_t)(chi - clo) * CIN * 4);
        };
        int next_out = U.oy0;
        auto prefetch_out = [&](int upto) {
          for (; next_out < min(upto, U.oy1); ++next_out) {
            const size_t off = ((size_t)next_out * a.Wo + ox0) * COUT;
            if (HS_TC_PREF_OUT && add) prefetch_l2(add + off, out_bytes);
            if (HS_TC_PREF_OUT && res) prefetch_l2(res + off, out_bytes);
          }
        };
        for (int g = U.glo; g < U.glo + kPrefetch; ++g) prefetch_in(g);
        prefetch_out(U.oy0 + kPrefetch);
        for (int g = U.glo; g <= U.ghi; ++g, ++seq) {
          const int i = g - U.glo;
          prefetch_in(g + kPrefetch);
          prefetch_out(U.oy0 + (MODE == 0 ? i : (MODE == 1 ? i / 2 : 2 * i)) + kPrefetch);
          const int s = (int)(seq % NR);
          const uint32_t use = seq / NR;
          if (use > 0) mbar_wait(smem_u32(&raw_empty[s]), (uint32_t)((use - 1) & 1));
          const uint32_t bar = smem_u32(&raw_full[s]);
          if (g >= 0 && g < a.H && chi > clo && !(kProbe & 128)) {
            const uint32_t bytes = (uint32_t)(chi - clo) * CIN * 4;
            mbar_arrive_tx(bar, bytes);
            bulk_g2s(smem_u32(raw + (size_t)s * C::RAW_BYTES + (size_t)(clo - x0) * CIN * 4),
                     img + ((size_t)g * a.W + clo) * CIN, bytes, bar);
          } else {
            mbar_arrive(bar);
          }
        }
      }
    }
  } else if (warp >= kCvtWarp0 && warp < kCvtWarp0 + C::NCVT) {
    // ================= converters: raw fp32 -> staged bf16x3
    const int cg = (warp - kCvtWarp0) / C::NCVT_BASE;              // converter group: rows seq % NCG == cg
    const int ct = tid - 32 * kCvtWarp0 - cg * C::GCVT_THREADS;    // thread within the group
    uint32_t seq = 0;  // 32-bit ring bookkeeping
    if constexpr (C::PAIR) {
      // Two input rows per round: both rows' raw loads and conversions interleave, one group barrier
      // covers both, and both rows' TMEM writes follow (the converters had one warp per SM
      // sub-partition and spent most of a row in load / conversion latencies and the barrier)
      constexpr int NEL = (kProbe & 1) ? 0 : C::RW * KC;
      constexpr int TRIPS = (NEL + C::GCVT_THREADS - 1) / C::GCVT_THREADS;
      const int q = warp & 3, m = 32 * q + lane;
      for (long long u = blockIdx.x; u < nunits; u += gridDim.x) {
        Unit U;
        if (!unit_at<MODE, MT>(a, NSPLIT, u, U)) continue;
        const int x0 = raw_x0<MODE, MT>(U.xb);
        const int clo = max(x0, 0) - x0, chi = min(x0 + C::RW, a.W) - x0;
        for (int g = U.glo; g <= U.ghi;) {
          const int np = g + 1 <= U.ghi ? 2 : 1;
          float4 va[2][TRIPS > 0 ? TRIPS : 1][2];
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            if (r >= np) break;
            const uint32_t sq = seq + r;
            mbar_wait(smem_u32(&raw_full[sq % NR]), (sq / NR) & 1);
            const bool row_ok = g + r >= 0 && g + r < a.H;
            const unsigned char* src = raw + (size_t)(sq % NR) * C::RAW_BYTES;
#pragma unroll
            for (int t = 0; t < TRIPS; ++t) {
              const int e = ct + t * C::GCVT_THREADS;
              const int p = e / KC, c = e - p * KC;
              va[r][t][0] = va[r][t][1] = make_float4(0.f, 0.f, 0.f, 0.f);
              if (e < NEL && row_ok && p >= clo && p < chi) {
                load_chunk<HS_TC_RAW_SWZ && !C::ATM>(src + ((size_t)p * CIN + 8 * c) * 4, e, va[r][t][0], va[r][t][1]);
              }
            }
          }
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            if (r >= np) break;
            const int ss = (int)((seq + r) % NS);
#pragma unroll
            for (int t = 0; t < TRIPS; ++t) {
              const int e = ct + t * C::GCVT_THREADS;
              if (e < NEL) {
                const int p = e / KC, c = e - p * KC;
                const float v[8] = {va[r][t][0].x, va[r][t][0].y, va[r][t][0].z, va[r][t][0].w,
                                    va[r][t][1].x, va[r][t][1].y, va[r][t][1].z, va[r][t][1].w};
                uint4 p3[3];
                split_bf16x3(v, p3[0], p3[1], p3[2]);
                const size_t off = ((size_t)c * C::XPL + ss * C::RW + p) * 16;
#pragma unroll
                for (int part = 0; part < 3; ++part) *reinterpret_cast<uint4*>(xp[part] + off) = p3[part];
              }
            }
          }
          __syncwarp();
          if (lane == 0)
            for (int r = 0; r < np; ++r) mbar_arrive(smem_u32(&raw_empty[(seq + r) % NR]));
          asm volatile("bar.sync %0, %1;" ::"r"(1), "n"(C::GCVT_THREADS) : "memory");  // staged rows complete
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            if (r >= np) break;
            const uint32_t sq = seq + r, as = sq % C::NSA, ause = sq / C::NSA;
            if (ause > 0) mbar_wait(smem_u32(&a_empty[as]), (ause - 1) & 1);
            tc_fence_after();
            const int ss = (int)(sq % NS);
            const uint32_t tcol = tmem + ((uint32_t)(32 * q) << 16) + C::AOFF + as * C::SLOT_COLS;
#pragma unroll
            for (int kx = 0; kx < 3; ++kx)
#pragma unroll
              for (int part = 0; part < 3; ++part) {
                const unsigned char* b0 = xp[part] + ((size_t)ss * C::RW + m + kx) * 16;
                const uint4 lo = *reinterpret_cast<const uint4*>(b0);
                const uint4 hi = *reinterpret_cast<const uint4*>(b0 + (size_t)C::XPL * 16);
                asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                                 tcol + (kx * 3 + part) * 8),
                             "r"(lo.x), "r"(lo.y), "r"(lo.z), "r"(lo.w), "r"(hi.x), "r"(hi.y), "r"(hi.z), "r"(hi.w));
              }
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&a_full[as]));
          }
          seq += np;
          g += np;
        }
      }
    } else
    for (long long u = blockIdx.x; u < nunits; u += gridDim.x) {
      Unit U;
      if (!unit_at<MODE, MT>(a, NSPLIT, u, U)) continue;
      const int x0 = raw_x0<MODE, MT>(U.xb);
      const int clo = max(x0, 0) - x0, chi = min(x0 + C::RW, a.W) - x0;  // valid raw pixels [clo, chi)
      for (int g = U.glo; g <= U.ghi; ++g, ++seq) {
        if (C::NCG > 1 && (int)(seq % C::NCG) != cg) continue;
        const int rs = (int)(seq % NR);
        const int ss = C::ATM ? (int)(2 * cg + (seq / C::NCG) % 2) : (int)(seq % NS);
        const uint32_t suse = seq / NS;
        if (!C::ATM && suse > 0) mbar_wait(smem_u32(&stg_empty[ss]), (uint32_t)((suse - 1) & 1));
        mbar_wait(smem_u32(&raw_full[rs]), (uint32_t)((seq / NR) & 1));
        const bool row_ok = g >= 0 && g < a.H;
        const unsigned char* src = raw + (size_t)rs * C::RAW_BYTES;
        // elements (pixel, 8-channel chunk) in batches of up to three per thread: the batch's raw-row
        // loads are issued before any of its conversions and stores (a rolled loop paid one
        // shared-memory round trip per element, and the compiler cannot hoist loads across the stores
        // to the staged ring; one converter warp per SM sub-partition has no other warps to hide it)
        constexpr int NEL = (kProbe & 1) ? 0 : C::RW * KC;
        constexpr int TRIPS = (NEL + C::GCVT_THREADS - 1) / C::GCVT_THREADS;
        constexpr int NBW = (MODE == 2 || MT == 64) ? 1 : 3;  // batch width (the M = 64 and transposed tiles: no registers to spare)
        constexpr int NB = TRIPS < NBW ? (TRIPS > 0 ? TRIPS : 1) : NBW;
#pragma unroll 1
        for (int t0 = 0; t0 < TRIPS; t0 += NB) {
          float4 va[NB][2];
#pragma unroll
          for (int t = 0; t < NB; ++t) {
            const int e = ct + (t0 + t) * C::GCVT_THREADS;
            const int p = e / KC, c = e - p * KC;  // chunk fastest: conflict-free raw reads
            va[t][0] = va[t][1] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (t0 + t < TRIPS && e < NEL && row_ok && p >= clo && p < chi) {
              load_chunk<HS_TC_RAW_SWZ && !C::ATM>(src + ((size_t)p * CIN + 8 * c) * 4, e, va[t][0], va[t][1]);
            }
          }
#pragma unroll
          for (int t = 0; t < NB; ++t) {
            const int e = ct + (t0 + t) * C::GCVT_THREADS;
            if (t0 + t < TRIPS && e < NEL) {
              const int p = e / KC, c = e - p * KC;
              const float v[8] = {va[t][0].x, va[t][0].y, va[t][0].z, va[t][0].w,
                                  va[t][1].x, va[t][1].y, va[t][1].z, va[t][1].w};
              uint4 p3[3];
              split_bf16x3(v, p3[0], p3[1], p3[2]);
              const size_t off = ((size_t)c * C::XPL + ss * C::RW + staged_px<MODE, MT>(p)) * 16;
#pragma unroll
              for (int part = 0; part < 3; ++part) *reinterpret_cast<uint4*>(xp[part] + off) = p3[part];
            }
          }
        }
        if constexpr (C::ATM) {
          // every converter thread owns TMEM lane m = tile row m (a warp may only
          // write its own lane quarter): write the row's three tap views x three
          // parts of pixel m + kx from the staged row into TMEM slot `as`
          __syncwarp();  // barriers count warps: a waiter wakes once per warp, not once per thread
          if (lane == 0) mbar_arrive(smem_u32(&raw_empty[rs]));
          asm volatile("bar.sync %0, %1;" ::"r"(1 + cg), "n"(C::GCVT_THREADS) : "memory");  // staged row complete
          const uint32_t as = (uint32_t)(seq % C::NSA), ause = (uint32_t)(seq / C::NSA);
          if (ause > 0) mbar_wait(smem_u32(&a_empty[as]), (ause - 1) & 1);
          tc_fence_after();
          const int q = warp & 3, m = 32 * q + lane;
          const uint32_t tcol = tmem + ((uint32_t)(32 * q) << 16) + C::AOFF + as * C::SLOT_COLS;
#pragma unroll
          for (int kx = 0; kx < 3; ++kx)
#pragma unroll
            for (int part = 0; part < 3; ++part) {
              const unsigned char* b0 = xp[part] + ((size_t)ss * C::RW + m + kx) * 16;
              const uint4 lo = *reinterpret_cast<const uint4*>(b0);                          // channels 0-7
              const uint4 hi = *reinterpret_cast<const uint4*>(b0 + (size_t)C::XPL * 16);  // channels 8-15
              asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                               tcol + (kx * 3 + part) * 8),
                           "r"(lo.x), "r"(lo.y), "r"(lo.z), "r"(lo.w), "r"(hi.x), "r"(hi.y), "r"(hi.z), "r"(hi.w));
            }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(&a_full[as]));
        } else {
          fence_async_smem();
          __syncwarp();
          if (lane == 0) {
            mbar_arrive(smem_u32(&raw_empty[rs]));
            mbar_arrive(smem_u32(&stg_full[ss]));
          }
        }
      }
    }
  } else if (warp >= C::MMAW && warp < C::MMAW + C::NMW) {
    // ================= MMA issuer
    {  // the whole warp walks the schedule; mma_bf16 / mma_commit elect one lane
      DescBase db;
#pragma unroll
      for (int part = 0; part < 3; ++part) db.x[part] = desc_lo(smem_u32(xp[part]), C::XPL * 16);
      db.w = desc_lo(smem_u32(wst), NW * 16);
      // 32-bit, warp-uniform bookkeeping: ptxas keeps MMA operands in uniform registers
      const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
      uint32_t seq0 = 0;  // staged sequence number of the unit's first row
      uint32_t tile = 0;
      if constexpr (C::ATM) {
        // A in TMEM: the converters write each input row once into a TMEM slot
        // (a_full); the MMAs read the slots and release them (a_empty)
        constexpr uint32_t WT = C::KC * C::NW;
        constexpr uint32_t I0 = idesc_bf16(MT, 3 * CS), I1 = idesc_bf16(MT, 2 * CS), I2 = idesc_bf16(MT, CS);
        for (long long u = blockIdx.x; u < nunits; u += gridDim.x) {
          Unit U;
          if (!unit_at<MODE, MT>(a, NSPLIT, u, U)) continue;
          auto tslot = [&](int g) { return (seq0 + (uint32_t)(g - U.glo)) % C::NSA; };   // TMEM A slot
          int loaded = U.glo - 1;   // highest input row known to be in TMEM
          int retired = U.glo - 1;  // highest input row whose TMEM slot was released
          for (int oy = U.oy0; oy < U.oy1; ++oy, ++tile) {
            int lo, hi;
            tile_rows<MODE>(oy, lo, hi);
            for (int g = loaded + 1; g <= hi; ++g) {
              const uint32_t sq = seq0 + (uint32_t)(g - U.glo);
              mbar_wait(smem_u32(&a_full[sq % C::NSA]), (sq / C::NSA) & 1);
            }
            loaded = max(loaded, hi);
            const uint32_t acc = tile % C::NA;  // barrier pair / epilogue group
            // the TMEM accumulator was last written by tile - NTA: wait until its group drained it
            if (tile >= (uint32_t)C::NTA) {
              const uint32_t prev = tile - C::NTA;
              mbar_wait(smem_u32(&acc_empty[prev % C::NA]), (prev / C::NA) & 1);
            }
            tc_fence_after();
            const uint32_t d0 = tm + (tile % C::NTA) * C::ACOLS;
            if (!(kProbe & 2)) {
#pragma unroll
              for (int ky = 0; ky < 3; ++ky)
                mma_row9_tm<I0, I1, I2, WT>(d0, tm + C::AOFF + tslot(oy - 1 + ky) * C::SLOT_COLS,
                                            db.w + ky * 3 * WT, ky ? 1u : 0u);
            }
            mma_commit(smem_u32(&acc_full[acc]));
            int keep_lo = U.ghi + 1;
            if (oy + 1 < U.oy1) {
              int nl, nh;
              tile_rows<MODE>(oy + 1, nl, nh);
              keep_lo = nl;
            }
            for (int g = retired + 1; g < keep_lo && g <= loaded; ++g) mma_commit(smem_u32(&a_empty[tslot(g)]));
            retired = max(retired, min(keep_lo - 1, loaded));
          }
          seq0 += U.ghi - U.glo + 1;
        }
      } else
      for (long long u = blockIdx.x; u < nunits; u += gridDim.x) {
        Unit U;
        if (!unit_at<MODE, MT>(a, NSPLIT, u, U)) continue;
        auto slot = [&](int g) { return (int)((seq0 + (uint32_t)(g - U.glo)) % NS); };
        int waited = U.glo - 1;   // highest input row known to be staged
        int retired = U.glo - 1;  // highest input row released back to the converters
        const int mw = warp - C::MMAW;  // this issuer takes the tiles with tile % NMW == mw
        for (int oy = U.oy0; oy < U.oy1; ++oy, ++tile) {
          if ((int)(tile % C::NMW) != mw) continue;
          int lo, hi;
          tile_rows<MODE>(oy, lo, hi);
          for (int g = waited + 1; g <= hi; ++g) {
            const uint32_t sq = seq0 + (uint32_t)(g - U.glo);
            mbar_wait(smem_u32(&stg_full[sq % NS]), (sq / NS) & 1);
            waited = g;
            // rows below this tile were only read by the other issuer: release them at once,
            // or the ring (3 slots on the 64-channel layers) cannot stage this tile's rows
            for (; retired + 1 < lo && retired + 1 <= waited; ++retired) mma_commit(smem_u32(&stg_empty[slot(retired + 1)]));
          }
          waited = max(waited, hi);
          const uint32_t acc = tile % C::NA;
          const uint32_t ause = tile / C::NA;
          if (ause > 0) mbar_wait(smem_u32(&acc_empty[acc]), (ause - 1) & 1);
          tc_fence_after();
          if (!(kProbe & 2)) issue_mmas<C, MODE, MT>(oy, tm + acc * C::ACOLS, db, slot);
          mma_commit(smem_u32(&acc_full[acc]));
          // release rows this issuer's next tile of the unit no longer reads (a row is
          // released only after it was seen staged: an early arrival would complete the
          // slot's previous phase)
          int keep_lo = U.ghi + 1;
          if (oy + C::NMW < U.oy1) {
            int nl, nh;
            tile_rows<MODE>(oy + C::NMW, nl, nh);
            keep_lo = nl;
          }
          for (int g = retired + 1; g < keep_lo && g <= waited; ++g) mma_commit(smem_u32(&stg_empty[slot(g)]));
          retired = max(retired, min(keep_lo - 1, waited));
        }
        // unit end: rows this issuer never read still need its release
        for (int g = waited + 1; g <= U.ghi; ++g) {
          const uint32_t sq = seq0 + (uint32_t)(g - U.glo);
          mbar_wait(smem_u32(&stg_full[sq % NS]), (sq / NS) & 1);
        }
        waited = max(waited, U.ghi);
        for (int g = retired + 1; g <= U.ghi; ++g) mma_commit(smem_u32(&stg_empty[slot(g)]));
        seq0 += U.ghi - U.glo + 1;
      }
    }
  } else {
    if constexpr (C::ATM) {
      // ================= epilogue of the 16-channel stride-1 layers: warp group hg = warp / 4 drains
      // the tiles with tile % 2 == hg (TMEM accumulator hg), all 16 channels of its lane quarter's 32
      // pixels.  A 4x4 transpose of 16-byte chunks inside each group of four lanes (shuffles) makes
      // every store instruction write whole 64-byte pixels (two full sectors each): the per-lane
      // layout wrote half sectors, which measured 0.38 ms of a 1.73 ms C3 level-0 conv.
      static_assert(CS == 16 && COUT == 16 && C::NACC == 1 && C::NA == 2, "tile-split epilogue");
      const int q4 = warp & 3, hg = warp >> 2;
      const int m = q4 * 32 + lane;
      const int gi = lane & 3;  // position inside the group of four lanes
      uint32_t tile = 0;
      for (long long u = blockIdx.x; u < nunits; u += gridDim.x) {
        Unit U;
        if (!unit_at<MODE, MT>(a, NSPLIT, u, U)) continue;
        const float* add = a.addend ? a.addend + (a.addend_per_model ? (a.model_of ? a.model_of[U.b] : 0) : U.b) *
                                                     a.addend_bstride
                                    : nullptr;
        for (int oy = U.oy0; oy < U.oy1; ++oy, ++tile) {
          if ((int)(tile & 1) != hg) continue;
          const int acc = hg;                                  // barrier pair
          const uint32_t tcol = (uint32_t)(tile % C::NTA) * C::ACOLS;  // TMEM accumulator
          const size_t pix = (size_t)oy * a.Wo + (size_t)U.xb * MT + m;
          // side inputs in the layout the stores use after the 4x4 transpose below (chunk gi of the four
          // pixels of this lane's group): each load instruction reads whole 64-byte pixels, coalesced,
          // and they are requested before the accumulator wait
          const size_t gpix = pix - lane + (lane & ~3);
          float4 sd[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) sd[q] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (add && !(kProbe & 256)) {
            const float4* ap = reinterpret_cast<const float4*>(add + gpix * COUT);
#pragma unroll
            for (int j = 0; j < 4; ++j) sd[j] = __ldg(ap + j * 4 + gi);
          }
          if (a.residual) {
            const float4* rp = reinterpret_cast<const float4*>(a.residual + ((size_t)U.b * a.Ho * a.Wo + gpix) * COUT);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const float4 r = __ldg(rp + j * 4 + gi);
              const uint64_t s01 = add2(pkf(sd[j].x, sd[j].y), pkf(r.x, r.y)), s23 = add2(pkf(sd[j].z, sd[j].w), pkf(r.z, r.w));
              sd[j] = make_float4(lo_f(s01), hi_f(s01), lo_f(s23), hi_f(s23));
            }
          }
          mbar_wait(smem_u32(&acc_full[acc]), (uint32_t)((tile / C::NA) & 1));
          tc_fence_after();
          float o[16];
#pragma unroll
          for (int n0 = 0; n0 < 16; n0 += 8) {
            uint32_t r0[8], r1[8], r2[8];
            const uint32_t col = tmem + ((uint32_t)(q4 * 32) << 16) + tcol + n0;
            tmem_ld8(col, r0);
            tmem_ld8(col + CS, r1);
            tmem_ld8(col + 2 * CS, r2);
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
          if (kProbe & 4) continue;
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
          // now ch[j] holds chunk gi of pixel (lane & ~3) + j: add the side inputs (same layout), and
          // store j writes whole pixels
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint64_t q01 = add2(pkf(ch[j].x, ch[j].y), pkf(sd[j].x, sd[j].y));
            const uint64_t q23 = add2(pkf(ch[j].z, ch[j].w), pkf(sd[j].z, sd[j].w));
            ch[j] = make_float4(lo_f(q01), hi_f(q01), lo_f(q23), hi_f(q23));
          }
          if (!(kProbe & 64)) {
            float4* yb = reinterpret_cast<float4*>(a.y + ((size_t)U.b * a.Ho * a.Wo + pix - lane + (lane & ~3)) * COUT);
#pragma unroll
            for (int j = 0; j < 4; ++j) yb[j * 4 + gi] = ch[j];  // pixel j of the group, chunk gi
          }
        }
      }
    } else {
    // ================= epilogue warps 0-7: TMEM lane quarter q = warp % 4 (the
    // only lanes a warp may read), channel half h = warp / 4 of the slice.
    // M = 128: tile row m = TMEM lane m.  M = 64: rows 16q..16q+15 sit in the
    // first 16 lanes of quarter q (the other 16 lanes are idle).
    constexpr int EH = CS / 2;
    const int q4 = warp & 3, h = warp >> 2;
    const bool lane_ok = MT == 128 || lane < 16;
    const int m = MT == 128 ? q4 * 32 + lane : q4 * 16 + (lane & 15);
    uint32_t tile = 0;
    for (long long u = blockIdx.x; u < nunits; u += gridDim.x) {
      Unit U;
      if (!unit_at<MODE, MT>(a, NSPLIT, u, U)) continue;
      const int n_base = U.split * CS + h * EH;
      const float* add = a.addend ? a.addend + (a.addend_per_model ? (a.model_of ? a.model_of[U.b] : 0) : U.b) *
                                                   a.addend_bstride
                                  : nullptr;
      // addend and residual do not depend on the accumulator: row oy + 1's are
      // loaded while row oy waits on its MMAs, and only added at the store (an
      // add right after the load would stall on it)
      // (wide transposed tiles have no registers to spare: there the two are summed at load)
      constexpr bool SPLIT = C::NACC * EH <= 16;
      constexpr int RK = SPLIT ? C::NACC : 1, RQ = SPLIT ? EH / 4 : 1;
      // TR (16 channels per warp-half at M = 128, one accumulator): the four lanes of a group transpose
      // their pixels' 16-byte chunks before storing, so every store writes whole 64-byte pixel halves,
      // and the side inputs are loaded in that layout (lane: chunk gi of the group's pixels 0..3)
      // (M = 64: lanes 16-31 mirror lanes 0-15 and do not store).
      // TR2 (transposed, 8 channels per warp-half, two output-column accumulators): lane pairs swap
      // chunks so that each store writes whole 32-byte pixel halves (a full sector per lane pair)
      constexpr bool TR = EH == 16 && C::NACC == 1;
      constexpr bool TR2 = MODE == 2 && EH == 8 && C::NACC == 2 && MT == 128;
      const bool tr = (TR || TR2) && !a.planar;
      const int gi = lane & 3, pi = lane & 1;
      auto fetch = [&](int oy, float4(&pa)[C::NACC][EH / 4], float4(&pr)[RK][RQ]) {
        if (TR2 && tr) {  // pixel P + j (P = the pair's first output column), chunk pi
          const size_t prow = (size_t)oy * a.Wo + 2 * (U.xb * MT + m - pi);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const size_t off = (prow + j) * COUT + n_base + 4 * pi;
            float4 ad = make_float4(0.f, 0.f, 0.f, 0.f), r = make_float4(0.f, 0.f, 0.f, 0.f);
            if (add && !(kProbe & 256)) ad = __ldg(reinterpret_cast<const float4*>(add + off));
            if (a.residual) r = __ldg(reinterpret_cast<const float4*>(a.residual + (size_t)U.b * a.Ho * a.Wo * COUT + off));
            pa[(j >> 1) % C::NACC][(j & 1) % (EH / 4)] = ad;
            pr[SPLIT ? (j >> 1) % RK : 0][SPLIT ? (j & 1) % RQ : 0] = r;
          }
          return;
        }
        if (TR && tr) {
          const size_t gpix = (size_t)oy * a.Wo + U.xb * MT + m - gi;
#pragma unroll
          for (int j = 0; j < EH / 4; ++j) {
            const size_t off = (gpix + j) * COUT + n_base + 4 * gi;
            pa[0][j] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (add && !(kProbe & 256)) pa[0][j] = __ldg(reinterpret_cast<const float4*>(add + off));
            float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
            if (a.residual) r = __ldg(reinterpret_cast<const float4*>(a.residual + (size_t)U.b * a.Ho * a.Wo * COUT + off));
            pr[0][SPLIT ? j : 0] = r;
          }
          return;
        }
#pragma unroll
        for (int k = 0; k < C::NACC; ++k) {
          const int ox = MODE == 2 ? 2 * (U.xb * MT + m) + k : U.xb * MT + m;
          const size_t pix = (size_t)oy * a.Wo + ox;
          const size_t obase = (size_t)U.b * a.Ho * a.Wo * COUT + pix * COUT + n_base;
#pragma unroll
          for (int q = 0; q < EH / 4; ++q) {
            pa[k][q] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (add && lane_ok && !(kProbe & 256)) pa[k][q] = __ldg(reinterpret_cast<const float4*>(add + pix * COUT + n_base) + q);
            float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
            if (a.residual && lane_ok) r = __ldg(reinterpret_cast<const float4*>(a.residual + obase) + q);
            if constexpr (SPLIT) {
              pr[k][q] = r;
            } else {
              pa[k][q].x += r.x;
              pa[k][q].y += r.y;
              pa[k][q].z += r.z;
              pa[k][q].w += r.w;
            }
          }
        }
      };
      float4 pre_a[C::NACC][EH / 4], nxt_a[C::NACC][EH / 4], pre_r[RK][RQ], nxt_r[RK][RQ];
      fetch(U.oy0, pre_a, pre_r);
      for (int oy = U.oy0; oy < U.oy1; ++oy, ++tile) {
        const int acc = (int)(tile % C::NA);
        if (oy + 1 < U.oy1) fetch(oy + 1, nxt_a, nxt_r);
        mbar_wait(smem_u32(&acc_full[acc]), (uint32_t)((tile / C::NA) & 1));
        tc_fence_after();
        // the three column groups hold the x0-, x1- and x2-weighted partial sums:
        // sum them while draining TMEM (8 columns of each group per round trip)
        float t[C::NACC][EH];
#pragma unroll
        for (int k = 0; k < C::NACC; ++k)
#pragma unroll
          for (int n0 = 0; n0 < EH; n0 += 8) {
            uint32_t r0[8], r1[8], r2[8];
            const uint32_t col = tmem + ((uint32_t)(q4 * 32) << 16) + acc * C::ACOLS + k * NW + h * EH + n0;
            tmem_ld8(col, r0);
            tmem_ld8(col + CS, r1);
            tmem_ld8(col + 2 * CS, r2);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 8; j += 2) {  // (x0 + x1) + x2 partial sums, channel pairs packed (FADD2)
              const uint64_t s = add2(add2(pk2(r0[j], r0[j + 1]), pk2(r1[j], r1[j + 1])), pk2(r2[j], r2[j + 1]));
              t[k][n0 + j] = __uint_as_float((uint32_t)s);
              t[k][n0 + j + 1] = __uint_as_float((uint32_t)(s >> 32));
            }
          }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&acc_empty[acc]));  // TMEM free; finish from registers
        if (TR2 && tr && !(kProbe & 4)) {
          // chunks A, B (column 2m: channels 0-3, 4-7 of the half) and C, D (column 2m + 1)
          float4 ch[4];
#pragma unroll
          for (int k = 0; k < 2; ++k)
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const int k2 = k % C::NACC;
              const float4 bs = *reinterpret_cast<const float4*>(s_bias + h * EH + 4 * q);
              const uint64_t o01 = add2(pkf(t[k2][4 * q], t[k2][4 * q + 1]), pkf(bs.x, bs.y));
              const uint64_t o23 = add2(pkf(t[k2][4 * q + 2], t[k2][4 * q + 3]), pkf(bs.z, bs.w));
              float4 o = make_float4(lo_f(o01), hi_f(o01), lo_f(o23), hi_f(o23));
              if (a.softplus) {
                o.x = softplus_fast(o.x);
                o.y = softplus_fast(o.y);
                o.z = softplus_fast(o.z);
                o.w = softplus_fast(o.w);
              }
              ch[2 * k + q] = o;
            }
          // even lane keeps A, C and receives the odd lane's A, C; odd keeps B, D and receives the even's
          float4 s0 = pi ? ch[0] : ch[1], s1 = pi ? ch[2] : ch[3], g0, g1;
          g0.x = __shfl_xor_sync(0xffffffffu, s0.x, 1);
          g0.y = __shfl_xor_sync(0xffffffffu, s0.y, 1);
          g0.z = __shfl_xor_sync(0xffffffffu, s0.z, 1);
          g0.w = __shfl_xor_sync(0xffffffffu, s0.w, 1);
          g1.x = __shfl_xor_sync(0xffffffffu, s1.x, 1);
          g1.y = __shfl_xor_sync(0xffffffffu, s1.y, 1);
          g1.z = __shfl_xor_sync(0xffffffffu, s1.z, 1);
          g1.w = __shfl_xor_sync(0xffffffffu, s1.w, 1);
          float4 outv[4];  // chunk pi of output columns P .. P + 3
          outv[0] = pi ? g0 : ch[0];
          outv[1] = pi ? g1 : ch[2];
          outv[2] = pi ? ch[1] : g0;
          outv[3] = pi ? ch[3] : g1;
          const size_t prow = (size_t)oy * a.Wo + 2 * (U.xb * MT + m - pi);
          float* yb = a.y + (size_t)U.b * a.Ho * a.Wo * COUT + n_base + 4 * pi;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float4 ad = pre_a[(j >> 1) % C::NACC][(j & 1) % (EH / 4)];
            const float4 rs = SPLIT ? pre_r[SPLIT ? (j >> 1) % RK : 0][SPLIT ? (j & 1) % RQ : 0]
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
            const uint64_t a01 = add2(pkf(ad.x, ad.y), pkf(rs.x, rs.y)), a23 = add2(pkf(ad.z, ad.w), pkf(rs.z, rs.w));
            const uint64_t q01 = add2(pkf(outv[j].x, outv[j].y), a01), q23 = add2(pkf(outv[j].z, outv[j].w), a23);
            if (!(kProbe & 64))
              *reinterpret_cast<float4*>(yb + (prow + j) * COUT) = make_float4(lo_f(q01), hi_f(q01), lo_f(q23), hi_f(q23));
          }
        } else if (TR && tr && !(kProbe & 4)) {
          float4 ch[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float4 bs = *reinterpret_cast<const float4*>(s_bias + h * EH + 4 * q);
            const uint64_t o01 = add2(pkf(t[0][4 * q], t[0][4 * q + 1]), pkf(bs.x, bs.y));
            const uint64_t o23 = add2(pkf(t[0][4 * q + 2], t[0][4 * q + 3]), pkf(bs.z, bs.w));
            float4 o = make_float4(lo_f(o01), hi_f(o01), lo_f(o23), hi_f(o23));
            if (a.softplus) {
              o.x = softplus_fast(o.x);
              o.y = softplus_fast(o.y);
              o.z = softplus_fast(o.z);
              o.w = softplus_fast(o.w);
            }
            ch[q] = o;
          }
          group4_transpose(ch, gi);
          const size_t gpix = (size_t)oy * a.Wo + U.xb * MT + m - gi;
          float* yb = a.y + (size_t)U.b * a.Ho * a.Wo * COUT + n_base + 4 * gi;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float4 ad = pre_a[0][j];
            const float4 rs = SPLIT ? pre_r[0][SPLIT ? j : 0] : make_float4(0.f, 0.f, 0.f, 0.f);
            const uint64_t a01 = add2(pkf(ad.x, ad.y), pkf(rs.x, rs.y)), a23 = add2(pkf(ad.z, ad.w), pkf(rs.z, rs.w));
            const uint64_t q01 = add2(pkf(ch[j].x, ch[j].y), a01), q23 = add2(pkf(ch[j].z, ch[j].w), a23);
            if (lane_ok && !(kProbe & 64))
              *reinterpret_cast<float4*>(yb + (gpix + j) * COUT) = make_float4(lo_f(q01), hi_f(q01), lo_f(q23), hi_f(q23));
          }
        } else if (lane_ok && !(kProbe & 4)) {
#pragma unroll
          for (int k = 0; k < C::NACC; ++k) {
            const int ox = MODE == 2 ? 2 * (U.xb * MT + m) + k : U.xb * MT + m;
            const size_t pix = (size_t)oy * a.Wo + ox;
            const size_t obase = (size_t)U.b * a.Ho * a.Wo * COUT + pix * COUT + n_base;
#pragma unroll
            for (int n0 = 0; n0 < EH; n0 += 4) {
              const float4 bs = *reinterpret_cast<const float4*>(s_bias + h * EH + n0);
              const uint64_t o01 = add2(pkf(t[k][n0], t[k][n0 + 1]), pkf(bs.x, bs.y));
              const uint64_t o23 = add2(pkf(t[k][n0 + 2], t[k][n0 + 3]), pkf(bs.z, bs.w));
              float4 o = make_float4(lo_f(o01), hi_f(o01), lo_f(o23), hi_f(o23));
              if (a.softplus) {
                o.x = softplus_fast(o.x);
                o.y = softplus_fast(o.y);
                o.z = softplus_fast(o.z);
                o.w = softplus_fast(o.w);
              }
              const float4 ad = pre_a[k][n0 / 4];
              const float4 rs = SPLIT ? pre_r[SPLIT ? k : 0][SPLIT ? n0 / 4 : 0] : make_float4(0.f, 0.f, 0.f, 0.f);
              {  // o + (addend + residual), packed
                const uint64_t a01 = add2(pkf(ad.x, ad.y), pkf(rs.x, rs.y)), a23 = add2(pkf(ad.z, ad.w), pkf(rs.z, rs.w));
                const uint64_t q01 = add2(pkf(o.x, o.y), a01), q23 = add2(pkf(o.z, o.w), a23);
                o = make_float4(lo_f(q01), hi_f(q01), lo_f(q23), hi_f(q23));
              }
              if (a.planar) {  // two complex channels, each a coalesced float2 plane store
                float2* yp = reinterpret_cast<float2*>(a.y) +
                             ((size_t)U.b * (COUT / 2) + (n_base + n0) / 2) * ((size_t)a.Ho * a.Wo) + pix;
                yp[0] = make_float2(o.x, o.y);
                yp[(size_t)a.Ho * a.Wo] = make_float2(o.z, o.w);
              } else if (!(kProbe & 64)) {
                *reinterpret_cast<float4*>(a.y + obase + n0) = o;
              }
            }
          }
        }
#pragma unroll
        for (int k = 0; k < C::NACC; ++k)
#pragma unroll
          for (int q = 0; q < EH / 4; ++q) {
            pre_a[k][q] = nxt_a[k][q];
            if constexpr (SPLIT) pre_r[k][q] = nxt_r[k][q];
          }
      }
    }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::NCOLS));
  }
}

template <int CIN, int COUT, int MODE, int MT, int CS>
void launch_tc(const TcArgs& a, cudaStream_t st) {
  using C = Cfg<CIN, COUT, MODE, MT, CS>;
  static_assert(C::TOTAL <= kSmemMax, "shared memory budget");
  static_assert(C::NCOLS_RAW <= 512, "TMEM budget");
  static_assert(COUT % CS == 0 && CS % 16 == 0, "cout slices");
  static int sms = 0;
  if (!sms) {
    cudaFuncSetAttribute(k_conv_tc<CIN, COUT, MODE, MT, CS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)C::TOTAL);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  long long grid = (sms / C::NSPLIT) * C::NSPLIT;  // a multiple of NSPLIT: fixed slice per CTA
  // Band height: tall bands re-read fewer halo rows, but units are handed out
  // round-robin, so with few units per CTA the last wave idles.  Halve the band
  // (down to 8 rows) until the RHS still iterating give every CTA >= 6 units.
  TcArgs b = a;
  const double act = prof::active_hint(a.B);
  const int xblocks = MODE == 2 ? a.W / MT : a.Wo / MT;
  b.band = HS_TC_BAND_MAX;
  while (b.band > 8 && C::NSPLIT * act * xblocks * ((a.Ho + b.band - 1) / b.band) < 6.0 * grid) b.band /= 2;
  const long long nunits = num_units<MODE, MT>(b, C::NSPLIT);
  if (nunits < grid) grid = nunits;
  constexpr bool pdl = HS_TC_PDL != 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(C::NT);
  cfg.dynamicSmemBytes = C::TOTAL;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, k_conv_tc<CIN, COUT, MODE, MT, CS>, b);
}

// (cin, cout, mode) -> cout slice per CTA, or 0 if not on the tensor-core path
int slice_for(int cin, int cout, int mode) {
  if (mode == 0 && cin == 16 && cout == 16) return 16;
  if (mode == 0 && cin == 32 && cout == 32) return 32;
  if (mode == 0 && cin == 64 && cout == 64) return 32;
  if (mode == 1 && cin == 16 && cout == 32) return 32;
  if (mode == 1 && cin == 32 && cout == 64) return 32;
  if (mode == 2 && cin == 32 && cout == 16) return 16;
  if (mode == 2 && cin == 64 && cout == 32) return 32;
  return 0;
}

}  // namespace

bool conv_tc_enabled = true;

bool conv_tc_supported(int cin, int cout, int stride, int transposed, int H, int W, int Wo, int planar) {
  (void)H;
  if (!conv_tc_enabled) return false;
  const int mode = transposed ? 2 : (stride == 2 ? 1 : 0);
  const int width = mode == 2 ? W : Wo;
  if (!planar && mode == 0 && cin == cout && ((HS_TC_SHIFT && cin == 16) || (HS_TC_SHIFT32 && cin == 32)))
    return true;  // conv_shift.cu: 30-pixel segments, any width
  if (HS_TC_SHIFT_S2 && !planar && mode == 1 && cin == 16 && cout == 32) return true;
  if (HS_TC_SHIFT_T && !planar && mode == 2 && cin == 32 && cout == 16) return true;
  if (HS_TC_SHIFT_T64 && !planar && mode == 2 && cin == 64 && cout == 32) return true;
  if (width % 64) return false;
  return slice_for(cin, cout, mode) > 0;
}

bool conv_tc_launch(const float* x, int H, int W, int cin, float* y, int Ho, int Wo, int cout, int stride,
                    int transposed, const float* w, const float* bias, int softplus, const float* addend,
                    long long addend_bstride, int addend_per_model, const int* model_of, const float* residual,
                    const void* const* active, int B, cudaStream_t st, int planar) {
  TcArgs a{x, H, W, y, Ho, Wo, w, bias, softplus, addend, addend_bstride, addend_per_model, model_of, residual,
           active, B, 32, planar};
  const int mode = transposed ? 2 : (stride == 2 ? 1 : 0);
  if (!planar && !kProbe && mode == 0 && cin == cout && ((HS_TC_SHIFT && cin == 16) || (HS_TC_SHIFT32 && cin == 32)))
    return conv_shift_launch(cin, x, H, W, y, w, bias, softplus, addend, addend_bstride, addend_per_model, model_of,
                             residual, active, B, st);
  if (HS_TC_SHIFT_S2 && !planar && !kProbe && mode == 1 && cin == 16 && cout == 32)
    return conv_shift_s2_launch(x, H, W, y, Ho, Wo, w, bias, softplus, addend, addend_bstride, addend_per_model,
                                model_of, residual, active, B, st);
  if (!planar && !kProbe && mode == 2 && ((HS_TC_SHIFT_T && cin == 32 && cout == 16) || (HS_TC_SHIFT_T64 && cin == 64 && cout == 32)))
    return conv_shift_t_launch(cin, x, H, W, y, w, bias, softplus, addend, addend_bstride, addend_per_model, model_of,
                               residual, active, B, st);
  const bool m128 = ((mode == 2 ? W : Wo) % 128) == 0 && !(kProbe & 32);
#define HS_TC(CI, CO, MD, CSL)                                           \
  if (mode == MD && cin == CI && cout == CO) {                           \
    if (m128) launch_tc<CI, CO, MD, 128, CSL>(a, st);                    \
    else launch_tc<CI, CO, MD, 64, CSL>(a, st);                          \
    return true;                                                         \
  }
  HS_TC(16, 16, 0, 16)
  HS_TC(32, 32, 0, 32)
  HS_TC(16, 32, 1, 32)
  HS_TC(32, 16, 2, 16)
  // 64-channel inputs / outputs: M = 64 tiles only (the M = 128 staging does not fit next to the weights)
  if (mode == 0 && cin == 64 && cout == 64) return launch_tc<64, 64, 0, 64, 32>(a, st), true;
  if (mode == 1 && cin == 32 && cout == 64) return launch_tc<32, 64, 1, 64, 32>(a, st), true;
  if (mode == 2 && cin == 64 && cout == 32) return launch_tc<64, 32, 2, 64, 32>(a, st), true;
#undef HS_TC
  return false;
}

}  // namespace hs
