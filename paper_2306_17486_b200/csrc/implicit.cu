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
#include <cooperative_groups.h>

#include <cstdlib>

#include "common.cuh"
#include "implicit.h"

namespace hs {
namespace {

constexpr int kImpThreads = 256;

HS_DEV int br5(int l) { return __brev(l) >> 27; }

// a * W_E^m, W_E = exp(-2 pi i / E), E in {2, 4, 8, 16}, m a compile-time constant
// after unrolling: multiples of pi/2 are swaps / negations, odd multiples of
// pi/4 one scaled add (no multiplications by 0 or 1 survive), odd multiples of
// pi/8 (E = 16) one complex multiply by a constant
template <int E>
HS_DEV float2 mul_wE(float2 a, int m) {
  if constexpr (E == 16) {
    const int k = m & 15;
    if ((k & 1) == 0) return mul_wE<8>(a, k >> 1);
    constexpr float C1 = 0.92387953251128675613f, S1 = 0.38268343236508977173f;  // cos, sin of pi/8
    float c, sn;
    switch (k) {  // W_16^k = cos(pi k / 8) - i sin(pi k / 8)
      case 1: c = C1, sn = S1; break;
      case 3: c = S1, sn = C1; break;
      case 5: c = -S1, sn = C1; break;
      case 7: c = -C1, sn = S1; break;
      case 9: c = -C1, sn = -S1; break;
      case 11: c = -S1, sn = -C1; break;
      case 13: c = S1, sn = -C1; break;
      default: c = C1, sn = -S1; break;
    }
    return make_float2(a.x * c + a.y * sn, a.y * c - a.x * sn);
  } else {
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

// ---------------------------------------------------------------------------------------------
// Four-step variant for square grids (N = 32 E, E in {2, 4}): a line of N points is split as
// n = l + 32 j (l < 32, j < E) and k = k1 + E m (k1 < E, m < 32):
//   X[k1 + E m] = sum_l W_32^(l m) [ W_N^(l k1) sum_j x[l + 32 j] W_E^(j k1) ]
// Step (a): one warp per line, lane l does the E-point DFT over j and the twiddle (registers).
// Step (c): one THREAD per (line, k1) does the 32-point DFT over l entirely in registers
// (radix-2, compile-time twiddles), through a padded shared-memory transpose.  No shuffles:
// the warp-shuffle version spends most of its issue slots on the 5 cross-lane stages.
// The column pass runs forward FFT, spectrum multiply and inverse FFT in the same thread's
// registers; all data stay in natural frequency order (the spectrum is used as stored).

// a * W_32^(+-k) for a compile-time k in [0, 16)
template <bool INV>
HS_DEV float2 tw32(float2 a, int k) {
  constexpr float C[9] = {1.f,
                          0.98078528040323044913f,
                          0.92387953251128675613f,
                          0.83146961230254523708f,
                          0.70710678118654752440f,
                          0.55557023301960222474f,
                          0.38268343236508977173f,
                          0.19509032201612826785f,
                          0.f};
  if (k == 0) return a;
  if (k == 8) return INV ? make_float2(-a.y, a.x) : make_float2(a.y, -a.x);
  const float c = k < 8 ? C[k] : -C[16 - k];
  const float sn = k < 8 ? C[8 - k] : C[k - 8];  // sin(pi k / 16)
  // W^k = c - i sn (forward), c + i sn (inverse)
  return INV ? make_float2(a.x * c - a.y * sn, a.y * c + a.x * sn) : make_float2(a.x * c + a.y * sn, a.y * c - a.x * sn);
}

HS_DEV constexpr int brev5(int m) {
  return ((m & 1) << 4) | ((m & 2) << 2) | (m & 4) | ((m & 8) >> 2) | ((m & 16) >> 4);
}

// in-place 32-point DFT of v (natural order in, natural order out), unnormalised
template <bool INV>
HS_DEV void fft32(float2 (&v)[32]) {
#pragma unroll
  for (int hs = 16; hs >= 1; hs >>= 1) {  // radix-2 DIF stages
#pragma unroll
    for (int blk = 0; blk < 32; blk += 2 * hs)
#pragma unroll
      for (int j = 0; j < hs; ++j) {
        const float2 a = v[blk + j], b = v[blk + j + hs];
        v[blk + j] = cadd(a, b);
        v[blk + j + hs] = tw32<INV>(csub(a, b), j * (16 / hs));
      }
  }
  // bit-reversed -> natural (a compile-time register permutation)
  float2 t[32];
#pragma unroll
  for (int m = 0; m < 32; ++m) t[m] = v[brev5(m)];
#pragma unroll
  for (int m = 0; m < 32; ++m) v[m] = t[m];
}

template <int E>
struct Imp2 {
  static constexpr int THREADS = 128;
  static constexpr int N = 32 * E, h = N / 2, NZ = E / 2, LD = N + 1, TL = 33, LINES = THREADS / E;
  static constexpr size_t SMEM = ((size_t)h * LD + (size_t)LINES * E * TL + N) * sizeof(float2);
};

template <int E>
__global__ void __launch_bounds__(Imp2<E>::THREADS) k_implicit2(ImpArgs a) {
  using G = Imp2<E>;
  constexpr int N = G::N, h = G::h, NZ = G::NZ, LD = G::LD, TL = G::TL, LINES = G::LINES, NT = G::THREADS;
  constexpr int NW = NT / 32;
  extern __shared__ float2 smem_imp2[];
  float2* S = smem_imp2;           // [h][LD]  row spectra (rows >= h of the padded input are zero)
  float2* T = S + h * LD;          // [E][LINES][TL] transpose buffer
  float2* tw = T + LINES * E * TL; // W_N^m
  const int b = blockIdx.y, k = blockIdx.x;
  if (a.active && a.active[b] == nullptr) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int m = threadIdx.x; m < N; m += NT) {
    float sn, cs;
    sincospif(-2.f * m / N, &sn, &cs);
    tw[m] = make_float2(cs, sn);
  }
  const float2* xin = a.x + b * a.xb + k * a.xk;
  float2* yout = a.y + b * a.yb + k * a.yk;
  const float2* sp = a.spec + (long long)k * N * N;
  const int tk = threadIdx.x / LINES, tl = threadIdx.x % LINES;  // step (c): (k1, line), lines fastest (banks)
  __syncthreads();
  // step (a) forward on a line held as q[j] = x[lane + 32 j] (j < NZ non-zero) -> T line
  auto fwd_a = [&](float2(&q)[E], int line) {
#pragma unroll
    for (int k1 = 0; k1 < E; ++k1) {
      float2 s = q[0];
#pragma unroll
      for (int j = 1; j < NZ; ++j) s = cadd(s, mul_wE<E>(q[j], j * k1));
      T[(k1 * LINES + line) * TL + lane] = k1 == 0 ? s : cmul(s, tw[lane * k1]);
    }
  };
  // step (a) inverse: T line -> q[j] = N x[lane + 32 j] for j < NZ
  auto inv_a = [&](float2(&q)[E], int line) {
    float2 y[E];
#pragma unroll
    for (int k1 = 0; k1 < E; ++k1) {
      y[k1] = T[(k1 * LINES + line) * TL + lane];
      if (k1) y[k1] = cmulc(y[k1], tw[lane * k1]);
    }
#pragma unroll
    for (int j = 0; j < NZ; ++j) {
      float2 s = y[0];
#pragma unroll
      for (int k1 = 1; k1 < E; ++k1) s = cadd(s, mul_wE<E>(y[k1], (E - (j * k1) % E) % E));
      q[j] = s;
    }
  };
  // 1. forward row transforms (h rows, LINES per chunk).  All of a warp's rows of a
  // chunk are loaded together, and the next chunk's rows are requested before this
  // chunk's barrier and step (c), so their latency overlaps the FFT work.
  constexpr int RPW = LINES / NW;
  float2 q[RPW][E];
  auto load_rows = [&](int r0) {
    const int nl = min(LINES, h - r0);
#pragma unroll
    for (int i = 0; i < RPW; ++i) {
      const int rr = warp + i * NW;
#pragma unroll
      for (int j = 0; j < E; ++j)
        q[i][j] = (j < NZ && rr < nl) ? xin[(long long)((r0 + rr) * h + lane + 32 * j) * a.xp] : make_float2(0.f, 0.f);
    }
  };
  load_rows(0);
  for (int r0 = 0; r0 < h; r0 += LINES) {
    const int nl = min(LINES, h - r0);
#pragma unroll
    for (int i = 0; i < RPW; ++i)
      if (warp + i * NW < nl) fwd_a(q[i], warp + i * NW);
    if (r0 + LINES < h) load_rows(r0 + LINES);
    __syncthreads();
    if (tl < nl) {
      float2 v[32];
#pragma unroll
      for (int l = 0; l < 32; ++l) v[l] = T[(tk * LINES + tl) * TL + l];
      fft32<false>(v);
#pragma unroll
      for (int m = 0; m < 32; ++m) S[(r0 + tl) * LD + tk + E * m] = v[m];
    }
    __syncthreads();
  }
  // 2. columns: forward, spectrum, inverse (rows < h kept)
  for (int c0 = 0; c0 < N; c0 += LINES) {
    const int nl = min(LINES, N - c0);
    // this thread's 32 spectrum values, requested before step (a) and the barrier
    // (the compiler does not move loads across __syncthreads; shared memory, not
    // registers, bounds this kernel's occupancy)
    float2 spv[32];
    if (tl < nl) {
      const float2* spc = sp + c0 + tl;
#pragma unroll
      for (int m = 0; m < 32; ++m) spv[m] = __ldg(spc + (long long)(tk + E * m) * N);
    }
    for (int cc = warp; cc < nl; cc += NW) {
      float2 q[E];
#pragma unroll
      for (int j = 0; j < E; ++j) q[j] = j < NZ ? S[(lane + 32 * j) * LD + c0 + cc] : make_float2(0.f, 0.f);
      fwd_a(q, cc);
    }
    __syncthreads();
    if (tl < nl) {
      float2 v[32];
#pragma unroll
      for (int l = 0; l < 32; ++l) v[l] = T[(tk * LINES + tl) * TL + l];
      fft32<false>(v);
#pragma unroll
      for (int m = 0; m < 32; ++m) v[m] = cmul(v[m], spv[m]);
      fft32<true>(v);
#pragma unroll
      for (int l = 0; l < 32; ++l) T[(tk * LINES + tl) * TL + l] = v[l];
    }
    __syncthreads();
    for (int cc = warp; cc < nl; cc += NW) {
      float2 q[E];
      inv_a(q, cc);
#pragma unroll
      for (int j = 0; j < NZ; ++j) S[(lane + 32 * j) * LD + c0 + cc] = q[j];
    }
    __syncthreads();
  }
  // 3. inverse row transforms (columns < h kept), 1 / N^2
  const float inv = 1.f / ((float)N * (float)N);
  for (int r0 = 0; r0 < h; r0 += LINES) {
    const int nl = min(LINES, h - r0);
    if (tl < nl) {
      float2 v[32];
#pragma unroll
      for (int m = 0; m < 32; ++m) v[m] = S[(r0 + tl) * LD + tk + E * m];
      fft32<true>(v);
#pragma unroll
      for (int l = 0; l < 32; ++l) T[(tk * LINES + tl) * TL + l] = v[l];
    }
    __syncthreads();
    for (int rr = warp; rr < nl; rr += NW) {
      float2 q[E];
      inv_a(q, rr);
#pragma unroll
      for (int j = 0; j < NZ; ++j)
        yout[(long long)((r0 + rr) * h + lane + 32 * j) * a.yp] = make_float2(q[j].x * inv, q[j].y * inv);
    }
    __syncthreads();
  }
}

template <int E>
void launch_imp2(const ImpArgs& a, int B, cudaStream_t st) {
  const size_t sm = Imp2<E>::SMEM;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_implicit2<E>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    attr = true;
  }
  k_implicit2<E><<<dim3((unsigned)a.C, (unsigned)B), Imp2<E>::THREADS, sm, st>>>(a);
}

// ---------------------------------------------------------------------------------------------
// Four-step transform on a 2-CTA cluster (rectangular grids, and 128 x 128): the (RHS, channel)
// pair is split by spectrum COLUMNS between the two CTAs of a cluster, so each CTA keeps only
// h x (W2 / 2) row spectra in shared memory (the single-CTA kernels keep h x W2, which left 8 warps
// per SM at C3's 64 x 128 coarsest grid and did not fit 128 x 128 at all).
//   1. CTA r transforms the rows [r h/2, (r+1) h/2) (four-step, length W2 = 32 EW); each thread's
//      32 outputs are column frequencies k1 + EW m, written to the owning CTA's shared memory
//      (distributed shared memory for the partner's half)                       -> cluster barrier
//   2. each CTA runs forward column FFT, spectrum multiply, inverse column FFT on its W2 / 2 columns
//      (length H2 = 32 EH, h rows kept), all local                               -> cluster barrier
//   3. CTA r inverse-transforms its rows, reading the partner's columns through DSMEM, and writes
//      the w kept outputs                                                         -> cluster barrier
// The spectrum is used in its natural [C][H2][W2] order, like k_implicit2.
template <int EW, int EH, int NCL>
struct ImpC {
  static constexpr int THREADS = 128, NWARP = THREADS / 32;
  static constexpr int W2 = 32 * EW, H2 = 32 * EH, h = H2 / 2, w = W2 / 2;
  static constexpr int HALF = W2 / NCL, LDS = HALF + 1;  // columns per CTA, S row pitch (odd: conflict-free)
  static constexpr int HR = h / NCL;                     // rows per CTA in the row passes
  static constexpr int RL = THREADS / EW, CL = THREADS / EH, TL = 33;
  static constexpr size_t SMEM = ((size_t)h * LDS + (size_t)THREADS * TL + W2 + H2) * sizeof(float2);
};

template <int EW, int EH, int NCL>
__global__ void __cluster_dims__(NCL, 1, 1) __launch_bounds__(ImpC<EW, EH, NCL>::THREADS) k_implicit_cl(ImpArgs a) {
  using G = ImpC<EW, EH, NCL>;
  constexpr int W2 = G::W2, H2 = G::H2, h = G::h, HALF = G::HALF, LDS = G::LDS, RL = G::RL, CL = G::CL,
                TL = G::TL, NT = G::THREADS, NWP = G::NWARP;
  constexpr int NZW = EW / 2, NZH = EH / 2;  // non-zero 32-blocks of a padded row / column
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int r = (int)cluster.block_rank();
  extern __shared__ float2 smem_cl[];
  float2* S = smem_cl;                      // [h][LDS]: this CTA's HALF spectrum columns, all rows
  float2* T = S + h * LDS;                  // [E][lines][TL] four-step transpose buffer
  float2* twW = T + NT * TL;                // W_W2^m
  float2* twH = twW + W2;                   // W_H2^m
  float2* Sp[NCL];  // every CTA's column slice
#pragma unroll
  for (int q = 0; q < NCL; ++q) Sp[q] = q == r ? S : cluster.map_shared_rank(S, q);
  const int b = blockIdx.y, k = blockIdx.x / NCL;
  const bool skip = a.active && a.active[b] == nullptr;  // both CTAs of the pair agree
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int m = threadIdx.x; m < W2; m += NT) {
    float sn, cs;
    sincospif(-2.f * m / W2, &sn, &cs);
    twW[m] = make_float2(cs, sn);
  }
  for (int m = threadIdx.x; m < H2; m += NT) {
    float sn, cs;
    sincospif(-2.f * m / H2, &sn, &cs);
    twH[m] = make_float2(cs, sn);
  }
  __syncthreads();
  if (!skip) {
    const float2* xin = a.x + b * a.xb + k * a.xk;
    const int row0 = r * G::HR;
    // ---- 1. forward row transforms of rows [row0, row0 + HR)
    for (int c0 = 0; c0 < G::HR; c0 += RL) {
      const int nl = min(RL, G::HR - c0);  // rows of this chunk (RL may exceed the CTA's HR rows)
      for (int line = warp; line < nl; line += NWP) {  // step (a): E-point DFT over j, twiddle
        const int row = row0 + c0 + line;
        float2 q[EW];
#pragma unroll
        for (int j = 0; j < EW; ++j)
          q[j] = j < NZW ? xin[(long long)(row * G::w + lane + 32 * j) * a.xp] : make_float2(0.f, 0.f);
#pragma unroll
        for (int k1 = 0; k1 < EW; ++k1) {
          float2 sm = q[0];
#pragma unroll
          for (int j = 1; j < NZW; ++j) sm = cadd(sm, mul_wE<EW>(q[j], j * k1));
          T[(k1 * RL + line) * TL + lane] = k1 == 0 ? sm : cmul(sm, twW[lane * k1]);
        }
      }
      __syncthreads();
      if (threadIdx.x % RL < nl) {  // step (c): 32-point DFT over l per (k1, line); column f = k1 + EW m
        const int tk = threadIdx.x / RL, tl = threadIdx.x % RL;
        float2 v[32];
#pragma unroll
        for (int l = 0; l < 32; ++l) v[l] = T[(tk * RL + tl) * TL + l];
        fft32<false>(v);
        const int row = row0 + c0 + tl;
#pragma unroll
        for (int m = 0; m < 32; ++m) {
          const int f = tk + EW * m;
          Sp[f / HALF][row * LDS + f % HALF] = v[m];
        }
      }
      __syncthreads();
    }
  }
  cluster.sync();  // every row spectrum is in its owner's shared memory
  if (!skip) {
    // ---- 2. this CTA's columns: forward, spectrum, inverse (rows < h kept)
    const float2* sp = a.spec + (long long)k * H2 * W2;
    const int tk = threadIdx.x / CL, tl = threadIdx.x % CL;
    static_assert(HALF % CL == 0, "column chunks");
    for (int c0 = 0; c0 < HALF; c0 += CL) {
      float2 spv[32];  // requested before the barrier
      {
        const float2* spc = sp + r * HALF + c0 + tl;
#pragma unroll
        for (int m = 0; m < 32; ++m) spv[m] = __ldg(spc + (long long)(tk + EH * m) * W2);
      }
      for (int cc = warp; cc < CL; cc += NWP) {
        float2 q[EH];
#pragma unroll
        for (int j = 0; j < EH; ++j) q[j] = j < NZH ? S[(lane + 32 * j) * LDS + c0 + cc] : make_float2(0.f, 0.f);
#pragma unroll
        for (int k1 = 0; k1 < EH; ++k1) {
          float2 sm = q[0];
#pragma unroll
          for (int j = 1; j < NZH; ++j) sm = cadd(sm, mul_wE<EH>(q[j], j * k1));
          T[(k1 * CL + cc) * TL + lane] = k1 == 0 ? sm : cmul(sm, twH[lane * k1]);
        }
      }
      __syncthreads();
      {
        float2 v[32];
#pragma unroll
        for (int l = 0; l < 32; ++l) v[l] = T[(tk * CL + tl) * TL + l];
        fft32<false>(v);
#pragma unroll
        for (int m = 0; m < 32; ++m) v[m] = cmul(v[m], spv[m]);
        fft32<true>(v);
#pragma unroll
        for (int l = 0; l < 32; ++l) T[(tk * CL + tl) * TL + l] = v[l];
      }
      __syncthreads();
      for (int cc = warp; cc < CL; cc += NWP) {  // inverse step (a): rows < h kept
        float2 y[EH];
#pragma unroll
        for (int k1 = 0; k1 < EH; ++k1) {
          y[k1] = T[(k1 * CL + cc) * TL + lane];
          if (k1) y[k1] = cmulc(y[k1], twH[lane * k1]);
        }
#pragma unroll
        for (int j = 0; j < NZH; ++j) {
          float2 sm = y[0];
#pragma unroll
          for (int k1 = 1; k1 < EH; ++k1) sm = cadd(sm, mul_wE<EH>(y[k1], (EH - (j * k1) % EH) % EH));
          S[(lane + 32 * j) * LDS + c0 + cc] = sm;
        }
      }
      __syncthreads();
    }
  }
  cluster.sync();  // both halves of every kept row are final
  if (!skip) {
    // ---- 3. inverse row transforms of this CTA's rows, the partner's columns through DSMEM
    float2* yout = a.y + b * a.yb + k * a.yk;
    const float inv = 1.f / ((float)H2 * (float)W2);
    const int row0 = r * G::HR;
    const int tk = threadIdx.x / RL, tl = threadIdx.x % RL;
    for (int c0 = 0; c0 < G::HR; c0 += RL) {
      const int nl = min(RL, G::HR - c0);
      if (tl < nl) {
        const int row = row0 + c0 + tl;
        float2 v[32];
#pragma unroll
        for (int m = 0; m < 32; ++m) {
          const int f = tk + EW * m;
          v[m] = Sp[f / HALF][row * LDS + f % HALF];
        }
        fft32<true>(v);
#pragma unroll
        for (int l = 0; l < 32; ++l) T[(tk * RL + tl) * TL + l] = v[l];
      }
      __syncthreads();
      for (int line = warp; line < nl; line += NWP) {
        const int row = row0 + c0 + line;
        float2 y[EW];
#pragma unroll
        for (int k1 = 0; k1 < EW; ++k1) {
          y[k1] = T[(k1 * RL + line) * TL + lane];
          if (k1) y[k1] = cmulc(y[k1], twW[lane * k1]);
        }
#pragma unroll
        for (int j = 0; j < NZW; ++j) {
          float2 sm = y[0];
#pragma unroll
          for (int k1 = 1; k1 < EW; ++k1) sm = cadd(sm, mul_wE<EW>(y[k1], (EW - (j * k1) % EW) % EW));
          yout[(long long)(row * G::w + lane + 32 * j) * a.yp] = make_float2(sm.x * inv, sm.y * inv);
        }
      }
      __syncthreads();
    }
  }
  cluster.sync();  // the partner may still be reading this CTA's shared memory
}

template <int EW, int EH, int NCL>
void launch_imp_cl(const ImpArgs& a, int B, cudaStream_t st) {
  using G = ImpC<EW, EH, NCL>;
  static_assert(G::HR % 1 == 0 && G::h % NCL == 0 && G::HALF % G::CL == 0, "cluster split");
  const size_t sm = G::SMEM;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_implicit_cl<EW, EH, NCL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    attr = true;
  }
  k_implicit_cl<EW, EH, NCL><<<dim3(NCL * (unsigned)a.C, (unsigned)B), G::THREADS, sm, st>>>(a);
}

// the cluster kernel: non-square grids with sides in {32, 64, 128}, 128 x 128 (2-CTA clusters), and
// the 128 x 256 coarsest grid of C4 / C5 (512-point rows, 4-CTA clusters)
bool use_cl(int h, int w) {
  if ((h == 128 && w == 256) || (h == 256 && w == 128)) return true;
  auto ok = [](int n) { return n == 32 || n == 64 || n == 128; };
  return ok(h) && ok(w) && (h != w || h == 128) && !(h == 128 && w == 32) && !(h == 32 && w == 128);
}

// the four-step kernel where it applies (square 64^2 / 128^2 padded grids)
bool use_v2(int h, int w) { return h == w && (h == 32 || h == 64); }

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
  if (use_cl(h, w)) return true;
  auto ok = [](int n) { return n == 32 || n == 64 || n == 128; };  // E = 2n / 32 in {2, 4, 8}
  return ok(h) && ok(w) && (use_v2(h, w) || smem_bytes(h, w) <= 200 * 1024);
}

void implicit_permute_spectrum(const void* spec, void* spec_perm, int C, int h, int w, cudaStream_t st) {
  const long long n = (long long)C * 4 * h * w;
  if (use_v2(h, w) || use_cl(h, w)) {  // the four-step kernels read the natural order
    cudaMemcpyAsync(spec_perm, spec, n * sizeof(float2), cudaMemcpyDeviceToDevice, st);
    return;
  }
  const unsigned g = (unsigned)((n + 255) / 256 > 4096 ? 4096 : (n + 255) / 256);
  k_permute_spec<<<g, 256, 0, st>>>(static_cast<const float2*>(spec), static_cast<float2*>(spec_perm), C, 2 * h,
                                    2 * w);
}

#ifndef HS_IMP_NCL_C3
#define HS_IMP_NCL_C3 2  // CTAs per (RHS, channel) cluster at C3's 64 x 128 grid (measured: 4 is slower, 1.62 vs 1.29 ms)
#endif
int implicit_fused(const void* x, long long xb, long long xk, long long xp, void* y, long long yb, long long yk,
                   long long yp, const void* spec_perm, const void* const* active, int B, int C, int h, int w,
                   cudaStream_t st) {
  if (!implicit_fused_supported(h, w)) return HS_ECONFIG;
  ImpArgs a{static_cast<const float2*>(x), xb, xk, xp, static_cast<float2*>(y), yb, yk, yp,
            static_cast<const float2*>(spec_perm), active, C};
  const int EW = w / 16, EH = h / 16;
  if (use_cl(h, w)) {
#define HS_IMPC(A, Bq, NC) \
  if (EW == A && EH == Bq) return launch_imp_cl<A, Bq, NC>(a, B, st), HS_OK;
    HS_IMPC(8, 4, HS_IMP_NCL_C3)
    HS_IMPC(4, 8, HS_IMP_NCL_C3)
    HS_IMPC(4, 2, 2)
    HS_IMPC(2, 4, 2)
    HS_IMPC(8, 8, 2)
    HS_IMPC(16, 8, 4)
    HS_IMPC(8, 16, 4)
#undef HS_IMPC
  }
  if (use_v2(h, w)) {
    if (EW == 2) return launch_imp2<2>(a, B, st), HS_OK;
    if (EW == 4) return launch_imp2<4>(a, B, st), HS_OK;
  }
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
