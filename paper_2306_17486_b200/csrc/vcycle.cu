// Shifted-Laplacian V(1,1)-cycle kernels (multigrid.py:218-274), batched over
// right-hand sides.  Each non-coarsest level costs two fused, shared-memory
// tiled passes over HBM:
//
//   k_vc_down : u1 = u0 + w_pre (rhs - A u0)/diag       (jacobi_relax, :218-229)
//               res = rhs - A u1                         (:270)
//               coarse_rhs = R res                       (restrict_full_weighting, :64-78)
//   k_vc_up   : u2 = u1 + P e_coarse                     (prolong_bilinear, :81-114, :273)
//               u3 = u2 + w_post (rhs - A u2)/diag       (:274)
//
// u1 is recomputed in k_vc_up instead of being stored (cheaper: it needs only
// rhs, the medium and u0, which k_vc_up reads anyway).
// The coarsest level runs k_coarse_gmres: the reference's 10-step GMRES with
// a damped-Jacobi preconditioner (coarse_solve, :232-244), one CTA per RHS,
// basis kept in an L2-resident workspace, fp64 reductions.
#include <algorithm>
#include <map>
#include <mutex>

#include "common.cuh"
#include "level.cuh"
#include "prof.h"
#include <cooperative_groups.h>

#include "vcycle.h"

namespace hs {

HS_DEV const float2* vin_ptr(const VecIn& v, int b) { return v.tab ? v.tab[b] : v.base + (long long)b * v.bstride; }
HS_DEV float2* vout_ptr(const VecOut& v, int b) { return v.tab ? v.tab[b] : v.base + (long long)b * v.bstride; }

// ------------------------------------------------------------------ row-marching warps
//
// Both legs run one warp per (column block, band of rows): every lane owns two
// adjacent columns (ja even, jb = ja + 1) and the warp marches down the rows,
// keeping the three-row stencil windows of every intermediate (u0, u1 / u2) in
// registers.  Left / right neighbours come from the adjacent lanes by shuffle,
// so each stencil stage shrinks the valid column range by one column per side;
// the warp's outermost lanes are halo lanes whose results are discarded.  Each
// input row is read once per warp (HBM once, the band and column halos hit L2),
// nothing is staged in shared memory and there are no block barriers.

struct Pair {
  float2 a, b;  // columns ja, jb = ja + 1
};

HS_DEV float2 shfl_up1(float2 v) {
  return make_float2(__shfl_up_sync(0xffffffffu, v.x, 1), __shfl_up_sync(0xffffffffu, v.y, 1));
}
HS_DEV float2 shfl_dn1(float2 v) {
  return make_float2(__shfl_down_sync(0xffffffffu, v.x, 1), __shfl_down_sync(0xffffffffu, v.y, 1));
}

// row i of a field at the lane's two columns, zero outside the grid, times s
HS_DEV Pair ld_pair(const float2* __restrict__ g, int nx, int ny, int i, int ja, float s) {
  Pair r{make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
  if (i >= 0 && i < nx) {
    const float2* p = g + (long long)i * ny;
    if (ja >= 0 && ja < ny) r.a = cscale(p[ja], s);
    if (ja + 1 >= 0 && ja + 1 < ny) r.b = cscale(p[ja + 1], s);
  }
  return r;
}

HS_DEV float2 sum4(float2 a, float2 b, float2 c, float2 d) {
  return make_float2((a.x + b.x) + (c.x + d.x), (a.y + b.y) + (c.y + d.y));
}

// neighbour sums of row i at both columns from rows up = i-1, mid = i, dn = i+1
HS_DEV Pair nbsum_pair(const Pair& up, const Pair& mid, const Pair& dn) {
  const float2 left = shfl_up1(mid.b), right = shfl_dn1(mid.a);
  return Pair{sum4(up.a, dn.a, mid.b, left), sum4(up.b, dn.b, right, mid.a)};
}

// one damped Jacobi sweep at row i (diagonal form, level.cuh), from u = 0 when !U0
template <bool U0>
HS_DEV Pair jacobi_pair(const Pair& dinv, const Pair& rhs, float inv_h2, const Pair& up, const Pair& mid,
                        const Pair& dn, float w) {
  if (U0) {
    const Pair nb = nbsum_pair(up, mid, dn);
    return Pair{jacobi_dd(dinv.a, inv_h2, w, mid.a, rhs.a, nb.a), jacobi_dd(dinv.b, inv_h2, w, mid.b, rhs.b, nb.b)};
  }
  return Pair{cscale(cmul(dinv.a, rhs.a), w), cscale(cmul(dinv.b, rhs.b), w)};
}

HS_DEV Pair mask_pair(Pair v, bool row_ok, bool oka, bool okb) {
  const float2 z = make_float2(0.f, 0.f);
  if (!(row_ok && oka)) v.a = z;
  if (!(row_ok && okb)) v.b = z;
  return v;
}

constexpr int kVcWarps = 4;          // warps per block (independent)
constexpr int kDownQ = 29;           // coarse columns per down-leg warp (lanes 1..29)
constexpr int kUpCols = 60;          // fine columns per up-leg warp (lanes 1..30)
#ifndef HS_VC_RING
#define HS_VC_RING 6
#endif
#ifndef HS_VC_WAVES
#define HS_VC_WAVES 0  // 0: ~32 warps per SM heuristic; n > 0: bands sized for n full waves of resident warps
#endif
constexpr int kRing = HS_VC_RING;    // rows in flight per warp (cp.async ring depth)

// Row staging: every lane copies its own two columns of a row into a per-warp
// shared-memory ring with 8-byte cp.async (zero-filled outside the grid) and
// reads them back after cp.async.wait_group, so kRing - 1 rows of every input
// stay in flight without holding registers.
HS_DEV void cpa8(uint32_t dst, const float2* src, bool ok) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(ok ? 8 : 0) : "memory");
}
HS_DEV void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
HS_DEV void cpa_wait_ring() { asm volatile("cp.async.wait_group %0;\n" ::"n"(kRing - 1) : "memory"); }

HS_DEV void issue_pair(uint32_t dst, const float2* __restrict__ g, int nx, int ny, int i, int ja) {
  const bool rok = i >= 0 && i < nx;
  const bool oka = rok && ja >= 0 && ja < ny, okb = rok && ja + 1 >= 0 && ja + 1 < ny;
  const long long off = (long long)i * ny + ja;
  cpa8(dst, oka ? g + off : g, oka);
  cpa8(dst + 8, okb ? g + off + 1 : g, okb);
}

// the same from a running row offset `off` (= i * ny + ja) and the row's validity
HS_DEV void issue_pair_at(uint32_t dst, const float2* __restrict__ g, int off, bool rok, bool oka, bool okb) {
  cpa8(dst, (rok && oka) ? g + off : g, rok && oka);
  cpa8(dst + 8, (rok && okb) ? g + off + 1 : g, rok && okb);
}

HS_DEV Pair read_pair(const float2* slot, float s) {
  const float4 v = *reinterpret_cast<const float4*>(slot);
  return Pair{make_float2(v.x * s, v.y * s), make_float2(v.z * s, v.w * s)};
}

// ------------------------------------------------------------------ down leg
//
//   u1 = u0 + w_pre (rhs - A u0)/diag      (jacobi_relax, multigrid.py:218-229)
//   r  = rhs - A u1                         (:270)
//   coarse_rhs = R r                        (restrict_full_weighting, :64-78)
//
// Lane l owns fine columns (2Q, 2Q+1) with Q = Q0 - 1 + l, so its odd column is
// the centre of coarse column Q; lanes 1..29 emit.  A warp covers coarse rows
// [K0, K1): u1 rows 2K0-1 .. 2K1+1, r rows 2K0 .. 2K1.  Ring slot of u1 row s:
// rhs, diag and dinv of row s, u0 row s + 1.

constexpr int kDownSlot = 4 * 64;  // float2 per warp and ring slot
constexpr int kUpSlot = 4 * 64;

template <bool U0>
__global__ void __launch_bounds__(kVcWarps * 32) k_vc_down(LevelDev L, int ncx, int ncy, VecIn rhs_in, VecIn u0_in,
                                                           const float2* const* active, const int* model_of,
                                                           float w_pre, float2* __restrict__ coarse_out, int ncb,
                                                           int band) {
  extern __shared__ __align__(16) float2 vc_smem[];
  const int lane = threadIdx.x & 31;
  const int wid = blockIdx.y * kVcWarps + (threadIdx.x >> 5);
  const int nbands = (ncx + band - 1) / band;
  if (wid >= ncb * nbands) return;
  const int b = blockIdx.x;
  if (active && active[b] == nullptr) return;
  const int Q0 = (wid % ncb) * kDownQ, K0 = (wid / ncb) * band, K1 = min(ncx, K0 + band);
  const int Q = Q0 - 1 + lane, ja = 2 * Q;
  const int nx = L.nx, ny = L.ny;
  const bool oka = ja >= 0 && ja < ny, okb = ja + 1 >= 0 && ja + 1 < ny;
  const bool emit = lane >= 1 && lane <= kDownQ && Q < ncy;
  const long long N = (long long)nx * ny;
  const long long moff = (model_of ? model_of[b] : 0) * N;
  const float2* __restrict__ dg = L.diag + moff;
  const float2* __restrict__ di = L.dinv + moff;
  const float ih2 = L.inv_h2;
  const float2* __restrict__ rhs = vin_ptr(rhs_in, b);
  const float rs = rhs_in.scale ? rhs_in.scale[b] : 1.f;
  const float2* __restrict__ u0 = U0 ? vin_ptr(u0_in, b) : nullptr;
  const float us = (U0 && u0_in.scale) ? u0_in.scale[b] : 1.f;
  float2* __restrict__ co = coarse_out + (long long)b * ncx * ncy;
  float2* ring = vc_smem + (threadIdx.x >> 5) * kRing * kDownSlot;
  const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring) + lane * 16;

  const int s0 = 2 * K0 - 1, s1 = 2 * K1 + 1;  // u1 rows
  // issue side: the next row, its ring slot and its in-field offset advance by one row per call
  // (no per-row multiplies or divisions by the ring depth)
  int is = s0, ioff = s0 * ny + ja;
  uint32_t islot = 0;
  auto issue_next = [&]() {
    if (is <= s1) {
      const uint32_t d = ring_s + islot * (kDownSlot * 8);
      const bool rok = is >= 0 && is < nx;
      issue_pair_at(d, rhs, ioff, rok, oka, okb);
      issue_pair_at(d + 512, dg, ioff, rok, oka, okb);
      issue_pair_at(d + 1024, di, ioff, rok, oka, okb);
      if (U0) issue_pair_at(d + 1536, u0, ioff + ny, is + 1 >= 0 && is + 1 < nx, oka, okb);
    }
    cpa_commit();
    ++is;
    ioff += ny;
    islot = islot + 1 == kRing ? 0 : islot + 1;
  };
#pragma unroll
  for (int k = 0; k < kRing - 1; ++k) issue_next();
  uint32_t cslot = 0;  // consume side
  const Pair z{make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
  Pair u0m = z, u0c = z, u0p = z;
  if (U0) {
    u0c = ld_pair(u0, nx, ny, s0 - 1, ja, us);
    u0p = ld_pair(u0, nx, ny, s0, ja, us);
  }
  Pair rh_m = z, dg_m = z, u1m2 = z, u1m1 = z;
  float2 acc = make_float2(0.f, 0.f);
  for (int s = s0; s <= s1; ++s) {
    issue_next();
    cpa_wait_ring();
    const float2* slot = ring + cslot * kDownSlot + 2 * lane;
    cslot = cslot + 1 == kRing ? 0 : cslot + 1;
    const Pair rh_c = read_pair(slot, rs), dg_c = read_pair(slot + 64, 1.f), di_c = read_pair(slot + 128, 1.f);
    if (U0) {
      u0m = u0c;
      u0c = u0p;
      u0p = read_pair(slot + 192, us);
    }
    const bool row_ok = s >= 0 && s < nx;
    const Pair u1 = mask_pair(jacobi_pair<U0>(di_c, rh_c, ih2, u0m, u0c, u0p, w_pre), row_ok, oka, okb);
    // residual of row i = s - 1 from u1 rows s-2, s-1, s
    const int i = s - 1;
    if (i >= 2 * K0) {
      const Pair nb = nbsum_pair(u1m2, u1m1, u1);
      Pair r;
      r.a = csub(rh_m.a, apply_dd(dg_m.a, ih2, u1m1.a, nb.a));
      r.b = csub(rh_m.b, apply_dd(dg_m.b, ih2, u1m1.b, nb.b));
      r = mask_pair(r, i < nx, oka, okb);
      // horizontal full weighting centred on the odd column jb
      const float2 rr = shfl_dn1(r.a);
      const float2 hr = cadd(cadd(cscale(r.a, 0.25f), cscale(r.b, 0.5f)), cscale(rr, 0.25f));
      if ((i & 1) == 0) {
        if (i > 2 * K0 && emit) co[(long long)(i / 2 - 1) * ncy + Q] = cadd(acc, cscale(hr, 0.25f));
        acc = cscale(hr, 0.25f);
      } else {
        acc = cadd(acc, cscale(hr, 0.5f));
      }
    }
    u1m2 = u1m1;
    u1m1 = u1;
    rh_m = rh_c;
    dg_m = dg_c;
  }
}

// ------------------------------------------------------------------ up leg
//
//   u2 = u1 + P e_coarse                    (prolong_bilinear, multigrid.py:81-114, :273)
//   u3 = u2 + w_post (rhs - A u2)/diag      (:274)
// with u1 recomputed from rhs and u0 (cheaper than storing it).  Lane l owns
// fine columns (c0 + 2l, c0 + 2l + 1), c0 = 60 cb - 2; lanes 1..30 emit.  A
// warp covers fine rows [R0, R1): u2 rows R0-1 .. R1.  Ring slot of u2 row s:
// rhs and dinv of row s, u0 row s + 1 and, for even s, coarse error row s / 2
// at coarse column Q = ja / 2.

// horizontally prolonged coarse row at the lane's columns from its value v at
// column Q = ja / 2: even column ja takes (e[Q-1] + e[Q]) / 2, odd jb takes e[Q]
HS_DEV Pair prolong_pair(float2 v) {
  const float2 vm = shfl_up1(v);
  return Pair{cscale(cadd(vm, v), 0.5f), v};
}

template <bool U0>
__global__ void __launch_bounds__(kVcWarps * 32) k_vc_up(LevelDev L, int ncx, int ncy, VecIn rhs_in, VecIn u0_in,
                                                         const float2* const* active, const int* model_of,
                                                         float w_pre, float w_post, const float2* __restrict__ ecoarse,
                                                         VecOut out, int ncb, int band) {
  extern __shared__ __align__(16) float2 vc_smem[];
  const int lane = threadIdx.x & 31;
  const int wid = blockIdx.y * kVcWarps + (threadIdx.x >> 5);
  const int nx = L.nx, ny = L.ny;
  const int nbands = (nx + band - 1) / band;
  if (wid >= ncb * nbands) return;
  const int b = blockIdx.x;
  if (active && active[b] == nullptr) return;
  const int c0 = (wid % ncb) * kUpCols - 2, R0 = (wid / ncb) * band, R1 = min(nx, R0 + band);
  const int ja = c0 + 2 * lane, Q = ja / 2;  // c0 even, so ja / 2 is exact (Q = -1 only on a halo lane)
  const bool oka = ja >= 0 && ja < ny, okb = ja + 1 >= 0 && ja + 1 < ny;
  const bool emit = lane >= 1 && lane <= 30;
  const bool okq = Q >= 0 && Q < ncy;
  const long long N = (long long)nx * ny;
  const float2* __restrict__ di = L.dinv + (model_of ? model_of[b] : 0) * N;
  const float ih2 = L.inv_h2;
  const float2* __restrict__ rhs = vin_ptr(rhs_in, b);
  const float rs = rhs_in.scale ? rhs_in.scale[b] : 1.f;
  const float2* __restrict__ u0 = U0 ? vin_ptr(u0_in, b) : nullptr;
  const float us = (U0 && u0_in.scale) ? u0_in.scale[b] : 1.f;
  const float2* __restrict__ e = ecoarse + (long long)b * ncx * ncy;
  float2* __restrict__ dst = vout_ptr(out, b);
  float2* ring = vc_smem + (threadIdx.x >> 5) * kRing * kUpSlot;
  const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring) + lane * 16;

  const int s0 = R0 - 1, s1 = R1;  // u2 rows
  int is = s0, ioff = s0 * ny + ja;
  uint32_t islot = 0;
  auto issue_next = [&]() {
    if (is <= s1) {
      const uint32_t d = ring_s + islot * (kUpSlot * 8);
      const bool rok = is >= 0 && is < nx;
      issue_pair_at(d, rhs, ioff, rok, oka, okb);
      issue_pair_at(d + 512, di, ioff, rok, oka, okb);
      if (U0) issue_pair_at(d + 1024, u0, ioff + ny, is + 1 >= 0 && is + 1 < nx, oka, okb);
      if ((is & 1) == 0) {
        const int K = is / 2;
        const bool ok = okq && K < ncx;
        cpa8(d + 1536, ok ? e + (long long)K * ncy + Q : e, ok);
      }
    }
    cpa_commit();
    ++is;
    ioff += ny;
    islot = islot + 1 == kRing ? 0 : islot + 1;
  };
#pragma unroll
  for (int k = 0; k < kRing - 1; ++k) issue_next();
  uint32_t cslot = 0;
  const Pair z{make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
  Pair u0m = z, u0c = z, u0p = z;
  if (U0) {
    u0c = ld_pair(u0, nx, ny, s0 - 1, ja, us);
    u0p = ld_pair(u0, nx, ny, s0, ja, us);
  }
  Pair rh_m = z, di_m = z, u2m2 = z, u2m1 = z;
  // hcur = prolonged coarse row below the first u2 row: K = (s0-1)/2 for odd s0,
  // s0/2 - 1 for even s0 (s0 >= -1; K = -1 is a zero row)
  Pair hcur = z;
  {
    const int K = (s0 & 1) ? (s0 - 1) / 2 : s0 / 2 - 1;
    float2 v = make_float2(0.f, 0.f);
    if (okq && K >= 0 && K < ncx) v = e[(long long)K * ncy + Q];
    hcur = prolong_pair(v);
  }
  for (int s = s0; s <= s1; ++s) {
    issue_next();
    cpa_wait_ring();
    const float2* slot = ring + cslot * kUpSlot + 2 * lane;
    cslot = cslot + 1 == kRing ? 0 : cslot + 1;
    const Pair rh_c = read_pair(slot, rs), di_c = read_pair(slot + 64, 1.f);
    if (U0) {
      u0m = u0c;
      u0c = u0p;
      u0p = read_pair(slot + 128, us);
    }
    // P e at row s: odd s = 2K+1 -> h(K); even s = 2K -> (h(K-1) + h(K)) / 2
    Pair pe;
    if ((s & 1) == 0) {
      const Pair hprev = hcur;
      hcur = prolong_pair(slot[192]);
      pe.a = cscale(cadd(hprev.a, hcur.a), 0.5f);
      pe.b = cscale(cadd(hprev.b, hcur.b), 0.5f);
    } else {
      pe = hcur;
    }
    Pair u2 = jacobi_pair<U0>(di_c, rh_c, ih2, u0m, u0c, u0p, w_pre);
    u2.a = cadd(u2.a, pe.a);
    u2.b = cadd(u2.b, pe.b);
    u2 = mask_pair(u2, s >= 0 && s < nx, oka, okb);
    // post-smoothing of row i = s - 1 from u2 rows s-2, s-1, s
    const int i = s - 1;
    if (i >= R0) {
      const Pair u3 = jacobi_pair<true>(di_m, rh_m, ih2, u2m2, u2m1, u2, w_post);
      if (emit) {
        float2* row = dst + (long long)i * ny;
        if (oka) row[ja] = u3.a;
        if (okb) row[ja + 1] = u3.b;
      }
    }
    u2m2 = u2m1;
    u2m1 = u2;
    rh_m = rh_c;
    di_m = di_c;
  }
}

// ------------------------------------------------------------ coarsest level
//
// GMRES(m) with M = damping/diag and x0 = 0, tol 1e-12 (coarse_solve,
// multigrid.py:232-244 -> krylov.py:39-146).  One CTA per RHS.  V_0 is the rhs
// itself (scale 1/beta0); V_k, k >= 1, live unnormalised in `vws` with their
// scales 1/h_{k,k-1} in shared memory.  Dot products accumulate in fp64 and
// are reduced deterministically; the Hessenberg/Givens work is fp64 on
// thread 0.  Breakdown / non-finite conditions are written to `status`.

constexpr int kCoarseThreads = 512;

template <int MI>  // iteration capacity (coarse_iters <= MI): sizes the register partials
__global__ void __launch_bounds__(kCoarseThreads) k_coarse_gmres(LevelDev L, const float2* __restrict__ rhs_base,
                                                                 float2* __restrict__ x_out, float2* vws,
                                                                 float2* sws, const float2* const* active,
                                                                 const int* model_of, int m, float damping,
                                                                 int* status) {
  constexpr int NACC = 2 * (MI + 1) + 1;
  __shared__ double red[NACC * (kCoarseThreads / 32 + 1)];
  __shared__ double2 H[(MI + 1) * MI];
  __shared__ double2 gv[MI + 1], sn[MI], yv[MI];
  __shared__ double cs[MI], vs[MI + 1];
  __shared__ double2 hc[MI + 1];
  __shared__ int s_flag, s_jend;
  const int b = blockIdx.x;
  if (active && active[b] == nullptr) return;
  const int nx = L.nx, ny = L.ny;
  const long long N = (long long)nx * ny;
  const float2* rhs = rhs_base + b * N;
  float2* V = vws + (long long)b * (m + 1) * N;  // slots 1..m used
  float2* S = sws + b * N;
  float2* x = x_out + b * N;
  const float2* mass = L.mass + (model_of ? model_of[b] : 0) * N;
  auto vec = [&](int k) -> const float2* { return k == 0 ? rhs : V + k * N; };

  // Jacobi scale s = damping / diag and beta0 = ||rhs||
  double acc[NACC];
  acc[0] = 0.0;
  for (long long p = threadIdx.x; p < N; p += blockDim.x) {
    int i = (int)(p / ny), j = (int)(p - (long long)i * ny);
    S[p] = cdiv(make_float2(damping, 0.f), level_diag(L, mass[p], i, j));
    float2 r = rhs[p];
    acc[0] += (double)r.x * r.x + (double)r.y * r.y;
  }
  block_sum_n<NACC>(acc, 1, red);  // (acc[0] only: before acc[] is used with constant indices)
  const double beta0 = sqrt(acc[0]);
  if (beta0 == 0.0) {
    for (long long p = threadIdx.x; p < N; p += blockDim.x) x[p] = make_float2(0.f, 0.f);
    return;
  }
  if (threadIdx.x == 0) {
    vs[0] = 1.0 / beta0;
    gv[0] = make_double2(beta0, 0.0);
    s_flag = 0;
    s_jend = m;
  }
  __syncthreads();  // S visible block-wide (global writes by this CTA, read via L1/L2)
  __threadfence_block();

  for (int j = 0; j < m; ++j) {
    const float2* vj = vec(j);
    float2* W = V + (j + 1) * N;
    const float sj = (float)vs[j];
    // pass A: w = A (S .* v_j), dots with v_0..v_j, ||w||^2
    // every acc[] index below is a compile-time constant (unrolled loops with
    // k <= j guards), which keeps the partial sums in registers
#pragma unroll
    for (int k = 0; k < NACC; ++k) acc[k] = 0.0;
    int bad = 0;
    for (long long p = threadIdx.x; p < N; p += blockDim.x) {
      int i = (int)(p / ny), jj = (int)(p - (long long)i * ny);
      auto zat = [&](int ii, int jq) -> float2 {
        if (ii < 0 || ii >= nx || jq < 0 || jq >= ny) return make_float2(0.f, 0.f);
        long long q = (long long)ii * ny + jq;
        return cscale(cmul(S[q], vj[q]), sj);
      };
      float2 w = level_apply(L, mass[p], i, jj, zat(i, jj), zat(i + 1, jj), zat(i - 1, jj), zat(i, jj + 1),
                             zat(i, jj - 1));
      if (!isfinite(w.x) || !isfinite(w.y)) bad = 1;
      W[p] = w;
      double2 wd = f2d(w);
      acc[0] += wd.x * wd.x + wd.y * wd.y;
#pragma unroll
      for (int k = 0; k <= MI; ++k) {
        if (k <= j) {
          double2 d = zcmul(f2d(vec(k)[p]), wd);
          acc[1 + 2 * k] += d.x;
          acc[2 + 2 * k] += d.y;
        }
      }
    }
    if (bad) atomicOr(&s_flag, 1);
    block_sum<NACC>(acc, red);
    if (s_flag) {
      if (threadIdx.x == 0) atomicCAS(status + b, 0, HS_ENONFINITE);
      return;
    }
    const double wn = sqrt(acc[0]);
    if (threadIdx.x == 0)
#pragma unroll
      for (int k = 0; k <= MI; ++k)
        if (k <= j) {
          hc[k] = make_double2(acc[1 + 2 * k] * vs[k], acc[2 + 2 * k] * vs[k]);
          H[k * MI + j] = hc[k];
        }
    __syncthreads();
    double hn2 = 0.0;
    for (int pass = 0; pass < 2; ++pass) {
      // w -= sum_k hc_k v_k ; ||w||^2   (hc = first-pass coefficients, then the extra part)
      acc[0] = 0.0;
      for (long long p = threadIdx.x; p < N; p += blockDim.x) {
        float2 w = W[p];
        for (int k = 0; k <= j; ++k) {
          double2 hk = hc[k];
          float2 coef = make_float2((float)(hk.x * vs[k]), (float)(hk.y * vs[k]));
          w = csub(w, cmul(coef, vec(k)[p]));
        }
        W[p] = w;
        acc[0] += (double)w.x * w.x + (double)w.y * w.y;
      }
      block_sum<1>(*reinterpret_cast<double(*)[1]>(acc), red);
      hn2 = acc[0];
      if (pass == 1 || sqrt(hn2) >= 0.25 * wn) break;
      // one re-orthogonalisation pass (krylov.py:105-111): extra = V^H w
#pragma unroll
      for (int k = 0; k < NACC; ++k) acc[k] = 0.0;
      for (long long p = threadIdx.x; p < N; p += blockDim.x) {
        double2 wd = f2d(W[p]);
#pragma unroll
        for (int k = 0; k <= MI; ++k)
          if (k <= j) {
            double2 d = zcmul(f2d(vec(k)[p]), wd);
            acc[2 * k] += d.x;
            acc[2 * k + 1] += d.y;
          }
      }
      block_sum<NACC>(acc, red);
      if (threadIdx.x == 0)
#pragma unroll
        for (int k = 0; k <= MI; ++k)
          if (k <= j) {
            hc[k] = make_double2(acc[2 * k] * vs[k], acc[2 * k + 1] * vs[k]);
            H[k * MI + j] = zadd(H[k * MI + j], hc[k]);
          }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      const double hn = sqrt(hn2);
      double2 col[MI + 1];
      for (int k = 0; k <= j; ++k) col[k] = H[k * MI + j];
      for (int k = 0; k < j; ++k) {
        double2 a = col[k], bb = col[k + 1];
        double2 s = sn[k];
        col[k] = zadd(zscale(a, cs[k]), zmul(s, bb));
        col[k + 1] = zadd(zmul(make_double2(-s.x, s.y), a), zscale(bb, cs[k]));
      }
      double2 a = col[j];
      double c;
      double2 s, rr;
      double mag = hypot(a.x, a.y);
      if (mag == 0.0) {
        c = 0.0;
        s = make_double2(1.0, 0.0);
        rr = make_double2(hn, 0.0);
      } else {
        double t = hypot(mag, hn);
        double2 ph = make_double2(a.x / mag, a.y / mag);
        c = mag / t;
        s = zscale(ph, hn / t);
        rr = zscale(ph, t);
      }
      cs[j] = c;
      sn[j] = s;
      col[j] = rr;
      for (int k = 0; k <= j; ++k) H[k * MI + j] = col[k];
      double2 gj = gv[j];
      gv[j] = zscale(gj, c);
      gv[j + 1] = zmul(make_double2(-s.x, s.y), gj);
      const double est = hypot(gv[j + 1].x, gv[j + 1].y) / beta0;
      if (est <= 1e-12) {
        s_jend = j + 1;
        s_flag = 2;
      } else if (hn <= 1e-14 * fmax(1.0, wn)) {
        s_flag = 3;
      }
      vs[j + 1] = 1.0 / hn;
    }
    __syncthreads();
    if (s_flag == 2) break;
    if (s_flag == 3) {
      if (threadIdx.x == 0) atomicCAS(status + b, 0, HS_EBREAKDOWN);
      return;
    }
  }
  // y = R^{-1} g ; x = sum_k y_k S v_k
  const int jend = s_jend;
  if (threadIdx.x == 0) {
    for (int i = jend - 1; i >= 0; --i) {
      double2 acc2 = gv[i];
      for (int k = i + 1; k < jend; ++k) acc2 = zsub(acc2, zmul(H[i * MI + k], yv[k]));
      double2 d = H[i * MI + i];
      double den = d.x * d.x + d.y * d.y;
      yv[i] = make_double2((acc2.x * d.x + acc2.y * d.y) / den, (acc2.y * d.x - acc2.x * d.y) / den);
    }
  }
  __syncthreads();
  for (long long p = threadIdx.x; p < N; p += blockDim.x) {
    float2 sum = make_float2(0.f, 0.f);
    for (int k = 0; k < jend; ++k) {
      float2 yk = make_float2((float)(yv[k].x * vs[k]), (float)(yv[k].y * vs[k]));
      sum = cadd(sum, cmul(yk, vec(k)[p]));
    }
    x[p] = cmul(S[p], sum);
  }
}

// Small coarsest grids (N <= 512 * 8 nodes: C1's 32^2, C2's 64^2): the same
// GMRES with the vector being expanded kept on chip.  Each thread owns nodes
// p = t + 512 u (u < 8) and keeps the unnormalised V_j of those nodes in
// registers; z_j = S v_j / h is staged in shared memory so the stencil reads
// its neighbours on chip; the operator is the diagonal form (diag / dinv
// planes, level.cuh); the stored basis V_1..V_j is read back from the
// L2-resident workspace two nodes x every k at a time, so each Gram-Schmidt
// pass costs a few L2 round trips instead of one per node and vector.
// Gram-Schmidt passes of the fast coarse GMRES over the thread's nodes, with
// the number of basis vectors JJ a compile-time constant (dispatched on the
// window position), so every loop is unrolled without guards.
// dots: acc[1 + 2k] + i acc[2 + 2k] += conj(v_k) w, k < JJ (v_0 = rhs)
#ifndef HS_COARSE_UNROLL
#define HS_COARSE_UNROLL 1  // measured: 1, 2, 4 and 8 equal at C3 (the coarse solve is issue-bound, not L2-latency-bound)
#endif
constexpr int kCoarseUnroll = HS_COARSE_UNROLL;
// The node loop is unrolled (HS_COARSE_UNROLL nodes per trip) so the basis loads of several nodes are
// in flight together: the basis lives in L2, and a trip per node paid one L2 round trip each.
template <int JJ, int NACC>
HS_DEV void coarse_dots(double (&acc)[NACC], const float2* __restrict__ rhs, const float2* __restrict__ V, int N,
                        const float2* ws) {
#pragma unroll kCoarseUnroll
  for (int p = threadIdx.x; p < N; p += blockDim.x) {
    float2 q[JJ];
    q[0] = rhs[p];
#pragma unroll
    for (int k = 1; k < JJ; ++k) q[k] = V[k * N + p];
    const double2 wd = f2d(ws[p]);
#pragma unroll
    for (int k = 0; k < JJ; ++k) {
      const double2 d = zcmul(f2d(q[k]), wd);
      acc[1 + 2 * k] += d.x;
      acc[2 + 2 * k] += d.y;
    }
  }
}
// orth: w -= sum_k coef_k v_k, k < JJ; returns the thread's part of ||w||^2
template <int JJ>
HS_DEV double coarse_orth(const float2* __restrict__ rhs, const float2* __restrict__ V, int N, float2* ws,
                          const float2* coef) {
  float2 c[JJ];
#pragma unroll
  for (int k = 0; k < JJ; ++k) c[k] = coef[k];
  double nn = 0.0;
#pragma unroll kCoarseUnroll
  for (int p = threadIdx.x; p < N; p += blockDim.x) {
    float2 q[JJ];
    q[0] = rhs[p];
#pragma unroll
    for (int k = 1; k < JJ; ++k) q[k] = V[k * N + p];
    float2 wv = ws[p];
#pragma unroll
    for (int k = 0; k < JJ; ++k) wv = csub(wv, cmul(c[k], q[k]));
    ws[p] = wv;
    nn += (double)wv.x * wv.x + (double)wv.y * wv.y;
  }
  return nn;
}

#define HS_COARSE_SWITCH(J, CALL) \
  switch (J) {                    \
    case 1: CALL(1); break;       \
    case 2: CALL(2); break;       \
    case 3: CALL(3); break;       \
    case 4: CALL(4); break;       \
    case 5: CALL(5); break;       \
    case 6: CALL(6); break;       \
    case 7: CALL(7); break;       \
    case 8: CALL(8); break;       \
    case 9: CALL(9); break;       \
    default: CALL(10); break;     \
  }

constexpr int kCoarseFastMax = kCoarseThreads * 16;  // C3's 4-level coarsest grid, 64 x 128

template <int MI, int NPT>
__global__ void __launch_bounds__(kCoarseThreads, 1)
    k_coarse_gmres_fast(LevelDev L, const float2* __restrict__ rhs_base, float2* __restrict__ x_out, float2* vws,
                        const float2* const* active, const int* model_of, int m, float damping, int* status) {
  constexpr int NACC = 2 * (MI + 1) + 1;
  __shared__ double red[NACC * (kCoarseThreads / 32 + 1)];
  extern __shared__ __align__(16) float2 coarse_dyn[];
  float2* zs = coarse_dyn;                           // z_j = S v_j / h_j
  float2* ws = coarse_dyn + kCoarseThreads * NPT;  // unnormalised V_j, then w
  __shared__ double2 H[(MI + 1) * MI];
  __shared__ double2 gv[MI + 1], sn[MI], yv[MI];
  __shared__ double cs[MI], vs[MI + 1];
  __shared__ double2 hc[MI + 1];
  __shared__ float2 scoef[MI + 1];
  __shared__ int s_flag, s_jend;
  const int b = blockIdx.x;
  if (active && active[b] == nullptr) return;
  const int nx = L.nx, ny = L.ny, N = nx * ny;
  const float ih2 = L.inv_h2;
  const float2* rhs = rhs_base + (long long)b * N;
  float2* V = vws + (long long)b * (m + 1) * N;  // slots 1..m used
  float2* x = x_out + (long long)b * N;
  const long long moff = (long long)(model_of ? model_of[b] : 0) * N;
  const float2* __restrict__ dg = L.diag + moff;
  const float2* __restrict__ di = L.dinv + moff;
  auto vec = [&](int k) -> const float2* { return k == 0 ? rhs : V + (long long)k * N; };
  const int t = threadIdx.x;

  double acc[NACC];
  acc[0] = 0.0;
#pragma unroll
  for (int u = 0; u < NPT; ++u) {
    const int p = t + u * kCoarseThreads;
    const float2 r = p < N ? rhs[p] : make_float2(0.f, 0.f);
    if (p < N) ws[p] = r;
    acc[0] += (double)r.x * r.x + (double)r.y * r.y;
  }
  block_sum_n<NACC>(acc, 1, red);
  const double beta0 = sqrt(acc[0]);
  if (beta0 == 0.0) {
#pragma unroll
    for (int u = 0; u < NPT; ++u) {
      const int p = t + u * kCoarseThreads;
      if (p < N) x[p] = make_float2(0.f, 0.f);
    }
    return;
  }
  if (t == 0) {
    vs[0] = 1.0 / beta0;
    gv[0] = make_double2(beta0, 0.0);
    s_flag = 0;
    s_jend = m;
  }
  __syncthreads();

  for (int j = 0; j < m; ++j) {
    const float sj = (float)vs[j];
    // z_j = S v_j (S = damping / diag) into shared memory
#pragma unroll
    for (int u = 0; u < NPT; ++u) {
      const int p = t + u * kCoarseThreads;
      if (p < N) zs[p] = cscale(cmul(di[p], ws[p]), damping * sj);
    }
    __syncthreads();
    // w = A z_j (diagonal form), ||w||^2
#pragma unroll
    for (int k = 0; k < NACC; ++k) acc[k] = 0.0;
    int bad = 0;
#pragma unroll
    for (int u = 0; u < NPT; ++u) {
      const int p = t + u * kCoarseThreads;
      float2 r = make_float2(0.f, 0.f);
      if (p < N) {
        const int i = p / ny, q = p - i * ny;
        const float2 zero = make_float2(0.f, 0.f);
        const float2 xp = i + 1 < nx ? zs[p + ny] : zero, xm = i > 0 ? zs[p - ny] : zero;
        const float2 yp = q + 1 < ny ? zs[p + 1] : zero, ym = q > 0 ? zs[p - 1] : zero;
        const float2 nb = make_float2((xp.x + xm.x) + (yp.x + ym.x), (xp.y + xm.y) + (yp.y + ym.y));
        r = apply_dd(dg[p], ih2, zs[p], nb);
      }
      if (!isfinite(r.x) || !isfinite(r.y)) bad = 1;
      if (p < N) ws[p] = r;
      acc[0] += (double)r.x * r.x + (double)r.y * r.y;
    }
    // dots with v_0..v_j
#define HS_DOTS(JJ) coarse_dots<JJ>(acc, rhs, V, N, ws)
    HS_COARSE_SWITCH(j + 1, HS_DOTS)
#undef HS_DOTS
    __syncthreads();  // every thread is done with zs before the next step rewrites it
    if (bad) atomicOr(&s_flag, 1);
    // reduce only the 2(j+1)+1 live partial sums
#define HS_RED(JJ) block_sum<2 * JJ + 1>(*reinterpret_cast<double(*)[2 * JJ + 1]>(acc), red)
    HS_COARSE_SWITCH(j + 1, HS_RED)
#undef HS_RED
    if (s_flag) {
      if (t == 0) atomicCAS(status + b, 0, HS_ENONFINITE);
      return;
    }
    const double wn = sqrt(acc[0]);
    if (t == 0)
#pragma unroll
      for (int k = 0; k <= MI; ++k)
        if (k <= j) {
          hc[k] = make_double2(acc[1 + 2 * k] * vs[k], acc[2 + 2 * k] * vs[k]);
          H[k * MI + j] = hc[k];
        }
    __syncthreads();
    double hn2 = 0.0;
    for (int pass = 0; pass < 2; ++pass) {
      // w -= sum_k hc_k v_k ; ||w||^2  (coefficients from shared memory)
      if (t <= j) scoef[t] = make_float2((float)(hc[t].x * vs[t]), (float)(hc[t].y * vs[t]));
      __syncthreads();
#define HS_ORTH(JJ) acc[0] = coarse_orth<JJ>(rhs, V, N, ws, scoef)
      HS_COARSE_SWITCH(j + 1, HS_ORTH)
#undef HS_ORTH
      block_sum<1>(*reinterpret_cast<double(*)[1]>(acc), red);
      hn2 = acc[0];
      if (pass == 1 || sqrt(hn2) >= 0.25 * wn) break;
      // one re-orthogonalisation pass (krylov.py:105-111): extra = V^H w
#pragma unroll
      for (int k = 0; k < NACC; ++k) acc[k] = 0.0;
#pragma unroll 1
      for (int u = 0; u < NPT; ++u) {
        const int p = t + u * kCoarseThreads;
        if (p >= N) continue;
        const double2 wd = f2d(ws[p]);
#pragma unroll
        for (int k = 0; k <= MI; ++k)
          if (k <= j) {
            const double2 d = zcmul(f2d(vec(k)[p]), wd);
            acc[2 * k] += d.x;
            acc[2 * k + 1] += d.y;
          }
      }
      block_sum<NACC>(acc, red);
      if (t == 0)
#pragma unroll
        for (int k = 0; k <= MI; ++k)
          if (k <= j) {
            hc[k] = make_double2(acc[2 * k] * vs[k], acc[2 * k + 1] * vs[k]);
            H[k * MI + j] = zadd(H[k * MI + j], hc[k]);
          }
      __syncthreads();
    }
    // store the unnormalised V_{j+1} for the later passes and the solution
    if (j + 1 < m) {
#pragma unroll
      for (int u = 0; u < NPT; ++u) {
        const int p = t + u * kCoarseThreads;
        if (p < N) V[(long long)(j + 1) * N + p] = ws[p];
      }
    }
    if (t == 0) {
      const double hn = sqrt(hn2);
      double2 col[MI + 1];
      for (int k = 0; k <= j; ++k) col[k] = H[k * MI + j];
      for (int k = 0; k < j; ++k) {
        double2 a = col[k], bb = col[k + 1];
        double2 s = sn[k];
        col[k] = zadd(zscale(a, cs[k]), zmul(s, bb));
        col[k + 1] = zadd(zmul(make_double2(-s.x, s.y), a), zscale(bb, cs[k]));
      }
      double2 a = col[j];
      double c;
      double2 s, rr;
      double mag = hypot(a.x, a.y);
      if (mag == 0.0) {
        c = 0.0;
        s = make_double2(1.0, 0.0);
        rr = make_double2(hn, 0.0);
      } else {
        double tt = hypot(mag, hn);
        double2 ph = make_double2(a.x / mag, a.y / mag);
        c = mag / tt;
        s = zscale(ph, hn / tt);
        rr = zscale(ph, tt);
      }
      cs[j] = c;
      sn[j] = s;
      col[j] = rr;
      for (int k = 0; k <= j; ++k) H[k * MI + j] = col[k];
      double2 gj = gv[j];
      gv[j] = zscale(gj, c);
      gv[j + 1] = zmul(make_double2(-s.x, s.y), gj);
      const double est = hypot(gv[j + 1].x, gv[j + 1].y) / beta0;
      if (est <= 1e-12) {
        s_jend = j + 1;
        s_flag = 2;
      } else if (hn <= 1e-14 * fmax(1.0, wn)) {
        s_flag = 3;
      }
      vs[j + 1] = 1.0 / hn;
    }
    __syncthreads();
    if (s_flag == 2) break;
    if (s_flag == 3) {
      if (t == 0) atomicCAS(status + b, 0, HS_EBREAKDOWN);
      return;
    }
  }
  // y = R^{-1} g ; x = S sum_k y_k v_k
  const int jend = s_jend;
  if (t == 0) {
    for (int i = jend - 1; i >= 0; --i) {
      double2 acc2 = gv[i];
      for (int k = i + 1; k < jend; ++k) acc2 = zsub(acc2, zmul(H[i * MI + k], yv[k]));
      double2 d = H[i * MI + i];
      double den = d.x * d.x + d.y * d.y;
      yv[i] = make_double2((acc2.x * d.x + acc2.y * d.y) / den, (acc2.y * d.x - acc2.x * d.y) / den);
    }
  }
  __syncthreads();
#pragma unroll 1
  for (int u = 0; u < NPT; ++u) {
    const int p = t + u * kCoarseThreads;
    if (p >= N) continue;
    float2 sum = make_float2(0.f, 0.f);
#pragma unroll
    for (int k = 0; k < MI; ++k)
      if (k < jend) {
        const float2 yk = make_float2((float)(yv[k].x * vs[k]), (float)(yv[k].y * vs[k]));
        sum = cadd(sum, cmul(yk, vec(k)[p]));
      }
    x[p] = cmul(cscale(di[p], damping), sum);
  }
}

// the reference's coarse solve runs 10 steps (multigrid.py:243); 16 is the supported maximum
// ---------------------------------------------------------------------------------------------
// The same GMRES-Jacobi coarse solve (multigrid.py:232-244) on a 2-CTA cluster per RHS.  One CTA
// per RHS left most SMs idle at C3 (64 RHS on 148 SMs) with each CTA walking 8192 nodes serially;
// here CTA r owns the rows [r nx0, ...) of the coarsest grid, reads the partner's boundary row of
// z_j through distributed shared memory for the stencil, and every reduction is a block sum
// followed by an exchange of the two block totals (added in rank order in both CTAs, so both hold
// bit-identical coefficients and run identical Givens / stopping logic).
namespace cgc = cooperative_groups;
#ifndef HS_COARSE_CLUSTER
#define HS_COARSE_CLUSTER 0
#endif

template <int MI>
struct ClRed {  // double-buffered exchange slots for the cluster reductions
  static constexpr int NMAX = 2 * (MI + 1) + 2;
};

// (all N_ entries, compile-time indices: the accumulators stay in registers)
template <int N_, int MI>
HS_DEV void cluster_sum(double (&v)[N_], double* red, double* cred, int& parity, cgc::cluster_group& cl, int r) {
  static_assert(N_ <= ClRed<MI>::NMAX, "exchange slots");
  block_sum<N_>(v, red);  // every thread holds this CTA's totals
  double* mine = cred + parity * ClRed<MI>::NMAX;
  if (threadIdx.x == 0)
#pragma unroll
    for (int i = 0; i < N_; ++i) mine[i] = v[i];
  cl.sync();
  const double* other = cl.map_shared_rank(cred, 1 - r) + parity * ClRed<MI>::NMAX;
#pragma unroll
  for (int i = 0; i < N_; ++i) v[i] = r == 0 ? mine[i] + other[i] : other[i] + mine[i];
  parity ^= 1;
}

template <int MI, int NPT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kCoarseThreads, 1)
    k_coarse_gmres_cl(LevelDev L, const float2* __restrict__ rhs_base, float2* __restrict__ x_out, float2* vws,
                      const float2* const* active, const int* model_of, int m, float damping, int* status) {
  constexpr int NACC = 2 * (MI + 1) + 2;  // |w|^2, the dots, and the non-finite count
  __shared__ double red[NACC * (kCoarseThreads / 32 + 1)];
  __shared__ double cred[2 * ClRed<MI>::NMAX];
  extern __shared__ __align__(16) float2 coarse_dyn[];
  float2* zs = coarse_dyn;                         // z_j = S v_j / h_j on this CTA's rows
  float2* ws = coarse_dyn + kCoarseThreads * NPT;  // unnormalised V_j, then w
  __shared__ double2 H[(MI + 1) * MI];
  __shared__ double2 gv[MI + 1], sn[MI], yv[MI];
  __shared__ double cs[MI], vs[MI + 1];
  __shared__ double2 hc[MI + 1];
  __shared__ float2 scoef[MI + 1];
  __shared__ int s_flag, s_jend;
  cgc::cluster_group cl = cgc::this_cluster();
  const int r = (int)cl.block_rank();
  const int b = blockIdx.x >> 1;
  if (active && active[b] == nullptr) return;  // both CTAs of the pair
  const int nx = L.nx, ny = L.ny, N = nx * ny;
  const int nx0 = nx / 2, rows = r ? nx - nx0 : nx0, row0 = r ? nx0 : 0;
  const int Nr = rows * ny, p0 = row0 * ny;  // this CTA's nodes [p0, p0 + Nr)
  const float ih2 = L.inv_h2;
  const float2* rhs = rhs_base + (long long)b * N;
  float2* V = vws + (long long)b * (m + 1) * N;  // slots 1..m used
  float2* x = x_out + (long long)b * N;
  const long long moff = (long long)(model_of ? model_of[b] : 0) * N;
  const float2* __restrict__ dg = L.diag + moff;
  const float2* __restrict__ di = L.dinv + moff;
  const float2* zo = cl.map_shared_rank(zs, 1 - r);  // the partner's z (its boundary row)
  const int orows = r ? nx0 : nx - nx0;
  auto vec = [&](int k) -> const float2* { return k == 0 ? rhs : V + (long long)k * N; };
  const int t = threadIdx.x;
  int par = 0;

  double acc[NACC];
#pragma unroll
  for (int k = 0; k < NACC; ++k) acc[k] = 0.0;
#pragma unroll
  for (int u = 0; u < NPT; ++u) {
    const int pl = t + u * kCoarseThreads;
    const float2 v = pl < Nr ? rhs[p0 + pl] : make_float2(0.f, 0.f);
    if (pl < Nr) ws[pl] = v;
    acc[0] += (double)v.x * v.x + (double)v.y * v.y;
  }
  cluster_sum<NACC, MI>(acc, red, cred, par, cl, r);
  const double beta0 = sqrt(acc[0]);
  if (beta0 == 0.0) {
#pragma unroll
    for (int u = 0; u < NPT; ++u) {
      const int pl = t + u * kCoarseThreads;
      if (pl < Nr) x[p0 + pl] = make_float2(0.f, 0.f);
    }
    cl.sync();
    return;
  }
  if (t == 0) {
    vs[0] = 1.0 / beta0;
    gv[0] = make_double2(beta0, 0.0);
    s_flag = 0;
    s_jend = m;
  }
  __syncthreads();

  for (int j = 0; j < m; ++j) {
    const float sj = (float)vs[j];
#pragma unroll
    for (int u = 0; u < NPT; ++u) {
      const int pl = t + u * kCoarseThreads;
      if (pl < Nr) zs[pl] = cscale(cmul(di[p0 + pl], ws[pl]), damping * sj);
    }
    cl.sync();  // both halves of z_j written (the partner reads this CTA's boundary row)
#pragma unroll
    for (int k = 0; k < NACC; ++k) acc[k] = 0.0;
    double bad = 0.0;
#pragma unroll
    for (int u = 0; u < NPT; ++u) {
      const int pl = t + u * kCoarseThreads;
      float2 w = make_float2(0.f, 0.f);
      if (pl < Nr) {
        const int il = pl / ny, q = pl - il * ny, i = row0 + il;
        const float2 zero = make_float2(0.f, 0.f);
        const float2 xp = i + 1 < nx ? (il + 1 < rows ? zs[pl + ny] : zo[q]) : zero;
        const float2 xm = i > 0 ? (il > 0 ? zs[pl - ny] : zo[(orows - 1) * ny + q]) : zero;
        const float2 yp = q + 1 < ny ? zs[pl + 1] : zero, ym = q > 0 ? zs[pl - 1] : zero;
        const float2 nb = make_float2((xp.x + xm.x) + (yp.x + ym.x), (xp.y + xm.y) + (yp.y + ym.y));
        w = apply_dd(dg[p0 + pl], ih2, zs[pl], nb);
      }
      if (!isfinite(w.x) || !isfinite(w.y)) bad = 1.0;
      if (pl < Nr) ws[pl] = w;
      acc[0] += (double)w.x * w.x + (double)w.y * w.y;
    }
    // dots with v_0..v_j over this CTA's nodes
#pragma unroll 1
    for (int u = 0; u < NPT; ++u) {
      const int pl = t + u * kCoarseThreads;
      if (pl >= Nr) continue;
      const double2 wd = f2d(ws[pl]);
#pragma unroll
      for (int k = 0; k <= MI; ++k)
        if (k <= j) {
          const double2 d = zcmul(f2d(vec(k)[p0 + pl]), wd);
          acc[1 + 2 * k] += d.x;
          acc[2 + 2 * k] += d.y;
        }
    }
    acc[NACC - 1] = bad;
    cluster_sum<NACC, MI>(acc, red, cred, par, cl, r);
    if (acc[NACC - 1] > 0.0) {  // non-finite A z in either half: both CTAs stop here
      if (t == 0 && r == 0) atomicCAS(status + b, 0, HS_ENONFINITE);
      cl.sync();
      return;
    }
    const double wn = sqrt(acc[0]);
    if (t == 0)
#pragma unroll
      for (int k = 0; k <= MI; ++k)
        if (k <= j) {
          hc[k] = make_double2(acc[1 + 2 * k] * vs[k], acc[2 + 2 * k] * vs[k]);
          H[k * MI + j] = hc[k];
        }
    __syncthreads();
    double hn2 = 0.0;
    for (int pass = 0; pass < 2; ++pass) {
      // w -= sum_k hc_k v_k ; ||w||^2
      if (t <= j) scoef[t] = make_float2((float)(hc[t].x * vs[t]), (float)(hc[t].y * vs[t]));
      __syncthreads();
      double nn[1] = {0.0};
#pragma unroll 1
      for (int u = 0; u < NPT; ++u) {
        const int pl = t + u * kCoarseThreads;
        if (pl >= Nr) continue;
        float2 wv = ws[pl];
#pragma unroll
        for (int k = 0; k <= MI; ++k)
          if (k <= j) wv = csub(wv, cmul(scoef[k], vec(k)[p0 + pl]));
        ws[pl] = wv;
        nn[0] += (double)wv.x * wv.x + (double)wv.y * wv.y;
      }
      cluster_sum<1, MI>(nn, red, cred, par, cl, r);
      hn2 = nn[0];
      if (pass == 1 || sqrt(hn2) >= 0.25 * wn) break;
      // one re-orthogonalisation pass (krylov.py:105-111): extra = V^H w
#pragma unroll
      for (int k = 0; k < NACC; ++k) acc[k] = 0.0;
#pragma unroll 1
      for (int u = 0; u < NPT; ++u) {
        const int pl = t + u * kCoarseThreads;
        if (pl >= Nr) continue;
        const double2 wd = f2d(ws[pl]);
#pragma unroll
        for (int k = 0; k <= MI; ++k)
          if (k <= j) {
            const double2 d = zcmul(f2d(vec(k)[p0 + pl]), wd);
            acc[2 * k] += d.x;
            acc[2 * k + 1] += d.y;
          }
      }
      cluster_sum<NACC, MI>(acc, red, cred, par, cl, r);
      if (t == 0)
#pragma unroll
        for (int k = 0; k <= MI; ++k)
          if (k <= j) {
            hc[k] = make_double2(acc[2 * k] * vs[k], acc[2 * k + 1] * vs[k]);
            H[k * MI + j] = zadd(H[k * MI + j], hc[k]);
          }
      __syncthreads();
    }
    // the unnormalised V_{j+1} (this CTA's rows) for the later passes and the solution
    if (j + 1 < m) {
#pragma unroll
      for (int u = 0; u < NPT; ++u) {
        const int pl = t + u * kCoarseThreads;
        if (pl < Nr) V[(long long)(j + 1) * N + p0 + pl] = ws[pl];
      }
    }
    if (t == 0) {  // identical inputs in both CTAs: identical rotations and decisions
      const double hn = sqrt(hn2);
      double2 col[MI + 1];
      for (int k = 0; k <= j; ++k) col[k] = H[k * MI + j];
      for (int k = 0; k < j; ++k) {
        double2 a = col[k], bb = col[k + 1];
        double2 sk = sn[k];
        col[k] = zadd(zscale(a, cs[k]), zmul(sk, bb));
        col[k + 1] = zadd(zmul(make_double2(-sk.x, sk.y), a), zscale(bb, cs[k]));
      }
      double2 a = col[j];
      double c;
      double2 sv, rr;
      double mag = hypot(a.x, a.y);
      if (mag == 0.0) {
        c = 0.0;
        sv = make_double2(1.0, 0.0);
        rr = make_double2(hn, 0.0);
      } else {
        double tt = hypot(mag, hn);
        double2 ph = make_double2(a.x / mag, a.y / mag);
        c = mag / tt;
        sv = zscale(ph, hn / tt);
        rr = zscale(ph, tt);
      }
      cs[j] = c;
      sn[j] = sv;
      col[j] = rr;
      for (int k = 0; k <= j; ++k) H[k * MI + j] = col[k];
      double2 gj = gv[j];
      gv[j] = zscale(gj, c);
      gv[j + 1] = zmul(make_double2(-sv.x, sv.y), gj);
      const double est = hypot(gv[j + 1].x, gv[j + 1].y) / beta0;
      if (est <= 1e-12) {
        s_jend = j + 1;
        s_flag = 2;
      } else if (hn <= 1e-14 * fmax(1.0, wn)) {
        s_flag = 3;
      }
      vs[j + 1] = 1.0 / hn;
    }
    __syncthreads();
    if (s_flag == 2) break;
    if (s_flag == 3) {
      if (t == 0 && r == 0) atomicCAS(status + b, 0, HS_EBREAKDOWN);
      cl.sync();
      return;
    }
  }
  // y = R^{-1} g ; x = S sum_k y_k v_k on this CTA's rows
  const int jend = s_jend;
  if (t == 0) {
    for (int i = jend - 1; i >= 0; --i) {
      double2 acc2 = gv[i];
      for (int k = i + 1; k < jend; ++k) acc2 = zsub(acc2, zmul(H[i * MI + k], yv[k]));
      double2 d = H[i * MI + i];
      double den = d.x * d.x + d.y * d.y;
      yv[i] = make_double2((acc2.x * d.x + acc2.y * d.y) / den, (acc2.y * d.x - acc2.x * d.y) / den);
    }
  }
  __syncthreads();
#pragma unroll 1
  for (int u = 0; u < NPT; ++u) {
    const int pl = t + u * kCoarseThreads;
    if (pl >= Nr) continue;
    float2 sum = make_float2(0.f, 0.f);
#pragma unroll
    for (int k = 0; k < MI; ++k)
      if (k < jend) {
        const float2 yk = make_float2((float)(yv[k].x * vs[k]), (float)(yv[k].y * vs[k]));
        sum = cadd(sum, cmul(yk, vec(k)[p0 + pl]));
      }
    x[p0 + pl] = cmul(cscale(di[p0 + pl], damping), sum);
  }
  cl.sync();  // the partner may still read this CTA's exchange slots
}

void launch_coarse(LevelDev L, const float2* rhs, float2* x, float2* vws, float2* sws, const float2* const* active,
                   const int* model_of, int m, float damping, int* status, int B, cudaStream_t stream) {
  const long long nc = (long long)L.nx * L.ny;
  // 2-CTA clusters once a half fits 8 nodes per thread: a measurement variant only (HS_COARSE_CLUSTER=1).
  // Measured at C3 (64 RHS, 64 x 128): 352 us per V-cycle vs 301 us for one CTA per RHS -- the per-step
  // chain of reductions, now with cluster barriers, sets the pace, not the node loops.
  if (HS_COARSE_CLUSTER && m <= 10 && L.dinv && nc >= 2048 &&
      (L.nx - L.nx / 2) * (long long)L.ny <= kCoarseThreads * 8 && L.nx >= 2) {
    const int smem = 2 * kCoarseThreads * 8 * (int)sizeof(float2);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_coarse_gmres_cl<10, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      attr = true;
    }
    k_coarse_gmres_cl<10, 8><<<2 * B, kCoarseThreads, smem, stream>>>(L, rhs, x, vws, active, model_of, m, damping,
                                                                       status);
    return;
  }
  if (m <= 10 && L.dinv && nc <= kCoarseFastMax) {
    auto launch = [&](auto kern, int npt) {
      const int smem = 2 * kCoarseThreads * npt * (int)sizeof(float2);
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      kern<<<B, kCoarseThreads, smem, stream>>>(L, rhs, x, vws, active, model_of, m, damping, status);
    };
    if (nc <= kCoarseThreads * 8)
      launch(k_coarse_gmres_fast<10, 8>, 8);
    else
      launch(k_coarse_gmres_fast<10, 16>, 16);
  }
  else if (m <= 10)
    k_coarse_gmres<10><<<B, kCoarseThreads, 0, stream>>>(L, rhs, x, vws, sws, active, model_of, m, damping, status);
  else
    k_coarse_gmres<kCoarseMaxIters>
        <<<B, kCoarseThreads, 0, stream>>>(L, rhs, x, vws, sws, active, model_of, m, damping, status);
}

}  // namespace hs

// ------------------------------------------------------------------ host side

namespace hs {

namespace {
constexpr int kDownSmem = kVcWarps * kRing * kDownSlot * 8;
constexpr int kUpSmem = kVcWarps * kRing * kUpSlot * 8;

// rows per warp band: enough (column block, band) warps to fill every SM
// ~32 warps deep over the batch, but never bands shorter than `min_rows`
// (each band re-reads a few halo rows)
int band_rows(int rows, int ncb, int B, int min_rows, const void* kern, int smem) {
  static std::mutex mu;
  static std::map<const void*, int> cache;  // resident blocks per SM of each leg kernel
  int resident;
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(kern);
    if (it == cache.end()) {
      int nb = 0;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, kVcWarps * 32, smem);
      it = cache.emplace(kern, nb > 0 ? nb : 1).first;
    }
    resident = it->second;
  }
  const long target = HS_VC_WAVES > 0 ? (long)HS_VC_WAVES * 148 * resident * kVcWarps : 148L * 32;
  long nb = HS_VC_WAVES > 0 ? target / ((long)ncb * B) : (target + (long)ncb * B - 1) / ((long)ncb * B);
  const long cap = rows / min_rows;
  if (nb > cap) nb = cap;
  if (nb < 1) nb = 1;
  return (int)((rows + nb - 1) / nb);
}

__global__ void k_gather_scaled(VecIn in, const float2* const* active, float2* out, long long N) {
  const int b = blockIdx.y;
  if (active && active[b] == nullptr) return;
  const float2* src = vin_ptr(in, b);
  const float s = in.scale ? in.scale[b] : 1.f;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < N; p += (long long)gridDim.x * blockDim.x)
    out[b * N + p] = cscale(src[p], s);
}

__global__ void k_scatter(const float2* in, const float2* const* active, VecOut out, long long N) {
  const int b = blockIdx.y;
  if (active && active[b] == nullptr) return;
  float2* dst = vout_ptr(out, b);
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < N; p += (long long)gridDim.x * blockDim.x)
    dst[p] = in[b * N + p];
}

size_t align_up(size_t v) { return (v + 255) & ~size_t(255); }

// diag / dinv planes of every level (vcycle_prepare), at the head of the workspace
size_t planes_bytes(const Hierarchy& H) {
  size_t total = 0;
  for (int l = 0; l < H.num_levels; ++l) total += 2 * align_up((size_t)H.n_models * H.lv[l].nx * H.lv[l].ny * sizeof(float2));
  return total;
}

// diag = 4/h^2 - c + wall (level_diag, fp32 as before) and dinv = 1 / diag
// (fp64 division, rounded once) for every model of a level
__global__ void k_level_planes(LevelDev L, int n_models, float2* diag, float2* dinv) {
  const long long N = (long long)L.nx * L.ny, total = N * n_models;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    const long long p = q % N;
    const int i = (int)(p / L.ny), j = (int)(p - (long long)i * L.ny);
    const float2 d = level_diag(L, L.mass[q], i, j);
    const double den = (double)d.x * d.x + (double)d.y * d.y;
    diag[q] = d;
    dinv[q] = make_float2((float)(d.x / den), (float)(-d.y / den));
  }
}
}  // namespace

size_t vcycle_workspace_bytes(const Hierarchy& H, int B) {
  size_t total = planes_bytes(H);
  for (int l = 1; l < H.num_levels; ++l) {
    size_t n = (size_t)H.lv[l].nx * H.lv[l].ny;
    total += 2 * align_up(n * B * sizeof(float2));  // rhs_l and e_l
  }
  const LevelDev& C = H.lv[H.num_levels - 1];
  size_t nc = (size_t)C.nx * C.ny;
  total += align_up(nc * B * (H.coarse_iters + 1) * sizeof(float2));  // coarse basis
  total += align_up(nc * B * sizeof(float2));                          // coarse Jacobi scale
  if (H.num_levels == 1) total += 2 * align_up(nc * B * sizeof(float2));
  return total;
}

void vcycle_prepare(Hierarchy& H, void* ws, cudaStream_t stream) {
  char* p = static_cast<char*>(ws);
  for (int l = 0; l < H.num_levels; ++l) {
    LevelDev& L = H.lv[l];
    const size_t n = (size_t)H.n_models * L.nx * L.ny;
    float2* dg = reinterpret_cast<float2*>(p);
    p += align_up(n * sizeof(float2));
    float2* di = reinterpret_cast<float2*>(p);
    p += align_up(n * sizeof(float2));
    k_level_planes<<<(unsigned)std::min<size_t>(cdiv_u((long)n, 256), 4 * 148), 256, 0, stream>>>(L, H.n_models, dg, di);
    L.diag = dg;
    L.dinv = di;
  }
}

void vcycle(const Hierarchy& H_in, VecIn rhs, VecIn u0, VecOut out, const float2* const* active,
            const int* model_of, int B, void* ws, int* status, cudaStream_t stream) {
  Hierarchy H = H_in;
  if (!H.lv[0].dinv) vcycle_prepare(H, ws, stream);  // stand-alone call: derive the planes now
  char* p = static_cast<char*>(ws) + planes_bytes(H);
  float2* lrhs[kMaxLevels] = {nullptr};
  float2* lerr[kMaxLevels] = {nullptr};
  for (int l = 1; l < H.num_levels; ++l) {
    size_t n = (size_t)H.lv[l].nx * H.lv[l].ny;
    lrhs[l] = reinterpret_cast<float2*>(p);
    p += align_up(n * B * sizeof(float2));
    lerr[l] = reinterpret_cast<float2*>(p);
    p += align_up(n * B * sizeof(float2));
  }
  const int Lc = H.num_levels - 1;
  const LevelDev& C = H.lv[Lc];
  size_t nc = (size_t)C.nx * C.ny;
  float2* cV = reinterpret_cast<float2*>(p);
  p += align_up(nc * B * (H.coarse_iters + 1) * sizeof(float2));
  float2* cS = reinterpret_cast<float2*>(p);
  p += align_up(nc * B * sizeof(float2));

  if (H.num_levels == 1) {
    // multigrid.py:266-267: a one-level hierarchy is just the coarse solve (u0 ignored)
    float2* tmp_in = reinterpret_cast<float2*>(p);
    p += align_up(nc * B * sizeof(float2));
    float2* tmp_out = reinterpret_cast<float2*>(p);
    dim3 g(cdiv_u(nc, 256 * 4), B);
    k_gather_scaled<<<g, 256, 0, stream>>>(rhs, active, tmp_in, (long long)nc);
    launch_coarse(C, tmp_in, tmp_out, cV, cS, active, model_of, H.coarse_iters, H.coarse_damping, status, B, stream);
    k_scatter<<<g, 256, 0, stream>>>(tmp_out, active, out, (long long)nc);
    return;
  }
  // Algorithmic HBM bytes: per RHS and non-coarsest level,
  // down = rhs 8N + coarse 2N, up = rhs 8N + e 2N + out 8N (+ u0 8N twice at
  // level 0); the complex64 diag / dinv planes (16N down, 8N up) are read once
  // per slowness model per kernel (shared by every RHS of that model, L2-hot).
  const bool has_u0 = (u0.tab || u0.base);
  const double nact = prof::active_hint(B);
  double vc_bytes = 0.0;
  const int vslot = prof::start(prof::VCYCLE, stream);
  // down legs
  for (int l = 0; l < Lc; ++l) {
    const LevelDev& F = H.lv[l];
    const int ncx = H.lv[l + 1].nx, ncy = H.lv[l + 1].ny;
    VecIn in = l == 0 ? rhs : VecIn{nullptr, lrhs[l], (long long)F.nx * F.ny, nullptr};
    VecIn uz = l == 0 ? u0 : VecIn{nullptr, nullptr, 0, nullptr};
    const int ncb = (int)cdiv_u(ncy, kDownQ);
    const int band = band_rows(ncx, ncb, B, 4, (uz.tab || uz.base) ? (const void*)k_vc_down<true> : (const void*)k_vc_down<false>, kDownSmem);
    dim3 g(B, cdiv_u((long)ncb * cdiv_u(ncx, band), kVcWarps));  // RHS fastest: the planes stay L2-hot
    if (uz.tab || uz.base)
      k_vc_down<true><<<g, kVcWarps * 32, kDownSmem, stream>>>(F, ncx, ncy, in, uz, active, model_of, H.w_pre, lrhs[l + 1],
                                                       ncb, band);
    else
      k_vc_down<false><<<g, kVcWarps * 32, kDownSmem, stream>>>(F, ncx, ncy, in, uz, active, model_of, H.w_pre,
                                                        lrhs[l + 1], ncb, band);
    const double N = (double)F.nx * F.ny;
    vc_bytes += nact * (10.0 * N + ((l == 0 && has_u0) ? 8.0 * N : 0.0)) + H.n_models * 16.0 * N;
  }
  // coarsest
  launch_coarse(C, lrhs[Lc], lerr[Lc], cV, cS, active, model_of, H.coarse_iters, H.coarse_damping, status, B, stream);
  vc_bytes += nact * 16.0 * (double)nc + H.n_models * 8.0 * (double)nc;
  // up legs
  for (int l = Lc - 1; l >= 0; --l) {
    const LevelDev& F = H.lv[l];
    const int ncx = H.lv[l + 1].nx, ncy = H.lv[l + 1].ny;
    VecIn in = l == 0 ? rhs : VecIn{nullptr, lrhs[l], (long long)F.nx * F.ny, nullptr};
    VecIn uz = l == 0 ? u0 : VecIn{nullptr, nullptr, 0, nullptr};
    VecOut o = l == 0 ? out : VecOut{nullptr, lerr[l], (long long)F.nx * F.ny};
    const int ncb = (int)cdiv_u(F.ny, kUpCols);
    const int band = band_rows(F.nx, ncb, B, 8, (uz.tab || uz.base) ? (const void*)k_vc_up<true> : (const void*)k_vc_up<false>, kUpSmem);
    dim3 g(B, cdiv_u((long)ncb * cdiv_u(F.nx, band), kVcWarps));
    const double N = (double)F.nx * F.ny;
    const double up_bytes = nact * (18.0 * N + ((l == 0 && has_u0) ? 8.0 * N : 0.0)) + H.n_models * 8.0 * N;
    const int uslot = l == 0 ? prof::start(prof::VC_UP0, stream) : -1;
    if (uz.tab || uz.base)
      k_vc_up<true><<<g, kVcWarps * 32, kUpSmem, stream>>>(F, ncx, ncy, in, uz, active, model_of, H.w_pre, H.w_post,
                                                     lerr[l + 1], o, ncb, band);
    else
      k_vc_up<false><<<g, kVcWarps * 32, kUpSmem, stream>>>(F, ncx, ncy, in, uz, active, model_of, H.w_pre, H.w_post,
                                                      lerr[l + 1], o, ncb, band);
    prof::stop(uslot, stream, up_bytes);
    vc_bytes += up_bytes;
  }
  prof::stop(vslot, stream, vc_bytes);
  prof::count(2 * Lc + 1);
}

}  // namespace hs
