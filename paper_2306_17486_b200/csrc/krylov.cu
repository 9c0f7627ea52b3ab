// Batched device-resident flexible GMRES (krylov.py:39-146) for the outer
// Helmholtz solve.  Every RHS carries its own window position, Hessenberg
// matrix, Givens rotations and history, so RHS that converge (or restart
// after the drift guard, krylov.py:140-141) simply drop out of later steps.
//
// Precision recipe: the basis V and Z are complex64, the
// true-operator matvec A z and the true residual b - A x are evaluated in
// fp64 from the stored values, every reduction accumulates in fp64, the
// Hessenberg/Givens work is fp64 and the iterate x is complex128.
//
// w = A z_j is never stored: each Gram-Schmidt pass recomputes it in fp64
// registers from z_j (8 B/node) and the L2-resident medium.  V_{j+1} is written
// unnormalised with its scale 1/h_{j+1,j} kept per RHS, saving the
// normalisation sweep.
#include <algorithm>

#include "common.cuh"
#include "krylov.h"
#include "prof.h"

namespace hs {

namespace {

constexpr int NT = 128;
constexpr int KC = 10;            // basis vectors per chunk in a dot pass (registers vs w recomputes)
constexpr int PST = 2 * KC + 1;   // doubles per partial record
constexpr int kChunks = (kMaxRestart + KC - 1) / KC;
// The fused orthogonalisation + re-dot pass for windows of KC < J <= KCF vectors runs as ONE chunk of
// KCF (k_arnoldi<ORTH, KCF>): with chunks of KC every chunk's blocks recomputed w from all J vectors,
// so each vector was read once per chunk; one chunk reads each once, and w is formed from the same
// registers the dots use (more registers, fewer warps).
constexpr int KCF = 20;

// ORTH is the orthogonalisation pass fused with the re-dot (for RHS predicted
// to re-orthogonalise), ORTHP the plain one (the rest)
enum Mode { DOT = 0, ORTH = 1, REDOT = 2, ORTH2 = 3, ORTHP = 4 };

HS_DEV double2 ldz(const float2* p) {
  float2 v = *p;
  return make_double2((double)v.x, (double)v.y);
}

// (A u)(p) of the TRUE operator (shift 1 + 0i, no wall), fp64, summation
// order of neg_laplacian (fields.py:191-199) then minus c u (fields.py:208-210).
// Division by h2 becomes a multiply by its exact reciprocal when h2 is a power
// of two (bitwise identical; inv_h2 == 0 otherwise).
template <typename LD>
HS_DEV double2 apply_true(LD ld, const double2* __restrict__ c, int nx, int ny, int p, int i, int j, double h2,
                          double inv_h2) {
  double2 u = ld(p);
  double2 z0 = make_double2(0.0, 0.0);
  double2 xp = i + 1 < nx ? ld(p + ny) : z0;
  double2 xm = i > 0 ? ld(p - ny) : z0;
  double2 yp = j + 1 < ny ? ld(p + 1) : z0;
  double2 ym = j > 0 ? ld(p - 1) : z0;
  double lr = __dsub_rn(__dsub_rn(__dsub_rn(__dsub_rn(4.0 * u.x, xp.x), xm.x), yp.x), ym.x);
  double li = __dsub_rn(__dsub_rn(__dsub_rn(__dsub_rn(4.0 * u.y, xp.y), xm.y), yp.y), ym.y);
  double2 cu = zmul(c[p], u);
  const double qr = inv_h2 != 0.0 ? __dmul_rn(lr, inv_h2) : __ddiv_rn(lr, h2);
  const double qi = inv_h2 != 0.0 ? __dmul_rn(li, inv_h2) : __ddiv_rn(li, h2);
  return make_double2(__dsub_rn(qr, cu.x), __dsub_rn(qi, cu.y));
}

// Deterministic two-level reduction: block partials, then the last block of
// each RHS folds them in block order and runs `finish`.
HS_DEV bool arrive_last(int* counter, int total) {
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(counter, 1) == total - 1);
  __syncthreads();
  if (s_last) {
    __threadfence();
    if (threadIdx.x == 0) *counter = 0;
  }
  return s_last;
}

struct ArnArgs {
  const float2* Vb;
  const float2* zb;
  const double2* c;
  const double2* coef;  // shared memory
  int N, J, k0, chunk, p0, stride;
};

// One field sweep of a Gram-Schmidt pass.  NV is the number of basis vectors
// the pass touches per node, fixed at compile time so their loads are issued
// together: DOT / REDOT dot v_{k0} .. v_{k0+NV-1} (REDOT first subtracts every
// k < J with a runtime loop; it runs only where krylov.py:105 triggers), ORTH /
// ORTH2 subtract v_0 .. v_{NV-1} (NV = 0: runtime J).
template <int MODE, int NV, int KCT = KC>
HS_DEV void arn_sweep(const SolveDims& d, const ArnArgs& g, double (&acc)[2 * KCT + 1], int& bad) {
  const long long N = g.N;
  auto ldz_b = [&](int q) { return ldz(g.zb + q); };
  for (int p = g.p0; p < g.N; p += g.stride) {
    const int i = p / d.ny, jj = p - i * d.ny;
    if constexpr (MODE == DOT || MODE == REDOT || MODE == ORTH) {
      float2 v[NV > 0 ? NV : 1];
#pragma unroll
      for (int kk = 0; kk < NV; ++kk) v[kk] = g.Vb[(long long)(g.k0 + kk) * N + p];
      double2 w = apply_true(ldz_b, g.c, d.nx, d.ny, p, i, jj, d.h2, d.inv_h2);
      if (MODE == DOT) {
        if (!isfinite(w.x) || !isfinite(w.y)) bad = 1;
        if (g.chunk == 0) acc[2 * KCT] += w.x * w.x + w.y * w.y;
      } else {
        bool done = false;
        if constexpr (KCT == KCF && NV > 0) {  // the 20-vector chunk holds every vector: subtract from registers
          if (NV == g.J) {
#pragma unroll
            for (int k = 0; k < NV; ++k) w = zsub(w, zmul(g.coef[k], f2d(v[k])));
            done = true;
          }
        }
        if (!done)
          for (int k = 0; k < g.J; ++k) w = zsub(w, zmul(g.coef[k], ldz(g.Vb + (long long)k * N + p)));
        if (MODE == ORTH && g.chunk == 0) {
          const_cast<float2*>(g.Vb)[(long long)g.J * N + p] = d2f(w);
          acc[2 * KCT] += w.x * w.x + w.y * w.y;
        }
      }
#pragma unroll
      for (int kk = 0; kk < NV; ++kk) {
        const double2 dv = zcmul(f2d(v[kk]), w);
        acc[2 * kk] += dv.x;
        acc[2 * kk + 1] += dv.y;
      }
    } else {
      double2 w = apply_true(ldz_b, g.c, d.nx, d.ny, p, i, jj, d.h2, d.inv_h2);
      if constexpr (NV > 0) {
        float2 v[NV > 0 ? NV : 1];
#pragma unroll
        for (int k = 0; k < NV; ++k) v[k] = g.Vb[(long long)k * N + p];
#pragma unroll
        for (int k = 0; k < NV; ++k) w = zsub(w, zmul(g.coef[k], f2d(v[k])));
      } else {
        for (int k = 0; k < g.J; ++k) w = zsub(w, zmul(g.coef[k], ldz(g.Vb + (long long)k * N + p)));
      }
      const_cast<float2*>(g.Vb)[(long long)g.J * N + p] = d2f(w);
      acc[2 * KCT] += w.x * w.x + w.y * w.y;
    }
  }
}

// arn_sweep with the chunk's vector count as a compile-time constant 1..NV (the 20-vector fused pass)
template <int MODE, int KCT, int NV>
HS_DEV void arn_dispatch(int nv, const SolveDims& d, const ArnArgs& g, double (&acc)[2 * KCT + 1], int& bad) {
  if constexpr (NV > 1) {
    if (nv < NV) {
      arn_dispatch<MODE, KCT, NV - 1>(nv, d, g, acc, bad);
      return;
    }
  }
  arn_sweep<MODE, NV, KCT>(d, g, acc, bad);
}


template <int MODE, int KCT = KC>
__global__ void __launch_bounds__(NT) k_arnoldi(SolveDims d, SolveBuffers s, int nchunks) {
  constexpr int PT = 2 * KCT + 1;  // doubles per partial record
  __shared__ double red[PT * (NT / 32 + 1)];
  __shared__ double2 s_coef[kMaxRestart + 1];
  const int blk = blockIdx.x, chunk = blockIdx.y, b = blockIdx.z;
  RhsState& S = s.st[b];
  const int active = S.active;
  const int reorth = S.reorth;
  if (!active) return;
  if ((MODE == REDOT || MODE == ORTH2) && !reorth) return;
  if (MODE == REDOT && S.fused) return;  // the fused ORTH pass already added the re-dot
  if ((MODE == ORTH && !S.fuse) || (MODE == ORTHP && S.fuse)) return;
  const int j = S.j, J = j + 1, m = d.restart;
  if (MODE == ORTH && ((J > KC && J <= KCF) != (KCT == KCF))) return;  // the other fused-pass kernel's RHS
  // dot passes: only the chunks holding v_0..v_j do work (and take part in the
  // last-block count); the rest exit before touching memory
  const int live = (MODE == DOT || MODE == REDOT || MODE == ORTH) ? min(nchunks, (J + KCT - 1) / KCT) : nchunks;
  if (chunk >= live) return;
  const int N = (int)d.N;
  const float2* Vb = s.V + (long long)b * (m + 1) * N;
  const float2* zb = s.Z + ((long long)b * m + j) * N;
  const double2* c = s.c_true + (long long)(s.model_of ? s.model_of[b] : 0) * N;
  if (MODE != DOT) {
    for (int k = threadIdx.x; k < J; k += NT) s_coef[k] = zscale(S.hcol[k], S.vscale[k]);
    __syncthreads();
  }
  const int k0 = chunk * KCT;
  double acc[PT];
#pragma unroll
  for (int t = 0; t < PT; ++t) acc[t] = 0.0;
  int bad = 0;
  ArnArgs g{Vb, zb, c, s_coef, N, J, k0, chunk, blk * NT + (int)threadIdx.x, d.nblk * NT};
  if (MODE == DOT || MODE == REDOT || MODE == ORTH) {
    // vectors of this chunk, a compile-time count
    if constexpr (KCT != KC) {
      arn_dispatch<MODE, KCT, KCT>(min(KCT, J - k0), d, g, acc, bad);
    } else
    switch (min(KC, J - k0)) {
      case 1: arn_sweep<MODE, 1>(d, g, acc, bad); break;
      case 2: arn_sweep<MODE, 2>(d, g, acc, bad); break;
      case 3: arn_sweep<MODE, 3>(d, g, acc, bad); break;
      case 4: arn_sweep<MODE, 4>(d, g, acc, bad); break;
      case 5: arn_sweep<MODE, 5>(d, g, acc, bad); break;
      case 6: arn_sweep<MODE, 6>(d, g, acc, bad); break;
      case 7: arn_sweep<MODE, 7>(d, g, acc, bad); break;
      case 8: arn_sweep<MODE, 8>(d, g, acc, bad); break;
      case 9: arn_sweep<MODE, 9>(d, g, acc, bad); break;
      default: arn_sweep<MODE, 10>(d, g, acc, bad); break;
    }
  } else {
    // w -= sum_k coef_k v_k over every k < J: the runtime loop measured faster
    // than the fully unrolled one (159 vs 139 us per pass at C2)
    arn_sweep<MODE, 0, KCT>(d, g, acc, bad);
  }
  if (MODE == DOT && bad) atomicOr(&S.nonfinite, 1);
  block_sum<PT>(acc, red);
  double* part = s.partial + (((long long)b * nchunks + chunk) * d.nblk + blk) * PT;
#pragma unroll
  for (int t = 0; t < PT; ++t)  // constant indices keep acc[] in registers
    if (threadIdx.x == t) part[t] = acc[t];
  if (!arrive_last(&s.counter[b], live * d.nblk)) return;
  // ---- finish (one block per RHS)
  const double* pb = s.partial + (long long)b * nchunks * d.nblk * PT;
  if (MODE == DOT || MODE == REDOT) {
    for (int t = threadIdx.x; t < 2 * J; t += NT) {
      const int k = t >> 1, ch = k / KCT, slot = 2 * (k % KCT) + (t & 1);
      double sum = 0.0;
      for (int q = 0; q < d.nblk; ++q) sum += pb[((long long)ch * d.nblk + q) * PT + slot];
      red[t] = sum * S.vscale[k];
    }
    if (MODE == DOT && threadIdx.x == 0) {
      double nn = 0.0;
      for (int q = 0; q < d.nblk; ++q) nn += pb[(long long)q * PT + 2 * KCT];
      S.wn = sqrt(nn);
    }
    __syncthreads();
    for (int k = threadIdx.x; k < J; k += NT) {
      double2 v = make_double2(red[2 * k], red[2 * k + 1]);
      S.hcol[k] = MODE == DOT ? v : zadd(S.hcol[k], v);
    }
  } else if (MODE == ORTH) {
    // ||w||, the re-orthogonalisation test (krylov.py:105) and, when it fires,
    // the second-pass coefficients V^H w: this pass formed exactly the w the
    // re-dot would recompute (same operations, same order), so it dots it here
    for (int t = threadIdx.x; t < 2 * J; t += NT) {
      const int k = t >> 1, ch = k / KCT, slot = 2 * (k % KCT) + (t & 1);
      double sum = 0.0;
      for (int q = 0; q < d.nblk; ++q) sum += pb[((long long)ch * d.nblk + q) * PT + slot];
      red[t] = sum * S.vscale[k];
    }
    if (threadIdx.x == 0) {
      double nn = 0.0;
      for (int q = 0; q < d.nblk; ++q) nn += pb[(long long)q * PT + 2 * KCT];
      S.hn = sqrt(nn);
      S.reorth = S.hn < 0.25 * S.wn;
      S.fused = 1;
    }
    __syncthreads();
    if (S.reorth)
      for (int k = threadIdx.x; k < J; k += NT) S.hcol[k] = zadd(S.hcol[k], make_double2(red[2 * k], red[2 * k + 1]));
  } else if (threadIdx.x == 0) {
    double nn = 0.0;
    for (int q = 0; q < d.nblk; ++q) nn += pb[(long long)q * PT + 2 * KCT];
    S.hn = sqrt(nn);
    if (MODE == ORTHP) {
      S.reorth = S.hn < 0.25 * S.wn;  // krylov.py:105
      S.fused = 0;
    }
  }
}

// Hessenberg column, Givens rotation, estimate, stopping tests (krylov.py:112-135)
__global__ void k_givens(SolveDims d, SolveBuffers s) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= d.B) return;
  RhsState& S = s.st[b];
  if (!S.active) return;
  S.fuse = S.reorth;  // predict the next step's re-orthogonalisation from this one
  if (s.vstatus && s.vstatus[b]) {  // this RHS's coarse solve failed: only it stops (the reference raises per solve)
    S.status = s.vstatus[b];
    S.active = 0;
    return;
  }
  if (S.nonfinite) {
    S.status = HS_ENONFINITE;
    S.active = 0;
    return;
  }
  const int j = S.j;
  double2 col[kMaxRestart + 1];
  for (int k = 0; k <= j; ++k) col[k] = S.hcol[k];
  for (int k = 0; k < j; ++k) {
    double2 a = col[k], bb = col[k + 1], sk = S.sn[k];
    col[k] = zadd(zscale(a, S.cs[k]), zmul(sk, bb));
    col[k + 1] = zadd(zmul(make_double2(-sk.x, sk.y), a), zscale(bb, S.cs[k]));
  }
  const double hn = S.hn;
  double2 a = col[j];
  double cr;
  double2 sr, rr;
  const double mag = hypot(a.x, a.y);  // krylov.py:29-36
  if (mag == 0.0) {
    cr = 0.0;
    sr = make_double2(1.0, 0.0);
    rr = make_double2(hn, 0.0);
  } else {
    const double t = hypot(mag, hn);
    const double2 ph = make_double2(a.x / mag, a.y / mag);
    cr = mag / t;
    sr = zscale(ph, hn / t);
    rr = zscale(ph, t);
  }
  S.cs[j] = cr;
  S.sn[j] = sr;
  col[j] = rr;
  for (int k = 0; k <= j; ++k) S.H[k * kMaxRestart + j] = col[k];
  const double2 gj = S.g[j];
  S.g[j] = zscale(gj, cr);
  S.g[j + 1] = zmul(make_double2(-sr.x, sr.y), gj);
  S.iter += 1;
  S.j = j + 1;
  const double est = hypot(S.g[j + 1].x, S.g[j + 1].y) / S.beta0;
  s.hist[(long long)b * d.hist_stride + S.iter] = est;
  S.hist_len = S.iter + 1;
  if (est <= S.tol) {
    S.conv_est = 1;
    S.window_end = 1;
  } else if (hn <= 1e-14 * fmax(1.0, S.wn)) {
    S.status = HS_EBREAKDOWN;  // krylov.py:130-134
    S.active = 0;
    return;
  } else {
    S.vscale[j + 1] = 1.0 / hn;
    if (S.j == S.m) S.window_end = 1;
  }
  if (S.window_end) {  // y = R^{-1} g (krylov.py:149-153)
    const int n = S.j;
    for (int r = n - 1; r >= 0; --r) {
      double2 acc = S.g[r];
      for (int k = r + 1; k < n; ++k) acc = zsub(acc, zmul(S.H[r * kMaxRestart + k], S.y[k]));
      const double2 dd = S.H[r * kMaxRestart + r];
      const double den = dd.x * dd.x + dd.y * dd.y;
      S.y[r] = make_double2((acc.x * dd.x + acc.y * dd.y) / den, (acc.y * dd.x - acc.x * dd.y) / den);
    }
  }
}

// x += Z y at the end of a window (krylov.py:136-137)
__global__ void __launch_bounds__(NT) k_xupdate(SolveDims d, SolveBuffers s) {
  __shared__ double2 s_y[kMaxRestart];
  const int b = blockIdx.y;
  RhsState& S = s.st[b];
  if (!S.active || !S.window_end) return;
  const int n = S.j, N = (int)d.N;
  for (int k = threadIdx.x; k < n; k += NT) s_y[k] = S.y[k];
  __syncthreads();
  const float2* Zb = s.Z + (long long)b * d.restart * N;
  double2* xb = s.x + (long long)b * N;
  for (int p = blockIdx.x * NT + threadIdx.x; p < N; p += d.nblk * NT) {
    double2 t = make_double2(0.0, 0.0);
    for (int k = 0; k < n; ++k) t = zadd(t, zmul(s_y[k], ldz(Zb + (long long)k * N + p)));
    xb[p] = zadd(xb[p], t);
  }
}

HS_DEV void start_window(RhsState& S, const SolveDims& d, double beta) {
  S.m = min(min(d.restart, S.cap), S.cap - S.iter);  // krylov.py:79,83
  S.j = 0;
  S.vscale[0] = 1.0 / beta;
  S.g[0] = make_double2(beta, 0.0);
  for (int k = 1; k <= kMaxRestart; ++k) S.g[k] = make_double2(0.0, 0.0);
  S.window_end = 0;
  S.conv_est = 0;
  S.reorth = 0;
}

// r = b - A x (fp64), V_0 = r (unnormalised); INIT: beta0 and the first window,
// else the drift guard and restart logic of krylov.py:138-143.
template <bool INIT>
__global__ void __launch_bounds__(NT) k_residual(SolveDims d, SolveBuffers s, int use_x) {
  __shared__ double red[NT / 32 + 1];
  const int blk = blockIdx.x, b = blockIdx.y;
  RhsState& S = s.st[b];
  if (!S.active) return;
  if (!INIT && !S.window_end) return;
  const int N = (int)d.N, m = d.restart;
  const double2* xb = s.x + (long long)b * N;
  const double2* bb = s.b + (long long)b * N;
  const double2* c = s.c_true + (long long)(s.model_of ? s.model_of[b] : 0) * N;
  float2* V0 = s.V + (long long)b * (m + 1) * N;
  double acc[1] = {0.0};
  auto ldx = [&](int q) { return xb[q]; };
  for (int p = blk * NT + threadIdx.x; p < N; p += d.nblk * NT) {
    double2 r = bb[p];
    if (use_x) {
      const int i = p / d.ny, jj = p - i * d.ny;
      r = zsub(r, apply_true(ldx, c, d.nx, d.ny, p, i, jj, d.h2, d.inv_h2));
    }
    V0[p] = d2f(r);
    acc[0] += r.x * r.x + r.y * r.y;
  }
  block_sum<1>(acc, red);
  double* part = s.partial + (long long)b * kChunks * d.nblk * PST + blk;
  if (threadIdx.x == 0) part[0] = acc[0];
  if (!arrive_last(&s.counter[b], d.nblk)) return;
  if (threadIdx.x != 0) return;
  const double* pb = s.partial + (long long)b * kChunks * d.nblk * PST;
  double rr = 0.0;
  for (int q = 0; q < d.nblk; ++q) rr += pb[q];
  const double rn = sqrt(rr);
  double* hist = s.hist + (long long)b * d.hist_stride;
  if (INIT) {
    S.beta0 = rn;
    hist[0] = 1.0;
    S.hist_len = 1;
    if (rn == 0.0) {  // krylov.py:73-75
      hist[1] = 0.0;
      S.hist_len = 2;
      S.converged = 1;
      S.active = 0;
      return;
    }
    if (1.0 <= S.tol) {  // krylov.py:76-77
      S.converged = 1;
      S.active = 0;
      return;
    }
    start_window(S, d, rn);
    return;
  }
  const double true_rel = rn / S.beta0;
  if (S.conv_est && true_rel > S.tol) S.conv_est = 0;  // drift guard
  if (S.conv_est) {
    hist[S.iter] = true_rel;
    S.converged = 1;
    S.active = 0;
  } else if (S.iter >= S.cap) {
    S.active = 0;
  } else {
    start_window(S, d, rn);
  }
}

__global__ void k_init_state(SolveDims d, SolveBuffers s, const double* tol, const int* iter_cap) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= d.B) return;
  RhsState& S = s.st[b];
  S.active = 1;
  S.j = 0;
  S.m = 0;
  S.iter = 0;
  S.status = 0;
  S.nonfinite = 0;
  S.reorth = 0;
  S.fuse = 0;
  S.fused = 0;
  S.window_end = 0;
  S.conv_est = 0;
  S.converged = 0;
  S.hist_len = 0;
  S.tol = tol[b];
  S.cap = iter_cap ? min(max(iter_cap[b], 1), d.max_iter) : d.max_iter;
  S.beta0 = 0.0;
  s.counter[b] = 0;
}

__global__ void k_zero_x(SolveDims d, SolveBuffers s) {
  long long n = (long long)d.B * d.N;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x)
    s.x[p] = make_double2(0.0, 0.0);
}

__global__ void k_prep(SolveDims d, SolveBuffers s) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= d.B) return;
  const RhsState& S = s.st[b];
  const long long N = d.N;
  if (S.active) {
    s.vin[b] = s.V + ((long long)b * (d.restart + 1) + S.j) * N;
    s.vin_scale[b] = (float)S.vscale[S.j];
    s.zout[b] = s.Z + ((long long)b * d.restart + S.j) * N;
  } else {
    s.vin[b] = nullptr;
    s.vin_scale[b] = 0.f;
    s.zout[b] = nullptr;
  }
}

__global__ void k_count_active(SolveDims d, SolveBuffers s) {
  __shared__ int cnt;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  for (int b = threadIdx.x; b < d.B; b += blockDim.x)
    if (s.st[b].active) atomicAdd(&cnt, 1);
  __syncthreads();
  if (threadIdx.x == 0) *s.n_active = cnt;
}

}  // namespace

size_t krylov_partial_doubles(const SolveDims& d) { return (size_t)d.B * kChunks * d.nblk * PST; }

void krylov_init(const SolveDims& d, const SolveBuffers& s, const double* tol, const int* iter_cap, bool have_x0,
                 cudaStream_t stream) {
  k_init_state<<<cdiv_u(d.B, 128), 128, 0, stream>>>(d, s, tol, iter_cap);
  if (!have_x0) k_zero_x<<<592, 256, 0, stream>>>(d, s);
  k_residual<true><<<dim3(d.nblk, d.B), NT, 0, stream>>>(d, s, have_x0 ? 1 : 0);
}

void krylov_prep(const SolveDims& d, const SolveBuffers& s, cudaStream_t stream) {
  k_prep<<<cdiv_u(d.B, 128), 128, 0, stream>>>(d, s);
}

void krylov_after_precond(const SolveDims& d, const SolveBuffers& s, int j_hint, cudaStream_t stream) {
  const int nch = (std::min(d.restart, d.max_iter) + KC - 1) / KC;
  // algorithmic bytes of the dot pass: z_j (8N) + v_0..v_j (8N each) per RHS,
  // the complex128 true-operator mass (16N) once per model
  const double N = (double)d.N;
  const double dot_bytes = prof::active_hint(d.B) * 8.0 * N * (j_hint + 2) + d.n_models * 16.0 * N;
  const int slot = prof::start(prof::ARNOLDI, stream);
  k_arnoldi<DOT><<<dim3(d.nblk, nch, d.B), NT, 0, stream>>>(d, s, nch);
  prof::stop(slot, stream, dot_bytes);
  prof::count(8);
  // the other kernels of the step, each timed under tag KRYLOV with its own label when profiling is on
  auto timed = [&](int label, auto&& launch) {
    prof::set_label(label);
    const int sl = prof::start(prof::KRYLOV, stream);
    launch();
    prof::stop(sl, stream, 0.0);
  };
  timed(ORTH, [&] {  // + the re-dot (windows of up to KC vectors, and beyond KCF)
    k_arnoldi<ORTH><<<dim3(d.nblk, nch, d.B), NT, 0, stream>>>(d, s, nch);
  });
  if (d.restart > KC)  // windows of KC < J <= KCF vectors: one 20-vector chunk
    timed(5, [&] { k_arnoldi<ORTH, KCF><<<dim3(d.nblk, 1, d.B), NT, 0, stream>>>(d, s, 1); });
  timed(ORTHP, [&] { k_arnoldi<ORTHP><<<dim3(d.nblk, 1, d.B), NT, 0, stream>>>(d, s, 1); });
  timed(REDOT, [&] { k_arnoldi<REDOT><<<dim3(d.nblk, nch, d.B), NT, 0, stream>>>(d, s, nch); });
  timed(ORTH2, [&] { k_arnoldi<ORTH2><<<dim3(d.nblk, 1, d.B), NT, 0, stream>>>(d, s, 1); });
  timed(10, [&] { k_givens<<<cdiv_u(d.B, 64), 64, 0, stream>>>(d, s); });
  timed(11, [&] { k_xupdate<<<dim3(d.nblk, d.B), NT, 0, stream>>>(d, s); });
  timed(12, [&] { k_residual<false><<<dim3(d.nblk, d.B), NT, 0, stream>>>(d, s, 1); });
}

void krylov_count_active(const SolveDims& d, const SolveBuffers& s, cudaStream_t stream) {
  k_count_active<<<1, 256, 0, stream>>>(d, s);
}

}  // namespace hs
