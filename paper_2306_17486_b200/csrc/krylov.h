// Batched, device-resident flexible GMRES (krylov.py:39-146).
#pragma once
#include "vcycle.h"

namespace hs {

// Per-RHS solver state, device resident.  Field meanings follow the local
// variables of the reference fgmres loop (krylov.py:79-143).
struct RhsState {
  int active;       // still iterating
  int j;            // position inside the current restart window
  int m;            // length of the current window (krylov.py:83)
  int iter;         // total iterations (preconditioner applications)
  int status;       // HsStatus; 0 while fine
  int nonfinite;    // set by the Arnoldi pass when A z has a NaN/Inf
  int reorth;       // second Gram-Schmidt pass needed this step
  int fuse;         // predicted re-orthogonalisation: the ORTH pass also forms the re-dot
  int fused;        // whether this step's ORTH pass did
  int window_end;   // x update + true residual due this step
  int conv_est;     // the Givens estimate met tol this window
  int converged;    // final flag (SolveReport.converged)
  int hist_len;     // entries written to the history
  int cap;          // this RHS's iteration cap (<= SolveDims::max_iter)
  double beta0, tol, wn, hn;
  double vscale[kMaxRestart + 1];   // v_k = vscale[k] * V_k (V stored unnormalised)
  double2 hcol[kMaxRestart + 1];    // Gram-Schmidt coefficients of this step (total)
  double2 g[kMaxRestart + 1];
  double cs[kMaxRestart];
  double2 sn[kMaxRestart];
  double2 H[(kMaxRestart + 1) * kMaxRestart];  // H[row * kMaxRestart + col]
  double2 y[kMaxRestart];
};

struct SolveDims {
  int B, nx, ny, n_models;
  long long N;
  double h2;          // h*h of the finest grid
  double inv_h2;      // 1/h2 when h2 is a power of two (x / h2 == x * inv_h2 exactly), else 0
  int restart;        // window length parameter (krylov.py:79)
  int max_iter;
  int nblk;           // blocks per RHS for the field-sweeping kernels
  int hist_stride;    // max_iter + 2
};

struct SolveBuffers {
  float2* V;          // (B, restart+1, N) complex64, unnormalised basis
  float2* Z;          // (B, restart, N)   complex64, preconditioned basis
  double2* x;         // (B, N) complex128 iterate
  const double2* b;   // (B, N) complex128 right-hand sides
  const double2* c_true;  // (n_models, N) complex128 mass term of the true operator
  const int* model_of;    // (B,) or null
  RhsState* st;       // (B,)
  double* hist;       // (B, hist_stride)
  double* partial;    // reduction scratch
  int* counter;       // (B,) last-block counters, zero-initialised
  // per-step pointer tables for the preconditioner
  const float2** vin;
  float* vin_scale;
  float2** zout;
  int* n_active;      // device scalar
  const int* vstatus; // (B,) V-cycle status of each RHS (coarse GMRES), or null
};

size_t krylov_partial_doubles(const SolveDims& d);

// initial residual: x <- x0 (or 0), r = b - A x, beta0, first window
void krylov_init(const SolveDims& d, const SolveBuffers& s, const double* tol, const int* iter_cap, bool have_x0,
                 cudaStream_t stream);
// pointer tables for the preconditioner of the current step
void krylov_prep(const SolveDims& d, const SolveBuffers& s, cudaStream_t stream);
// everything after z_j = M v_j: Arnoldi, Givens, window end
void krylov_after_precond(const SolveDims& d, const SolveBuffers& s, int j_hint, cudaStream_t stream);
void krylov_count_active(const SolveDims& d, const SolveBuffers& s, cudaStream_t stream);

}  // namespace hs
