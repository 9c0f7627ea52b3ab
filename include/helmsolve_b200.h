/*
 * helmsolve_b200 — C ABI of the B200-native Helmholtz FGMRES hot path.
 *
 * The reference (helmsolve, pure numpy) exposes this path as Python
 * callables: fgmres(apply_A, apply_M, ...) with apply_A = the Helmholtz
 * operator and apply_M = the V-cycle, optionally preceded by the network
 * (krylov.py:39-47, :156-246).  Each entry point below replaces one of those
 * reference interfaces; the citation is given per function.  A reference
 * maintainer binds them with ctypes.
 *
 * Conventions
 *  - All pointers are DEVICE pointers unless stated; the caller allocates every
 *    buffer (the library never frees caller memory).  Fields are (B, nx, ny)
 *    row-major (iy fastest), the reference's data[ix, iy] C order
 *    (fields.py:5-12).  complex64 = interleaved float2, complex128 = double2.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  Calls are
 *    asynchronous on it except hs_fgmres_solve, which polls for completion.
 *  - Return codes: HS_OK or one of the HS_E* codes; hs_last_error() gives the
 *    message of the calling thread's last failure.  Per-RHS solver failures
 *    are reported through the status array (same codes).
 */
#ifndef HELMSOLVE_B200_H
#define HELMSOLVE_B200_H

#include <stddef.h>

#ifdef __cplusplus
#define HS_EXTERN extern "C"
#else
#define HS_EXTERN
#endif
#define HS_API HS_EXTERN __attribute__((visibility("default")))

enum {
  HS_OK = 0,
  HS_EDIMENSION = 1, /* errors.DimensionError   (errors.py:4)  */
  HS_ESINGULAR = 2,  /* errors.SingularityError (errors.py:8)  */
  HS_EBREAKDOWN = 3, /* errors.SolverError      (errors.py:12) */
  HS_ENONFINITE = 4, /* errors.NumericalError   (errors.py:16) */
  HS_ECONFIG = 5,    /* errors.ConfigurationError (errors.py:24) */
  HS_ECUDA = 6
};

/* hs_helm_apply modes */
enum {
  HS_APPLY_C64_F32 = 0,  /* u c64, mass c64,  out c64,  fp32 math (V-cycle levels) */
  HS_APPLY_C64_F64 = 1,  /* u c64, mass c128, out c128, fp64 math (outer operator on the basis) */
  HS_APPLY_C128 = 2      /* u c128, mass c128, out c128, fp64 math (reference arithmetic) */
};

/* One grid level (multigrid.Level, multigrid.py:128-150).  `mass` holds the
 * complex per-node factor c = omega^2 kappa^2 (alpha - i(beta + gamma))
 * (fields.mass_coefficient, fields.py:186-188) for each slowness model:
 * complex64 (n_models, nx, ny).  The wall re-alignment term
 * (multigrid.py:153-163) is wall_x on row nx-1 and wall_y on column ny-1. */
typedef struct {
  int nx, ny;
  double h;
  double wall_x, wall_y;
  const void* mass;
} hs_level_t;

/* multigrid.GridHierarchy (multigrid.py:166-182). */
typedef struct {
  int num_levels;
  int n_models;
  hs_level_t levels[8];
  int relax_pre, relax_post;       /* only 1/1 (the reference default) is fused */
  double damping_pre, damping_post;
  int coarse_iters;                /* <= 16 */
  double coarse_damping;           /* 0.8, multigrid.py:233 */
} hs_hierarchy_t;

/* Encoder-solver network prepared for the device (ARCH.md); opaque. */
typedef struct hs_net hs_net_t;

/* Arguments of one batched FGMRES solve (krylov.fgmres, krylov.py:39-146,
 * with apply_A = the true operator and apply_M = V-cycle or net->V-cycle). */
typedef struct {
  int B;                 /* right-hand sides */
  int max_iter;          /* krylov.py:45 */
  int restart;           /* krylov.py:46 (<= 32) */
  const void* b;         /* complex128 (B, nx, ny) */
  const void* x0;        /* complex128 (B, nx, ny) or NULL (zero guess) */
  void* x;               /* complex128 (B, nx, ny) out */
  const double* tol;     /* (B,) relative tolerance per RHS */
  const void* c_true;    /* complex128 (n_models, nx, ny): mass of the TRUE operator */
  const int* model_of;   /* (B,) slowness-model index per RHS, or NULL (all 0) */
  double* hist;          /* (B, max_iter + 2) relative-residual history out */
  int* hist_len;         /* (B,) out */
  int* iterations;       /* (B,) out */
  int* converged;        /* (B,) out */
  int* status;           /* (B,) out: HS_OK / HS_EBREAKDOWN / HS_ENONFINITE */
} hs_solve_args_t;

/* version of the ABI (bumped on incompatible changes) */
HS_API int hs_abi_version(void);
HS_API const char* hs_last_error(void);

/* fields.apply_helmholtz_array / multigrid.Level.apply (fields.py:202-210,
 * multigrid.py:146-150): out = -Lap_h u - c u + wall u for B fields. */
HS_API int hs_helm_apply(const void* u, void* out, const void* mass, const int* model_of, int B, int nx,
                         int ny, double h, double wall_x, double wall_y, int mode, void* stream);

/* multigrid.restrict_full_weighting (multigrid.py:64-78); complex64 (f64 = 0)
 * or complex128 (f64 = 1) fields. */
HS_API int hs_restrict(const void* fine, void* coarse, int B, int nx, int ny, int f64, void* stream);
/* multigrid.prolong_bilinear (multigrid.py:81-114); complex64 / complex128. */
HS_API int hs_prolong(const void* coarse, void* fine, int B, int ncx, int ncy, int nx, int ny, int f64,
                      void* stream);
/* multigrid.jacobi_relax, one sweep (multigrid.py:218-229); complex64. */
HS_API int hs_jacobi(const void* u, const void* rhs, void* out, const hs_level_t* level, const int* model_of,
                     int B, double damping, void* stream);

/* multigrid.v_cycle (multigrid.py:247-274) over B right-hand sides;
 * rhs/u0/out complex64 (B, nx0, ny0); u0 may be NULL.  A one-level hierarchy
 * is multigrid.coarse_solve (multigrid.py:232-244). `status` (device int,
 * may be NULL) receives HS_EBREAKDOWN / HS_ENONFINITE from the coarse GMRES. */
HS_API size_t hs_vcycle_workspace_bytes(const hs_hierarchy_t* h, int B);
HS_API int hs_vcycle(const hs_hierarchy_t* h, const void* rhs, const void* u0, void* out, const int* model_of,
                     int B, void* ws, size_t ws_bytes, int* status, void* stream);

/* krylov.fgmres specialised to the Helmholtz solve (krylov.py:39-146), the
 * engine behind krylov.solve_helmholtz (:156-177) and both phases of
 * krylov.solve_with_learned_preconditioner (:180-246).  net == NULL: apply_M
 * = v_cycle(r, None); otherwise apply_M = v_cycle(r, net(r)) (krylov.py:225-226).
 * Blocks until every RHS has converged, hit max_iter or failed. */
HS_API size_t hs_fgmres_workspace_bytes(const hs_hierarchy_t* h, const hs_net_t* net, int B, int nx, int ny,
                                        int restart, int max_iter);
HS_API int hs_fgmres_solve(const hs_hierarchy_t* h, const hs_net_t* net, const hs_solve_args_t* args, void* ws,
                           size_t ws_bytes, void* stream);

#endif
