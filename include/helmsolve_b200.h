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

/* One 3x3 convolution of the network with batch norm folded in
 * (autodiff.conv2d / conv_transpose2d + batchnorm2d inference + softplus,
 * autodiff.py:472-607): y = act(conv(x, w) + b).  w is device float32
 * [cout][3][3][cin]; a transposed layer (stride 2) uses the same order. */
typedef struct {
  int cin, cout, stride, transposed, softplus;
  const float* w;
  const float* b;
} hs_conv_t;

/* Layer table of the ARCH.md network (the network.py the reference imports
 * at krylov.py:201 but never shipped).  Index l of the per-level arrays is
 * level l (0 = finest); down[0] / up[0] are unused. */
typedef struct {
  int levels;
  int channels[8];
  int ix, iy;            /* network grid (nx-1, ny-1) */
  int nx, ny;            /* PDE grid */
  float out_scale;       /* h^2/64 */
  hs_conv_t enc_stem, enc_res_a[8], enc_res_b[8], enc_down[8];
  hs_conv_t sol_stem, sol_res_a[8], sol_res_b[8], sol_down[8];
  hs_conv_t sol_up[8], sol_ures_a[8], sol_ures_b[8], sol_head;
  const void* implicit_w; /* complex64 (C_{L-1}/2, 3, 3) */
} hs_net_desc_t;

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
  const int* iter_cap;   /* (B,) device, per-RHS iteration cap (<= max_iter), or NULL: max_iter for every RHS
                            (training-pair generation runs k ~ U{2..20} iterations per sample in one solve) */
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
 * is multigrid.coarse_solve (multigrid.py:232-244). */
HS_API size_t hs_vcycle_workspace_bytes(const hs_hierarchy_t* h, int B);
HS_API int hs_vcycle(const hs_hierarchy_t* h, const void* rhs, const void* u0, void* out, const int* model_of,
                     int B, void* ws, size_t ws_bytes, int* status, void* stream);
/* status: B device ints, zeroed by the caller; status[b] receives HS_EBREAKDOWN / HS_ENONFINITE when RHS b's
   coarse-grid GMRES fails (multigrid.py:232-244 -> krylov.py:96-99, :130-134) */

/* krylov.fgmres specialised to the Helmholtz solve (krylov.py:39-146), the
 * engine behind krylov.solve_helmholtz (:156-177) and both phases of
 * krylov.solve_with_learned_preconditioner (:180-246).  net == NULL: apply_M
 * = v_cycle(r, None); otherwise apply_M = v_cycle(r, net(r)) (krylov.py:225-226).
 * Blocks until every RHS has converged, hit max_iter or failed. */
HS_API size_t hs_fgmres_workspace_bytes(const hs_hierarchy_t* h, const hs_net_t* net, int B, int nx, int ny,
                                        int restart, int max_iter);
HS_API int hs_fgmres_solve(const hs_hierarchy_t* h, const hs_net_t* net, const hs_solve_args_t* args, void* ws,
                           size_t ws_bytes, void* stream);

/* ---- network (ARCH.md; the missing helmsolve.network, krylov.py:201) ---- */

/* Build the device network; also computes the implicit layer's Green
 * spectrum once (green.ImplicitKernel.spectrum, green.py:139-146).  The
 * layer weights stay owned by the caller and must outlive the network. */
HS_API int hs_net_create(hs_net_t** net, const hs_net_desc_t* desc, void* stream);
HS_API void hs_net_destroy(hs_net_t* net);
/* network.precompute_encodings (krylov.py:205-206): media is float32 NHWC
 * (n_models, ix, iy, 2) = (kappa^2, gamma); enc[l] receives the level-l
 * encodings, float32 NHWC (n_models, ix/2^l, iy/2^l, channels[l]), and the
 * network keeps pointers to them for later forwards. */
HS_API size_t hs_net_encode_workspace_bytes(const hs_net_t* net, int n_models);
HS_API int hs_net_encode(hs_net_t* net, const float* media, int n_models, float* const* enc, void* ws,
                         size_t ws_bytes, void* stream);
/* ---- tracing (the reference only reports SolveReport.wall_time) ---- */
/* tags: 0 every conv (work = flops), 1 level-0 16-channel convs, 2 V-cycle
 * (work = algorithmic bytes), 3 Gram-Schmidt dot pass (bytes), 4 network
 * forward, 5 implicit layer, 6 finest-level V-cycle up-leg kernel (bytes). */
HS_API void hs_profile_enable(unsigned tag_mask);
HS_API void hs_profile_reset(void);
HS_API int hs_profile_query(int tag, double* total_ms, double* total_work, long long* count);
/* kernels launched by the library since the last hs_profile_reset */
HS_API long long hs_launch_count(void);
/* per-launch records of the enabled tags (tracing; no reference counterpart) */
HS_API int hs_profile_records(int* tags, int* labels, double* ms, int max);
/* 1 (default): tcgen05 BF16x3 convolutions (exact three-way bf16 split, fp32 accumulate) where the shape
   allows; 0: SIMT fp32 only (a test switch for A/B parity; it never skips work) */
HS_API void hs_set_conv_path(int tensor_cores);

/* ---- slowness-model preparation (SPEC.md datagen: load_slowness_corpus / gaussian_smooth,
 *      reference SPEC.md:404-417,441).  fp64 fields (B, rows, cols), device pointers. */
/* corner-aligned bilinear resize (B, hin, win) -> (B, hout, wout) */
HS_API int hs_resize_bilinear(const double* in, double* out, int B, int hin, int win, int hout, int wout,
                              void* stream);
/* separable truncated Gaussian, radius ceil(3 sigma), edge-replicated; sigma = 0 is the identity.
 * tmp: (B, nx, ny) scratch.  Blocks until done. */
HS_API int hs_gaussian_smooth(const double* in, double* out, double* tmp, int B, int nx, int ny, double sigma,
                              void* stream);
/* affine map of each field onto [lo, hi]; a constant field maps to lo.  minmax: (B, 2) scratch out. */
HS_API int hs_normalise_range(const double* in, double* out, double* minmax, int B, long long n, double lo,
                              double hi, void* stream);

/* use caller-held encodings (same layout as hs_net_encode's output) */
HS_API int hs_net_set_encodings(hs_net_t* net, int levels, const float* const* enc);
/* network.preconditioner_estimate (krylov.py:225-226): u0 = (h^2/64) net(r),
 * r and u0 complex64 (B, nx, ny); model_of selects each RHS's encodings. */
HS_API size_t hs_net_workspace_bytes(const hs_net_t* net, int B);
HS_API int hs_net_forward(const hs_net_t* net, const void* r, void* u0, const int* model_of, int B, void* ws,
                          size_t ws_bytes, void* stream);
/* green.green_function (green.py:55-82): kernel complex64 (C, 3, 3) ->
 * spectrum complex128 (C, 2h, 2w), the reference's numpy-2 dtype flow. */
HS_API int hs_green_spectrum(const void* kernel, int C, int h, int w, void* spectrum, void* stream);
/* the same with the regulariser as an argument (green.py:55, green_function(..., eps=SPECTRUM_EPS));
 * hs_green_spectrum is this with eps = 1e-5 (green.py:19) */
HS_API int hs_green_spectrum_eps(const void* kernel, int C, int h, int w, double eps, void* spectrum, void* stream);
/* green.implicit_apply (green.py:85-107): x complex64 (B, C, h, w),
 * spectrum complex64 (C, 2h, 2w) -> y complex64 (B, C, h, w). */
HS_API int hs_implicit_apply(const void* x, const void* spectrum, void* y, int B, int C, int h, int w,
                             void* stream);
/* one network convolution on float32 NHWC tensors (autodiff.conv2d /
 * conv_transpose2d, pad 1): y = act(conv(x) + b) [+ addend] [+ residual]. */
HS_API int hs_conv2d(const float* x, const hs_conv_t* conv, const float* addend, const float* residual, float* y,
                     int B, int H, int W, void* stream);

/* ---- network training (SPEC.md `[MODULE] trainer`, reference SPEC.md:454-507).
 * The reference has no trainer; one step is the SPEC mse_loss of u0 = (h^2/64) net(r) against the
 * true error e, backward through the reference autodiff's rules (autodiff.py: conv2d :472-507,
 * conv_transpose2d :510-544, batchnorm2d training :547-592, softplus :243-252, green.py:55-107),
 * then Adam.  Parameters are one float32 vector in netparams.param_spec order (complex implicit
 * kernels as (re, im) pairs), running batch-norm statistics included and updated in place. */
typedef struct hs_trainer hs_trainer_t;
typedef struct {
  int levels;      /* L >= 2 */
  int channels[8]; /* C_0 .. C_{L-1}, powers of two <= 256, C_{L-1} even */
  int nx, ny;      /* node grid; the network grid is (nx-1, ny-1), divisible by 2^(L-1) */
  int batch;       /* samples per step */
  double h;        /* grid spacing of the u0 scale h^2/64 */
} hs_train_desc_t;
typedef struct {
  float lr, beta1, beta2, eps; /* torch.optim.Adam defaults: 1e-3, 0.9, 0.999, 1e-8 */
} hs_adam_t;
/* floats in the flat parameter vector (0 for an invalid descriptor) */
HS_API size_t hs_train_param_count(const hs_train_desc_t* desc);
/* params: host float32 vector of hs_train_param_count floats */
HS_API int hs_trainer_create(hs_trainer_t** out, const hs_train_desc_t* desc, const float* params, void* stream);
HS_API void hs_trainer_destroy(hs_trainer_t* t);
/* media: device float32 (n_models, 2, nx-1, ny-1) (kappa^2, gamma); model_of: HOST int (batch,);
 * r, e: device complex128 (batch, nx, ny).  adam NULL = gradients only (no update).  loss (host,
 * optional) receives the batch MSE and makes the call synchronous; HS_ENONFINITE on a non-finite loss. */
HS_API int hs_trainer_step(hs_trainer_t* t, const float* media, int n_models, const int* model_of, const void* r,
                           const void* e, const hs_adam_t* adam, double* loss, void* stream);
/* data-parallel training: copy the flat float32 gradient vector to (to_trainer = 0) or from (1)
 * a caller DEVICE buffer, so an all-reduce can run between the backward pass (hs_trainer_step with
 * adam = NULL) and hs_trainer_apply. */
HS_API int hs_trainer_grads(hs_trainer_t* t, void* dev, int to_trainer, void* stream);
/* one Adam step on the trainer's current gradient vector */
HS_API int hs_trainer_apply(hs_trainer_t* t, const hs_adam_t* adam, void* stream);
/* which: 0 parameters, 1 last gradients, 2 Adam m, 3 Adam v; host float32 out */
HS_API int hs_trainer_read(const hs_trainer_t* t, int which, float* host, void* stream);
/* which: 0 parameters, 2 Adam m, 3 Adam v (checkpoint restore); step >= 0 sets Adam's step counter */
HS_API int hs_trainer_write(hs_trainer_t* t, int which, const float* host, int step, void* stream);

#endif
