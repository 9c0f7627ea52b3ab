// C ABI (include/helmsolve_b200.h) and the host driver of the batched solve.
#include <cstdio>
#include <cstring>
#include <string>

#include "../../include/helmsolve_b200.h"
#include "cnn.h"
#include <cmath>

#include "common.cuh"
#include "krylov.h"
#include "prof.h"
#include "stencil.h"
#include "vcycle.h"

namespace hs {
thread_local std::string g_last_error;
int set_error(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}
}  // namespace hs

namespace {

int fail(int code, const std::string& msg) { return hs::set_error(code, msg); }

int check_cuda(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(HS_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return HS_OK;
}

size_t align_up(size_t v) { return (v + 255) & ~size_t(255); }

int to_hierarchy(const hs_hierarchy_t* h, hs::Hierarchy& H) {
  if (!h) return fail(HS_ECONFIG, "null hierarchy");
  if (h->num_levels < 1 || h->num_levels > hs::kMaxLevels)
    return fail(HS_ECONFIG, "num_levels must lie in [1, 8]");
  if (h->relax_pre != 1 || h->relax_post != 1)
    return fail(HS_ECONFIG, "the fused V-cycle implements relax_pre = relax_post = 1 (the reference default)");
  if (h->coarse_iters < 1 || h->coarse_iters > hs::kCoarseMaxIters)
    return fail(HS_ECONFIG, "coarse_iters must lie in [1, 16]");
  H.num_levels = h->num_levels;
  H.n_models = h->n_models;
  for (int l = 0; l < h->num_levels; ++l) {
    const hs_level_t& s = h->levels[l];
    if (l > 0 && (s.nx != h->levels[l - 1].nx / 2 || s.ny != h->levels[l - 1].ny / 2))
      return fail(HS_EDIMENSION, "level shapes must halve (multigrid.py:55-56)");
    if (l + 1 < h->num_levels && (s.nx < 5 || s.ny < 5))
      return fail(HS_EDIMENSION, "grid too small to coarsen");
    H.lv[l] = LevelDev{s.nx, s.ny, (float)(1.0 / (s.h * s.h)), (float)s.wall_x, (float)s.wall_y,
                           static_cast<const float2*>(s.mass)};
  }
  H.w_pre = (float)h->damping_pre;
  H.w_post = (float)h->damping_post;
  H.coarse_iters = h->coarse_iters;
  H.coarse_damping = (float)h->coarse_damping;
  return HS_OK;
}

__global__ void k_table(const float2* base, long long stride, const float2** tab, int B) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < B) tab[b] = base + b * stride;
}

__global__ void k_finalize(hs::SolveDims d, hs::SolveBuffers s, int* hist_len, int* iters, int* conv, int* status,
                           const int* vstatus) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= d.B) return;
  const hs::RhsState& S = s.st[b];
  hist_len[b] = S.hist_len;
  iters[b] = S.iter;
  conv[b] = S.converged;
  int st = S.status;
  if (st == 0 && vstatus && vstatus[b]) st = vstatus[b];  // this RHS's coarse-grid GMRES failed
  status[b] = st;
}

int choose_nblk(long long N, int B) {
  long long want = (16LL * 148 + B - 1) / B;
  long long cap = (N + 256 * 8 - 1) / (256 * 8);
  long long n = want < cap ? want : cap;
  return (int)(n < 1 ? 1 : n);
}

struct SolveLayout {
  size_t V, Z, st, partial, counter, vin, vin_scale, zout, n_active, vstatus, vws, netws, u0, total;
};

SolveLayout layout(const hs::Hierarchy& H, const hs_net_t* net, int B, long long N, int restart, int max_iter) {
  SolveLayout L{};
  hs::SolveDims d{};
  d.B = B;
  d.N = N;
  d.nblk = choose_nblk(N, B);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += align_up(bytes);
    return o;
  };
  L.V = take((size_t)B * (restart + 1) * N * sizeof(float2));
  L.Z = take((size_t)B * restart * N * sizeof(float2));
  L.st = take((size_t)B * sizeof(hs::RhsState));
  L.partial = take(hs::krylov_partial_doubles(d) * sizeof(double));
  L.counter = take((size_t)B * sizeof(int));
  L.vin = take((size_t)B * sizeof(void*));
  L.vin_scale = take((size_t)B * sizeof(float));
  L.zout = take((size_t)B * sizeof(void*));
  L.n_active = take(sizeof(int));
  L.vstatus = take((size_t)B * sizeof(int));  // per-RHS V-cycle status (coarse GMRES breakdown / NaN)
  L.vws = take(hs::vcycle_workspace_bytes(H, B));
  L.netws = net ? take(hs::cnn_workspace_bytes(net, B)) : 0;
  L.u0 = net ? take((size_t)B * N * sizeof(float2)) : 0;
  L.total = off;
  (void)max_iter;
  return L;
}

int* pinned_flag() {
  static thread_local int* p = nullptr;
  if (!p) cudaHostAlloc(&p, sizeof(int), cudaHostAllocDefault);
  return p;
}

}  // namespace

HS_API int hs_abi_version(void) { return 2; }  // 2: hs_solve_args_t.iter_cap
HS_API const char* hs_last_error(void) { return hs::g_last_error.c_str(); }

HS_API int hs_helm_apply(const void* u, void* out, const void* mass, const int* model_of, int B, int nx, int ny,
                         double h, double wall_x, double wall_y, int mode, void* stream) {
  if (B < 1 || nx < 1 || ny < 1) return fail(HS_EDIMENSION, "empty field");
  if (mode < 0 || mode > 2) return fail(HS_ECONFIG, "unknown apply mode");
  hs::helm_apply(u, out, mass, model_of, B, nx, ny, h, wall_x, wall_y, mode, (cudaStream_t)stream);
  return check_cuda("hs_helm_apply");
}

HS_API int hs_restrict(const void* fine, void* coarse, int B, int nx, int ny, int f64, void* stream) {
  if (nx < 5 || ny < 5) return fail(HS_EDIMENSION, "grid " + std::to_string(nx) + "x" + std::to_string(ny) + " too small to coarsen");
  hs::restrict_fw(fine, coarse, B, nx, ny, f64, (cudaStream_t)stream);
  return check_cuda("hs_restrict");
}

HS_API int hs_prolong(const void* coarse, void* fine, int B, int ncx, int ncy, int nx, int ny, int f64,
                      void* stream) {
  if (!(2 * ncx <= nx && nx <= 2 * ncx + 1 && 2 * ncy <= ny && ny <= 2 * ncy + 1))
    return fail(HS_EDIMENSION, "cannot prolong onto that shape; expected about 2x");
  hs::prolong_bl(coarse, fine, B, ncx, ncy, nx, ny, f64, (cudaStream_t)stream);
  return check_cuda("hs_prolong");
}

HS_API int hs_jacobi(const void* u, const void* rhs, void* out, const hs_level_t* lv, const int* model_of, int B,
                     double damping, void* stream) {
  LevelDev L{lv->nx, lv->ny, (float)(1.0 / (lv->h * lv->h)), (float)lv->wall_x, (float)lv->wall_y,
                 static_cast<const float2*>(lv->mass)};
  hs::jacobi(u, rhs, out, L, model_of, B, (float)damping, (cudaStream_t)stream);
  return check_cuda("hs_jacobi");
}

HS_API size_t hs_vcycle_workspace_bytes(const hs_hierarchy_t* h, int B) {
  hs::Hierarchy H;
  if (to_hierarchy(h, H) != HS_OK) return 0;
  return hs::vcycle_workspace_bytes(H, B) + align_up(3 * (size_t)B * sizeof(void*));
}

HS_API int hs_vcycle(const hs_hierarchy_t* h, const void* rhs, const void* u0, void* out, const int* model_of,
                     int B, void* ws, size_t ws_bytes, int* status, void* stream) {
  hs::Hierarchy H;
  int rc = to_hierarchy(h, H);
  if (rc != HS_OK) return rc;
  if (ws_bytes < hs_vcycle_workspace_bytes(h, B)) return fail(HS_ECONFIG, "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  const long long N = (long long)H.lv[0].nx * H.lv[0].ny;
  char* p = static_cast<char*>(ws);
  const float2** act = reinterpret_cast<const float2**>(p);
  p += align_up(3 * (size_t)B * sizeof(void*));
  k_table<<<cdiv_u(B, 128), 128, 0, st>>>(static_cast<const float2*>(rhs), N, act, B);
  hs::VecIn in{act, nullptr, 0, nullptr};
  hs::VecIn uz{nullptr, static_cast<const float2*>(u0), u0 ? N : 0, nullptr};
  hs::VecOut o{nullptr, static_cast<float2*>(out), N};
  hs::vcycle(H, in, uz, o, act, model_of, B, p, status, st);
  return check_cuda("hs_vcycle");
}

HS_API size_t hs_fgmres_workspace_bytes(const hs_hierarchy_t* h, const hs_net_t* net, int B, int nx, int ny,
                                        int restart, int max_iter) {
  hs::Hierarchy H;
  if (to_hierarchy(h, H) != HS_OK) return 0;
  int window = restart < max_iter ? restart : max_iter;
  return layout(H, net, B, (long long)nx * ny, window, max_iter).total;
}

HS_API int hs_fgmres_solve(const hs_hierarchy_t* h, const hs_net_t* net, const hs_solve_args_t* a, void* ws,
                           size_t ws_bytes, void* stream) {
  hs::Hierarchy H;
  int rc = to_hierarchy(h, H);
  if (rc != HS_OK) return rc;
  if (!a || a->B < 1) return fail(HS_EDIMENSION, "no right-hand sides");
  if (a->max_iter < 1) return fail(HS_ECONFIG, "max_iter must be >= 1");
  if (a->restart < 1) return fail(HS_ECONFIG, "restart must be >= 1");
  const int window = a->restart < a->max_iter ? a->restart : a->max_iter;
  if (window > hs::kMaxRestart) return fail(HS_ECONFIG, "restart window longer than 32 is not supported");
  cudaStream_t st = (cudaStream_t)stream;
  const int nx = H.lv[0].nx, ny = H.lv[0].ny;
  const long long N = (long long)nx * ny;
  SolveLayout L = layout(H, net, a->B, N, window, a->max_iter);
  if (ws_bytes < L.total) return fail(HS_ECONFIG, "workspace too small");
  char* base = static_cast<char*>(ws);

  hs::SolveDims d{};
  d.B = a->B;
  d.nx = nx;
  d.ny = ny;
  d.n_models = H.n_models;
  d.N = N;
  const double h0 = h->levels[0].h;
  d.h2 = h0 * h0;
  {
    int e = 0;
    d.inv_h2 = std::frexp(d.h2, &e) == 0.5 ? 1.0 / d.h2 : 0.0;  // exact reciprocal of a power of two
  }
  d.restart = window;
  d.max_iter = a->max_iter;
  d.nblk = choose_nblk(N, a->B);
  d.hist_stride = a->max_iter + 2;

  hs::SolveBuffers s{};
  s.V = reinterpret_cast<float2*>(base + L.V);
  s.Z = reinterpret_cast<float2*>(base + L.Z);
  s.x = static_cast<double2*>(a->x);
  s.b = static_cast<const double2*>(a->b);
  s.c_true = static_cast<const double2*>(a->c_true);
  s.model_of = a->model_of;
  s.st = reinterpret_cast<hs::RhsState*>(base + L.st);
  s.hist = a->hist;
  s.partial = reinterpret_cast<double*>(base + L.partial);
  s.counter = reinterpret_cast<int*>(base + L.counter);
  s.vin = reinterpret_cast<const float2**>(base + L.vin);
  s.vin_scale = reinterpret_cast<float*>(base + L.vin_scale);
  s.zout = reinterpret_cast<float2**>(base + L.zout);
  s.n_active = reinterpret_cast<int*>(base + L.n_active);
  int* vstatus = reinterpret_cast<int*>(base + L.vstatus);
  void* vws = base + L.vws;
  float2* u0 = net ? reinterpret_cast<float2*>(base + L.u0) : nullptr;

  cudaMemsetAsync(vstatus, 0, (size_t)a->B * sizeof(int), st);
  s.vstatus = vstatus;
  hs::vcycle_prepare(H, vws, st);
  if (a->x0) cudaMemcpyAsync(a->x, a->x0, (size_t)a->B * N * sizeof(double2), cudaMemcpyDeviceToDevice, st);
  hs::krylov_init(d, s, a->tol, a->iter_cap, a->x0 != nullptr, st);
  if ((rc = check_cuda("fgmres init")) != HS_OK) return rc;

  int* flag = pinned_flag();
  const int kCheckEvery = 4;
  int done_steps = 0;
  for (int step = 0; step <= a->max_iter + 2 * kCheckEvery; step += kCheckEvery) {
    hs::krylov_count_active(d, s, st);
    hs::prof::count(1);
    cudaMemcpyAsync(flag, s.n_active, sizeof(int), cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return check_cuda("fgmres poll");
    if (*flag == 0) break;
    hs::prof::active_now.store(*flag);
    for (int k = 0; k < kCheckEvery; ++k, ++done_steps) {
      hs::prof::count(1);
      hs::krylov_prep(d, s, st);
      hs::VecIn vin{s.vin, nullptr, 0, s.vin_scale};
      hs::VecOut zout{s.zout, nullptr, 0};
      hs::VecIn uz{nullptr, nullptr, 0, nullptr};
      if (net) {
        if ((rc = hs::cnn_preconditioner_estimate(net, vin, s.vin, u0, a->model_of, a->B, base + L.netws, st)) !=
            HS_OK)
          return fail(rc, "network forward");
        uz = hs::VecIn{nullptr, u0, N, nullptr};
      }
      hs::vcycle(H, vin, uz, zout, s.vin, a->model_of, a->B, vws, vstatus, st);
      hs::krylov_after_precond(d, s, done_steps % window, st);
    }
    if ((rc = check_cuda("fgmres step")) != HS_OK) return rc;
  }
  hs::prof::active_now.store(0);
  hs::prof::count(1);
  k_finalize<<<cdiv_u(a->B, 128), 128, 0, st>>>(d, s, a->hist_len, a->iterations, a->converged, a->status, vstatus);
  return check_cuda("fgmres finalize");
}
