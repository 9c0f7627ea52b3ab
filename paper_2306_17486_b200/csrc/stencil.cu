// Stand-alone operator, transfer and smoother kernels: the C-ABI versions of
// fields.apply_helmholtz_array, multigrid.restrict_full_weighting,
// prolong_bilinear and jacobi_relax.  The solve itself uses the fused
// kernels in vcycle.cu / krylov.cu; these serve the drop-in Python API and
// the parity tests.
#include "common.cuh"
#include "level.cuh"
#include "stencil.h"

namespace hs {

namespace {

template <typename T>
HS_DEV double2 ld2(const T* p, long long q);
template <>
HS_DEV double2 ld2<float2>(const float2* p, long long q) {
  float2 v = p[q];
  return make_double2(v.x, v.y);
}
template <>
HS_DEV double2 ld2<double2>(const double2* p, long long q) {
  return p[q];
}

// fp64 operator with complex128 mass, summation order of fields.py:191-199
template <typename TIN>
__global__ void k_apply_f64(const TIN* __restrict__ u, double2* __restrict__ out, const double2* __restrict__ mass,
                            const int* model_of, int nx, int ny, double h2, double wall_x, double wall_y) {
  const int b = blockIdx.y;
  const long long N = (long long)nx * ny;
  const TIN* ub = u + b * N;
  const double2* c = mass + (model_of ? model_of[b] : 0) * N;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < N; p += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(p / ny), j = (int)(p - (long long)i * ny);
    double2 z0 = make_double2(0.0, 0.0);
    double2 uu = ld2(ub, p);
    double2 xp = i + 1 < nx ? ld2(ub, p + ny) : z0;
    double2 xm = i > 0 ? ld2(ub, p - ny) : z0;
    double2 yp = j + 1 < ny ? ld2(ub, p + 1) : z0;
    double2 ym = j > 0 ? ld2(ub, p - 1) : z0;
    double lr = __dsub_rn(__dsub_rn(__dsub_rn(__dsub_rn(4.0 * uu.x, xp.x), xm.x), yp.x), ym.x);
    double li = __dsub_rn(__dsub_rn(__dsub_rn(__dsub_rn(4.0 * uu.y, xp.y), xm.y), yp.y), ym.y);
    double2 cu = zmul(c[p], uu);
    double2 r = make_double2(__dsub_rn(__ddiv_rn(lr, h2), cu.x), __dsub_rn(__ddiv_rn(li, h2), cu.y));
    double wl = (i == nx - 1 ? wall_x : 0.0) + (j == ny - 1 ? wall_y : 0.0);
    if (wl != 0.0) r = zadd(r, zscale(uu, wl));
    out[b * N + p] = r;
  }
}

__global__ void k_apply_f32(const float2* __restrict__ u, float2* __restrict__ out, LevelDev L,
                            const int* model_of) {
  const int b = blockIdx.y;
  const int nx = L.nx, ny = L.ny;
  const long long N = (long long)nx * ny;
  const float2* ub = u + b * N;
  const float2* c = L.mass + (model_of ? model_of[b] : 0) * N;
  const float2 z0 = make_float2(0.f, 0.f);
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < N; p += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(p / ny), j = (int)(p - (long long)i * ny);
    out[b * N + p] = level_apply(L, c[p], i, j, ub[p], i + 1 < nx ? ub[p + ny] : z0, i > 0 ? ub[p - ny] : z0,
                                 j + 1 < ny ? ub[p + 1] : z0, j > 0 ? ub[p - 1] : z0);
  }
}

__global__ void k_jacobi(const float2* __restrict__ u, const float2* __restrict__ rhs, float2* __restrict__ out,
                         LevelDev L, const int* model_of, float w) {
  const int b = blockIdx.y;
  const int nx = L.nx, ny = L.ny;
  const long long N = (long long)nx * ny;
  const float2* ub = u + b * N;
  const float2* c = L.mass + (model_of ? model_of[b] : 0) * N;
  const float2 z0 = make_float2(0.f, 0.f);
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < N; p += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(p / ny), j = (int)(p - (long long)i * ny);
    float2 au = level_apply(L, c[p], i, j, ub[p], i + 1 < nx ? ub[p + ny] : z0, i > 0 ? ub[p - ny] : z0,
                            j + 1 < ny ? ub[p + 1] : z0, j > 0 ? ub[p - 1] : z0);
    out[b * N + p] = cadd(ub[p], cscale(cdiv(csub(rhs[b * N + p], au), level_diag(L, c[p], i, j)), w));
  }
}

template <typename T, typename R>
__global__ void k_restrict(const T* __restrict__ f, T* __restrict__ cout, int nx, int ny, int ncx, int ncy) {
  const int b = blockIdx.y;
  const long long N = (long long)nx * ny, Nc = (long long)ncx * ncy;
  const R fw[3] = {R(0.25), R(0.5), R(0.25)};
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < Nc; q += (long long)gridDim.x * blockDim.x) {
    const int K = (int)(q / ncy), L = (int)(q - (long long)K * ncy);
    T acc{};
    for (int u = 0; u < 3; ++u)
      for (int v = 0; v < 3; ++v) {
        int i = 2 * K + u, j = 2 * L + v;
        if (i < nx && j < ny) {
          const T x = f[b * N + (long long)i * ny + j];
          const R w = fw[u] * fw[v];
          acc.x += w * x.x;
          acc.y += w * x.y;
        }
      }
    cout[b * Nc + q] = acc;
  }
}

template <typename T, typename R>
__global__ void k_prolong(const T* __restrict__ c, T* __restrict__ f, int ncx, int ncy, int nx, int ny) {
  const int b = blockIdx.y;
  const long long N = (long long)nx * ny, Nc = (long long)ncx * ncy;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < N; p += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(p / ny), j = (int)(p - (long long)i * ny);
    int kxa = (i & 1) ? (i - 1) / 2 : i / 2 - 1, kxb = (i & 1) ? kxa : i / 2;
    int kya = (j & 1) ? (j - 1) / 2 : j / 2 - 1, kyb = (j & 1) ? kya : j / 2;
    T acc{};
    for (int K = kxa; K <= kxb; ++K) {
      if (K < 0 || K >= ncx) continue;
      for (int Q = kya; Q <= kyb; ++Q) {
        if (Q < 0 || Q >= ncy) continue;
        const T x = c[b * Nc + (long long)K * ncy + Q];
        const R w = R(prolong_w(i - 2 * K)) * R(prolong_w(j - 2 * Q));
        acc.x += w * x.x;
        acc.y += w * x.y;
      }
    }
    f[b * N + p] = acc;
  }
}

dim3 grid_for(long long n, int B) {
  long long blocks = (n + 255) / 256;
  if (blocks > 1184) blocks = 1184;
  return dim3((unsigned)blocks, (unsigned)B);
}

}  // namespace

void helm_apply(const void* u, void* out, const void* mass, const int* model_of, int B, int nx, int ny, double h,
                double wall_x, double wall_y, int mode, cudaStream_t stream) {
  dim3 g = grid_for((long long)nx * ny, B);
  const double h2 = h * h;
  if (mode == 2) {
    k_apply_f64<double2><<<g, 256, 0, stream>>>((const double2*)u, (double2*)out, (const double2*)mass, model_of, nx,
                                                ny, h2, wall_x, wall_y);
  } else if (mode == 1) {
    k_apply_f64<float2><<<g, 256, 0, stream>>>((const float2*)u, (double2*)out, (const double2*)mass, model_of, nx,
                                               ny, h2, wall_x, wall_y);
  } else {
    LevelDev L{nx, ny, (float)(1.0 / h2), (float)wall_x, (float)wall_y, (const float2*)mass};
    k_apply_f32<<<g, 256, 0, stream>>>((const float2*)u, (float2*)out, L, model_of);
  }
}

void restrict_fw(const void* fine, void* coarse, int B, int nx, int ny, int f64, cudaStream_t stream) {
  dim3 g = grid_for((long long)(nx / 2) * (ny / 2), B);
  if (f64)
    k_restrict<double2, double><<<g, 256, 0, stream>>>((const double2*)fine, (double2*)coarse, nx, ny, nx / 2, ny / 2);
  else
    k_restrict<float2, float><<<g, 256, 0, stream>>>((const float2*)fine, (float2*)coarse, nx, ny, nx / 2, ny / 2);
}

void prolong_bl(const void* coarse, void* fine, int B, int ncx, int ncy, int nx, int ny, int f64,
                cudaStream_t stream) {
  dim3 g = grid_for((long long)nx * ny, B);
  if (f64)
    k_prolong<double2, double><<<g, 256, 0, stream>>>((const double2*)coarse, (double2*)fine, ncx, ncy, nx, ny);
  else
    k_prolong<float2, float><<<g, 256, 0, stream>>>((const float2*)coarse, (float2*)fine, ncx, ncy, nx, ny);
}

void jacobi(const void* u, const void* rhs, void* out, const LevelDev& L, const int* model_of, int B, float w,
            cudaStream_t stream) {
  k_jacobi<<<grid_for((long long)L.nx * L.ny, B), 256, 0, stream>>>((const float2*)u, (const float2*)rhs,
                                                                     (float2*)out, L, model_of, w);
}

}  // namespace hs
