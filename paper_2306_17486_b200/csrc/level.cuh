// Grid-level operator descriptors and the pointwise stencil algebra of the
// shifted-Laplacian hierarchy (multigrid.py:128-163, fields.py:186-224).
#pragma once
#include "common.cuh"

// One multigrid level as the kernels see it.  `mass` holds, per slowness
// model, c = omega^2 kappa^2 (alpha - i (beta + gamma)) in complex64 for the
// V-cycle's shifted operator (computed on the host in float64, fields.py:186-188).
// The wall re-alignment term (multigrid.py:153-163) is a constant per high
// edge: wall_x on row nx-1, wall_y on column ny-1 (both at the corner).
struct LevelDev {
  int nx, ny;
  float inv_h2;   // 1 / h^2
  float wall_x;   // 0 when the level has no wall on that axis
  float wall_y;
  const float2* mass;  // (n_models, nx, ny)
  // derived once per solve by vcycle_prepare (null until then), (n_models, nx, ny):
  const float2* diag;  // 4/h^2 - c + wall
  const float2* dinv;  // 1 / diag
};

HS_DEV float wall_at(const LevelDev& L, int i, int j) {
  float w = 0.f;
  if (i == L.nx - 1) w += L.wall_x;
  if (j == L.ny - 1) w += L.wall_y;
  return w;
}

// diag = 4/h^2 - c + wall  (stencil_diagonal + wall, multigrid.py:137-142)
HS_DEV float2 level_diag(const LevelDev& L, float2 c, int i, int j) {
  return make_float2(4.f * L.inv_h2 - c.x + wall_at(L, i, j), -c.y);
}

// (A u)(p) given u at p and its four neighbours (zero outside the grid):
// (4u - u[x+1] - u[x-1] - u[y+1] - u[y-1]) / h^2 - c u + wall u
HS_DEV float2 level_apply(const LevelDev& L, float2 c, int i, int j, float2 u, float2 xp, float2 xm,
                          float2 yp, float2 ym) {
  float2 lap = make_float2(4.f * u.x - xp.x - xm.x - yp.x - ym.x, 4.f * u.y - xp.y - xm.y - yp.y - ym.y);
  float wl = wall_at(L, i, j);
  float2 cu = cmul(c, u);
  return make_float2(lap.x * L.inv_h2 - cu.x + wl * u.x, lap.y * L.inv_h2 - cu.y + wl * u.y);
}

// The same operator in diagonal form: (A u)(p) = diag u - (sum of the four
// neighbours) / h^2, and one damped Jacobi sweep
//   u + w (rhs - A u) / diag = (1 - w) u + w dinv (rhs + nb / h^2).
HS_DEV float2 apply_dd(float2 d, float inv_h2, float2 u, float2 nb) {
  return make_float2(fmaf(d.x, u.x, fmaf(-d.y, u.y, -nb.x * inv_h2)), fmaf(d.x, u.y, fmaf(d.y, u.x, -nb.y * inv_h2)));
}
HS_DEV float2 jacobi_dd(float2 di, float inv_h2, float w, float2 u, float2 rhs, float2 nb) {
  const float2 t = make_float2(fmaf(nb.x, inv_h2, rhs.x), fmaf(nb.y, inv_h2, rhs.y));
  const float2 q = cmul(di, t);
  return make_float2(fmaf(1.f - w, u.x, w * q.x), fmaf(1.f - w, u.y, w * q.y));
}

// 1D prolongation weights of P = 4 R^T for fine index i against coarse K
// (multigrid.py:81-114): 1 at i = 2K+1, 1/2 at i = 2K or 2K+2, else 0.
HS_DEV float prolong_w(int a) { return a == 1 ? 1.f : 0.5f; }
