// Internal (C++) interface of the V-cycle and Krylov kernels.  The public
// C ABI lives in include/helmsolve_b200.h.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

#include "level.cuh"

namespace hs {

constexpr int kCoarseMaxIters = 16;  // coarse_iters supported by k_coarse_gmres
constexpr int kMaxLevels = 8;
constexpr int kMaxRestart = 32;      // FGMRES restart supported by the device loop

// A batch of complex64 vectors: either a per-RHS pointer table (entries may be
// null = RHS inactive) or a base pointer with a per-RHS stride.  `scale`
// (optional, per RHS) multiplies every value on load.
struct VecIn {
  const float2* const* tab;
  const float2* base;
  long long bstride;
  const float* scale;
};
struct VecOut {
  float2* const* tab;
  float2* base;
  long long bstride;
};

struct Hierarchy {
  int num_levels;
  int n_models;
  LevelDev lv[kMaxLevels];
  float w_pre, w_post;
  int coarse_iters;
  float coarse_damping;
};

// Workspace (bytes) for a V-cycle over B right-hand sides.
size_t vcycle_workspace_bytes(const Hierarchy& H, int B);

// Derive the per-level diag / dinv planes into the head of `ws` and point H's
// levels at them.  vcycle() does this itself when H is not prepared; a solve
// that runs many V-cycles with one workspace prepares once.
void vcycle_prepare(Hierarchy& H, void* ws, cudaStream_t stream);

// z = V-cycle(rhs, u0) for every RHS whose `active` entry is non-null (or all
// RHS when active == nullptr).  Asynchronous on `stream`.
void vcycle(const Hierarchy& H, VecIn rhs, VecIn u0, VecOut out, const float2* const* active,
            const int* model_of, int B, void* ws, int* status, cudaStream_t stream);

}  // namespace hs
