// Launch counting and CUDA-event timing of tagged kernels (the tracing
// subsystem; the reference only has SolveReport.wall_time, krylov.py:19-26).
// Tags are timed only when enabled through hs_profile_enable, so the solve
// pays nothing by default.  Work units (bytes or flops) are attached per
// launch so callers can compute achieved bandwidth / throughput.
#pragma once
#include <cuda_runtime.h>

#include <atomic>

namespace hs {
namespace prof {

enum Tag {
  CONV = 0,       // every network convolution (work = flops)
  CONV_L0 = 1,    // 16-channel level-0 stride-1 convolutions (work = flops)
  VCYCLE = 2,     // one whole V-cycle (work = algorithmic bytes)
  ARNOLDI = 3,    // Gram-Schmidt dot pass (work = algorithmic bytes)
  CNN = 4,        // one whole network forward
  IMPLICIT = 5,   // implicit layer (work = algorithmic bytes: complex input + output)
  VC_UP0 = 6,     // finest-level up-leg kernel (work = algorithmic bytes)
  TRAIN_WGRAD = 7,  // training weight-gradient reductions (work = flops)
  CONV_WIDE = 8,  // 3x3 convolutions with >= 64 input or output channels, tensor-bound (work = flops)
  KRYLOV = 9,     // the other Krylov kernels of a step (orthogonalisation passes, Givens, x update, residual)
  NTAGS = 10
};

extern std::atomic<long long> launches;
inline void count(int n) { launches.fetch_add(n, std::memory_order_relaxed); }

// RHS still iterating, as last polled by the solve driver (B outside a solve);
// only used to attribute work units to timed launches.
extern std::atomic<int> active_now;
inline double active_hint(int B) {
  int a = active_now.load(std::memory_order_relaxed);
  return (double)(a > 0 && a < B ? a : B);
}

bool on(int tag);
// label attached to the records this thread starts next (per-layer breakdowns)
void set_label(int label);
// returns an opaque slot (or -1) to close with stop()
int start(int tag, cudaStream_t st);
void stop(int slot, cudaStream_t st, double work);

}  // namespace prof
}  // namespace hs
