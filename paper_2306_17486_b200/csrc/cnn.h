// Encoder-solver CNN on the device (ARCH.md).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

#include "../../include/helmsolve_b200.h"
#include "vcycle.h"

namespace hs {
size_t cnn_workspace_bytes(const hs_net_t* net, int B);
// u0[b] = (h^2/64) net(scale_b * vin[b]) zero-padded, for RHS with active[b] != null
void cnn_preconditioner_estimate(const hs_net_t* net, VecIn vin, const float2* const* active, float2* u0,
                                 const int* model_of, int B, void* ws, cudaStream_t stream);
}  // namespace hs
