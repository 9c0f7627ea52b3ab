// Encoder-solver CNN on the device (ARCH.md).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

#include "../../include/helmsolve_b200.h"
#include "vcycle.h"

namespace hs {

// One 3x3 convolution (pad 1) with batch norm folded into weights/bias:
//   y = act(conv(x, w) + b) [+ addend] [+ residual]
// Weights are stored [cout][3][3][cin] (K-major: tap-major, then cin); a
// transposed layer (stride 2, weight (cin, cout, 3, 3) in the reference) is
// stored in the same [cout][ky][kx][cin] order.
struct ConvDesc {
  int cin, cout, stride, transposed, softplus;
  const float* w;
  const float* b;
};

size_t cnn_workspace_bytes(const hs_net_t* net, int B);
// u0[b] = (h^2/64) net(scale_b * vin[b]) zero-padded, for RHS with active[b] != null
int cnn_preconditioner_estimate(const hs_net_t* net, VecIn vin, const float2* const* active, float2* u0,
                                 const int* model_of, int B, void* ws, cudaStream_t stream);
}  // namespace hs
