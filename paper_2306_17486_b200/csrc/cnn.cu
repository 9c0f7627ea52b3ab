#include "cnn.h"

struct hs_net {
  int levels;
};

namespace hs {
size_t cnn_workspace_bytes(const hs_net_t*, int) { return 0; }
void cnn_preconditioner_estimate(const hs_net_t*, VecIn, const float2* const*, float2*, const int*, int, void*,
                                 cudaStream_t) {}
}  // namespace hs
