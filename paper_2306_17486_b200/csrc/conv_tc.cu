#include "conv_tc.h"

namespace hs {
bool conv_tc_supported(int, int, int) { return false; }
void conv_tc_launch(const float*, int, int, int, float*, int, int, int, int, const float*, const float*, int,
                    const float*, long long, const int*, const float*, const void* const*, int, cudaStream_t) {}
}  // namespace hs
