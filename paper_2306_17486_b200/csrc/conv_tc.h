// tcgen05 (5th-gen tensor core) implicit-GEMM convolution, 3xTF32.
#pragma once
#include <cuda_runtime.h>

namespace hs {
bool conv_tc_supported(int cin, int cout, int stride);
void conv_tc_launch(const float* x, int H, int W, int cin, float* y, int Ho, int Wo, int cout, int stride,
                    const float* w, const float* bias, int softplus, const float* addend, long long addend_bstride,
                    const int* model_of, const float* residual, const void* const* active, int B, cudaStream_t st);
}  // namespace hs
