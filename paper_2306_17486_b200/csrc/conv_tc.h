// tcgen05 (5th-gen tensor core) implicit-GEMM 3x3 convolution, BF16x3 (exact three-way bf16 split, six products, fp32 accumulate).
#pragma once
#include <cuda_runtime.h>

namespace hs {
extern bool conv_tc_enabled;  // hs_set_conv_path() toggles it (tests compare both paths)
bool conv_tc_supported(int cin, int cout, int stride, int transposed, int H, int W, int Wo, int planar = 0);
bool conv_tc_launch(const float* x, int H, int W, int cin, float* y, int Ho, int Wo, int cout, int stride,
                    int transposed, const float* w, const float* bias, int softplus, const float* addend,
                    long long addend_bstride, int addend_per_model, const int* model_of, const float* residual,
                    const void* const* active, int B, cudaStream_t st, int planar = 0);
// 16 -> 16 and 32 -> 32 stride-1 layers (conv_shift.cu): A operand in TMEM, horizontal taps by tcgen05.shift; any
// width.  conv_tc_launch routes those shapes here (NHWC output only).
bool conv_shift_launch(int channels, const float* x, int H, int W, float* y, const float* w, const float* bias,
                       int softplus, const float* addend, long long addend_bstride, int addend_per_model,
                       const int* model_of, const float* residual, const void* const* active, int B,
                       cudaStream_t st);
// 16 -> 32 stride-2 layer on the same scheme (lanes hold input pixel pairs; one shift per input row); any size
bool conv_shift_s2_launch(const float* x, int H, int W, float* y, int Ho, int Wo, const float* w, const float* bias,
                          int softplus, const float* addend, long long addend_bstride, int addend_per_model,
                          const int* model_of, const float* residual, const void* const* active, int B,
                          cudaStream_t st);
// 32 -> 16 and 64 -> 32 transposed layers on the same scheme (lanes hold input pixels; one shift for the odd output
// columns; 64 -> 32: one 16-channel output half per CTA, the input channels in two halves)
bool conv_shift_t_launch(int cin, const float* x, int H, int W, float* y, const float* w, const float* bias,
                         int softplus, const float* addend, long long addend_bstride, int addend_per_model,
                         const int* model_of, const float* residual, const void* const* active, int B,
                         cudaStream_t st);
// K-streamed tcgen05 kernel for the >= 64-channel layers (conv_wide.cu): 64->64 / 128->128 stride 1,
// 32->64 / 64->128 / 128->128 stride 2, 128->64 and 128->128 (two 64-channel slices) transposed, widths
// (transposed: input widths) that are multiples of 128.  Same arguments and epilogue as conv_tc_launch.
bool conv_wide_supported(int cin, int cout, int stride, int transposed, int H, int W, int Wo);
bool conv_wide_launch(const float* x, int H, int W, int cin, float* y, int Ho, int Wo, int cout, int stride,
                      int transposed, const float* w, const float* bias, int softplus, const float* addend,
                      long long addend_bstride, int addend_per_model, const int* model_of, const float* residual,
                      const void* const* active, int B, cudaStream_t st, int planar);
// The network's wide layers are split into bf16x3 pieces once, at hs_net_create (conv_wide_register,
// keyed by the device weight pointer; conv_wide_unregister at hs_net_destroy).  Unregistered weights are
// split into a stream-ordered temporary on every launch.
bool conv_wide_eligible(int cin, int cout);
int conv_wide_register(const float* w, int cin, int cout, cudaStream_t st);
void conv_wide_unregister(const float* w);
// planar != 0: the output is stored complex-planar, channel pair (2c, 2c+1) of pixel p at
// float2 index (b * cout/2 + c) * Ho * Wo + p (the implicit layer's coalesced input)
}  // namespace hs
