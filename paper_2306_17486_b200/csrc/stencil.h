#pragma once
#include <cuda_runtime.h>

#include "level.cuh"

namespace hs {
void helm_apply(const void* u, void* out, const void* mass, const int* model_of, int B, int nx, int ny, double h,
                double wall_x, double wall_y, int mode, cudaStream_t stream);
void restrict_fw(const void* fine, void* coarse, int B, int nx, int ny, int f64, cudaStream_t stream);
void prolong_bl(const void* coarse, void* fine, int B, int ncx, int ncy, int nx, int ny, int f64,
                cudaStream_t stream);
void jacobi(const void* u, const void* rhs, void* out, const LevelDev& L, const int* model_of, int B, float w,
            cudaStream_t stream);
}  // namespace hs
