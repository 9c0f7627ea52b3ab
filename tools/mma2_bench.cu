// Microbenchmark + layout probe for tcgen05.mma.cta_group::2 (a CTA pair on one TPC),
// the groundwork for 2-CTA convolution tiles (DESIGN.md "Known gaps" 1).
//
// Each CTA of a 2-CTA cluster holds its half of A (MH = M/2 rows x K = 16, bf16,
// K-major, no swizzle) and its half of B (NH = N/2 columns).  Rank 0 issues one
// MMA D = A B^T; the commit is multicast to both CTAs' mbarriers; every CTA then
// dumps its 128 TMEM lanes x N columns.  The host checks which lanes hold which
// rows of D against an exact integer reference, then times NMMA back-to-back
// MMAs (cycles per MMA) for the pair.
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mma2_bench tools/mma2_bench.cu
#include <cuda_bf16.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}

__host__ __device__ inline float aval(int m, int k) { return (float)((m + 2 * k) % 5 - 2); }
__host__ __device__ inline float bval(int n, int k) { return (float)((3 * n + k) % 7 - 3); }

template <int M, int N, int NMMA>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k_pair(float* dump, long long* cycles) {
  constexpr int MH = M / 2, NH = N / 2;
  __shared__ __align__(1024) unsigned char sa[MH * 32];
  __shared__ __align__(1024) unsigned char sb[NH * 32];
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) uint64_t bar;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // operands: element (row, k) at chunk (k / 8) * LBO + (row / 8) * 128 + (row % 8) * 16 + (k % 8) * 2
  for (int e = threadIdx.x; e < MH * 16; e += blockDim.x) {
    const int r = e / 16, k = e % 16;
    reinterpret_cast<__nv_bfloat16*>(sa)[((k / 8) * MH * 16 + (r / 8) * 128 + (r % 8) * 16 + (k % 8) * 2) / 2] =
        __float2bfloat16(aval((int)rank * MH + r, k));
  }
  for (int e = threadIdx.x; e < NH * 16; e += blockDim.x) {
    const int r = e / 16, k = e % 16;
    reinterpret_cast<__nv_bfloat16*>(sb)[((k / 8) * NH * 16 + (r / 8) * 128 + (r % 8) * 16 + (k % 8) * 2) / 2] =
        __float2bfloat16(bval((int)rank * NH + r, k));
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s_tmem;
  const uint32_t id = idesc_bf16(M, N);
  long long t0 = 0;
  if (rank == 0 && warp == 0) {
    const uint64_t da = desc(smem_u32(sa), MH * 16, 128), db = desc(smem_u32(sb), NH * 16, 128);
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < NMMA; ++i) {
      asm volatile(
          "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
          "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, 0;\n\t}\n" ::"r"(tmem),
          "l"(da), "l"(db), "r"(id));
    }
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}\n"
        ::"r"(smem_u32(&bar)), "h"((uint16_t)3));
  }
  // every thread of both CTAs waits for the multicast commit
  asm volatile(
      "{\n\t.reg .pred P;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n\t@!P bra W;\n\t}\n" ::"r"(
          smem_u32(&bar)));
  if (rank == 0 && warp == 0 && lane == 0) cycles[0] = clock64() - t0;
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // dump lanes 32 warp .. 32 warp + 31, N columns
  for (int c = 0; c < N; c += 8) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(tmem + ((uint32_t)(32 * warp) << 16) + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 8; ++j) dump[((size_t)rank * 128 + threadIdx.x) * N + c + j] = __uint_as_float(r[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int M, int N, int NMMA>
void run(const char* label) {
  float* dump;
  long long* cyc;
  cudaMalloc(&dump, 2 * 128 * N * sizeof(float));
  cudaMalloc(&cyc, sizeof(long long));
  cudaMemset(dump, 0, 2 * 128 * N * sizeof(float));
  k_pair<M, N, NMMA><<<2, 128>>>(dump, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("%s: %s\n", label, cudaGetErrorString(e));
    exit(1);
  }
  std::vector<float> h(2 * 128 * N);
  long long c = 0;
  cudaMemcpy(h.data(), dump, h.size() * sizeof(float), cudaMemcpyDeviceToHost);
  cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  // exact reference D[m][n] = sum_k A[m][k] B[n][k]; find, for each (CTA, lane), the row of D it holds
  auto Dref = [&](int m, int n) {
    float s = 0.f;
    for (int k = 0; k < 16; ++k) s += aval(m, k) * bval(n, k);
    return s;
  };
  int mapped = 0, first_row[2][128];
  for (int r = 0; r < 2; ++r)
    for (int l = 0; l < 128; ++l) {
      first_row[r][l] = -1;
      for (int m = 0; m < M && first_row[r][l] < 0; ++m) {
        bool ok = true;
        for (int n = 0; n < N && ok; ++n) ok = h[((size_t)r * 128 + l) * N + n] == Dref(m, n);
        if (ok) first_row[r][l] = m;
      }
      if (first_row[r][l] >= 0) ++mapped;
    }
  printf("%s: %d of 256 (CTA, lane) hold a full row of D (all N = %d columns); %.1f cycles per MMA (%d MMAs)\n",
         label, mapped, N, (double)c / NMMA, NMMA);
  for (int r = 0; r < 2; ++r) {
    printf("  CTA %d lanes 0,1,15,16,31,32,63,64,127 -> rows", r);
    const int ls[] = {0, 1, 15, 16, 31, 32, 63, 64, 127};
    for (int l : ls) printf(" %d", first_row[r][l]);
    printf("\n");
  }
  cudaFree(dump);
  cudaFree(cyc);
}

int main() {
  run<256, 64, 1>("M=256 N=64 (pair)");
  run<128, 64, 1>("M=128 N=64 (pair)");
  run<256, 192, 1>("M=256 N=192 (pair)");
  run<256, 96, 256>("timing M=256 N=96");
  run<256, 192, 256>("timing M=256 N=192");
  run<128, 192, 256>("timing M=128 N=192");
  return 0;
}
