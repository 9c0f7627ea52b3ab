// Microbenchmark: cycles per tcgen05.mma.kind::f16 (cta_group::1) as a function
// of M, N and where A lives (shared memory descriptor or TMEM), issued back to
// back by one elected thread into one accumulator.  Operand contents are
// irrelevant (zeros); only the issue/execution rate is measured.
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mma_bench tools/mma_bench.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}

template <int M, int N, bool ATMEM, int NMMA, int ND, int NWI = 1>
__global__ void k_bench(long long* out) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) uint64_t bar[4];
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s_tmem;
  if ((threadIdx.x & 31) == 0 && warp < NWI) {
    const uint64_t da = desc(smem_u32(smem), 128 * 16, 128);
    const uint64_t db = desc(smem_u32(smem + 32768), N * 16, 128);
    const uint32_t id = idesc_bf16(M, N);
    const uint32_t ta = tmem + 256;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < NMMA; i += 16) {
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const uint32_t d = tmem + (uint32_t)(warp * 64) + (uint32_t)((k % ND) * (64 / ND));  // per-warp accumulators
        if (ATMEM)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
                       "r"(ta), "l"(db), "r"(id), "r"(i + k));
        else
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
                       "l"(da), "l"(db), "r"(id), "r"(i + k));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar[warp]))
                 : "memory");
    asm volatile(
        "{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@P1 bra D;\n\tbra W;\n\tD:\n\t}\n" ::"r"(
            smem_u32(&bar[warp])));
    long long t1 = clock64();
    if (warp == 0) out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int M, int N, bool ATMEM, int ND = 1, int NWI = 1>
void run(long long* d) {
  constexpr int NMMA = 4096;
  auto k = k_bench<M, N, ATMEM, NMMA, ND, NWI>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  k<<<1, 128, 64 * 1024>>>(d);
  k<<<1, 128, 64 * 1024>>>(d);
  long long h = 0;
  cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
  cudaError_t e = cudaDeviceSynchronize();
  printf("M=%3d N=%3d A=%s acc=%d warps=%d: %6.1f cycles per MMA per warp (%s)\n", M, N, ATMEM ? "tmem" : "smem", ND, NWI, (double)h / NMMA,
         cudaGetErrorString(e));
}

int main() {
  long long* d;
  cudaMalloc(&d, 1024 * sizeof(long long));
  run<128, 48, false, 1, 1>(d);
  run<128, 48, false, 1, 2>(d);
  run<128, 48, false, 1, 4>(d);
  run<128, 16, false, 1, 2>(d);
  run<128, 16, false, 1, 4>(d);
  run<128, 96, false, 1, 2>(d);
  run<128, 48, true, 1, 2>(d);
  run<128, 48, true, 1, 4>(d);
  run<128, 256, false, 1, 2>(d);
  return 0;
}
