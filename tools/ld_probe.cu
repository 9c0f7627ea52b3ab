// Probe of tcgen05.ld.16x256b (sm_100a): which (lane, column) each thread's registers hold.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/ld_probe tools/ld_probe.cu
#include <cstdio>
#include <vector>

#include "../paper_2306_17486_b200/csrc/tc_util.cuh"
using namespace hs::tc;

__global__ void __launch_bounds__(128) k_probe(uint32_t* out) {
  __shared__ uint32_t s_tmem;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)), "r"(64));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  const uint32_t lane_base = tmem + ((uint32_t)(32 * warp) << 16);
  for (int c0 = 0; c0 < 32; c0 += 8) {  // value = TMEM lane << 8 | column
    uint32_t r[8];
    for (int j = 0; j < 8; ++j) r[j] = ((uint32_t)tid << 8) | (uint32_t)(c0 + j);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(lane_base + c0), "r"(r[0]),
                 "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]));
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  for (int hh = 0; hh < 2; ++hh) {  // lanes 16 hh .. 16 hh + 15 of the warp's quarter, columns 0..15 (x2)
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(lane_base + ((uint32_t)(16 * hh) << 16)));
    tmem_wait_ld();
    for (int j = 0; j < 8; ++j) out[(tid * 2 + hh) * 8 + j] = r[j];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(64));
}

int main() {
  uint32_t* out;
  cudaMalloc(&out, 128 * 16 * 4);
  k_probe<<<1, 128>>>(out);
  cudaError_t e = cudaDeviceSynchronize();
  printf("sync: %s\n", cudaGetErrorString(e));
  std::vector<uint32_t> h(128 * 16);
  cudaMemcpy(h.data(), out, h.size() * 4, cudaMemcpyDeviceToHost);
  for (int t : {0, 1, 2, 3, 4, 5, 31, 32, 33, 37, 127}) {
    for (int hh = 0; hh < 2; ++hh) {
      printf("thread %3d half %d:", t, hh);
      for (int j = 0; j < 8; ++j) printf(" r%d=(%3u,c%02u)", j, h[(t * 2 + hh) * 8 + j] >> 8, h[(t * 2 + hh) * 8 + j] & 0xff);
      printf("\n");
    }
  }
  // check the expected rule: reg j of thread T (lane l = T % 32, warp w): row 32 w + 16 hh + l / 4 + 8 ((j / 2) % 2), column 8 (j / 4) + 2 (l % 4) + j % 2
  int bad = 0;
  for (int t = 0; t < 128; ++t)
    for (int hh = 0; hh < 2; ++hh)
      for (int j = 0; j < 8; ++j) {
        const int l = t % 32, w = t / 32;
        const uint32_t want = ((uint32_t)(32 * w + 16 * hh + l / 4 + 8 * ((j / 2) % 2)) << 8) | (uint32_t)(8 * (j / 4) + 2 * (l % 4) + j % 2);
        bad += h[(t * 2 + hh) * 8 + j] != want;
      }
  printf("rule mismatches: %d\n", bad);
  return 0;
}
