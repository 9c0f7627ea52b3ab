// Probe of tcgen05.shift (sm_100a): what one shift does to a TMEM block, and whether
// MMA -> shift -> MMA issued by one thread execute in issue order (A operand in TMEM).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/shift_probe tools/shift_probe.cu
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2306_17486_b200/csrc/tc_util.cuh"

using namespace hs::tc;

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]));
}
__device__ __forceinline__ void shift_down(uint32_t taddr) {
  asm volatile("tcgen05.shift.cta_group::1.down [%0];" ::"r"(taddr) : "memory");
}

// out[0]: 128 x 32 words after one shift at column 0 (columns 0..31 written as lane << 8 | col)
// out[1]: same after a second shift issued at column 8 with lane base 32
// out[2]: D of MMA / shift / MMA / shift / MMA (3 x 128 x 16 floats), repeated `reps` times; mismatch count in flag
__global__ void __launch_bounds__(128) k_probe(uint32_t* out, int reps, int nmma, int* flag) {
  __shared__ __align__(128) unsigned char bsm[3 * 48 * 32];
  __shared__ uint64_t bar;
  __shared__ uint32_t s_tmem;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(smem_u32(&bar), 1);
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  const uint32_t lane_base = tmem + ((uint32_t)(32 * warp) << 16);
  uint32_t phase = 0;
  // ---- part 1: what moves
  for (int c0 = 0; c0 < 32; c0 += 8) {
    uint32_t r[8];
    for (int j = 0; j < 8; ++j) r[j] = ((uint32_t)tid << 8) | (uint32_t)(c0 + j);
    tmem_st8(lane_base + c0, r);
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  if (tid == 0) {
    tc_fence_after();
    shift_down(tmem + 0);
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
  }
  mbar_wait(smem_u32(&bar), phase);
  phase ^= 1;
  tc_fence_after();
  for (int c0 = 0; c0 < 32; c0 += 8) {
    uint32_t r[8];
    tmem_ld8(lane_base + c0, r);
    tmem_wait_ld();
    for (int j = 0; j < 8; ++j) out[tid * 32 + c0 + j] = r[j];
  }
  tc_fence_before();
  __syncthreads();
  if (tid == 0) {
    tc_fence_after();
    shift_down(tmem + (32u << 16) + 8);  // lane base 32, column 8
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
  }
  mbar_wait(smem_u32(&bar), phase);
  phase ^= 1;
  tc_fence_after();
  for (int c0 = 0; c0 < 32; c0 += 8) {
    uint32_t r[8];
    tmem_ld8(lane_base + c0, r);
    tmem_wait_ld();
    for (int j = 0; j < 8; ++j) out[4096 + tid * 32 + c0 + j] = r[j];
  }
  tc_fence_before();
  __syncthreads();
  // ---- part 2: MMA / shift / MMA ordering.  A[m][k] = (k == 0) ? m + 1 : 0 (bf16, exact); B[n][k] = (k == 0) ? 1 : 0,
  // so D[m][n] = m + 1, then m + 2, then m + 3 after the shifts (a shift moves lane m + 1 to lane m inside each 32-lane quarter).  N = 48 MMAs, `nmma` of them per view (accumulating).
  for (int e = tid; e < 3 * 48 * 2; e += 128) {  // B: (chunk c, row n) x 16 B, three copies
    const int c = (e / 48) % 2;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (c == 0) v.x = 0x3F80u;  // bf16 1.0 at k = 0
    *reinterpret_cast<uint4*>(bsm + (size_t)e * 16) = v;
  }
  fence_async_smem();
  __syncthreads();
  const uint32_t idesc = idesc_bf16(128, 48);
  int bad = 0;
  for (int rep = 0; rep < reps; ++rep) {
    uint32_t r[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    __nv_bfloat16 hv = __float2bfloat16((float)(tid + 1));
    r[0] = (uint32_t)(*reinterpret_cast<unsigned short*>(&hv));
    tmem_st8(lane_base + 0, r);  // A at columns 0..7
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
      tc_fence_after();
      const uint32_t blo = desc_lo(smem_u32(bsm), 48 * 16);
      for (int v = 0; v < 3; ++v) {
        for (int i = 0; i < nmma; ++i) {
          asm volatile(
              "{\n\t.reg .pred p, e;\n\t.reg .b64 db;\n\t"
              "mov.b64 db, {%2, %3};\n\tsetp.ne.b32 p, %5, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], db, %4, p;\n\t}\n" ::"r"(tmem + 64 + 48 * v),
              "r"(tmem + 0), "r"(blo), "r"(kDescHi), "r"(idesc), "r"(i ? 1u : 0u));
        }
        if (v < 2) {
          asm volatile(
              "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
              "@e tcgen05.shift.cta_group::1.down [%0];\n\t}\n" ::"r"(tmem + 0)
              : "memory");
        }
      }
      mma_commit(smem_u32(&bar));
    }
    mbar_wait(smem_u32(&bar), phase);
    phase ^= 1;
    tc_fence_after();
    for (int v = 0; v < 3; ++v)
      for (int c0 = 0; c0 < 16; c0 += 8) {
        uint32_t q[8];
        tmem_ld8(lane_base + 64 + 48 * v + c0, q);
        tmem_wait_ld();
        for (int j = 0; j < 8; ++j) {
          const float got = __uint_as_float(q[j]);
          const float want = (float)nmma * (float)(tid + 1 + v);
          if (rep == 0) out[8192 + (v * 128 + tid) * 16 + c0 + j] = q[j];
          if ((tid & 31) <= 31 - v && got != want) ++bad;
        }
      }
    tc_fence_before();
    __syncthreads();
  }
  if (bad) atomicAdd(flag, bad);
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

int main(int argc, char** argv) {
  const int reps = argc > 1 ? atoi(argv[1]) : 200, nmma = argc > 2 ? atoi(argv[2]) : 9;
  uint32_t* out;
  int* flag;
  const size_t n = 8192 + 3 * 128 * 16;
  cudaMalloc(&out, n * 4);
  cudaMalloc(&flag, 4);
  cudaMemset(out, 0xff, n * 4);
  cudaMemset(flag, 0, 4);
  k_probe<<<1, 128>>>(out, reps, nmma, flag);
  cudaError_t e = cudaDeviceSynchronize();
  printf("sync: %s\n", cudaGetErrorString(e));
  if (e != cudaSuccess) return 1;
  std::vector<uint32_t> h(n);
  int hf = 0;
  cudaMemcpy(h.data(), out, n * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(&hf, flag, 4, cudaMemcpyDeviceToHost);
  for (int part = 0; part < 2; ++part) {
    printf("after shift %d: source lane of (lane, column block)\n", part + 1);
    for (int m = 0; m < 128; ++m) {
      if (!(m < 4 || (m % 32) < 2 || (m % 32) > 29)) continue;
      printf("  lane %3d:", m);
      for (int c = 0; c < 32; c += 4) printf(" c%02d<-(%3u,c%02u)", c, h[part * 4096 + m * 32 + c] >> 8, h[part * 4096 + m * 32 + c] & 0xff);
      printf("\n");
    }
  }
  printf("MMA/shift/MMA (nmma %d, reps %d): mismatches %d\n", nmma, reps, hf);
  for (int v = 0; v < 3; ++v) {
    printf("  view %d D[m][0], m = 0..5, 31..34, 126, 127:", v);
    const int ms[] = {0, 1, 2, 3, 4, 5, 31, 32, 33, 34, 126, 127};
    for (int m : ms) printf(" %g", *reinterpret_cast<float*>(&h[8192 + (v * 128 + m) * 16]));
    printf("\n");
  }
  return 0;
}
