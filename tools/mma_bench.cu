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

template <int M, int N, bool ATMEM, int NMMA, int ND, int NWI = 1, bool CONSTP = false, int AOFS = 0>
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
  if (warp < NWI) {  // converged issuing warps; one elected lane issues, 8 MMAs per asm block
    const uint32_t da = (uint32_t)(desc(smem_u32(smem) + AOFS, 128 * 16 + AOFS, 128) & 0xffffffffu);
    const uint32_t db = (uint32_t)(desc(smem_u32(smem + 32768), N * 16, 128) & 0xffffffffu);
    const uint32_t hi = (uint32_t)(desc(0, 0, 128) >> 32);
    const uint32_t id = idesc_bf16(M, N);
    const uint32_t ta = tmem + 256;
    const uint32_t d = tmem + (uint32_t)(warp * 64);
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < NMMA; i += 8) {
      if (ATMEM)
        asm volatile(
            "{\n\t.reg .pred e;\n\t.reg .b64 db;\n\t"
            "elect.sync _|e, 0xffffffff;\n\tmov.b64 db, {%2, %3};\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], db, %4, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], db, %4, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], db, %4, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], db, %4, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], db, %4, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], db, %4, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], db, %4, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], db, %4, 1;\n\t}\n" ::"r"(d),
            "r"(ta), "r"(db), "r"(hi), "r"(id));
      else
        asm volatile(
            "{\n\t.reg .pred e;\n\t.reg .b64 da, db;\n\t"
            "elect.sync _|e, 0xffffffff;\n\tmov.b64 db, {%2, %3};\n\tmov.b64 da, {%1, %3};\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %4, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %4, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %4, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %4, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %4, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %4, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %4, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %4, 1;\n\t}\n" ::"r"(d),
            "r"(da), "r"(db), "r"(hi), "r"(id));
    }
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(
            smem_u32(&bar[warp]))
        : "memory");
    asm volatile(
        "{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@P1 bra D;\n\tbra W;\n\tD:\n\t}\n" ::"r"(
            smem_u32(&bar[warp])));
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int M, int N, bool ATMEM, int ND = 1, int NWI = 1, bool CONSTP = false, int AOFS = 0>
void run(long long* d) {
  constexpr int NMMA = 4096;
  auto k = k_bench<M, N, ATMEM, NMMA, ND, NWI, CONSTP, AOFS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  k<<<1, 128, 64 * 1024>>>(d);
  k<<<1, 128, 64 * 1024>>>(d);
  long long h = 0;
  cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
  cudaError_t e = cudaDeviceSynchronize();
  printf("M=%3d N=%3d A=%s acc=%d warps=%d aofs=%d: %6.1f cycles per MMA per warp (%s)\n", M, N, ATMEM ? "tmem" : "smem", ND, NWI, AOFS, (double)h / NMMA,
         cudaGetErrorString(e));
}


// tcgen05.cp 128x256b (4 KB smem -> TMEM) rate, and tcgen05.st 32x32b.x8 (1 KB per warp) rate
template <int NCP>
__global__ void k_cp(long long* out) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s_tmem;
  if (warp == 0) {
    const uint32_t sl = (uint32_t)(desc(smem_u32(smem), 128 * 16, 128) & 0xffffffffu);
    const uint32_t hi = (uint32_t)(desc(0, 0, 128) >> 32);
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < NCP; i += 8)
      asm volatile(
          "{\n\t.reg .pred e;\n\t.reg .b64 ds;\n\telect.sync _|e, 0xffffffff;\n\tmov.b64 ds, {%1, %2};\n\t"
          "@e tcgen05.cp.cta_group::1.128x256b [%0], ds;\n\t@e tcgen05.cp.cta_group::1.128x256b [%0], ds;\n\t"
          "@e tcgen05.cp.cta_group::1.128x256b [%0], ds;\n\t@e tcgen05.cp.cta_group::1.128x256b [%0], ds;\n\t"
          "@e tcgen05.cp.cta_group::1.128x256b [%0], ds;\n\t@e tcgen05.cp.cta_group::1.128x256b [%0], ds;\n\t"
          "@e tcgen05.cp.cta_group::1.128x256b [%0], ds;\n\t@e tcgen05.cp.cta_group::1.128x256b [%0], ds;\n\t}\n" ::"r"(
              tmem + 256),
          "r"(sl), "r"(hi));
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(smem_u32(&bar))
        : "memory");
    asm volatile(
        "{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@P1 bra D;\n\tbra W;\n\tD:\n\t}\n" ::"r"(
            smem_u32(&bar)));
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = t1 - t0;
  }
  // tcgen05.st: 4 warps (all lane quarters) each store x8 (32 lanes x 8 columns = 1 KB) NCP times
  __syncthreads();
  if (warp < 4) {
    uint32_t r[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) r[i] = i;
    const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + 256;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < NCP / 4; ++i)
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
          "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(ta + (i & 3) * 32),
          "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
          "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]),
          "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]),
          "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    long long t1 = clock64();
    if (threadIdx.x == 0) out[1] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

void run_cp(long long* d) {
  constexpr int NCP = 4096;
  cudaFuncSetAttribute(k_cp<NCP>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  k_cp<NCP><<<1, 128, 64 * 1024>>>(d);
  k_cp<NCP><<<1, 128, 64 * 1024>>>(d);
  long long h[2] = {0, 0};
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("tcgen05.cp 128x256b: %.1f cycles each (%.0f B/clk); tcgen05.st x32 per warp, 4 warps: %.1f cycles each "
         "(%.0f B/clk aggregate)\n",
         (double)h[0] / NCP, 4096.0 * NCP / h[0], (double)h[1] / (NCP / 4), 4.0 * 4096 * (NCP / 4) / h[1]);
}


constexpr uint32_t kDescHi = ((128u >> 4) & 0x3FFFu) | (1u << 14);
template <uint32_t I0, uint32_t I1, uint32_t I2, uint32_t PX0, uint32_t PX1, uint32_t PX2, uint32_t WT, uint32_t PS>
__device__ __forceinline__ void mma_row9(uint32_t d, uint32_t xbase, uint32_t wbase, uint32_t accumulate) {
#define HS_MMA_PARTS(PX, P0)                                             \
  "add.u32 al, %1, " PX ";\n\tmov.b64 da, {al, hi};\n\t"              \
  "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, i0, " P0 ";\n\t" \
  "add.u32 al, al, %12;\n\tmov.b64 da, {al, hi};\n\t"                 \
  "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, i1, t;\n\t"      \
  "add.u32 al, al, %12;\n\tmov.b64 da, {al, hi};\n\t"                 \
  "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, i2, t;\n\t"
  asm volatile(
      "{\n\t.reg .pred p, t, e;\n\t.reg .b64 da, db;\n\t.reg .b32 hi, i0, i1, i2, al, bl;\n\t"
      "mov.b32 hi, %4;\n\tmov.b32 i0, %5;\n\tmov.b32 i1, %6;\n\tmov.b32 i2, %7;\n\t"
      "setp.ne.b32 p, %3, 0;\n\tsetp.eq.b32 t, %3, %3;\n\telect.sync _|e, 0xffffffff;\n\t"
      "mov.b64 db, {%2, hi};\n\t" HS_MMA_PARTS("%8", "p")
      "add.u32 bl, %2, %11;\n\tmov.b64 db, {bl, hi};\n\t" HS_MMA_PARTS("%9", "t")
      "add.u32 bl, %2, %13;\n\tmov.b64 db, {bl, hi};\n\t" HS_MMA_PARTS("%10", "t") "}\n" ::"r"(d),
      "r"(xbase), "r"(wbase), "r"(accumulate), "n"(kDescHi), "n"(I0), "n"(I1), "n"(I2), "n"(PX0), "n"(PX1),
      "n"(PX2), "n"(WT), "n"(PS), "n"(2 * WT));
#undef HS_MMA_PARTS
}

// the conv kernel's issue pattern: filter-row asm blocks of nine MMAs (N = 3cs, 2cs, cs)
template <int CS, int COMMIT_EVERY>
__global__ void k_row9(long long* out, int reps) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(8) uint64_t bar2[4];
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar2[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s_tmem;
  if (warp == 0) {
    constexpr uint32_t I0 = idesc_bf16(128, 3 * CS), I1 = idesc_bf16(128, 2 * CS), I2 = idesc_bf16(128, CS);
    const uint32_t xb = (uint32_t)(desc(smem_u32(smem), 400 * 16, 128) & 0xffffffffu);
    const uint32_t wb = (uint32_t)(desc(smem_u32(smem + 65536), 3 * CS * 16, 128) & 0xffffffffu);
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < reps; ++i) {
      mma_row9<I0, I1, I2, 0, 1, 2, 2 * 3 * CS, 1200>(tmem + (i / COMMIT_EVERY % 4) * 96, xb + (i & 3) * 130, wb, 1);
      if (COMMIT_EVERY && i % COMMIT_EVERY == COMMIT_EVERY - 1) {
        asm volatile(
            "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(
                smem_u32(&bar2[(i / COMMIT_EVERY) & 3]))
            : "memory");
        asm volatile(
            "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(
                smem_u32(&bar2[(i / COMMIT_EVERY + 1) & 3]))
            : "memory");
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      }
    }
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(smem_u32(&bar))
        : "memory");
    asm volatile(
        "{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@P1 bra D;\n\tbra W;\n\tD:\n\t}\n" ::"r"(
            smem_u32(&bar)));
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int CS, int CE = 0>
void run_row9(long long* d) {
  const int reps = 1024;
  cudaFuncSetAttribute(k_row9<CS, CE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  k_row9<CS, CE><<<1, 128, 200 * 1024>>>(d, reps);
  k_row9<CS, CE><<<1, 128, 200 * 1024>>>(d, reps);
  long long h = 0;
  cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("row9 asm, cs=%d (N = %d/%d/%d), 2 commits+fence every %d blocks: %.1f cycles per MMA (%s)\n", CS, 3 * CS, 2 * CS, CS, CE, (double)h / (9 * reps),
         cudaGetErrorString(cudaDeviceSynchronize()));
}


// the tcgen05.shift conv's issue pattern (conv_shift.cu): per input row 27 MMAs (N = 48 / 32 / 16) into three
// accumulators and 6 shifts of the row's TMEM A slot, all from one elected thread
constexpr uint32_t WT = 96;
#define HS_SH_TAP(D, E, P0, WOFF)                                                   \
  "add.u32 bl, %4, " WOFF ";\n\tmov.b64 db, {bl, hi};\n\t"                         \
  "@" E " tcgen05.mma.cta_group::1.kind::f16 [" D "], [%3], db, i0, " P0 ";\n\t"    \
  "@" E " tcgen05.mma.cta_group::1.kind::f16 [" D "], [ta1], db, i1, pt;\n\t"       \
  "@" E " tcgen05.mma.cta_group::1.kind::f16 [" D "], [ta2], db, i2, pt;\n\t"
#define HS_SH_SHIFT                                                                 \
  "@es tcgen05.shift.cta_group::1.down [%3];\n\t"                                   \
  "@es tcgen05.shift.cta_group::1.down [ta1];\n\t"                                  \
  "@es tcgen05.shift.cta_group::1.down [ta2];\n\t"
#define HS_SH_KX(E0, E1, E2, P0, W0, W1, W2, SH) \
  HS_SH_TAP("%0", E0, P0, W0) HS_SH_TAP("%1", E1, "pt", W1) HS_SH_TAP("%2", E2, "pt", W2) SH
#define HS_SH_ROW(E0, E1, E2)                                                       \
  HS_SH_KX(E0, E1, E2, "pz", "%10", "%13", "%16", HS_SH_SHIFT)                      \
  HS_SH_KX(E0, E1, E2, "pt", "%11", "%14", "%17", HS_SH_SHIFT)                      \
  HS_SH_KX(E0, E1, E2, "pt", "%12", "%15", "%18", "")
#define HS_SH_OPERANDS                                                                                          \
  "r"(d0), "r"(d1), "r"(d2), "r"(abase), "r"(wlo), "r"(valid), "n"(kDescHi), "n"(I0), "n"(I1), "n"(I2), "n"(0 * WT), \
      "n"(1 * WT), "n"(2 * WT), "n"(3 * WT), "n"(4 * WT), "n"(5 * WT), "n"(6 * WT), "n"(7 * WT), "n"(8 * WT)
#define HS_SH_HEAD                                                                                              \
  "{\n\t.reg .pred e, es, e0, e1, e2, pz, pt;\n\t.reg .b64 db;\n\t.reg .b32 hi, i0, i1, i2, ta1, ta2, bl, m;\n\t" \
  "mov.b32 hi, %6;\n\tmov.b32 i0, %7;\n\tmov.b32 i1, %8;\n\tmov.b32 i2, %9;\n\t"                                  \
  "elect.sync _|e, 0xffffffff;\n\t"                                                                             \
  "setp.ne.b32 pz, %5, %5;\n\tsetp.eq.b32 pt, %5, %5;\n\t"                                                       \
  "add.u32 ta1, %3, 8;\n\tadd.u32 ta2, %3, 16;\n\t"


template <int SAMEACC, int NOSHIFT, int NCOMMIT = 0>
__global__ void k_rowpat(long long* out, int rows) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(8) uint64_t cbar[2];
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    for (int i = 0; i < 2; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&cbar[i])));
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
  if (warp == 0) {
    constexpr uint32_t I0 = idesc_bf16(128, 48), I1 = idesc_bf16(128, 32), I2 = idesc_bf16(128, 16);
    const uint32_t wlo = (uint32_t)(desc(smem_u32(smem), 48 * 16, 128) & 0xffffffffu);
    const uint32_t valid = NOSHIFT ? 0u : 1u;
    long long t0 = clock64();
    uint32_t s = 0, as = 0;
#pragma unroll 1
    for (int r = 0; r < rows; ++r) {
      const uint32_t d0 = tmem + s * 48, d1 = SAMEACC ? d0 : tmem + ((s + 5) % 6) * 48, d2 = SAMEACC ? d0 : tmem + ((s + 4) % 6) * 48;
      const uint32_t abase = tmem + 288 + as * 24;
      asm volatile(HS_SH_HEAD
                   "@!e bra SH_SKIP_%=;\n\t"
                   "setp.ne.b32 es, %5, 0;\n\t" HS_SH_ROW("pt", "pt", "pt") "SH_SKIP_%=:\n\t}\n" ::HS_SH_OPERANDS
                   : "memory");
      __syncwarp();
      for (int c = 0; c < NCOMMIT; ++c)
        asm volatile(
            "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(smem_u32(&cbar[c]))
            : "memory");
      s = s + 1 == 6 ? 0 : s + 1;
      as = as + 1 == 9 ? 0 : as + 1;
    }
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(smem_u32(&bar))
        : "memory");
    asm volatile(
        "{\n\t.reg .pred P1;\n\tW2:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@P1 bra D2;\n\tbra W2;\n\tD2:\n\t}\n" ::"r"(
            smem_u32(&bar)));
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int SAMEACC, int NOSHIFT, int NCOMMIT = 0>
void run_rowpat(long long* d) {
  auto k = k_rowpat<SAMEACC, NOSHIFT, NCOMMIT>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  k<<<1, 128, 64 * 1024>>>(d, 2000);
  k<<<1, 128, 64 * 1024>>>(d, 2000);
  long long h = 0;
  cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
  cudaError_t e = cudaDeviceSynchronize();
  printf("shift-conv row pattern (27 MMAs + 6 shifts), same accumulator %d, no shifts %d, commits per row %d: %.1f cycles per row (%s)\n", SAMEACC,
         NOSHIFT, NCOMMIT, (double)h / 2000, cudaGetErrorString(e));
}

int main(int argc, char** argv) {
  long long* d;
  cudaMalloc(&d, 1024 * sizeof(long long));
  if (argc > 1) {  // "tm": A in TMEM, cycles per MMA against N (one accumulator, back to back)
    run_rowpat<0, 0>(d);
    run_rowpat<0, 0, 1>(d);
    run_rowpat<0, 0, 2>(d);
    run_rowpat<1, 0>(d);
    run_rowpat<0, 1>(d);
    run_rowpat<1, 1>(d);
    run<128, 16, true>(d);
    run<128, 32, true>(d);
    run<128, 48, true>(d);
    run<128, 64, true>(d);
    run<128, 96, true>(d);
    run<128, 128, true>(d);
    run<128, 144, true>(d);
    run<128, 192, true>(d);
    run<128, 256, true>(d);
    return 0;
  }
  run_row9<16>(d);
  run_row9<32>(d);
  run_row9<32, 6>(d);
  run_row9<16, 3>(d);
  run<128, 48, false, 1, 1, false, 0>(d);
  run<128, 48, false, 1, 1, false, 16>(d);
  run<128, 48, false, 1, 1, false, 32>(d);
  run<128, 96, false, 1, 1, false, 0>(d);
  run<128, 96, false, 1, 1, false, 16>(d);
  run<128, 96, false, 1, 1, false, 48>(d);
  return 0;
}
