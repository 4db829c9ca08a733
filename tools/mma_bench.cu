// Microbenchmark: back-to-back tcgen05.mma issue rate (no loads), 1-CTA M=128 and 2-CTA M=256.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo, int layout) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | ((uint64_t)layout << 61);
}

template <int CG, int N, int UNROLL, bool MNB>
__global__ void __launch_bounds__(128, 1) bench(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sm);
  sbase = (sbase + 1023) & ~1023u;
  const int warp = __shfl_sync(0xffffffff, threadIdx.x >> 5, 0);
  uint32_t rank = 0;
  if (CG == 2) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (warp == 0) {
    if (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&slot)), "r"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&slot)), "r"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
  }
  if (threadIdx.x == 32) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  if (CG == 2) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;");
  else __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  // A: 128 rows x 64 bf16 (K-major SW128) at sbase; B at sbase + 16K
  const uint32_t M = 128 * CG;
  uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((MNB ? 1u : 0u) << 16) | ((uint32_t)(N >> 3) << 17) | ((M >> 4) << 24);
  uint64_t ad = desc(sbase, 16, 1024, 2);
  uint64_t bd = MNB ? desc(sbase + 16384, 64 * 128, 1024, 2) : desc(sbase + 16384, 16, 1024, 2);
  long long t0 = 0, t1 = 0;
  if (warp == 1 && rank == 0) {
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        uint32_t pred = 0;
        asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(pred));
        if (pred) {
          if (CG == 1)
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                         ::"r"(tmem), "l"(ad + (u & 3) * 2), "l"(bd), "r"(idesc), "r"(1));
          else
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                         ::"r"(tmem), "l"(ad + (u & 3) * 2), "l"(bd), "r"(idesc), "r"(1));
        }
        __syncwarp();
      }
    }
    uint32_t pred = 0;
    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(pred));
    if (pred) {
      if (CG == 1)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
      else
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)), "h"((uint16_t)1));
    }
    __syncwarp();
    asm volatile("{\n\t.reg .pred P;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n\t@!P bra W;\n\t}" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
    t1 = clock64();
    if (threadIdx.x == 32) out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  if (CG == 2) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;");
  else __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) {
    if (CG == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    else asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

template <int CG, int N, int UNROLL, bool MNB>
void run(const char* name) {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  cudaMemset(d, 0, 148 * sizeof(long long));
  auto fn = bench<CG, N, UNROLL, MNB>;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = 80000;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CG;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const int iters = 512;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaError_t err = cudaLaunchKernelEx(&cfg, fn, d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    if (err != cudaSuccess || cudaGetLastError() != cudaSuccess) { printf("%s: launch error %s\n", name, cudaGetErrorString(err)); return; }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    const double mmas = (double)iters * UNROLL;
    const double flops = 2.0 * 128 * CG * N * 16 * mmas * (148 / CG);
    printf("%-28s cycles/MMA %.1f  (%.1f TF/s over %.3f ms)\n", name, (double)h[0] / mmas, flops / (ms * 1e-3) / 1e12, ms);
  }
  cudaFree(d);
}

int main() {
  run<1, 256, 8, false>("1CTA M128 N256 Kmaj");
  run<1, 256, 8, true>("1CTA M128 N256 MNmaj");
  run<1, 128, 8, true>("1CTA M128 N128 MNmaj");
  run<2, 256, 8, false>("2CTA M256 N256 Kmaj");
  run<2, 256, 8, true>("2CTA M256 N256 MNmaj");
  run<2, 128, 8, true>("2CTA M256 N128 MNmaj");
  return 0;
}
