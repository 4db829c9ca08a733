// Microbenchmark: per-SM bulk-copy (TMA engine) ingest from L2 into shared memory, no compute.
// One CTA per SM streams `chunk`-byte cp.async.bulk copies of an L2-resident buffer into a
// 4-slot shared-memory ring (one elected thread issues, mbarrier complete_tx per slot, slots
// re-armed as soon as they land).  Printed: bytes per SM-clock per active SM and chip-wide GB/s
// for 148, 74 and 37 active CTAs -- a per-SM ceiling shows as a constant B/clk/SM, a chip-wide
// one as a B/clk/SM that rises when fewer SMs pull.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ingest tools/ingest_bench.cu && /tmp/ingest
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kSlots = 4;

__device__ __forceinline__ bool try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.b32 %0, 1, 0, P;\n\t}"
               : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
  return ok != 0;
}

__global__ void __launch_bounds__(32, 1) ingest(const uint8_t* src, size_t src_bytes, int chunk, int iters,
                                               long long* cycles, unsigned long long* bytes) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bars[kSlots];
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sm);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kSlots; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bars[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  if (threadIdx.x != 0) return;
  const size_t nchunks = src_bytes / chunk;
  size_t c = (size_t)blockIdx.x * 97 % nchunks;
  auto issue = [&](int s) {
    const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&bars[s]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(chunk) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(sbase + (uint32_t)(s * chunk)), "l"(src + c * chunk), "r"(chunk), "r"(bar) : "memory");
    c = (c + 148) % nchunks;
  };
  for (int s = 0; s < kSlots; ++s) issue(s);
  uint32_t phase[kSlots] = {0, 0, 0, 0};
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    const int s = i % kSlots;
    const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&bars[s]);
    while (!try_wait(bar, phase[s])) {
    }
    phase[s] ^= 1u;
    issue(s);
  }
  const long long t1 = clock64();
  for (int s = 0; s < kSlots; ++s) {                  // drain the copies still in flight
    const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&bars[s]);
    while (!try_wait(bar, phase[s])) {
    }
  }
  cycles[blockIdx.x] = t1 - t0;
  bytes[blockIdx.x] = (unsigned long long)iters * chunk;
}

int main() {
  const size_t src_bytes = 64ull << 20;              // 64 MiB: L2-resident after the first pass
  uint8_t* src;
  cudaMalloc(&src, src_bytes);
  cudaMemset(src, 1, src_bytes);
  long long* cyc;
  unsigned long long* by;
  cudaMalloc(&cyc, 148 * sizeof(long long));
  cudaMalloc(&by, 148 * sizeof(unsigned long long));
  cudaFuncSetAttribute(ingest, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  for (int chunk : {16384, 32768, 49152}) {
    for (int grid : {148, 74, 37, 8}) {
      const int iters = 4000;
      ingest<<<grid, 32, kSlots * chunk>>>(src, src_bytes, chunk, 200, cyc, by);   // warm L2
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      ingest<<<grid, 32, kSlots * chunk>>>(src, src_bytes, chunk, iters, cyc, by);
      cudaEventRecord(e1);
      cudaDeviceSynchronize();
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      long long hc[148];
      unsigned long long hb[148];
      cudaMemcpy(hc, cyc, grid * sizeof(long long), cudaMemcpyDeviceToHost);
      cudaMemcpy(hb, by, grid * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
      double bpc = 0, tot = 0;
      for (int g = 0; g < grid; ++g) {
        bpc += (double)hb[g] / (double)hc[g];
        tot += (double)hb[g];
      }
      printf("{\"chunk\": %d, \"ctas\": %d, \"bytes_per_sm_clock\": %.1f, \"chip_GBps\": %.0f, \"ms\": %.3f, \"err\": \"%s\"}\n",
             chunk, grid, bpc / grid, tot / (ms * 1e-3) / 1e9, ms, cudaGetErrorString(cudaGetLastError()));
    }
  }
  (void)clk_khz;
  return 0;
}
