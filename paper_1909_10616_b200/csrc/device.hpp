// Device-side entry points of libtiletune (kernel launchers; no torch types anywhere).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "space.hpp"

namespace tt {

// Launch binding (a5 of SURVEY §8a): factors -> grid, block, smem, stages, descriptors.
tt_status bind(const Space& sp, const State& s, tt_launch_info* info, std::string* err);

// K1 / K2 / K3 dispatch for a feasible config; asynchronous on `stream`.
tt_status launch_gemm(const Space& sp, const State& s, const void* A, const void* B, float* C,
                      cudaStream_t stream, std::string* err);

// Everything a launch does on the host except the launch itself (instance choice, plan, tensor
// maps, the shared-memory opt-in that loads the kernel's module), so a timed launch right after
// it spends no host time between its CUDA events.
tt_status prepare_gemm(const Space& sp, const State& s, const void* A, const void* B, float* C, std::string* err);

// K4: counter-based U[-1,1) operand generator.
tt_status launch_fill(void* dst, int dtype, uint64_t seed, uint64_t idx0, uint64_t count,
                      cudaStream_t stream, std::string* err);

// K5: im2col for conv-as-GEMM.
tt_status launch_im2col(int dtype, const void* x, int64_t Nb, int64_t C, int64_t H, int64_t W, int R, int S,
                        int stride, int pad, void* A, cudaStream_t stream, std::string* err);

// Family-specific launchers (gemm_simt.cu, gemm_umma.cu).
tt_status simt_bind(const Space& sp, const State& s, tt_launch_info* info, std::string* err);
tt_status simt_launch(const Space& sp, const State& s, const float* A, const float* B, float* C,
                      cudaStream_t stream, std::string* err, int64_t max_rows = 0);
// K1 launch shape for the partial-grid probe: total CTAs and co-resident CTA slots on the device.
tt_status simt_probe_shape(const Space& sp, const State& s, int64_t* ctas, int64_t* slots, std::string* err);
tt_status simt_prepare(const Space& sp, const State& s, std::string* err);
// Load every kernel of a family (the max-smem opt-in loads the module function), so no first
// launch of a search pays it.
tt_status simt_preload(std::string* err);
tt_status umma_preload(int family, std::string* err);
// 2-D fp32 tensor map without swizzle (gemm_umma.cu): dims {inner, outer}, box {box_in, box_out}.
bool encode_map_2d_f32(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint32_t box_in,
                       uint32_t box_out, std::string* err);
tt_status umma_bind(const Space& sp, const State& s, tt_launch_info* info, std::string* err);
// every cluster's work items (tile, kb0, kb1, order, split) x n of a tcgen05 launch, in walk order
tt_status umma_schedule(const Space& sp, const State& s, std::vector<std::vector<int32_t>>* per_worker,
                        int32_t* k0, std::string* err);
tt_status umma_prepare(const Space& sp, const State& s, const void* A, const void* B, float* C, std::string* err);
tt_status umma_launch(const Space& sp, const State& s, const void* A, const void* B, float* C,
                      cudaStream_t stream, std::string* err);

inline bool cuda_ok(cudaError_t e, std::string* err, const char* what) {
  if (e == cudaSuccess) return true;
  *err = std::string(what) + ": " + cudaGetErrorString(e);
  return false;
}

// Opt kernel `fn` into `bytes` of dynamic shared memory on the current device.  The attribute is
// per device context, so the "already set" cache is keyed by (device, fn) and guarded by a lock.
bool ensure_max_smem(const void* fn, int bytes, std::string* err);

}  // namespace tt
