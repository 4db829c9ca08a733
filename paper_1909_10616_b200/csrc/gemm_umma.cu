// K2 / K3: tcgen05 (5th-gen tensor core) tiled GEMM family for sm_100a, TF32 and BF16.
//
// The paper's tiling configuration (Eq. 1-4; d = (4,2,4)) is bound to a
// persistent, warp-specialised tcgen05 kernel (reading Z2):
//   m = [m0 cluster tiles along M, m1 = cta_group (1, or 2 = CTA pair sharing one UMMA_M=256
//        instruction), m2 = UMMA M-atoms per CTA (1|2), m3 = UMMA_M per CTA (128)]
//   n = [n0 cluster tiles along N, n1 = 1, n2 = UMMA N-atoms per CTA (1|2), n3 = UMMA_N]
//   k = [k0 main-loop trips, k1 = BK (K slab per pipeline stage)]
// Cluster tile = (m1 m2 128) x (n2 n3).  C[M][N] fp32 = A[M][K] . B[K][N] with A K-major and
// B MN-major (row-major B is read transposed by the descriptor; no copy).
//
// Warp roles (256 threads, 1 CTA per SM): warp 0 = TMA producer (A and B slabs into a
// `stages`-deep shared-memory ring guarded by full/empty mbarriers), warp 1 = MMA issuer
// (one elected thread, leader CTA only), warp 2 = TMEM allocator, warps 4-7 = epilogue
// (TMEM -> registers via tcgen05.ld -> swizzled smem -> TMA store of fp32 C).  Accumulators are double buffered in
// TMEM when m2 n2 n3 <= 256 columns so the epilogue of tile t overlaps the MMAs of tile t+1.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>

#include "device.hpp"

namespace tt {

namespace {

constexpr int kEpiBytes = 32768;   // minimum epilogue staging (the J_hw reserve)
constexpr int kEpiBoxBytes = 4096; // one 32 x 32 fp32 staging box
constexpr int kEpiMaxBufs = 8;     // boxes per epilogue warp
// Epilogue warps 4 .. 3 + kEpiWarps; kEpiWarps / 4 warps per TMEM lane quarter take its 32-column
// chunks round-robin.  8 warps measured no faster than 4 (the SM's write path bounds the drain,
// profiles/r3_epilogue.md) and cost ~3 % at 4096^3 by competing with the MMA phase for shared
// memory, so 4.
constexpr int kEpiWarps = 4;
constexpr int kEpiGroups = kEpiWarps / 4;
constexpr int kThreads = 32 * (4 + kEpiWarps);
static_assert(kEpiWarps % 4 == 0 && kEpiWarps * kEpiBoxBytes <= kEpiBytes, "the epilogue staging fits the J_hw reserve");

struct UmmaArgs {
  int64_t M, N, K;
  int m0, n0, k0;
  int m2, n2, n3, bk;
  int stages, acc_bufs, acc_cols;   // acc_cols = m2 n2 n3 (columns per accumulator buffer)
  int tmem_cols;
  int swz_a, swz_b;                 // swizzle bytes: 32 | 64 | 128
  int a_layout, b_layout;           // descriptor layout codes (SW128 2, SW64 4, SW32 6, SW128_BASE32B 1)
  int sbo_b;                        // B stride between K core-matrix groups (bytes)
  int a_mn;                         // A is MN-major: W = A^T row-major [K][M] (P:372 Y = W^T X)
  int a_cw;                         // MN-major A: M elements per TMA box (128 B)
  int a_chunk_bytes;                // bytes of one A K-chunk (rows x swz_a)
  int b_cw;                         // B columns per TMA box (swz_b / elem)
  int nb;                           // B columns per CTA per atom = n3 / cta_group
  int a_stage_bytes, stage_bytes;   // A part, total per stage (A + padded B)
  int epi_bufs;                     // 4 KB staging boxes per epilogue warp (1 .. kEpiMaxBufs)
  int n1;                           // CTA pairs (or CTAs) per cluster along N; 2 = A multicast
  int a_box_rows;                   // K-major A: rows per TMA box (m2 128 / n1: each pair loads its share)
  uint32_t idesc;
  uint32_t tx_bytes;                // bytes landing per stage per CTA
  // tail split: the last sk_tiles tiles' k-blocks are spread evenly over the
  // first sk_workers clusters; the remaining dp_tiles tiles go round-robin to all clusters.
  int dp_tiles, sk_tiles, sk_workers;
  int flag_group;                   // slice of g_split_flags this launch uses (per launch stream)
  uint64_t* trace;                  // debug (TT_UMMA_TRACE): per cluster x item timestamps, or null
};

// Debug instrumentation is compiled only into the trace build (python -m paper_1909_10616_b200.build
// --variant trace TT_UMMA_TRACE_BUILD; tools/umma_trace.py loads it): in the product kernel every
// `kTrace && ...` branch folds away, so the timing code costs neither instructions nor registers.
#ifdef TT_UMMA_TRACE_BUILD
constexpr bool kTrace = true;
#else
constexpr bool kTrace = false;
#endif

// TT_UMMA_TRACE layout: [cluster][kTraceItems][8] u64 = tile, kb0 | kb1 << 16 | order << 32,
// t(MMA start), t(MMA last issue), t(epilogue: accumulator ready), t(epilogue: flag ok), t(done),
// and in slot 7: kernel entry (item 0) / teardown barrier passed (item 1)
constexpr int kTraceItems = 16;

// Tail-split handshake words: per split tile and CTA rank, the number of epilogue warps of the
// tile's pieces that have landed.  A module-scope device array (zero at module load, one copy per
// device context), so tt_gemm never allocates or memsets; every launch leaves its words at zero
// (the top piece resets them), so back-to-back launches and CUDA-graph replays need no reset.
// Launches on different streams use different groups (host: split_flag_group).
constexpr int kFlagGroups = 64;
constexpr int kFlagWords = 1024;    // >= max split tiles (< 148 clusters) x CTAs per cluster (<= 4)
__device__ uint32_t g_split_flags[kFlagGroups * kFlagWords];

// ---------------------------------------------------------------- PTX helpers
// debug (TT_UMMA_TRACE): cycles since kernel entry on this SM, into slot 7 of item 8 + idx
__device__ __forceinline__ void trace_cycles(uint64_t* trace, int cluster, int idx, long long t_entry) {
  trace[((int64_t)cluster * 16 + 8 + idx) * 8 + 7] = (uint64_t)(clock64() - t_entry);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2, %3;\n\t"
      "selp.b32 %0, 1, 0, P;\n\t}" : "=r"(ok) : "r"(bar), "r"(parity), "r"(0x989680) : "memory");
  return ok != 0;
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Watchdog: a pipeline that has not advanced for 10 s traps (a launch error the host reports)
// instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  if (mbar_try(bar, parity)) return;
  const uint64_t t0 = globaltimer();
  while (!mbar_try(bar, parity)) {
    if (globaltimer() - t0 > 10000000000ull) __trap();
  }
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar, uint32_t cta) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\t"
      "mapa.shared::cluster.u32 ra, %0, %1;\n\t"
      "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n\t}" ::"r"(bar), "r"(cta) : "memory");
}
__device__ __forceinline__ void st_shared_v4(uint32_t addr, float a, float b, float c, float d) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, uint32_t src, int x, int y) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
               ::"l"(map), "r"(x), "r"(y), "r"(src) : "memory");
}
__device__ __forceinline__ void tma_reduce_add_2d(const CUtensorMap* map, uint32_t src, int x, int y) {
  asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2}], [%3];"
               ::"l"(map), "r"(x), "r"(y), "r"(src) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t atom_add_release(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.release.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
// Spin until *flag >= target (written by the lower-index clusters that own the lower k-blocks of
// the same tile, see Sched); the watchdog turns a lost writer into a trap instead of a hang.
__device__ __forceinline__ void wait_flag(const uint32_t* flag, uint32_t target) {
  if (ld_acquire(flag) >= target) return;
  const uint64_t t0 = globaltimer();
  while (ld_acquire(flag) < target) {
    if (globaltimer() - t0 > 10000000000ull) __trap();
  }
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
// wait until at most n bulk groups are still reading shared memory (n is warp-uniform)
__device__ __forceinline__ void bulk_wait_read_n(int n) {
  switch (n) {
    case 0: bulk_wait_read<0>(); break;
    case 1: bulk_wait_read<1>(); break;
    case 2: bulk_wait_read<2>(); break;
    case 3: bulk_wait_read<3>(); break;
    case 4: bulk_wait_read<4>(); break;
    case 5: bulk_wait_read<5>(); break;
    case 6: bulk_wait_read<6>(); break;
    default: bulk_wait_read<7>(); break;
  }
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int CG>
__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint32_t bar, uint32_t dst, int x, int y) {
  if constexpr (CG == 1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        ::"r"(dst), "l"(map), "r"(x), "r"(y), "r"(bar) : "memory");
  } else {
    // both CTAs of the pair signal the leader's barrier (peer bit cleared)
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        ::"r"(dst), "l"(map), "r"(x), "r"(y), "r"(bar & 0xFEFFFFFFu) : "memory");
  }
}

// Multicast load: the box lands at the same shared-memory offset in every CTA of `mask` and
// each destination's pair leader (peer bit cleared for cta_group::2) receives the complete_tx.
template <int CG>
__device__ __forceinline__ void tma_load_2d_mc(const CUtensorMap* map, uint32_t bar, uint32_t dst, int x, int y,
                                               uint16_t mask) {
  if constexpr (CG == 1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1, {%2, %3}], [%4], %5;"
        ::"r"(dst), "l"(map), "r"(x), "r"(y), "r"(bar), "h"(mask) : "memory");
  } else {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1, {%2, %3}], [%4], %5;"
        ::"r"(dst), "l"(map), "r"(x), "r"(y), "r"(bar & 0xFEFFFFFFu), "h"(mask) : "memory");
  }
}

__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo, int layout_code) {
  // tcgen05 shared-memory matrix descriptor: start>>4 [0,14), LBO>>4 [16,30), SBO>>4 [32,46),
  // version 1 [46,48), base offset 0, layout [61,64): SW128 = 2, SW64 = 4, SW32 = 6,
  // SW128 with 32-byte atoms (the only MN-major tf32 layout) = 1
  const uint64_t layout = (uint64_t)layout_code;
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (layout << 61);
}

template <int KIND, int CG>
__device__ __forceinline__ void umma(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if constexpr (KIND == 0 && CG == 1)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                 ::"r"(d_tmem), "l"(a), "l"(b), "r"(idesc), "r"(acc));
  else if constexpr (KIND == 0 && CG == 2)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                 ::"r"(d_tmem), "l"(a), "l"(b), "r"(idesc), "r"(acc));
  else if constexpr (KIND == 1 && CG == 1)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                 ::"r"(d_tmem), "l"(a), "l"(b), "r"(idesc), "r"(acc));
  else
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                 ::"r"(d_tmem), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

// Arrive (when the issued MMAs complete) on `bar` in every CTA of `mask`; mask 0 = this CTA only.
template <int CG>
__device__ __forceinline__ void umma_commit(uint32_t bar, uint16_t mask) {
  if constexpr (CG == 1) {
    if (mask == 0)
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
    else
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                   ::"r"(bar), "h"(mask) : "memory");
  } else {
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(bar), "h"(mask) : "memory");
  }
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

template <int KIND>
__device__ __forceinline__ constexpr uint32_t kind_sbo_mn() { return KIND == 1 ? 4u * 128u : 8u * 128u; }

// One unit of work for a cluster: k-blocks [kb0, kb1) of output tile `tile`.  A split tile's
// partial sums are combined in ascending-k order: the piece holding k-block 0 (order 0) stores C,
// each higher piece waits until every piece below it has landed and adds with a TMA reduce.
// Every role warp walks the identical sequence.
//
// Deadlock freedom.  Worker (cluster) w owns the contiguous k-block range [sk_begin(w),
// sk_begin(w+1)) of the tail tiles in tile-major order, so the pieces below a piece of w belong
// to clusters with a LOWER index.  A worker's range spans at most two tiles (its length is at most
// k0) and it processes them last tile first: the first item is the piece that starts at k-block 0
// of its tile (stores, waits on nobody) unless the range lies inside one tile, in which case it is
// the worker's only item.  Hence every piece waits only on the first item of lower-index clusters,
// which themselves wait only on lower indices: no cycles, and no wait on a cluster that is
// dispatched later.  Clusters are dispatched in index order, so the tail split needs no
// co-residency of the whole grid (concurrent kernels, MPS or green contexts that hold SMs only
// delay it) -- the property CUB's decoupled look-back scan also relies on.
struct Item {
  int tile, kb0, kb1, order;
  bool split;
};

struct Sched {
  // 32-bit throughout: the host enables a split only when sk_workers x sk_tiles x k0 < 2^32
  // (plan_of), and 64-bit divisions (a called subroutine each) cost ~1 us of prologue.
  int w, P, dp, nseg, seg;
  uint32_t b, e;
  __host__ __device__ __forceinline__ static uint32_t sk_begin(const UmmaArgs& p, int v) {
    return (uint32_t)v * ((uint32_t)p.sk_tiles * (uint32_t)p.k0) / (uint32_t)p.sk_workers;
  }
  __host__ __device__ __forceinline__ Sched(const UmmaArgs& p, int w_, int P_) : w(w_), P(P_), dp(w_), nseg(0), seg(0), b(0), e(0) {
    if (w < p.sk_workers) {
      b = sk_begin(p, w);
      e = sk_begin(p, w + 1);
      if (e > b) nseg = (int)((e - 1) / (uint32_t)p.k0 - b / (uint32_t)p.k0) + 1;
    }
  }
  // tail pieces first, last tile of the range first; then the data-parallel tiles
  __host__ __device__ __forceinline__ bool next(const UmmaArgs& p, Item* it) {
    if (seg < nseg) {
      const uint32_t k0 = (uint32_t)p.k0;
      const uint32_t t_rel = (e - 1) / k0 - (uint32_t)seg;
      const uint32_t ts = t_rel * k0;
      const uint32_t lo = b > ts ? b : ts;
      const uint32_t hi = e < ts + k0 ? e : ts + k0;
      it->tile = p.dp_tiles + (int)t_rel;
      it->kb0 = (int)(lo - ts);
      it->kb1 = (int)(hi - ts);
      it->split = !(it->kb0 == 0 && it->kb1 == p.k0);
      int order = 0;                                 // pieces of this tile below this one
      if (it->split)
        for (int v = w - 1; v >= 0; --v) {
          const uint32_t vb = sk_begin(p, v), ve = sk_begin(p, v + 1);
          if (ve <= ts) break;
          if (ve > vb) ++order;
        }
      it->order = order;
      ++seg;
      return true;
    }
    if (dp < p.dp_tiles) {
      *it = Item{dp, 0, p.k0, 0, false};
      dp += P;
      return true;
    }
    return false;
  }
};

struct MmaCtx {
  uint32_t sbase, full0, empty0, tfull0, tempty0, tmem_base;
  int cluster_id, num_clusters;
  uint16_t empty_mask, tfull_mask;   // CTAs whose empty / accumulator-ready barriers a commit feeds
  long long t_entry;                 // debug trace only
};

template <int KIND, int CG, int KS, int M2, int N2>
__device__ __forceinline__ void mma_role(const UmmaArgs& p, const MmaCtx& c) {
  constexpr int ELEM = KIND == 0 ? 2 : 4;
  constexpr int UK = KIND == 0 ? 16 : 8;
  // descriptor words: high halves are invariant; low halves = (start >> 4) | (LBO >> 4) << 16
  const uint32_t lbo_b = (uint32_t)(p.bk * p.swz_b);
  // K-major A: 128-row atoms of swz_a-byte rows; MN-major A (TN layout): BK x 128 B boxes of a_cw
  // rows each, atom mi = 128 / a_cw boxes, LBO = box stride, SBO = 8 (4 for tf32) K-rows x 128 B
  const uint32_t a_box = (uint32_t)(p.bk * 128);
  const uint64_t a_hi = (p.a_mn ? smem_desc(0, a_box, kind_sbo_mn<KIND>(), p.a_layout)
                                : smem_desc(0, 16u, 8u * (uint32_t)p.swz_a, p.a_layout)) & 0xFFFFFFFF00000000ull;
  const uint64_t b_hi = smem_desc(0, lbo_b, (uint32_t)p.sbo_b, p.b_layout) & 0xFFFFFFFF00000000ull;
  const uint32_t a_lbo = p.a_mn ? (((a_box >> 4) & 0x3FFFu) << 16) : (1u << 16);
  const uint32_t b_lbo = ((lbo_b >> 4) & 0x3FFFu) << 16;
  // At most 16 k-steps are unrolled with per-step offsets in registers; a 32-step stage (tf32,
  // BK = 256) replays them with a constant shift (+16 k-steps = +512 B along K in every layout).
  constexpr int KSU = KS > 16 ? 16 : KS;
  constexpr int REP = KS / KSU;
  uint32_t a_off[KSU][M2], b_off[KSU][N2], d_off[M2][N2];
#pragma unroll
  for (int ks = 0; ks < KSU; ++ks) {
    const uint32_t kbytes = (uint32_t)(ks * UK * ELEM);
#pragma unroll
    for (int mi = 0; mi < M2; ++mi)
      a_off[ks][mi] = p.a_mn
          ? (((uint32_t)(mi * (128 / p.a_cw)) * a_box + (uint32_t)(ks * UK * 128)) >> 4) | a_lbo
          : (((kbytes / p.swz_a) * p.a_chunk_bytes + kbytes % p.swz_a + mi * 128 * p.swz_a) >> 4) | a_lbo;
#pragma unroll
    for (int ni = 0; ni < N2; ++ni)
      b_off[ks][ni] = (((uint32_t)(ni * (p.nb / p.b_cw)) * lbo_b + (uint32_t)(ks * UK * p.swz_b)) >> 4) | b_lbo;
  }
  const uint32_t a_rep = (uint32_t)(p.a_mn ? (KSU * UK * 128) : ((KSU * UK * ELEM) / p.swz_a) * p.a_chunk_bytes) >> 4;
  const uint32_t b_rep = (uint32_t)(KSU * UK * p.swz_b) >> 4;
  (void)a_rep;
  (void)b_rep;
#pragma unroll
  for (int mi = 0; mi < M2; ++mi)
#pragma unroll
    for (int ni = 0; ni < N2; ++ni) d_off[mi][ni] = (uint32_t)((mi * N2 + ni) * p.n3);
  int stage = 0;
  uint32_t phase = 0;
  int acc = 0;
  uint32_t aphase = 0;
  Sched sch(p, c.cluster_id, c.num_clusters);
  Item it;
  int item_no = 0;
  if (kTrace && p.trace && elect_one())                                // debug: MMA role set up (item 5, slot 7)
    p.trace[((int64_t)c.cluster_id * kTraceItems + 5) * 8 + 7] = globaltimer();
  __syncwarp();
  while (sch.next(p, &it)) {
    mbar_wait(c.tempty0 + 8u * acc, aphase ^ 1u);
    tc_fence_after();
    uint64_t* tr = (kTrace && p.trace && item_no < kTraceItems) ? p.trace + ((int64_t)c.cluster_id * kTraceItems + item_no) * 8 : nullptr;
    ++item_no;
    if (kTrace && tr && elect_one()) tr[2] = globaltimer();
    __syncwarp();
    const uint32_t dbase = c.tmem_base + (uint32_t)(acc * p.acc_cols);
    for (int kb = it.kb0; kb < it.kb1; ++kb) {
      mbar_wait(c.full0 + 8u * stage, phase);
      tc_fence_after();
      if (kTrace && p.trace && item_no == 1 && kb == it.kb0 && elect_one()) {  // debug: first stage landed (item 7, slot 7)
        p.trace[((int64_t)c.cluster_id * kTraceItems + 7) * 8 + 7] = globaltimer();
        trace_cycles(p.trace, c.cluster_id, 4, c.t_entry);
      }
      __syncwarp();
      // descriptor start field = CTA-window byte address >> 4 (14 bits): the cvta result of a CTA
      // with cluster rank > 0 carries the rank above bit 24, which must not leak into LBO
      const uint32_t sa16 = ((c.sbase + (uint32_t)stage * p.stage_bytes) >> 4) & 0x3FFFu;
      const uint32_t sb16 = sa16 + ((uint32_t)p.a_stage_bytes >> 4);
      if (elect_one()) {
#pragma unroll
        for (int rep = 0; rep < REP; ++rep)
#pragma unroll
          for (int ks = 0; ks < KSU; ++ks)
#pragma unroll
            for (int mi = 0; mi < M2; ++mi)
#pragma unroll
              for (int ni = 0; ni < N2; ++ni)
                umma<KIND, CG>(dbase + d_off[mi][ni], a_hi | (uint64_t)(sa16 + rep * a_rep + a_off[ks][mi]),
                               b_hi | (uint64_t)(sb16 + rep * b_rep + b_off[ks][ni]), p.idesc,
                               (kb != it.kb0 || rep != 0 || ks != 0) ? 1u : 0u);
        umma_commit<CG>(c.empty0 + 8u * stage, c.empty_mask);  // frees the slot in every CTA that fills it
      }
      __syncwarp();
      if (++stage == p.stages) { stage = 0; phase ^= 1u; }
    }
    if (elect_one()) {
      umma_commit<CG>(c.tfull0 + 8u * acc, c.tfull_mask);   // accumulator ready for the epilogue
      if (kTrace && tr) tr[3] = globaltimer();
      if (kTrace && tr && item_no == 1) trace_cycles(p.trace, c.cluster_id, 5, c.t_entry);
    }
    __syncwarp();
    if (++acc == p.acc_bufs) { acc = 0; aphase ^= 1u; }
  }
}

// ---------------------------------------------------------------- the kernel
template <int KIND, int CG>
__global__ void __launch_bounds__(kThreads, 1)
k_umma(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
       const __grid_constant__ CUtensorMap tmC, float* __restrict__ C,
       const UmmaArgs p) {
  constexpr int UK = KIND == 0 ? 16 : 8;     // UMMA_K
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const uint32_t epi_base = sbase + (uint32_t)p.stages * p.stage_bytes;   // kEpiWarps x epi_bufs x 4 KB staging
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)p.stages * p.stage_bytes +
                                               (size_t)kEpiWarps * p.epi_bufs * kEpiBoxBytes);
  const uint32_t full0 = smem_u32(bars);
  const uint32_t empty0 = full0 + 8u * p.stages;
  const uint32_t tfull0 = empty0 + 8u * p.stages;
  const uint32_t tempty0 = tfull0 + 16u;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * p.stages + 4);

  // warp index made provably warp-uniform so role loops run on the uniform datapath
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  // cluster = n1 pairs (CG = 2) or n1 CTAs (CG = 1) side by side along N; they share A rows,
  // so with n1 = 2 each loads its half of the A slab and multicasts it to its counterpart
  const int csize = CG * p.n1;
  const uint32_t crank = csize > 1 ? cluster_rank() : 0u;
  const uint32_t rank = crank % CG;                 // CTA within the pair
  const uint32_t pj = crank / CG;                   // pair (or CTA) index along N
  const bool leader = rank == 0;
  const uint16_t all_mask = (uint16_t)((1u << csize) - 1u);
  const uint16_t pair_mask = (uint16_t)(((1u << CG) - 1u) << (pj * CG));

  const long long t_entry = (kTrace && p.trace) ? clock64() : 0;
  if (kTrace && p.trace && warp == 0 && lane == 0 && leader)          // debug: kernel entry (item 0, slot 7)
    p.trace[((int64_t)(blockIdx.x / CG) * kTraceItems) * 8 + 7] = globaltimer();
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmC) : "memory");
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(full0 + 8u * s, 1);     // leader arms with both CTAs' bytes
      mbar_init(empty0 + 8u * s, (uint32_t)p.n1);   // one MMA commit from each pair reading this slot
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(tfull0 + 8u * b, 1);
      mbar_init(tempty0 + 8u * b, kEpiWarps * CG);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (kTrace && p.trace && leader) {                                 // debug: barriers initialised (item 2, slot 7)
      p.trace[((int64_t)(blockIdx.x / CG) * kTraceItems + 2) * 8 + 7] = globaltimer();
      trace_cycles(p.trace, blockIdx.x / CG, 0, t_entry);
    }
  }
  if (warp == 2) {
    if constexpr (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "r"(p.tmem_cols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "r"(p.tmem_cols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    if (kTrace && p.trace && leader && lane == 0) {                    // debug: TMEM allocated (item 3, slot 7)
      p.trace[((int64_t)(blockIdx.x / CG) * kTraceItems + 3) * 8 + 7] = globaltimer();
      trace_cycles(p.trace, blockIdx.x / CG, 1, t_entry);
    }
  }
  tc_fence_before();
  if (csize > 1) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (kTrace && p.trace && warp == 0 && lane == 0 && leader) {        // debug: prologue barrier passed (item 4, slot 7)
    p.trace[((int64_t)(blockIdx.x / CG) * kTraceItems + 4) * 8 + 7] = globaltimer();
    trace_cycles(p.trace, blockIdx.x / CG, 2, t_entry);
  }

  const int rows_cta = p.m2 * 128;
  const int cluster_id = blockIdx.x / csize;
  const int num_clusters = gridDim.x / csize;

  if (warp == 0) {
    // ===== TMA producer: the whole warp walks the ring, one elected lane issues =====
    int stage = 0;
    uint32_t phase = 0;
    constexpr int ELEM = KIND == 0 ? 2 : 4;
    const int kchunks = p.bk * ELEM / p.swz_a;
    const int bboxes = p.nb / p.b_cw;
    const uint32_t bbox_bytes = (uint32_t)(p.bk * p.swz_b);
    const int a_kstep = p.swz_a / ELEM;
    Sched sch(p, cluster_id, num_clusters);
    Item it;
    bool tp_first = true;
    while (sch.next(p, &it)) {
      const int tm = it.tile % p.m0, tn = it.tile / p.m0;
      const int row = tm * (CG * rows_cta) + (int)rank * rows_cta;
      const int colt = tn * (p.n1 * p.n2 * p.n3) + (int)pj * (p.n2 * p.n3) + (int)rank * p.nb;
      const uint16_t a_mask = (uint16_t)((1u << rank) | (1u << (rank + CG)));   // n1 = 2: both pairs
      for (int kb = it.kb0; kb < it.kb1; ++kb) {
        mbar_wait(empty0 + 8u * stage, phase ^ 1u);
        const uint32_t fb = full0 + 8u * stage;
        if (elect_one()) {
          if (kTrace && p.trace && leader && tp_first) {             // debug: first TMA issued (item 6, slot 7)
            p.trace[((int64_t)cluster_id * kTraceItems + 6) * 8 + 7] = globaltimer();
            trace_cycles(p.trace, cluster_id, 3, t_entry);
            tp_first = false;
          }
          if (leader) mbar_arrive_expect_tx(fb, p.tx_bytes * CG);
          const uint32_t sa = sbase + (uint32_t)stage * p.stage_bytes;
          const uint32_t sb = sa + p.a_stage_bytes;
          if (p.a_mn) {                                    // W rows: boxes of a_cw M-elements x BK
            for (int c = 0; c < rows_cta / p.a_cw; ++c) {
              const uint32_t dst = sa + (uint32_t)c * (uint32_t)(p.bk * 128);
              if (p.n1 == 1) tma_load_2d<CG>(&tmA, fb, dst, row + c * p.a_cw, kb * p.bk);
              else if ((c & 1) == (int)pj) tma_load_2d_mc<CG>(&tmA, fb, dst, row + c * p.a_cw, kb * p.bk, a_mask);
            }
          } else {
            for (int kc = 0; kc < kchunks; ++kc) {
              if (p.n1 == 1) {
                tma_load_2d<CG>(&tmA, fb, sa + kc * p.a_chunk_bytes, kb * p.bk + kc * a_kstep, row);
              } else {                                     // rows [pj h, pj h + h) of the slab, h = a_box_rows
                tma_load_2d_mc<CG>(&tmA, fb, sa + kc * p.a_chunk_bytes + (uint32_t)((int)pj * p.a_box_rows * p.swz_a),
                                   kb * p.bk + kc * a_kstep, row + (int)pj * p.a_box_rows, a_mask);
              }
            }
          }
          for (int ni = 0; ni < p.n2; ++ni)
            for (int c = 0; c < bboxes; ++c)
              tma_load_2d<CG>(&tmB, fb, sb + (uint32_t)(ni * bboxes + c) * bbox_bytes, colt + ni * p.n3 + c * p.b_cw,
                              kb * p.bk);
        }
        __syncwarp();
        if (++stage == p.stages) { stage = 0; phase ^= 1u; }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      // ===== MMA issuer: specialised on (k-steps per stage, M atoms, N atoms) so the per-stage
      // MMA sequence is fully unrolled with loop-invariant descriptor words (issue stays far
      // below the 64-128 cycles one MMA occupies the tensor pipe).
      const int code = (p.bk / UK) * 4 + (p.m2 - 1) * 2 + (p.n2 - 1);
      MmaCtx c{sbase, full0, empty0, tfull0, tempty0, tmem_base, cluster_id, num_clusters,
               (uint16_t)(csize > 1 ? all_mask : 0), (uint16_t)(CG == 2 ? pair_mask : 0), t_entry};
      switch (code) {
#define TT_MMA_CASE(KS, M2, N2) \
  case KS * 4 + (M2 - 1) * 2 + (N2 - 1): mma_role<KIND, CG, KS, M2, N2>(p, c); break;
#define TT_MMA_KS(KS) TT_MMA_CASE(KS, 1, 1) TT_MMA_CASE(KS, 1, 2) TT_MMA_CASE(KS, 2, 1) TT_MMA_CASE(KS, 2, 2)
        TT_MMA_KS(1) TT_MMA_KS(2) TT_MMA_KS(4) TT_MMA_KS(8) TT_MMA_KS(16)
#undef TT_MMA_KS
#undef TT_MMA_CASE
        case 32 * 4 + 0: if constexpr (KIND == 1) mma_role<KIND, CG, 32, 1, 1>(p, c); break;
        case 32 * 4 + 1: if constexpr (KIND == 1) mma_role<KIND, CG, 32, 1, 2>(p, c); break;
        case 32 * 4 + 2: if constexpr (KIND == 1) mma_role<KIND, CG, 32, 2, 1>(p, c); break;
        case 32 * 4 + 3: if constexpr (KIND == 1) mma_role<KIND, CG, 32, 2, 2>(p, c); break;
        default: __trap();
      }
    }
  } else if (warp >= 4) {
    // ===== epilogue: TMEM -> registers -> swizzled smem box -> TMA bulk store =====
    // Warp w reads TMEM lanes [32q, 32q+32) (q = w mod 4, 32 output rows) and takes the
    // 32-column chunks of the tile with index = h mod kEpiGroups.  Each warp stages through its own
    // 4 KB boxes (32 rows x 32 fp32, 128B-swizzled like the C tensor map); one lane issues the
    // cp.async.bulk.tensor store, so C leaves the SM as full 128 B lines.
    const int q = warp & 3;
    const int h = (warp - 4) >> 2;
    const uint32_t stage0 = epi_base + (uint32_t)((warp - 4) * p.epi_bufs * kEpiBoxBytes);
    int acc = 0;
    uint32_t aphase = 0;
    int sbuf = 0;
    float v[32];
    Sched sch(p, cluster_id, num_clusters);
    Item it;
    int item_no = 0;
    while (sch.next(p, &it)) {
      uint64_t* tr = (kTrace && p.trace && warp == 4 && lane == 0 && leader && item_no < kTraceItems)
                         ? p.trace + ((int64_t)cluster_id * kTraceItems + item_no) * 8 : nullptr;
      ++item_no;
      const int tm = it.tile % p.m0, tn = it.tile / p.m0;
      uint32_t* flag = it.split ? g_split_flags + (size_t)p.flag_group * kFlagWords + (it.tile - p.dp_tiles) * csize + crank
                                : nullptr;
      const bool add = it.split && it.order > 0;           // higher k-blocks: add onto C
      mbar_wait(tfull0 + 8u * acc, aphase);
      tc_fence_after();
      if (kTrace && tr) {
        tr[0] = (uint64_t)it.tile;
        tr[1] = (uint64_t)it.kb0 | ((uint64_t)it.kb1 << 16) | ((uint64_t)it.order << 32);
        tr[4] = globaltimer();
      }
      if (add) {
        wait_flag(flag, (uint32_t)kEpiWarps * (uint32_t)it.order);   // every epilogue warp of each piece below
        fence_proxy_async_global();
      }
      if (kTrace && tr) tr[5] = globaltimer();
      const int row_cta = tm * (CG * rows_cta) + (int)rank * rows_cta;
      int chunk = 0;                                       // running chunk index over the tile
      for (int mi = 0; mi < p.m2; ++mi) {
        const int row0 = row_cta + mi * 128 + q * 32;
        for (int ni = 0; ni < p.n2; ++ni) {
          const uint32_t tcol = (uint32_t)(acc * p.acc_cols + (mi * p.n2 + ni) * p.n3);
          const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + tcol;
          const int col0 = tn * (p.n1 * p.n2 * p.n3) + (int)pj * (p.n2 * p.n3) + ni * p.n3;
          int c0 = 0;
          for (; c0 + 32 <= p.n3; c0 += 32, ++chunk) {
            if (chunk % kEpiGroups != h) continue;
            tmem_ld32(taddr + (uint32_t)c0, v);
            const uint32_t buf = stage0 + (uint32_t)(sbuf * kEpiBoxBytes);
            if (lane == 0) bulk_wait_read_n(p.epi_bufs - 1);  // the store that used `buf` has read it
            __syncwarp();
            const uint32_t rowp = buf + (uint32_t)lane * 128u;
#pragma unroll
            for (int j = 0; j < 8; ++j)
              st_shared_v4(rowp + (uint32_t)((j ^ (lane & 7)) << 4), v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) {
              if (add) tma_reduce_add_2d(&tmC, buf, col0 + c0, row0);
              else tma_store_2d(&tmC, buf, col0 + c0, row0);
              bulk_commit();
            }
            if (++sbuf == p.epi_bufs) sbuf = 0;
          }
          if (c0 < p.n3) {                                 // n3 = 16: direct 16-column stores
            if (chunk++ % kEpiGroups == h) {
              tmem_ld16(taddr + (uint32_t)c0, v);
              float4* dst = reinterpret_cast<float4*>(C + (int64_t)(row0 + lane) * p.N + col0 + c0);
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                float4 o = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
                if (add) {
                  const float4 c = dst[j];
                  o.x += c.x; o.y += c.y; o.z += c.z; o.w += c.w;
                }
                dst[j] = o;
              }
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {                                     // TMEM drained: MMA may reuse `acc`
        if (CG == 1 || leader) mbar_arrive(tempty0 + 8u * acc);
        else mbar_arrive_cluster(tempty0 + 8u * acc, pj * CG);
      }
      if (it.split) {                                      // publish this piece
        if (lane == 0) {
          bulk_wait_all();
          fence_proxy_async_global();
        }
        __threadfence();
        __syncwarp();
        if (lane == 0) {
          const uint32_t old = atom_add_release(flag, 1u);
          if (it.kb1 == p.k0 && old == (uint32_t)kEpiWarps * ((uint32_t)it.order + 1u) - 1u) *flag = 0u;   // top piece lands last: reset
        }
      }
      if (kTrace && tr) {
        bulk_wait_all();
        tr[6] = globaltimer();
        if (item_no == 1) trace_cycles(p.trace, cluster_id, 6, t_entry);
      }
      if (++acc == p.acc_bufs) { acc = 0; aphase ^= 1u; }
    }
    if (lane == 0) bulk_wait_all();                         // stores done before smem is released
    __syncwarp();
  }

  __syncwarp();                                            // reconverge role warps
  tc_fence_before();
  if (csize > 1) cluster_sync(); else __syncthreads();
  tc_fence_after();
  if (kTrace && p.trace && warp == 0 && lane == 0 && leader) {        // debug: teardown reached (item 1, slot 7)
    p.trace[((int64_t)(blockIdx.x / CG) * kTraceItems + 1) * 8 + 7] = globaltimer();
    trace_cycles(p.trace, blockIdx.x / CG, 7, t_entry);
  }
  if (warp == 2) {
    if constexpr (CG == 1)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(p.tmem_cols));
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(p.tmem_cols));
  }
}

// ---------------------------------------------------------------- host side
PFN_cuTensorMapEncodeTiled_v12000 encode_fn(std::string* err) {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  if (!fn) *err = "cuTensorMapEncodeTiled unavailable";
  return fn;
}

CUtensorMapSwizzle swz_enum(int s) {
  if (s == 0) return CU_TENSOR_MAP_SWIZZLE_NONE;
  if (s == -128) return CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B;   // 128B swizzle, 32B atoms (tf32 MN-major)
  return s == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : (s == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
}

bool make_map(CUtensorMap* m, int kind, const void* ptr, uint64_t inner, uint64_t outer, uint32_t box_in,
              uint32_t box_out, int swz, std::string* err) {
  auto fn = encode_fn(err);
  if (!fn) return false;
  const int elem = kind == 0 ? 2 : 4;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * (uint64_t)elem};
  cuuint32_t box[2] = {box_in, box_out};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, kind == 0 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                  const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz_enum(swz),
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    *err = "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")";
    return false;
  }
  return true;
}

int num_sms() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  return n > 0 ? n : 148;
}

// Tail split policy: at most kMaxPieces clusters share one tile, so the
// ascending-k chain of TMA reduce-adds per tile stays short.  TT_TAIL_SPLIT = 0 disables it,
// 2 forces it wherever tiles % clusters != 0 (tests), unset / 1 = the measured policy in plan_of.
// Read at every plan so a process can A/B both schedules.
constexpr int kMaxPieces = 4;

int tail_split_mode() {
  const char* e = std::getenv("TT_TAIL_SPLIT");
  if (!e || !e[0]) return 1;
  return (e[0] >= '0' && e[0] <= '4') ? e[0] - '0' : 1;
}

template <int KIND, int CG>
bool set_smem_attr(std::string* err) {
  return ensure_max_smem((const void*)&k_umma<KIND, CG>, kSmemPerCta, err);
}

template <int KIND, int CG>
int query_clusters(int smem, int csize) {
  std::string err;
  if (!set_smem_attr<KIND, CG>(&err)) return 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(num_sms() / csize * csize), 1, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = (size_t)smem;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = csize;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, (const void*)&k_umma<KIND, CG>, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

// Co-resident clusters of one CTA (1 CTA per SM: launch bounds, TMEM and smem); without a
// device (build host) the SM count.
int max_active_clusters(int kind, int cg, int csize, int smem) {
  static std::mutex mu;
  static std::map<std::tuple<int, int, int, int, int>, int> cache;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    return num_sms() / csize;
  }
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_tuple(dev, kind, cg, csize, smem);
  auto itc = cache.find(key);
  if (itc != cache.end()) return itc->second;
  int n = kind == 0 ? (cg == 1 ? query_clusters<0, 1>(smem, csize) : query_clusters<0, 2>(smem, csize))
                    : (cg == 1 ? query_clusters<1, 1>(smem, csize) : query_clusters<1, 2>(smem, csize));
  if (n <= 0) n = num_sms() / csize;
  n = std::min(n, num_sms() / csize);
  cache[key] = n;
  return n;
}

// Flag group of a launch stream (g_split_flags): streams are numbered round-robin on first use,
// per device.  Two split launches that may run concurrently must be on different streams (more
// than kFlagGroups live streams wrap around); a CUDA graph keeps the group of its capture stream,
// so replays of one graph must not overlap each other on several streams.
int split_flag_group(cudaStream_t stream) {
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, int> groups;
  static std::map<int, int> next;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  auto it = groups.find({dev, stream});
  if (it != groups.end()) return it->second;
  const int g = next[dev]++ % kFlagGroups;
  groups[{dev, stream}] = g;
  return g;
}

struct Plan {
  UmmaArgs a;
  int cg, csize, kind;    // cta_group, CTAs per cluster (cta_group x n1)
  int grid;
  int smem;
};

void plan_of(const Space& sp, const State& s, Plan* pl) {
  const int fam = sp.family;
  const int kind = fam == TT_FAM_BF16_UMMA ? 0 : 1;
  const int elem = kind == 0 ? 2 : 4;
  UmmaArgs& a = pl->a;
  std::memset(&a, 0, sizeof(a));
  a.M = sp.dim[0];
  a.K = sp.dim[1];
  a.N = sp.dim[2];
  const int m1 = (int)s.f[0][1];
  a.m0 = (int)s.f[0][0];
  a.m2 = (int)s.f[0][2];
  a.k0 = (int)s.f[1][0];
  a.bk = (int)s.f[1][1];
  a.n0 = (int)s.f[2][0];
  a.n1 = (int)s.f[2][1];
  a.n2 = (int)s.f[2][2];
  a.n3 = (int)s.f[2][3];
  a.nb = a.n3 / m1;
  a.swz_a = std::min(a.bk * elem, 128);
  a.swz_b = std::min(a.nb * elem, 128);
  a.b_cw = a.swz_b / elem;
  auto code = [](int swz) { return swz == 128 ? 2 : (swz == 64 ? 4 : 6); };
  a.a_layout = code(a.swz_a);
  if (kind == 1) {
    // MN-major tf32: 128B swizzle with 32B atoms (4 K-rows per core-matrix group)
    a.b_layout = 1;
    a.sbo_b = 4 * 128;
  } else {
    a.b_layout = code(a.swz_b);
    a.sbo_b = 8 * a.swz_b;
  }
  a.a_chunk_bytes = a.m2 * 128 * a.swz_a;
  a.a_box_rows = a.m2 * 128 / a.n1;
  a.a_stage_bytes = a.m2 * 128 * a.bk * elem;
  a.stage_bytes = (int)umma_stage_bytes(fam, s);
  a.tx_bytes = (uint32_t)(a.a_stage_bytes + a.n2 * a.nb * a.bk * elem);
  a.stages = std::min<int>(kUmmaMaxStages, kUmmaPipeSmem / a.stage_bytes);
  // leftover pipeline shared memory goes to the epilogue staging
  {
    const int spare = kUmmaPipeSmem - a.stages * a.stage_bytes;
    a.epi_bufs = std::min(kEpiMaxBufs, kEpiBytes / (kEpiWarps * kEpiBoxBytes) + std::max(0, spare) / (kEpiWarps * kEpiBoxBytes));
  }
  a.acc_cols = a.m2 * a.n2 * a.n3;
  a.acc_bufs = a.acc_cols <= 256 ? 2 : 1;
  int need = a.acc_cols * a.acc_bufs, cols = 32;
  while (cols < need) cols <<= 1;
  a.tmem_cols = cols;
  // instruction descriptor: F32 accum, A/B format, A K-major, B MN-major, N>>3, M>>4
  const uint32_t fmt = kind == 0 ? 1u : 2u;
  const uint32_t M_inst = 128u * (uint32_t)m1;
  a.a_mn = sp.layout == TT_LAYOUT_TN ? 1 : 0;
  a.a_cw = 128 / elem;
  if (a.a_mn) a.a_layout = kind == 1 ? 1 : 2;          // MN-major A: SW128 (tf32: 32B atoms)
  a.idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)a.a_mn << 15) | (1u << 16) | (((uint32_t)a.n3 >> 3) << 17) |
            ((M_inst >> 4) << 24);
  pl->cg = m1;
  pl->csize = m1 * a.n1;
  pl->kind = kind;
  pl->smem = a.stages * a.stage_bytes + kEpiWarps * a.epi_bufs * kEpiBoxBytes + 1024 /*align*/ + 8 * (2 * a.stages + 4) + 16;
  // persistent grid: as many clusters as can be co-resident (the tail split's cross-cluster
  // waits rely on it), never more than there are tiles unless the tail is split
  const int tiles = a.m0 * a.n0;
  const int P = max_active_clusters(kind, m1, pl->csize, pl->smem);
  a.dp_tiles = tiles;
  // Split only where it measured a win (profiles/r3_tail_split.md): at least one full
  // data-parallel wave behind which the pieces' extra epilogues (store, then reduce-add chain)
  // can hide, a double-buffered accumulator (with one buffer the next item's MMAs wait for the
  // previous piece's whole epilogue), and an estimated saving of >= 8 us (the idle fraction of
  // the last wave x one tile's MMA time at ~8192 (bf16) / 4096 (tf32) flop/clk/SM, 1.9 GHz).
  const int rem = tiles % P;
  const double tile_us = 2.0 * (128.0 * m1 * a.m2) * (double)(a.n1 * a.n2 * a.n3) * (double)a.K /
                         ((kind == 0 ? 8192.0 : 4096.0) * pl->csize * 1.9e3);
  const double gain_us = (1.0 - (double)rem / P) * tile_us;
  const int mode = tail_split_mode();
  // the device schedule computes k-block offsets in 32 bits (Sched)
  const bool fits32 = (uint64_t)P * (uint64_t)tiles * (uint64_t)a.k0 < (1ull << 32);
  const bool worth = tiles - rem >= P && a.acc_bufs == 2 && gain_us >= 8.0;
  if (!fits32) {
    pl->grid = std::min(tiles, P) * pl->csize;
  } else if (mode == 3 && a.k0 >= 2 && tiles * pl->csize <= kFlagWords) {
    // experiment: stream-K over every tile (each cluster gets tiles k0 / P k-blocks)
    a.sk_tiles = tiles;
    a.dp_tiles = 0;
    a.sk_workers = P;
    pl->grid = P * pl->csize;
  } else if (mode == 4 && rem != 0 && a.k0 >= 2 && tiles >= rem + P && (rem + P) * pl->csize <= kFlagWords) {
    // experiment: data-parallel waves, then the last full wave plus the remainder by stream-K
    a.sk_tiles = rem + P;
    a.dp_tiles = tiles - a.sk_tiles;
    a.sk_workers = P;
    pl->grid = P * pl->csize;
  } else if (mode != 0 && mode < 3 && rem != 0 && a.k0 >= 2 && (mode == 2 || worth)) {
    if (mode == 1 && tiles >= rem + P && (rem + P) * pl->csize <= kFlagWords) {
      // measured default (round 2): the last full data-parallel wave joins the remainder and
      // their k-blocks are spread evenly over all P clusters (stream-K over rem + P tiles): every
      // cluster ends within a fraction of a tile.  bf16 4096^3 bench config 1418 -> 1440 TF/s,
      // 3 interleaved runs each (profiles/r11_split_modes.txt).
      a.sk_tiles = rem + P;
      a.dp_tiles = tiles - a.sk_tiles;
      a.sk_workers = P;
    } else {
      a.sk_tiles = tiles % P;                            // == tiles when tiles < P
      a.dp_tiles = tiles - a.sk_tiles;
      a.sk_workers = std::min(P, a.sk_tiles * kMaxPieces);
    }
    pl->grid = P * pl->csize;
  } else {
    pl->grid = std::min(tiles, P) * pl->csize;
  }
}

template <int KIND, int CG>
tt_status launch_t(const Plan& pl, const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mc, float* C,
                   cudaStream_t stream,
                   std::string* err) {
  auto fn = &k_umma<KIND, CG>;
  if (!set_smem_attr<KIND, CG>(err)) return TT_E_CUDA;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)pl.grid, 1, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = (size_t)pl.smem;
  cfg.stream = stream;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = pl.csize;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  UmmaArgs a = pl.a;
  if (a.sk_tiles) {
    if (a.sk_tiles * pl.csize > kFlagWords) {
      *err = "tail split wider than the flag array";
      return TT_E_UNSUPPORTED;
    }
    a.flag_group = split_flag_group(stream);
  }
  static const char* trace_path = kTrace ? std::getenv("TT_UMMA_TRACE") : nullptr;   // trace build only
  const size_t trace_words = (size_t)(pl.grid / CG) * kTraceItems * 8;
  if (trace_path) {
    if (!cuda_ok(cudaMalloc(&a.trace, trace_words * 8), err, "cudaMalloc(trace)")) return TT_E_CUDA;
    cudaMemsetAsync(a.trace, 0, trace_words * 8, stream);
  }
  if (!cuda_ok(cudaLaunchKernelEx(&cfg, fn, ma, mb, mc, C, a), err, "k_umma launch")) return TT_E_CUDA;
  if (trace_path) {                                         // debug only: synchronous dump
    std::vector<uint64_t> h(trace_words);
    if (!cuda_ok(cudaStreamSynchronize(stream), err, "trace sync")) return TT_E_CUDA;
    cudaMemcpy(h.data(), a.trace, trace_words * 8, cudaMemcpyDeviceToHost);
    cudaFree(a.trace);
    if (FILE* f = std::fopen(trace_path, "ab")) {
      const uint64_t hdr[4] = {(uint64_t)(pl.grid / CG), (uint64_t)kTraceItems, (uint64_t)a.dp_tiles, (uint64_t)a.sk_tiles};
      std::fwrite(hdr, 8, 4, f);
      std::fwrite(h.data(), 8, h.size(), f);
      std::fclose(f);
    }
  }
  return TT_OK;
}

}  // namespace

tt_status umma_bind(const Space& sp, const State& s, tt_launch_info* info, std::string* err) {
  Plan pl;
  plan_of(sp, s, &pl);
  *info = tt_launch_info{};
  info->family = sp.family;
  info->grid_x = pl.grid;
  info->grid_y = 1;
  info->grid_z = 1;
  info->block_x = kThreads;
  info->cluster_x = pl.csize;
  info->smem_bytes = pl.smem;
  info->stages = pl.a.stages;
  info->tile_m = pl.cg * pl.a.m2 * 128;
  info->tile_n = pl.a.n1 * pl.a.n2 * pl.a.n3;
  info->tile_k = pl.a.bk;
  info->tmem_cols = pl.a.tmem_cols;
  info->acc_buffers = pl.a.acc_bufs;
  info->idesc = pl.a.idesc;
  info->split_tiles = pl.a.sk_tiles;
  info->split_workers = pl.a.sk_workers;
  (void)err;
  return TT_OK;
}

// Work items of every cluster of a config's tcgen05 launch, in the order the kernel's roles walk
// them: the same Sched code the kernel runs, evaluated on the host (tt_umma_schedule; CPU tests
// check coverage and the lower-index-only wait order of the split pieces).
tt_status umma_schedule(const Space& sp, const State& s, std::vector<std::vector<int32_t>>* per_worker,
                        int32_t* k0, std::string* err) {
  Plan pl;
  plan_of(sp, s, &pl);
  const int P = pl.grid / pl.csize;
  per_worker->assign(P, {});
  for (int w = 0; w < P; ++w) {
    Sched sch(pl.a, w, P);
    Item it;
    while (sch.next(pl.a, &it)) {
      auto& v = (*per_worker)[w];
      v.insert(v.end(), {it.tile, it.kb0, it.kb1, it.order, it.split ? 1 : 0});
    }
  }
  *k0 = pl.a.k0;
  (void)err;
  return TT_OK;
}

namespace {

// Host launch path cache: plan + three tensor maps per (device, problem, config, pointers,
// tail-split mode).  Encoding three tensor maps costs microseconds of host time per launch,
// as long as a small GEMM runs on the device; repeated launches of one config (the evaluator,
// a training loop) reuse them.  Bounded: cleared when it reaches kLaunchCacheMax entries.
struct LaunchKey {
  int dev, family, layout, split_mode;
  int64_t dims[3];
  int64_t f[3][TT_MAXD];
  const void *A, *B;
  float* C;
  bool operator<(const LaunchKey& o) const { return std::memcmp(this, &o, sizeof(LaunchKey)) < 0; }
};
struct LaunchEntry {
  Plan pl;
  CUtensorMap ma, mb, mc;
};
constexpr size_t kLaunchCacheMax = 512;

tt_status prepare(const Space& sp, const State& s, const void* A, const void* B, float* C, LaunchEntry* e,
                  std::string* err) {
  Plan& pl = e->pl;
  plan_of(sp, s, &pl);
  if (((uintptr_t)A % 16) || ((uintptr_t)B % 16) || ((uintptr_t)C % 16)) {
    *err = "UMMA family needs 16-byte aligned A, B, C";
    return TT_E_INVAL;
  }
  const int elem = pl.kind == 0 ? 2 : 4;
  if ((pl.a.K * elem) % 16 || (pl.a.N * elem) % 16 || (pl.a.a_mn && (pl.a.M * elem) % 16)) {
    *err = "UMMA family needs row pitches that are multiples of 16 bytes";
    return TT_E_UNSUPPORTED;
  }
  if (pl.a.a_mn) {
    if (!make_map(&e->ma, pl.kind, A, (uint64_t)pl.a.M, (uint64_t)pl.a.K, (uint32_t)pl.a.a_cw, (uint32_t)pl.a.bk,
                  pl.kind == 1 ? -128 : 128, err))
      return TT_E_CUDA;
  } else if (!make_map(&e->ma, pl.kind, A, (uint64_t)pl.a.K, (uint64_t)pl.a.M, (uint32_t)(pl.a.swz_a / elem),
                       (uint32_t)pl.a.a_box_rows, pl.a.swz_a, err)) {
    return TT_E_CUDA;
  }
  if (!make_map(&e->mb, pl.kind, B, (uint64_t)pl.a.N, (uint64_t)pl.a.K, (uint32_t)pl.a.b_cw, (uint32_t)pl.a.bk,
                pl.a.b_layout == 1 ? -128 : pl.a.swz_b, err))
    return TT_E_CUDA;
  // C: fp32 [M][N], 32 x 32 boxes, 128B swizzle (matches the epilogue staging layout)
  if (!make_map(&e->mc, 1, C, (uint64_t)pl.a.N, (uint64_t)pl.a.M, 32u, 32u, 128, err)) return TT_E_CUDA;
  return TT_OK;
}

}  // namespace

namespace {
// Plan + tensor maps of (problem, config, pointers) from the launch cache (inserted on a miss).
tt_status cached_entry(const Space& sp, const State& s, const void* A, const void* B, float* C, LaunchEntry* e,
                       std::string* err) {
  static std::mutex mu;
  static std::map<LaunchKey, LaunchEntry> cache;
  LaunchKey k;
  std::memset(&k, 0, sizeof(k));                          // padding bytes take part in the compare
  cudaGetDevice(&k.dev);
  k.family = sp.family;
  k.layout = sp.layout;
  k.split_mode = tail_split_mode();
  for (int a = 0; a < 3; ++a) {
    k.dims[a] = sp.dim[a];
    for (int i = 0; i < TT_MAXD; ++i) k.f[a][i] = s.f[a][i];
  }
  k.A = A;
  k.B = B;
  k.C = C;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(k);
    if (it != cache.end()) {
      *e = it->second;
      return TT_OK;
    }
  }
  tt_status st = prepare(sp, s, A, B, C, e, err);
  if (st != TT_OK) return st;
  std::lock_guard<std::mutex> lk(mu);
  if (cache.size() >= kLaunchCacheMax) cache.clear();
  cache.emplace(k, *e);
  return TT_OK;
}
}  // namespace

tt_status umma_preload(int family, std::string* err) {
  const bool ok = family == TT_FAM_BF16_UMMA ? (set_smem_attr<0, 1>(err) && set_smem_attr<0, 2>(err))
                                             : (set_smem_attr<1, 1>(err) && set_smem_attr<1, 2>(err));
  return ok ? TT_OK : TT_E_CUDA;
}

tt_status umma_prepare(const Space& sp, const State& s, const void* A, const void* B, float* C, std::string* err) {
  LaunchEntry e;
  tt_status st = cached_entry(sp, s, A, B, C, &e, err);
  if (st != TT_OK) return st;
  const bool ok = e.pl.kind == 0 ? (e.pl.cg == 1 ? set_smem_attr<0, 1>(err) : set_smem_attr<0, 2>(err))
                                 : (e.pl.cg == 1 ? set_smem_attr<1, 1>(err) : set_smem_attr<1, 2>(err));
  return ok ? TT_OK : TT_E_CUDA;
}

tt_status umma_launch(const Space& sp, const State& s, const void* A, const void* B, float* C, cudaStream_t stream,
                      std::string* err) {
  LaunchEntry e;
  tt_status st = cached_entry(sp, s, A, B, C, &e, err);
  if (st != TT_OK) return st;
  const Plan& pl = e.pl;
  if (pl.kind == 0) {
    return pl.cg == 1 ? launch_t<0, 1>(pl, e.ma, e.mb, e.mc, C, stream, err)
                      : launch_t<0, 2>(pl, e.ma, e.mb, e.mc, C, stream, err);
  }
  return pl.cg == 1 ? launch_t<1, 1>(pl, e.ma, e.mb, e.mc, C, stream, err)
                    : launch_t<1, 2>(pl, e.ma, e.mb, e.mc, C, stream, err);
}


// 2-D fp32 tensor map without swizzle (K1's TMA-fed B slabs, gemm_simt.cu): dims {inner, outer},
// row pitch inner x 4 bytes, box {box_in, box_out}.
bool encode_map_2d_f32(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint32_t box_in,
                       uint32_t box_out, std::string* err) {
  return make_map(m, 1, ptr, inner, outer, box_in, box_out, 0, err);
}

}  // namespace tt
