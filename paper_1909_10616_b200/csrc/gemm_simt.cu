// K1: fp32 CUDA-core tiled GEMM family, parameterised by the paper's per-axis split factors.
//
// PAPER.md P:124-125 ("iteratively splitting computation into smaller tiles ... A resulted
// matrix is initialized with zeros ... accumulates"), P:166 (m_i, k_l, n_j are loop trip
// counts), P:369 (d_m = 4, d_k = 2, d_n = 4).  Level mapping (reading Z2):
//   m = [m0 CTAs along M (grid.y), m1 thread groups per CTA along M, m2 lanes per group along
//        M, m3 register rows per thread]
//   n = [n0 CTAs along N (grid.x), n1 groups along N, n2 lanes along N, n3 register columns]
//   k = [k0 main-loop trips, k1 = BK (shared-memory K slab)]
// so the CTA tile is BM x BN = (m1 m2 m3) x (n1 n2 n3) and a thread owns an m3 x n3 register
// tile.  Each output element is one fmaf chain in ascending k (no split-K, no k-interleaved
// partial sums): the result is bit-identical to the oracle's sequential fmaf reference.
//
// B200 mapping: slabs are double buffered (2 stages) so the next slab's copy overlaps the FFMA
// work on the current one.  B slabs arrive by TMA (one thread issues a 2-D bulk tensor copy of
// the dense [BK][BN] box per slab, completing on the slot's mbarrier) when the shape allows it,
// else by cp.async (LDGSTS); A is staged by cp.async and transposed on the way in (As[k][m], rows
// padded by 4 floats so the strided LDGSTS stores are bank-conflict free for BK = 8 warps);
// register tiles are read with LDS.128 when m3/n3 are multiples of 4 and results are stored with
// STG.128.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>

#include "device.hpp"

namespace tt {

namespace {

struct SimtArgs {
  // B slabs by TMA (b_tma = 1): one thread issues one 2-D bulk tensor copy per slab into a dense
  // [BK][BN] box and the CTA waits on that slot's mbarrier; the compute warps issue no B copies
  // (those held 3.7 % / 5.7 % of the time at 2048^3 / 4096^3, profiles/r12_simt_nocopy_ab.txt).
  CUtensorMap tmB;
  int b_tma;
  const float* A;
  const float* B;
  float* C;
  int64_t M, N, K;
  int m1, m2, n1, n2, bk, k0;
  int bk_sh;  // log2(BK) if BK is a power of two, else -1
  int bq_sh;  // log2(BN / 4) if a power of two, else -1
  int stages; // shared-memory slots (2 or 3)
  int a_tn;   // A stored as W = A^T row-major [K][M] (the paper's Y = W^T X)
  int a_vec16;  // TN: 16-byte cp.async of W rows legal
  int c_vec;    // C rows 16-byte aligned (STG.128 legal)
  int b_vec;  // B rows 16-byte aligned (16-byte cp.async legal)
};

// Slab copies carry an L2 256-byte prefetch hint (whole lines on a cold miss after the bench's L2
// flush): measured +0.35 % at 4096^3, neutral at 512^3-2048^3 (profiles/r11_simt_l2pf_ab.txt).
__device__ __forceinline__ void cp_async4(float* dst, const float* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global.L2::256B [%0], [%1], 4;\n" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(float* dst, const float* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global.L2::256B [%0], [%1], 16;\n" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

constexpr int max_threads(int acc) { return acc <= 16 ? 1024 : (acc <= 64 ? 512 : 256); }

// Fragment of one k step.  A register tile of TM (TN) values is read as float4 chunks: chunk c of
// the thread's rows sits at as[c * SA + 0..3] (columns: bs[c * SB + 0..3]).  SA = SB = 4 is the
// contiguous tile; the interleaved layout (kernel below) spreads a thread's chunks one warp-row
// apart so that the lanes of a warp read adjacent 16-byte words (no shared-memory bank conflicts).
template <int TM, int TN, bool VECA>
__device__ __forceinline__ void load_frag(const float* as, const float* bs, int kk, int LDA, int LDB, int SA, int SB,
                                          float* a, float* b) {
  if constexpr (VECA) {
#pragma unroll
    for (int i = 0; i < TM; i += 4) {
      const float4 v = *reinterpret_cast<const float4*>(as + kk * LDA + (i >> 2) * SA);
      a[i] = v.x; a[i + 1] = v.y; a[i + 2] = v.z; a[i + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < TM; ++i) a[i] = as[kk * LDA + (i >> 2) * SA + (i & 3)];   // SA = 4: as[kk LDA + i]
  }
  if constexpr (TN % 4 == 0) {
#pragma unroll
    for (int j = 0; j < TN; j += 4) {
      const float4 v = *reinterpret_cast<const float4*>(bs + kk * LDB + (j >> 2) * SB);
      b[j] = v.x; b[j + 1] = v.y; b[j + 2] = v.z; b[j + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < TN; ++j) b[j] = bs[kk * LDB + (j >> 2) * SB + (j & 3)];
  }
}

// acc[i][j] = fma(a[i], b[j], acc[i][j]) for one k step.  With PAIR the update runs as FFMA2
// (two independent fused multiply-adds per instruction, each rounded once), so every output is
// still exactly the fmaf chain in ascending k.
template <int TM, int TN, bool PAIR>
__device__ __forceinline__ void fma_frag(const float* a, const float* b, float (&acc)[TM][TN],
                                         float2 (&acc2)[TM][PAIR ? TN / 2 : 1]) {
  if constexpr (PAIR) {
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const float2 ai = make_float2(a[i], a[i]);
#pragma unroll
      for (int j = 0; j < TN / 2; ++j) acc2[i][j] = __ffma2_rn(ai, make_float2(b[2 * j], b[2 * j + 1]), acc2[i][j]);
    }
  } else {
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
  }
}

// BKF > 0: the K slab is a compile-time constant, so the k-step loop unrolls completely and the
// compiler hoists the shared-memory fragment loads as far ahead as registers allow (small register
// tiles otherwise expose the LDS latency).  BKF = 0: the generic instance.
template <int TM, int TN, int BKF = 0, int LB = max_threads(TM * TN)>
__global__ void __launch_bounds__(LB)
k1_simt(const __grid_constant__ SimtArgs p) {
  extern __shared__ __align__(128) float smem[];
  const int BM = p.m1 * p.m2 * TM;
  const int BN = p.n1 * p.n2 * TN;
  const int BK = BKF > 0 ? BKF : p.bk;
  const int LDA = BM + 4, LDB = p.b_tma ? BN : BN + 4;   // TMA boxes are dense
  const int NS = p.stages;               // 2 or 3 smem slots (binder: 3 when occupancy allows)
  float* Bs = smem;                      // [NS][BK][LDB]
  float* As = smem + NS * BK * LDB;      // [NS][BK][LDA]
  // one mbarrier per slot for the TMA-fed B slabs, after the A slots (fits: the dense B rows free
  // 16 bytes per k-row of every slot, and the binder's smem counts padded rows)
  const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(As + NS * BK * LDA);
  if (p.b_tma) {
    if (threadIdx.x == 0) {
      for (int s2 = 0; s2 < NS; ++s2)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0 + 8u * s2) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
  }

  const int T = blockDim.x;
  const int t = threadIdx.x;
  const int G = p.m2 * p.n2;
  const int g = t / G, l = t - (t / G) * G;
  const int gm = g / p.n1, gn = g - (g / p.n1) * p.n1;
  const int lm = l / p.n2, ln = l - (l / p.n2) * p.n2;
  // Rows / columns of the thread's register tile.  Contiguous: rows row0 .. row0 + TM.  Interleaved
  // (TM or TN a multiple of 4 and >= 8): float4 chunk c at row0 + c * SA with row0 = 4 x (thread's
  // index along M) and SA = 4 x (threads along M) -- the same m1 m2 m3 x n1 n2 n3 tile and the same
  // fmaf chain per output, only the assignment of the tile's rows / columns to threads changes.
  // The interleaved layout removes the 2-way shared-memory bank conflicts of the 16 x 8 tiles
  // (profiles/r10_ncu_k1_simt_4096.md: 98.7 M per launch) but measured 6 % slower at 4096^3 and 4 %
  // at 2048^3 (profiles/r10_simt_ilv_ab.txt), so it is an experiment build (-DTT_SIMT_ILV) only.
#ifdef TT_SIMT_ILV
  constexpr bool kIlvA = (TM % 4 == 0) && TM >= 8;
  constexpr bool kIlvB = (TN % 4 == 0) && TN >= 8;
#else
  constexpr bool kIlvA = false, kIlvB = false;
#endif
  const int row0 = kIlvA ? (gm * p.m2 + lm) * 4 : gm * (p.m2 * TM) + lm * TM;
  const int col0 = kIlvB ? (gn * p.n2 + ln) * 4 : gn * (p.n2 * TN) + ln * TN;
  const int SA = kIlvA ? p.m1 * p.m2 * 4 : 4;
  const int SB = kIlvB ? p.n1 * p.n2 * 4 : 4;

  const int64_t K = p.K, N = p.N;
  const float* Ab = p.a_tn ? p.A + (int64_t)blockIdx.y * BM : p.A + (int64_t)blockIdx.y * BM * K;
  const int64_t M = p.M;
  const float* Bb = p.B + (int64_t)blockIdx.x * BN;

  // Strength-reduced slab copies: with power-of-two BK (A) / BN/4 (B) dividing the thread count,
  // a thread's k (A) or column (B) offset is the same in every iteration and its row advances by
  // a fixed step, so each cp.async costs two pointer increments instead of a divide / multiply
  // chain (the copy phase held 16 % of the stall samples at 2048^3, profiles/r11_ncu_k1_simt_2048.md).
  // Only the 128-accumulator tiles use it: they are register-bound at one occupancy level anyway,
  // while the smaller tiles' extra live registers cost them occupancy (measured -7 .. -23 % at
  // 512^3 / 1024^3, +1.4 % / +3.2 % at 2048^3 / 4096^3; profiles/r11_simt_copy_ab.txt).
  constexpr bool kFastCopy = TM * TN >= 128;
  const bool a_fast = kFastCopy && !p.a_tn && p.bk_sh >= 0 && (T & (BK - 1)) == 0 && BM % (T >> p.bk_sh) == 0;
  const int a_rstep = a_fast ? (T >> p.bk_sh) : 1;
  const int a_c = t & (BK - 1), a_r0 = a_fast ? (t >> p.bk_sh) : 0;
  const int q4 = BN >> 2;
  const bool b_fast = kFastCopy && p.b_vec && p.bq_sh >= 0 && (T & (q4 - 1)) == 0 && BK % (T >> p.bq_sh) == 0;
  const int b_rstep = b_fast ? (T >> p.bq_sh) : 1;
  const int b_c = (t & (q4 - 1)) << 2, b_r0 = b_fast ? (t >> p.bq_sh) : 0;

  auto load = [&](int kt, int buf) {
#ifdef TT_SIMT_EXP_NOCOPY
    // experiment build only (tools/ab_simt.sh): no slab copies -- the k-loop runs on whatever the
    // shared memory holds, to measure what the copy phase costs; results are meaningless
    return;
#endif
    float* as = As + buf * BK * LDA;
    float* bs = Bs + buf * BK * LDB;
    const int64_t kb = (int64_t)kt * BK;
    const int na = BM * BK;
#ifdef TT_SIMT_EXP_NOCOPY_A
    if (true) {                            // experiment build: no A slab copies
    } else
#endif
#ifdef TT_SIMT_EXP_A16
    // experiment build only: A rows copied as 16-byte chunks WITHOUT the transpose (results are
    // wrong), to time what the copy's form costs against the transposing 4-byte copies
    if (!p.a_tn) {
      const int q4a = BK >> 2;             // 16-byte chunks per A row of the slab
      const int rstep = T / q4a;
      const int c = (t % q4a) << 2;
      const float* src = Ab + (int64_t)(t / q4a) * K + kb + c;
      float* dst = as + (t / q4a) * BK + c;
      for (int r = t / q4a; r < BM; r += rstep) {
        cp_async16(dst, src);
        dst += rstep * BK;
        src += (int64_t)rstep * K;
      }
    } else
#endif
    if (a_fast) {                          // rows a_r0, a_r0 + a_rstep, ... of column k = kb + a_c
      const float* src = Ab + (int64_t)a_r0 * K + kb + a_c;
      float* dst = as + a_c * LDA + a_r0;
      const int64_t sstep = (int64_t)a_rstep * K;
#pragma unroll 4
      for (int r = a_r0; r < BM; r += a_rstep) {
        cp_async4(dst, src);
        dst += a_rstep;
        src += sstep;
      }
    } else if (p.a_tn) {                          // W rows are already k-major: As[k][m] needs no transpose
      if (p.a_vec16) {
        const int q = BM >> 2;
        for (int e = t; e < BK * q; e += T) {
          const int r = e / q, c = (e - (e / q) * q) << 2;
          cp_async16(as + r * LDA + c, Ab + (kb + r) * M + c);
        }
      } else {
        for (int e = t; e < BK * BM; e += T) {
          const int r = e / BM, c = e - (e / BM) * BM;
          cp_async4(as + r * LDA + c, Ab + (kb + r) * M + c);
        }
      }
    } else if (p.bk_sh >= 0) {             // power-of-two BK: shifts instead of divisions
      for (int e = t; e < na; e += T) {
        const int r = e >> p.bk_sh, c = e & (BK - 1);
        cp_async4(as + c * LDA + r, Ab + (int64_t)r * K + kb + c);
      }
    } else {
      for (int e = t; e < na; e += T) {
        const int r = e / BK, c = e - (e / BK) * BK;
        cp_async4(as + c * LDA + r, Ab + (int64_t)r * K + kb + c);
      }
    }
#ifdef TT_SIMT_EXP_NOCOPY_B
    return;
#endif
    if (p.b_tma) {                         // one thread: arm the slot's barrier, issue the box
      if (threadIdx.x == 0) {
        const uint32_t bar = bar0 + 8u * (uint32_t)buf;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // slot reads done (barrier) -> async writes
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                     "r"((uint32_t)(BK * BN * 4)) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
            ::"r"((uint32_t)__cvta_generic_to_shared(bs)), "l"(&p.tmB), "r"((int)(blockIdx.x * BN)), "r"((int)kb),
            "r"(bar) : "memory");
      }
    } else if (b_fast) {                          // rows b_r0, b_r0 + b_rstep, ... of 16-byte column b_c
      const float* src = Bb + (kb + b_r0) * N + b_c;
      float* dst = bs + b_r0 * LDB + b_c;
      const int64_t sstep = (int64_t)b_rstep * N;
      const int dstep = b_rstep * LDB;
#pragma unroll 4
      for (int r = b_r0; r < BK; r += b_rstep) {
        cp_async16(dst, src);
        dst += dstep;
        src += sstep;
      }
    } else if (p.b_vec) {
      const int q = BN >> 2;
      const int nb = BK * q;
      if (p.bq_sh >= 0) {
        for (int e = t; e < nb; e += T) {
          const int r = e >> p.bq_sh, c = (e & (q - 1)) << 2;
          cp_async16(bs + r * LDB + c, Bb + (kb + r) * N + c);
        }
      } else {
        for (int e = t; e < nb; e += T) {
          const int r = e / q, c = (e - (e / q) * q) << 2;
          cp_async16(bs + r * LDB + c, Bb + (kb + r) * N + c);
        }
      }
    } else {
      const int nb = BK * BN;
      for (int e = t; e < nb; e += T) {
        const int r = e / BN, c = e - (e / BN) * BN;
        cp_async4(bs + r * LDB + c, Bb + (kb + r) * N + c);
      }
    }
  };

  // kVecA: TM, TN multiples of 4 => BN % 4 == 0 => the As base (2 BK LDB floats) is 16 B aligned
  constexpr bool kVecA = (TM % 4 == 0) && (TN % 4 == 0);
  constexpr bool kPair = (TN % 2 == 0);
  float acc[TM][TN];
  float2 acc2[TM][kPair ? TN / 2 : 1];
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    if constexpr (kPair) {
#pragma unroll
      for (int j = 0; j < TN / 2; ++j) acc2[i][j] = make_float2(0.0f, 0.0f);
    } else {
#pragma unroll
      for (int j = 0; j < TN; ++j) acc[i][j] = 0.0f;
    }
  }

  // prologue: slots 0 .. NS-2 in flight; every iteration commits one group (possibly empty)
  for (int pk = 0; pk < NS - 1; ++pk) {
    if (pk < p.k0) load(pk, pk);
    cp_async_commit();
  }
  int buf = 0;
  // one_bar (register tiles of >= 64 accumulators): the copies of slab kt + NS - 1 go out right
  // after the slab's barrier and a second barrier is not needed; small tiles keep the round-1 loop
  // (copies issued before the wait, a barrier at the end of the slab), which starts each copy a
  // little earlier -- that matters when a slab's compute is short (measured as a compile-time
  // switch: one barrier -1.6 % at 4096^3, -1.1 % at 2048^3, -2 % at 1024^3, +2-5 % for the 8 x 2
  // tile of 512^3; as a runtime switch inside one instance it bought only 0.5 %, so it is a
  // compile-time property of the instance; profiles/r12_simt_1bar_ab.txt).
#ifdef TT_SIMT_TWO_BARRIERS
  constexpr bool one_bar = false;         // A/B build
#elif defined(TT_SIMT_ONE_BAR_MIN)
  constexpr bool one_bar = TM * TN >= TT_SIMT_ONE_BAR_MIN;   // A/B build
#else
  constexpr bool one_bar = TM * TN >= 64;
#endif
  for (int kt = 0; kt < p.k0; ++kt) {
    if constexpr (!one_bar) {
      const int nxt = kt + NS - 1;
      if (nxt < p.k0) load(nxt, nxt % NS);
      cp_async_commit();
      if (NS == 3) cp_async_wait<2>();
      else cp_async_wait<1>();
    } else {
      // my copies of slab kt have landed (groups of slabs kt .. kt + NS - 2 were outstanding)
      if (NS == 3) cp_async_wait<1>();
      else cp_async_wait<0>();
    }
    if (p.b_tma) {                         // slot buf's B box landed (its (kt / NS)-th fill)
      const uint32_t bar = bar0 + 8u * (uint32_t)buf, par = (uint32_t)(kt / NS) & 1u;
      uint32_t ok = 0;
      uint64_t t0 = 0;
      while (true) {
        asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
                     "selp.b32 %0, 1, 0, P;\n\t}" : "=r"(ok) : "r"(bar), "r"(par) : "memory");
        if (ok) break;
        // watchdog (as in the tcgen05 kernel): a box that never lands traps after 10 s -- a launch
        // error the host reports -- instead of hanging the GPU
        uint64_t now;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
        if (t0 == 0) t0 = now;
        else if (now - t0 > 10000000000ull) __trap();
      }
    }
    // Slab kt is now visible to every thread.  With one_bar every thread has also finished
    // computing on slab kt - 1, whose slot ((kt - 1) mod NS = (kt + NS - 1) mod NS) the copies of
    // slab kt + NS - 1 issued right after this barrier overwrite.
    __syncthreads();
    if constexpr (one_bar) {
      const int nxt = kt + NS - 1;
      if (nxt < p.k0) load(nxt, nxt % NS);
      cp_async_commit();
    }
    const float* as = As + buf * BK * LDA + row0;
    const float* bs = Bs + buf * BK * LDB + col0;
    // fragments for step kk+1 are loaded from shared memory while step kk's FMAs issue
    float a0[TM], b0[TN], a1[TM], b1[TN];
    load_frag<TM, TN, kVecA>(as, bs, 0, LDA, LDB, SA, SB, a0, b0);
    int kk = 0;
#pragma unroll(BKF > 0 ? BKF / 2 : 1)
    for (; kk + 2 <= BK; kk += 2) {
      load_frag<TM, TN, kVecA>(as, bs, kk + 1, LDA, LDB, SA, SB, a1, b1);
      fma_frag<TM, TN, kPair>(a0, b0, acc, acc2);
      if (kk + 2 < BK) load_frag<TM, TN, kVecA>(as, bs, kk + 2, LDA, LDB, SA, SB, a0, b0);
      fma_frag<TM, TN, kPair>(a1, b1, acc, acc2);
    }
    if (kk < BK) fma_frag<TM, TN, kPair>(a0, b0, acc, acc2);   // odd BK: last step
    if (++buf == NS) buf = 0;
    if constexpr (!one_bar) __syncthreads();
  }
  if constexpr (kPair) {
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN / 2; ++j) {
        acc[i][2 * j] = acc2[i][j].x;
        acc[i][2 * j + 1] = acc2[i][j].y;
      }
  }

  float* Cb = p.C + ((int64_t)blockIdx.y * BM + row0) * N + (int64_t)blockIdx.x * BN + col0;
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    float* Ci = Cb + (int64_t)((i >> 2) * SA + (i & 3)) * N;          // contiguous: SA = 4 -> row i
    if constexpr (TN % 4 == 0) {
      if (p.c_vec) {
#pragma unroll
        for (int j = 0; j < TN; j += 4)
          *reinterpret_cast<float4*>(Ci + (j >> 2) * SB) = make_float4(acc[i][j], acc[i][j + 1], acc[i][j + 2], acc[i][j + 3]);
        continue;
      }
#pragma unroll
      for (int j = 0; j < TN; ++j) Ci[(j >> 2) * SB + (j & 3)] = acc[i][j];
    } else {
#pragma unroll
      for (int j = 0; j < TN; ++j) Ci[j] = acc[i][j];
    }
  }
}

using KernelFn = void (*)(const SimtArgs);

template <int LM, int LN>
constexpr KernelFn kfn() {
  if constexpr ((1 << LM) * (1 << LN) <= 128) return &k1_simt<(1 << LM), (1 << LN)>;
  else return nullptr;
}

template <int LM, int... LNs>
constexpr void fill_row(KernelFn (&t)[7][7], std::integer_sequence<int, LNs...>) {
  ((t[LM][LNs] = kfn<LM, LNs>()), ...);
}
template <int... LMs>
constexpr void fill_all(KernelFn (&t)[7][7], std::integer_sequence<int, LMs...>) {
  (fill_row<LMs>(t, std::make_integer_sequence<int, 7>{}), ...);
}

// Fixed-slab instances (register tile, BK) for the small register tiles the searches pick at the
// paper's 512^3 / 1024^3 shapes (measured +9 % / +27 %, profiles/r3_epilogue.md); a config
// matching one exactly runs it, everything else the generic instance.
struct FixedInst {
  int tm, tn, bk, lb;   // lb: the instance's launch bound (configs with more threads use others)
  KernelFn fn;
};
#define TT_FIXED3(TM, TN)                                                                   \
  {TM, TN, 32, max_threads(TM * TN), &k1_simt<TM, TN, 32>},                            \
      {TM, TN, 64, max_threads(TM * TN), &k1_simt<TM, TN, 64>},                        \
      {TM, TN, 128, max_threads(TM * TN), &k1_simt<TM, TN, 128>}
// register tiles of <= 32 accumulators (larger ones spill at their launch bound when fully
// unrolled, and already cover the LDS latency with the generic loop)
// (8 x 8 tiles with BK 16/32 at launch bound 128/256 measured +8 % for 8 x 8 configs but left
// the best-found 2048^3 / 4096^3 results, which use 16 x 8 tiles, unchanged: not kept)
const FixedInst kFixed[] = {TT_FIXED3(4, 4), TT_FIXED3(4, 8), TT_FIXED3(8, 4)};
#undef TT_FIXED3

struct Table {
  KernelFn fn[7][7] = {};
  Table() { fill_all(fn, std::make_integer_sequence<int, 7>{}); }
};
Table& table() {
  static Table t;
  return t;
}

int ilog2(int64_t v) {
  int l = 0;
  while ((int64_t(1) << l) < v) ++l;
  return l;
}

}  // namespace

tt_status simt_bind(const Space& sp, const State& s, tt_launch_info* info, std::string* err) {
  const int64_t m0 = s.f[0][0], m1 = s.f[0][1], m2 = s.f[0][2], m3 = s.f[0][3];
  const int64_t k1 = s.f[1][1];
  const int64_t n0 = s.f[2][0], n1 = s.f[2][1], n2 = s.f[2][2], n3 = s.f[2][3];
  *info = tt_launch_info{};
  info->family = TT_FAM_F32_SIMT;
  info->grid_x = n0;
  info->grid_y = m0;
  info->grid_z = 1;
  info->block_x = (int32_t)(m1 * n1 * m2 * n2);
  info->cluster_x = 1;
  // J_hw guarantees 2 slots fit.  The kernel also runs 3 slots, but measured no faster on B200
  // (2048^3: 40.7 vs 42.3 TF/s, 4096^3: 47.7 vs 49.3), so the binder keeps 2.
  const int64_t slot = (m1 * m2 * m3 + n1 * n2 * n3 + 2 * kSimtPad) * k1 * 4;
  const int stages = kSimtStages;
  info->smem_bytes = (int32_t)(stages * slot);
  info->stages = stages;
  info->tile_m = (int32_t)(m1 * m2 * m3);
  info->tile_n = (int32_t)(n1 * n2 * n3);
  info->tile_k = (int32_t)k1;
  info->reg_tile_m = (int32_t)m3;
  info->reg_tile_n = (int32_t)n3;
  (void)sp;
  (void)err;
  return TT_OK;
}

// The instance a config runs and its resident CTAs per SM (occupancy), for the partial-grid probe.
namespace {
struct Pick {
  KernelFn fn;
  tt_launch_info li;
};
tt_status pick_instance(const Space& sp, const State& s, Pick* pk, std::string* err);
}  // namespace

tt_status simt_probe_shape(const Space& sp, const State& s, int64_t* ctas, int64_t* slots, std::string* err) {
  Pick pk;
  tt_status st = pick_instance(sp, s, &pk, err);
  if (st != TT_OK) return st;
  int occ = 0, dev = 0, sms = 0;
  if (!cuda_ok(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pk.fn, pk.li.block_x, pk.li.smem_bytes), err,
               "occupancy(k1_simt)") ||
      !cuda_ok(cudaGetDevice(&dev), err, "cudaGetDevice") ||
      !cuda_ok(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), err, "SM count"))
    return TT_E_CUDA;
  *ctas = pk.li.grid_x * pk.li.grid_y;
  *slots = (int64_t)std::max(occ, 1) * sms;
  return TT_OK;
}

namespace {
tt_status pick_instance(const Space& sp, const State& s, Pick* pk, std::string* err) {
  tt_launch_info& li = pk->li;
  simt_bind(sp, s, &li, err);
  const int lm = ilog2(li.reg_tile_m), ln = ilog2(li.reg_tile_n);
  Table& tb = table();
  KernelFn fn = tb.fn[lm][ln];
  if (!fn) {
    *err = "no SIMT kernel instance for this register tile";
    return TT_E_UNSUPPORTED;
  }
  if (!ensure_max_smem((const void*)fn, kSmemPerCta, err)) return TT_E_CUDA;
  // TT_SIMT_FIXED=0 (experiments) keeps the generic instance for every config
  static const bool use_fixed = [] {
    const char* e = std::getenv("TT_SIMT_FIXED");
    return !(e && e[0] == '0');
  }();
  if (use_fixed) {
    for (size_t i = 0; i < sizeof(kFixed) / sizeof(kFixed[0]); ++i) {
      const FixedInst& f = kFixed[i];
      if (f.tm == li.reg_tile_m && f.tn == li.reg_tile_n && f.bk == li.tile_k && li.block_x <= f.lb) {
        if (!ensure_max_smem((const void*)f.fn, kSmemPerCta, err)) return TT_E_CUDA;
        fn = f.fn;
        break;
      }
    }
  }
  pk->fn = fn;
  return TT_OK;
}
}  // namespace

tt_status simt_preload(std::string* err) {
  Table& tb = table();
  for (auto& row : tb.fn)
    for (KernelFn f : row)
      if (f && !ensure_max_smem((const void*)f, kSmemPerCta, err)) return TT_E_CUDA;
  for (const FixedInst& f : kFixed)
    if (!ensure_max_smem((const void*)f.fn, kSmemPerCta, err)) return TT_E_CUDA;
  return TT_OK;
}

tt_status simt_prepare(const Space& sp, const State& s, std::string* err) {
  Pick pk;
  return pick_instance(sp, s, &pk, err);
}

namespace {
// TT_SIMT_TMA=0 (A/B experiments) keeps the cp.async B copies; read at every launch
bool simt_tma_enabled() {
  const char* e = std::getenv("TT_SIMT_TMA");
  return !(e && e[0] == '0');
}

// Tensor map of B's slabs, cached per (device, pointer, N, K, box): a measurement replays the same
// launch many times and a search keeps its operands, so the encode runs once per config.
tt_status simt_b_map(const float* B, int64_t N, int64_t K, uint32_t bn, uint32_t bk, CUtensorMap* out,
                     std::string* err) {
  static std::mutex mu;
  static std::map<std::tuple<int, const float*, int64_t, int64_t, uint32_t, uint32_t>, CUtensorMap> cache;
  int dev = 0;
  if (!cuda_ok(cudaGetDevice(&dev), err, "cudaGetDevice")) return TT_E_CUDA;
  const auto key = std::make_tuple(dev, B, N, K, bn, bk);
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(key);
  if (it != cache.end()) {
    *out = it->second;
    return TT_OK;
  }
  if (!encode_map_2d_f32(out, B, (uint64_t)N, (uint64_t)K, bn, bk, err)) return TT_E_CUDA;
  if (cache.size() >= 4096) cache.clear();
  cache[key] = *out;
  return TT_OK;
}
}  // namespace

tt_status simt_launch(const Space& sp, const State& s, const float* A, const float* B, float* C,
                      cudaStream_t stream, std::string* err, int64_t max_rows) {
  Pick pk;
  tt_status pst = pick_instance(sp, s, &pk, err);
  if (pst != TT_OK) return pst;
  const tt_launch_info& li = pk.li;
  KernelFn fn = pk.fn;
  SimtArgs a;
  std::memset(&a, 0, sizeof(a));
  a.A = A;
  a.B = B;
  a.C = C;
  a.M = sp.dim[0];
  a.K = sp.dim[1];
  a.N = sp.dim[2];
  a.m1 = (int)s.f[0][1];
  a.m2 = (int)s.f[0][2];
  a.n1 = (int)s.f[2][1];
  a.n2 = (int)s.f[2][2];
  a.bk = (int)s.f[1][1];
  a.k0 = (int)s.f[1][0];
  const int64_t LDB = li.tile_n + 4;
  (void)LDB;
  auto lg = [](int64_t v) -> int { if (v <= 0 || (v & (v - 1))) return -1; int l = 0; while ((int64_t(1) << l) < v) ++l; return l; };
  a.bk_sh = lg(a.bk);
  a.bq_sh = (li.tile_n % 4 == 0) ? lg(li.tile_n / 4) : -1;
  a.b_vec = (li.tile_n % 4 == 0 && a.N % 4 == 0 && ((uintptr_t)B % 16) == 0) ? 1 : 0;
  a.a_tn = sp.layout == TT_LAYOUT_TN ? 1 : 0;
  a.c_vec = (a.N % 4 == 0 && ((uintptr_t)C % 16) == 0) ? 1 : 0;
  a.stages = li.stages;
  a.b_tma = 0;
  if (simt_tma_enabled() && a.b_vec && li.tile_n <= 256 && a.bk >= 8 && a.bk <= 256 &&
      ((int64_t)a.bk * li.tile_n * 4) % 128 == 0) {
    tt_status st = simt_b_map(B, a.N, a.K, (uint32_t)li.tile_n, (uint32_t)a.bk, &a.tmB, err);
    if (st != TT_OK) return st;
    a.b_tma = 1;
  }
  const int64_t ldb = a.b_tma ? li.tile_n : li.tile_n + 4;
  a.a_vec16 = (li.tile_m % 4 == 0 && a.M % 4 == 0 && ((uintptr_t)A % 16) == 0 &&
               ((2 * (int64_t)a.bk * ldb) % 4) == 0) ? 1 : 0;
  // max_rows > 0 (the partial-grid probe of tt_measure): only the first max_rows CTA rows run
  const int64_t rows = max_rows > 0 ? std::min<int64_t>(max_rows, li.grid_y) : li.grid_y;
  dim3 grid((unsigned)li.grid_x, (unsigned)rows, 1);
  fn<<<grid, li.block_x, li.smem_bytes, stream>>>(a);
  if (!cuda_ok(cudaGetLastError(), err, "k1_simt launch")) return TT_E_CUDA;
  return TT_OK;
}

}  // namespace tt
