/*
 * tiletune.h -- C-ABI of libtiletune, the B200 (sm_100a) hot path of arXiv 1909.10616
 * "Compiler-Level Matrix Multiplication Optimization for Deep Learning" (G-BFS / N-A2C).
 *
 * Citations: P:n = line n of the paper's PAPER.md; S:n = line n of SPEC.md; readings Z1..Z23
 * and the J_hw table are in DESIGN.md.
 *
 * Conventions (apply to every entry point):
 *  - Every function returns tt_status and never throws across the ABI.  On a non-OK status a
 *    thread-local message is available from tt_last_error().
 *  - Argument order: the ABI takes (M, N, K) for C[M x N] = A[M x K] . B[K x N].  The paper
 *    names problems (m, k, n) and orders the state [s_m, s_k, s_n];
 *    tt_config keeps that paper order (m, k, n).  M == m, N == n, K == k.
 *  - Matrices are dense row-major: A[M][K], B[K][N], C[M][N] (reading Z14); C is overwritten.
 *  - Ownership: the caller owns every buffer passed in (host arrays and device A/B/C).  The
 *    library keeps no pointer past return.  Only a tt_ctx owns device memory (measurement
 *    operands, events, an L2-flush buffer, host staging for tt_gemm_host).
 *  - Threading: the configuration-space functions (tt_count_configs .. tt_neighbors,
 *    tt_binding) are pure and thread-safe.  A tt_ctx is used by one thread at a time;
 *    measurement is serialised per device.
 */
#ifndef TILETUNE_H
#define TILETUNE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TT_VERSION 6
#define TT_MAXD 4  /* maximum loop depth per axis carried in tt_config */

typedef enum {
  TT_OK = 0,
  TT_E_INVAL = 1,          /* bad argument (null pointer, size, depth > TT_MAXD, illegitimate s0) */
  TT_E_ILLEGITIMATE = 2,   /* J_prod false: Eq. 2-4 products or positivity violated */
  TT_E_INFEASIBLE = 3,     /* J_hw false for the requested family */
  TT_E_OVERFLOW = 4,       /* space size does not fit uint64 */
  TT_E_CAPACITY = 5,       /* output buffer too small; *n_out holds the size needed */
  TT_E_CUDA = 6,           /* CUDA runtime / driver error (message in tt_last_error) */
  TT_E_EVALUATOR = 7,      /* cost source failed during a search; partial result + trace valid */
  TT_E_UNSUPPORTED = 8     /* family / depth combination has no kernel */
} tt_status;

/* Kernel families = J_hw tables. */
typedef enum {
  TT_FAM_NONE = 0,         /* J = J_prod only (the paper's space); no kernel */
  TT_FAM_F32_SIMT = 1,     /* K1: fp32 CUDA-core FFMA, the paper's arithmetic (reading Z13) */
  TT_FAM_TF32_UMMA = 2,    /* K2: tcgen05.mma kind::tf32, fp32 storage, fp32 accumulate */
  TT_FAM_BF16_UMMA = 3     /* K3: tcgen05.mma kind::f16 with bf16 A/B, fp32 accumulate */
} tt_family;
/* UMMA level map (reading Z2): m = [cluster tiles, cta_group 1|2, M atoms per CTA 1|2, 128],
 * n = [cluster tiles, pairs per cluster along N 1|2 (2 = A shared by TMA multicast), N atoms per
 * CTA 1|2, UMMA_N], k = [trips, BK].  SIMT: m / n = [CTAs, thread groups, lanes, register tile]. */

/* Storage of A.  NN: A row-major [M][K] (the plain definition, reading Z14).  TN: the paper's
 * perceptron workload Y = W^T X with W in R^(k x m): the caller passes W row-major
 * [K][M] and the product uses A = W^T.  B is always row-major [K][N]. */
typedef enum { TT_LAYOUT_NN = 0, TT_LAYOUT_TN = 1 } tt_layout;

/* Problem instance: the paper's cost(s; m,k,n,d_m,d_k,d_n), plus the J_hw family. */
typedef struct {
  int64_t M, N, K;         /* C[M x N] = A[M x K] B[K x N]; all >= 1 */
  int32_t dm, dk, dn;      /* loop depths d_m, d_k, d_n, 1..TT_MAXD; paper uses 4,2,4 */
  int32_t family;          /* tt_family */
  int32_t layout;          /* tt_layout of A (does not change the space or J_hw, only the kernel) */
} tt_space;

/* A state s = [s_m, s_k, s_n] (Eq. 5).  Factor vectors outer -> inner (reading Z1):
 * m[i] = trip count of the i-th m loop.  Slots >= d_x must be 1. */
typedef struct {
  int64_t m[TT_MAXD], k[TT_MAXD], n[TT_MAXD];
} tt_config;

/* Result of one measurement ("arithmetic mean for 10 repeated trials"; reading Z10). */
typedef struct {
  double cost_s;           /* median of per-repeat means (the score the searches use) */
  double mean_s, min_s, stdev_s;
  double probe_s;          /* one timed launch before the repeats */
  int32_t repeats;         /* R actually run (1 when the slow-candidate cut fired, Z12) */
  int32_t number;          /* back-to-back launches per repeat */
  int32_t device;          /* CUDA ordinal the sample was taken on */
  int32_t slow_cut;        /* 1 if cost_s = probe_s because probe_s > cut_s (Z12); 2 if cost_s is the
                              F32_SIMT partial-grid estimate (the first ~2 waves of CTA rows timed
                              and scaled by the wave count) and it exceeded cut_s */
  int32_t graph_nodes;     /* launches per captured CUDA graph the repeats replayed (0: direct launches) */
  int32_t raced;           /* 1 if the repeats stopped after race_repeats (tt_measure_opts.race_s) */
} tt_sample;

typedef struct {
  int32_t warmup;          /* untimed launches between the cold probe and the repeats (default 2;
                              none with l2_flush, where every timed launch starts cold) */
  int32_t repeats;         /* R (default 10) */
  double min_repeat_s;     /* each repeat lasts >= this: number = ceil(min_repeat_s / probe) (5e-4) */
  double cut_s;            /* if > 0 and probe > cut_s: cost = probe, repeats = 1 (Z12) */
  int32_t l2_flush;        /* 1: overwrite a >= 2 x L2 buffer before every timed launch */
  int32_t max_number;      /* cap on `number` (default 1000) */
  int32_t graph;           /* 1 (default): each repeat replays a CUDA graph of up to 32 captured
                              launches, so host launch overhead never enters the score; 0: direct
                              launches from the host loop.  Ignored with l2_flush. */
  double race_s;           /* if > 0: when the first race_repeats repeats all exceed race_s, stop
                              there (cost = their median, raced = 1) -- a candidate that cannot
                              beat the incumbent is not timed to full precision (reading Z12) */
  int32_t race_repeats;    /* default 2 */
} tt_measure_opts;

/* One row per measured state, in evaluation order (Fig. 7 axes P:352). */
typedef struct {
  uint64_t eval_index;     /* 0 = s0 */
  double t_wall_s;         /* host wall clock since the search started */
  tt_config cfg;
  double cost_s;
  double best_so_far_s;
} tt_trace_row;

typedef struct {
  tt_config best;          /* s* (Alg. 1 line 16 / Alg. 2 line 26) */
  double best_cost_s;      /* cost_min */
  uint64_t evals;          /* distinct states measured, s0 included (reading Z19) */
  uint64_t space_raw;      /* card(xi), the paper's denominator */
  uint64_t space_feasible; /* states with J_prod and J_hw */
  double frac_raw;         /* evals / space_raw ("fraction of visited configurations") */
  double frac_feasible;    /* evals / space_feasible */
  double wall_s;           /* tuning wall time ("searching time") */
  uint64_t trace_len;      /* rows written to the trace buffer (<= trace_cap) */
} tt_result;

/* Cost sources (how a search scores candidates). */
typedef enum {
  TT_COST_DEVICE = 0,      /* tt_measure on the ctx's device (the hardware test of P:231) */
  TT_COST_CALLBACK = 1,    /* cost_fn(cfg, user) per state (synthetic landscapes) */
  TT_COST_TABLE = 2,       /* table[rank(cfg)] (deterministic tables / trace replay) */
  TT_COST_BATCH = 3        /* batch_fn(cfgs, n, costs, user) per round (multi-GPU sharding) */
} tt_cost_source;

typedef double (*tt_cost_fn)(const tt_config* cfg, void* user);
/* Must fill costs[0..n) and return 0; nonzero aborts the search with TT_E_EVALUATOR. */
typedef int32_t (*tt_batch_eval_fn)(const tt_config* cfgs, int32_t n, double* costs, void* user);

typedef struct {
  int32_t family;          /* tt_family of the searched space */
  int32_t dm, dk, dn;      /* loop depths (default 4,2,4) */
  uint64_t seed;           /* SplitMix64 seed (reading O7) */
  int32_t has_s0;          /* 1: start from s0 below; 0: per-family default (P:369 / Z3) */
  tt_config s0;
  double budget_seconds;   /* T_max; <= 0: none */
  int32_t cost_source;     /* tt_cost_source */
  tt_cost_fn cost_fn;
  tt_batch_eval_fn batch_fn;
  void* user;
  const double* table;     /* TABLE source: cost by rank, length table_len (= space_raw) */
  uint64_t table_len;
  tt_measure_opts measure; /* DEVICE source */
  /* G-BFS (Alg. 1) */
  int32_t rho;             /* neighbours sampled per expansion (default 5) */
  int32_t width;           /* states popped per round W (default 1 = Alg. 1; Z9) */
  /* N-A2C (Alg. 2; defaults per reading Z18 / S:417-423) */
  int32_t steps_T;         /* exploration steps T (default 3) */
  double epsilon;          /* exploitation probability (default 0.8) */
  int32_t batch;           /* len(B_test) (default 16) */
  int32_t mem_capacity;    /* |M| FIFO capacity (default 4096) */
  double gamma, beta, lr, clip;   /* 0.9, 0.01, 0.01, 1.0 */
  int32_t epochs, minibatch, hidden;   /* 4, 64, 64 */
  int32_t rollout_cap_factor, max_t_increase;   /* 50, 16 */
  /* T schedule ("the exploration step T can have a decay process, i.e., starting with a
   * large value and gradually reducing to a small number"): episode e explores
   * T_e = max(steps_T_floor, steps_T - e / steps_T_decay_every) steps; decay_every = 0: constant T. */
  int32_t steps_T_floor, steps_T_decay_every;
  int32_t layout;          /* tt_layout of A for the DEVICE cost source (default NN) */
  /* Alg. 2 line 24 "Train actor's and critic's neural networks with M" sits inside the
   * "for s' in B_collect" loop.  1: train after every candidate, in that order;
   * 0 (default, reading Z18 / S:422): train once after each measured batch. */
  int32_t train_per_candidate;
  /* Scoring budget of the DEVICE / batch cost sources (reading Z12, "searching time" P:359):
   * cut_s = min(max(20 cost_min, 1 ms), max(1 ms, cut_roofline_x t_roof)), applied from s0 on
   * (t_roof = tt_roofline_seconds), and race_s = race_factor cost_min.  cut_roofline_x <= 0 drops the
   * absolute cut; race_factor <= 0 disables racing.  Defaults 50 and 1.1. */
  double cut_roofline_x;
  double race_factor;
} tt_search_opts;

/* How a config is bound to a launch (a5 of SURVEY §8a; for tests and reports). */
typedef struct {
  int32_t family;
  int64_t grid_x, grid_y, grid_z;
  int32_t block_x;
  int32_t cluster_x;       /* CTAs per cluster (UMMA: cta_group x n1) */
  int32_t smem_bytes;      /* dynamic shared memory */
  int32_t stages;          /* pipeline depth */
  int32_t tile_m, tile_n, tile_k;   /* per-cluster output tile and K step */
  int32_t tmem_cols;       /* UMMA: allocated TMEM columns (0 for SIMT) */
  int32_t acc_buffers;     /* UMMA: TMEM accumulator buffers */
  uint32_t idesc;          /* UMMA: instruction descriptor */
  int32_t reg_tile_m, reg_tile_n;   /* SIMT: per-thread register tile m3 x n3 */
  /* UMMA tail split: when the tile count is not a multiple of the co-resident
   * clusters, the last split_tiles tiles' k-blocks are shared by split_workers clusters (<= 4 per
   * tile) and combined in ascending-k order (the k-block-0 piece stores, the higher pieces TMA-reduce-add after every piece below them); 0 = none. */
  int32_t split_tiles, split_workers;
} tt_launch_info;

typedef struct tt_ctx tt_ctx;

int32_t tt_version(void);
const char* tt_last_error(void);
void tt_search_opts_default(tt_search_opts* opts);
void tt_measure_opts_default(tt_measure_opts* opts);

/* ---------------------------------------------------------------- configuration space (host) */

/* card(xi) = prod_x prod_{p^e || x} C(e + d_x - 1, d_x - 1) (Eq. 1-4; P:375 prints
 * 899756 for 1024^3).  *feasible (nullable) counts states with J_hw too (enumerates the raw
 * space: milliseconds up to ~3M states).  TT_E_OVERFLOW if raw does not fit uint64. */
tt_status tt_count_configs(const tt_space* sp, uint64_t* raw, uint64_t* feasible);

/* States with J_prod true, in rank order (lexicographic over m0.., k0.., n0..; reading O4),
 * ranks [first_rank, first_rank + cap).  *n_out = number written. */
tt_status tt_enumerate_configs(const tt_space* sp, uint64_t first_rank, uint64_t cap,
                               tt_config* out, uint64_t* n_out);

/* Every state with J = J_prod and J_hw, in rank order.  cfgs and/or ranks may be null (count
 * only).  TT_E_CAPACITY with *n_out = needed if cap is too small. */
tt_status tt_enumerate_feasible(const tt_space* sp, uint64_t cap, tt_config* cfgs,
                                uint64_t* ranks, uint64_t* n_out);

/* rank = (r_m |xi_k| + r_k) |xi_n| + r_n.  TT_E_ILLEGITIMATE if J_prod is false. */
tt_status tt_rank(const tt_space* sp, const tt_config* cfg, uint64_t* rank);
tt_status tt_unrank(const tt_space* sp, uint64_t rank, tt_config* out);

/* J of Eq. 5: *j_prod per Eq. 2-4 + P:191 footnote; *j_hw per the family table. */
tt_status tt_is_legitimate(const tt_space* sp, const tt_config* cfg, int32_t* j_prod, int32_t* j_hw);

/* Eq. 6-7: s' = step(s, a) for a = (axis 0=m/1=k/2=n, double slot i, halve slot j).
 * *legit = 1 if s' has J (J_prod and J_hw); s' is written only when the halved factor is even. */
tt_status tt_step(const tt_space* sp, const tt_config* cfg, int32_t axis, int32_t i, int32_t j,
                  tt_config* out, int32_t* legit);

/* g(s) of Eq. 9 restricted to legitimate results (reading Z4), in action order
 * (x = m,k,n; i ascending; j ascending).  At most sum_x d_x(d_x-1) (26) entries. */
tt_status tt_neighbors(const tt_space* sp, const tt_config* cfg, tt_config* out, int32_t cap,
                       int32_t* n_out);

/* Launch binding of a feasible config (grid, block, smem, stages, descriptors). */
tt_status tt_binding(const tt_space* sp, const tt_config* cfg, tt_launch_info* info);

/* Introspection of the tcgen05 families' persistent schedule (DESIGN.md §6 tail / wave+remainder
 * split): the work items cluster `worker` walks, in order, as the kernel computes them (the same
 * code, evaluated on the host under the current TT_TAIL_SPLIT policy; without a GPU the cluster
 * count is SMs / cluster size).  Each item is 5 int32: tile, first k-block, end k-block, order
 * (pieces of the tile below this one), split flag.  Writes min(cap, n) items to `items` (may be
 * null with cap 0), the item count to *n_items, the number of clusters to *workers and k0 (k-blocks
 * per tile) to *k0.  TT_E_UNSUPPORTED for the SIMT family. */
tt_status tt_umma_schedule(const tt_space* sp, const tt_config* cfg, int32_t worker, int32_t* items, int32_t cap,
                           int32_t* n_items, int32_t* workers, int32_t* k0);

/* ---------------------------------------------------------------- device: generator, GEMM */

/* K4: fill `count` elements with the counter-based U[-1,1) recipe of DESIGN.md §5 for matrix
 * seed `seed` at logical indices idx0 .. idx0+count-1.  dtype 0 = fp32, 1 = bf16 (RNE).
 * dst is device memory; launched on `stream` (cudaStream_t, null = legacy default stream). */
tt_status tt_fill_uniform(void* dst, int32_t dtype, uint64_t seed, uint64_t idx0, uint64_t count,
                          void* stream);

/* The tiled GEMM of the paper for config cfg of family `family`:
 * C[M][N] (fp32) = A[M][K] . B[K][N].  A/B are fp32 for F32_SIMT and TF32_UMMA, bf16 for
 * BF16_UMMA.  Device pointers; launched on `stream`; never allocates, never synchronises.
 * The config's trip counts must tile M, N, K exactly (J_prod) and satisfy J_hw.
 * F32_SIMT keeps one fmaf chain per output in k order (bit-exact vs the oracle's fmaf mode).
 * Alignment: A, B, C 16-byte aligned; UMMA families need K and N multiples of 8 (bf16) / 4.
 * UMMA tail split (tt_launch_info.split_tiles > 0): the pieces of a split tile hand off through
 * library-owned device words (a static array, one slice per launch stream, left zeroed by every
 * launch), and a piece waits only on clusters with a lower index, so the launch needs no
 * co-residency of its grid.  Two split launches that can overlap must use different streams; a
 * captured graph keeps its capture stream's slice, so do not replay one graph concurrently on
 * several streams (TT_TAIL_SPLIT=0 disables the split). */
tt_status tt_gemm(int64_t M, int64_t N, int64_t K, int32_t family, const void* A, const void* B,
                  float* C, const tt_config* cfg, void* stream);

/* tt_gemm with an explicit A storage (tt_layout): for TT_LAYOUT_TN, A points to W row-major
 * [K][M] and C = W^T B.  Alignment as tt_gemm (UMMA families also need M a multiple of 8). */
tt_status tt_gemm_ex(int64_t M, int64_t N, int64_t K, int32_t family, int32_t layout, const void* A,
                     const void* B, float* C, const tt_config* cfg, void* stream);

/* A prepared tt_gemm_ex: (M, N, K, family, layout, cfg) are checked and bound to the device
 * buffers (A, B, C) once, so tt_plan_launch is a kernel launch on `stream` with no argument
 * checking -- the repeated launch of one GEMM (a training step, bench.py's timed loop).  The plan
 * keeps the three pointers (the caller keeps the buffers alive until tt_plan_destroy); errors as
 * tt_gemm_ex at creation, TT_E_CUDA at launch. */
typedef struct tt_plan tt_plan;
tt_status tt_plan_create(int64_t M, int64_t N, int64_t K, int32_t family, int32_t layout, const void* A,
                         const void* B, float* C, const tt_config* cfg, tt_plan** out);
tt_status tt_plan_launch(tt_plan* plan, void* stream);
tt_status tt_plan_destroy(tt_plan* plan);

/* Same product through host buffers: copies A (stored per `layout`), B host->device, runs the
 * GEMM, copies C back, all on the ctx stream, and synchronises.  The ctx owns the device staging
 * buffers.  Host buffers should be pinned for asynchronous copies. */
tt_status tt_gemm_host(tt_ctx* ctx, int64_t M, int64_t N, int64_t K, int32_t family, int32_t layout,
                       const void* A_host, const void* B_host, float* C_host, const tt_config* cfg);

/* ---------------------------------------------------------------- measurement (B2) */

/* A context on CUDA device `device`: owns a stream, events, an L2-flush buffer and the
 * measurement operands (generated on first use per (M,N,K,dtype) with seeds input_seed (A) and
 * input_seed + 1 (B) by K4). */
tt_status tt_ctx_create(int32_t device, uint64_t input_seed, tt_ctx** out);
tt_status tt_ctx_destroy(tt_ctx* ctx);
/* The ctx stream (cudaStream_t) -- use it to order caller work with measurements. */
tt_status tt_ctx_stream(tt_ctx* ctx, void** stream);
/* Device pointers of the ctx operands for this problem (created if needed). */
tt_status tt_ctx_operands(tt_ctx* ctx, int64_t M, int64_t N, int64_t K, int32_t family,
                          const void** A, const void** B, float** C);

/* One-time setup of a ctx for a space, outside any timed search: the measurement operands, the
 * L2-flush buffer, and every kernel of the space's family loaded into the context (lazy module
 * loading otherwise lands in the first measurement of each kernel).  Synchronises the ctx stream. */
tt_status tt_ctx_prepare(tt_ctx* ctx, const tt_space* sp);

/* cost(s) on hardware ("test (i.e., run the configuration on target hardware)"):
 * one cold timed probe (if it exceeds opts->cut_s the candidate is scored by it, Z12), warmup
 * launches, a warm probe that sizes `number`, then R repeats of `number` launches between CUDA
 * events on the ctx stream (replayed from a captured CUDA graph unless opts->graph = 0, so the
 * score is device time, not host launch rate); cost = median of per-repeat means (Z10).  The measured operands are
 * the ctx's (K4 recipe); the space's layout selects the NN or TN kernel.  TT_E_ILLEGITIMATE / TT_E_INFEASIBLE for a config
 * without J; TT_E_CUDA on a launch error. */
tt_status tt_measure(tt_ctx* ctx, const tt_space* sp, const tt_config* cfg,
                     const tt_measure_opts* opts, tt_sample* out);

/* One GEMM of sp at the family's nominal peak on `device` (-1: the current device; no device:
 * 148 SMs at 1965 MHz): 2 M N K / (SMs x SM clock x flop/clk/SM), with 256 (fp32 FFMA: 128 lanes
 * x 2), 4096 (TF32) and 8192 (BF16) flop/clk/SM.  The scale of the slow-candidate cut. */
tt_status tt_roofline_seconds(const tt_space* sp, int32_t device, double* seconds);

/* The per-candidate measurement options a search uses (reading Z12): copies opts->measure and
 * sets cut_s and race_s from the incumbent cost_min (+inf before s0 is scored) as documented at
 * tt_search_opts.cut_roofline_x.  Shared by the in-library DEVICE source and sharded evaluators. */
tt_status tt_scoring_opts(const tt_space* sp, int32_t device, const tt_search_opts* opts, double cost_min,
                          tt_measure_opts* out);

/* Measure a set of candidates on the ctx device (the per-rank half of a sharded round, SURVEY
 * §8e): for j in [0, n) with mine == NULL or mine[j] != 0, costs[j] = tt_measure(cfgs[j]).cost_s
 * with `mo`, and secs[j] (nullable) = host wall seconds that measurement took; other entries are
 * set to 0.  Stops at the first failing candidate (its status is returned). */
tt_status tt_measure_set(tt_ctx* ctx, const tt_space* sp, const tt_config* cfgs, int32_t n, const uint8_t* mine,
                         const tt_measure_opts* mo, double* costs, double* secs);

/* Two-phase form of tt_measure_set for the sharded evaluator (reading Z12).  Splits
 * one measurement at its cold probe so that a round can be balanced over ranks with the probe
 * known: the probe alone decides whether a candidate is cut (one launch) and predicts whether
 * racing stops it after race_repeats, i.e. how long the rest takes.
 *   phase 1: for j with mine == NULL or mine[j] != 0, run the (partial-grid and) cold probe of
 *            cfgs[j].  If that decides the score (slow cut, tt_sample.slow_cut != 0) then
 *            values[j] = the score and final_[j] = 1; else values[j] = probe seconds, final_[j] = 0.
 *   phase 2: run the rest of tt_measure (warm-ups, warm probe, R repeats with racing) for
 *            cfgs[j] as if its cold probe had returned probes[j] (> 0, from phase 1, possibly on
 *            another device of the same model); values[j] = cost_s, final_[j] = 1.
 * Phase 1 then phase 2 on one device performs exactly the launches of one tt_measure and gives
 * the same statistic.  Other entries are set to 0; secs[j] (nullable) = host wall seconds of that
 * phase.  values, final_ (and probes for phase 2) hold n entries, caller-owned.  Errors as
 * tt_measure_set; TT_E_INVAL for another phase, or a phase-2 probe <= 0. */
tt_status tt_measure_phase(tt_ctx* ctx, const tt_space* sp, const tt_config* cfgs, int32_t n, const uint8_t* mine,
                           const tt_measure_opts* mo, int32_t phase, const double* probes, double* values,
                           uint8_t* final_, double* secs);

/* The statistic tt_measure reports ("the arithmetic mean for 10 repeated trials"; reading
 * Z10): from R >= 1 per-repeat mean launch times per_repeat[0..R) (seconds, host array), sets
 * out->cost_s = median (mean of the two middle values for even R), mean_s = arithmetic mean
 * (left-to-right sum / R), min_s, stdev_s = sample standard deviation (0 for R = 1) and
 * repeats = R; the other fields are left untouched.  Pure host function: tt_measure calls exactly
 * this on its event timings, and it is exported so the statistic can be checked on injected
 * samples ("fake clock").  TT_E_INVAL for a null pointer or R < 1. */
tt_status tt_aggregate(const double* per_repeat, int32_t R, tt_sample* out);

/* ---------------------------------------------------------------- searches (B4) */

/* G-BFS, Algorithm 1 with readings Z4-Z9.  budget_evals = max distinct states
 * measured including s0 (0 = unlimited).  trace (nullable) receives up to trace_cap rows.
 * TT_E_INVAL for an illegitimate s0 (before any evaluation); TT_E_EVALUATOR if the cost
 * source fails (out and trace hold the partial search). */
tt_status tt_gbfs_search(tt_ctx* ctx, int64_t M, int64_t N, int64_t K, uint64_t budget_evals,
                         const tt_search_opts* opts, tt_result* out, tt_trace_row* trace,
                         uint64_t trace_cap);

/* N-A2C, Algorithm 2 with readings Z18.  Same contract as tt_gbfs_search. */
tt_status tt_na2c_search(tt_ctx* ctx, int64_t M, int64_t N, int64_t K, uint64_t budget_evals,
                         const tt_search_opts* opts, tt_result* out, tt_trace_row* trace,
                         uint64_t trace_cap);

/* ---------------------------------------------------------------- conv layer as a GEMM */

/* im2col ("each depth-wise (channel) slice of input can be added into an input matrix as a
 * row; similarly each kernel can be added into a kernel matrix as a column"): x is NCHW
 * [Nb][C][H][W] (dtype 0 fp32, 1 bf16), A is written row-major [Nb*P*Q][C*R*S] with
 * P = (H + 2 pad - R) / stride + 1, Q = (W + 2 pad - S) / stride + 1, row = (n P + p) Q + q,
 * column = (c R + r) S + s; taps outside the image read 0.  Device pointers; async on stream. */
tt_status tt_im2col(int32_t dtype, const void* x, int64_t Nb, int64_t C, int64_t H, int64_t W, int32_t R, int32_t S,
                    int32_t stride, int32_t pad, void* A, void* stream);

/* Conv layer y = conv(x, w) as im2col + the tiled GEMM of family `family`:
 * y [Nb*P*Q][Kf] (fp32, i.e. NPQK) = im2col(x) [Nb*P*Q][C*R*S] . Wm, where Wm is the kernel matrix
 * [C*R*S][Kf] (column kf = kernel kf flattened in (c, r, s) order).  cfg tiles the GEMM
 * (M, N, K) = (Nb*P*Q, Kf, C*R*S).  workspace (device) holds the im2col matrix:
 * workspace_bytes >= Nb*P*Q*C*R*S*elem, else TT_E_CAPACITY. */
tt_status tt_conv2d(int32_t family, const void* x, int64_t Nb, int64_t C, int64_t H, int64_t W, const void* Wm,
                    int64_t Kf, int32_t R, int32_t S, int32_t stride, int32_t pad, float* y, void* workspace,
                    uint64_t workspace_bytes, const tt_config* cfg, void* stream);

/* Random-search comparator ("configurations are randomly selected to be tested"):
 * the first budget_evals states of a uniform random permutation (SplitMix64 partial Fisher-Yates
 * with opts->seed) of the feasible set in rank order, measured in batches of opts->width.  Not the
 * paper's method; the baseline the searches are compared against. */
tt_status tt_random_search(tt_ctx* ctx, int64_t M, int64_t N, int64_t K, uint64_t budget_evals,
                           const tt_search_opts* opts, tt_result* out, tt_trace_row* trace, uint64_t trace_cap);

#ifdef __cplusplus
}
#endif
#endif /* TILETUNE_H */
