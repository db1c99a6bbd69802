/*
 * kvr_oracle.h — plain, slow, single-threaded CPU ORACLE for the replay of the
 * online process of arxiv 2601.18999 (KV-cache-aware load balancing).
 *
 * THIS IS TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only tests/, the
 * __graft_entry__.smoke() check and bench.py's cpu_baseline / --impl reference
 * legs may load it.  It shares no code, header, table or constant generator
 * with the CUDA path (paper_2601_18999_b200/csrc, include/kvr.h): every struct
 * below is duplicated on purpose.
 *
 * Citation keys: P:n = PAPER.md line n (paper_2601_18999), SURVEY §8(c) = the
 * operation order and the ambiguity readings A1..A36 listed in DESIGN.md.
 *
 * What it computes (one replay = one "trial"):
 *   per query j (trace order), t = a_j
 *     1. catch-up per worker: decay ticks P~ <- rho*P~ every dt (Alg. 2 l.17,
 *        P:276-277) merged with FIFO completions -> OnlineUpdate(theta) (NLMS,
 *        A8; Alg. 2 l.12) and ReleaseLoad (A10)
 *     2. longest cached prefix match h_ij on every worker
 *     3. router score + argmin: LBGR Eq. 4-5 (Alg. 2 l.3-9), or the
 *        baselines RR / RANDOM / cache-aware THRESHOLD / STATIC linear
 *     4. UpdateCache on the chosen worker only (Eq. 3) with
 *        Leaf-LRU or RLT (Alg. 1)
 *     5. accounting: Eq. 1, Eq. 2, Eq. 6,
 *        single-server FIFO latency / TTFT (A12, A20)
 *     6. decision digest
 *   With kvro_config.batch_slots = beta >= 1 the same steps run in the
 *   continuous-batching engine (readings A30-A36):
 *   beta slots per worker, FIFO wait, UpdateCache at dequeue with the
 *   in-flight paths pinned, completions in time order (run_batched).
 *
 * Pins (tests/test_oracle_pins.py, tests/test_oracle_batching_pins.py; DESIGN.md
 * §2 P1-P32) fix every function here against the paper, closed forms, brute
 * force or textbook reductions.  Parity unpinned (only the oracle<->GPU
 * agreement checks them): LBGR theta trajectories and routing on
 * realistic traces beyond P4/P5/P14/P15/P18/P32, STATIC / THRESHOLD outcomes between
 * the extremes of P31, and absolute latency / TTFT / makespan magnitudes on the
 * synthetic workloads.
 *
 * Every function returns 0 on success, nonzero on a contract error; none throws.
 */
#ifndef KVR_ORACLE_H
#define KVR_ORACLE_H
#include <stdint.h>
#include <stddef.h>
#ifdef __cplusplus
extern "C" {
#endif

/* eviction / fallback / router codes (SURVEY §8b enums, duplicated) */
enum { KVRO_EVICT_LRU = 0, KVRO_EVICT_RLT = 1, KVRO_EVICT_OPT = 2 /* Belady; W = 1 only */ };
enum { KVRO_RLT_EARLY_RESET = 0, KVRO_RLT_UNIFORM_LEAF = 1, KVRO_RLT_LRU_MARKED = 2 };
enum { KVRO_ROUTE_LBGR = 0, KVRO_ROUTE_STATIC_LINEAR = 1, KVRO_ROUTE_THRESHOLD = 2,
       KVRO_ROUTE_ROUND_ROBIN = 3, KVRO_ROUTE_RANDOM = 4,
       KVRO_ROUTE_LBGR_RLS = 5 /* LBGR with the RLS reading of "0.992" (A8b) */,
       KVRO_ROUTE_CACHE_AWARE = 6 /* SGLang-style cache-aware rule (reading A38) */ };
#define KVRO_MAX_TRACKER_LAG 32u
/* per-trial status codes */
enum { KVRO_TRIAL_OK = 0, KVRO_TRIAL_RING_OVERFLOW = 1, KVRO_TRIAL_VICTIM_LOG_FULL = 2,
       KVRO_TRIAL_ADMISSION = 4 /* batched: full cache, every leaf in flight */ };

/* raw (un-chained) trace: host arrays.  Gamma_j = n_in input blocks then
 * n_out output blocks (A2); |q_j| = block_tokens*n_in (A1). */
typedef struct {
  uint32_t n_queries, block_tokens;
  uint64_t hash_salt;
  const double*   arrival_ms;     /* [N] */
  const uint32_t* n_in_blocks;    /* [N] */
  const uint32_t* n_out_blocks;   /* [N] */
  const uint32_t* out_tokens;     /* [N] |a_j| */
  const uint64_t* block_offsets;  /* [N+1] */
  const uint64_t* block_keys;     /* [offsets[N]] content keys c_{j,d} */
} kvro_trace;

typedef struct {
  uint32_t eviction, rlt_fallback, router, _pad;
  double est_alpha_cached_ms, est_alpha_miss_ms;
  double rho, delta_t_ms, mu, theta0[4];
  double tau;
  double w_hit, w_load;
  double rls_p0;                  /* LBGR_RLS: initial covariance P = rls_p0 * I */
  uint32_t tracker_lag;           /* A29: k = the router does not yet see the last k queries'
                                     cache updates (0..KVRO_MAX_TRACKER_LAG) */
  uint32_t tracker_grain;         /* A29: the router sees grain * floor(m / grain) matched blocks (>= 1) */
  double ca_balance_abs;          /* A38 cache-aware: imbalanced iff max-min pending > abs */
  double ca_balance_rel;          /*   and max pending > rel * min pending */
  double ca_cache_threshold;      /*   else highest match if its rate h~/|q| > threshold,
                                       else the worker with the fewest cached blocks */
  uint64_t _pad2;
} kvro_policy;

typedef struct {
  uint32_t W, capacity_blocks;
  double alpha_cached_ms, alpha_miss_ms, out_ms_per_token;   /* Eq. 1 truth */
  uint32_t pending_ring;        /* FIFO capacity per worker (0 = unbounded) */
  uint32_t latency_hist_bins;   /* 0 = no histogram */
  uint32_t batch_slots;         /* 0: beta = 1 model of A3/A12 (update at assignment);
                                   beta >= 1: continuous batching (A30-A35):
                                   update at dequeue, in-flight paths pinned */
  uint32_t _pad;
} kvro_config;

typedef struct {
  uint64_t queries, hit_tokens, input_tokens, probes, inserted_blocks, evictions,
           rlt_draws, rlt_resets, rlt_fallbacks, max_pending, decision_digest;
  double   sum_latency_ms, sum_ttft_ms, max_latency_ms, makespan_ms,
           last_completion_ms, sum_load_ms;
  int32_t  status; uint32_t _pad;
} kvro_result;

/* per-query record of a recorded trial; score = router score of i* (LBGR E^_i*j,
 * STATIC s_i*, 0 for the other routers) */
typedef struct { uint32_t worker, hit_tokens, n_victims, _pad; double ttft_ms, latency_ms, score;
                 uint64_t victim_offset; } kvro_query_record;

uint32_t kvro_version(void);

/* ---- primitives (pinned by KATs in tests) ---- */
uint64_t kvro_fmix64(uint64_t x);
void     kvro_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
/* chained block identities of every block of the trace (SURVEY §8c Definitions, A26) */
int      kvro_chain(const kvro_trace* tr, uint64_t* out_hashes /* [offsets[N]] */);

/* identity collisions: adjacent pairs (in (identity, occurrence) order) with equal
 * identity but a different (depth, parent identity, content key) */
int kvro_count_collisions(const kvro_trace* tr, uint64_t* count);

/* one RLS step of the LBGR_RLS residual model (reading A8b): P row-major 4x4,
 * e = target - prediction; exposed for the pins */
void kvro_rls_step(double P[16], double theta[4], const double phi[4], double e, double lam);

/* ---- the replay (one trial) ---- */
int kvro_run(const kvro_config* cfg, const kvro_trace* tr, const kvro_policy* pol,
             uint64_t philox_key, kvro_result* out,
             kvro_query_record* records /* [N] or NULL */,
             uint64_t* victims, uint64_t victims_cap,
             uint32_t* hist /* [bins] or NULL */,
             int check_invariants /* P13 full checks after every query */);

/* ---- single-cache analysis (W = 1, token paths; §3.2) ----
 * Replays the paths of tr (arrivals/costs ignored) through ONE cache of B
 * blocks with the given eviction (LRU / RLT / OPT=Belady).
 * miss_flags[k] = 1 if the k-th block access (flattened Gamma order) missed.
 * If choices != NULL (RLT only) the uniform draws are replaced by the given
 * choice indices (clamped), and arity[k] receives |U| of the k-th draw; used by
 * the exact-expectation enumerator.  n_draws receives the number of draws. */
int kvro_single_replay(const kvro_trace* tr, uint32_t B, uint32_t eviction, uint32_t rlt_fallback,
                       uint64_t philox_key, uint8_t* miss_flags, uint64_t* total_misses,
                       const uint32_t* choices, uint32_t* arity, uint32_t max_draws, uint32_t* n_draws);

/* Phase ledger: the flattened block-access sequence of
 * the complete paths is cut greedily into phases of exactly B distinct blocks (the
 * last possibly fewer), and the single-cache replay (same arguments as
 * kvro_single_replay, Philox draws) is counted per phase v:
 *   ledger[4v+0] distinct blocks of the phase ("new" tokens: first appearance in it)
 *   ledger[4v+1] misses
 *   ledger[4v+2] misses at first appearances (misses on "old" tokens = [1] - [2])
 *   ledger[4v+3] clean tokens: first appearances of blocks that were not in this
 *                eviction policy's cache at the end of phase v-1 (reading A39)
 * *n_phases receives the number of phases; returns 3 if it exceeds max_phases. */
int kvro_phase_ledger(const kvro_trace* tr, uint32_t B, uint32_t eviction, uint32_t rlt_fallback,
                      uint64_t philox_key, uint32_t* ledger, uint32_t max_phases,
                      uint32_t* n_phases);

/* exhaustive minimum number of misses over all leaf-eviction choices
 * (SPEC S:246-254); refuses (returns 3) when the instance is too large */
int kvro_bruteforce_min_misses(const kvro_trace* tr, uint32_t B, uint64_t* min_misses);

/* exact E[misses] and E[misses^2] of RLT by enumerating every uniform choice */
int kvro_rlt_exact_expectation(const kvro_trace* tr, uint32_t B, uint32_t rlt_fallback,
                               double* mean, double* second_moment, uint64_t* leaves);

#ifdef __cplusplus
}
#endif
#endif
