/*
 * kvr.h — C ABI of the B200 replay engine for arxiv 2601.18999
 * ("KV-cache-aware load balancing": randomized leaf-token eviction RLT, Alg. 1,
 * PAPER.md P:220-248; learning-based greedy routing LBGR, Alg. 2).
 *
 * The engine replays the paper's online process (§3.1) for many
 * independent trials on one GPU: for every query j in trace order, every
 * worker i matches the longest cached prefix of the query's block identities
 * (h_ij), the router scores the workers and takes the argmin
 * (Eq. 4-5), the chosen worker applies UpdateCache (Eq. 3,
 * P:115-122) with RLT or Leaf-LRU, and the queue load / latency /
 * TTFT are accounted (Eq. 1-2; Eq. 6).  The exact
 * operation order and every reading of an under-specified passage are listed
 * in DESIGN.md §3 (ids A1..A36).
 *
 * Conventions
 *   - Every function returns kvr_status (0 = OK) and never throws or exits;
 *     kvr_last_error() returns a thread-local message for the last failure.
 *   - The library allocates NO device memory.  Every device buffer (raw trace,
 *     packed trace, workspace, results) is owned by the caller; pointers marked
 *     DEVICE must be device (or managed) memory of the current device.
 *   - Handles (kvr_trace, kvr_sim) are small host objects that BORROW the
 *     caller's buffers; *_destroy frees only the handle.  A handle is
 *     immutable after creation and may be used from several streams, but
 *     concurrent kvr_sim_run calls need distinct workspaces.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *     stream).  Launches are asynchronous unless stated otherwise; argument
 *     validation is synchronous.  Problems found on the device inside one
 *     trial land in that trial's kvr_trial_result.status, never poisoning the
 *     other trials.
 */
#ifndef KVR_H
#define KVR_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define KVR_ABI_VERSION 8u   /* 2: OPT, next-use index, LBGR_RLS; 3: tracker_lag / tracker_grain;
                                4: kvr_sim_config.extended_policies;
                                5: kvr_sim_config.batch_slots (continuous batching);
                                6: kvr_trace_collision_bytes / kvr_trace_check_collisions;
                                7: KVR_TRIAL_BAD_TRACE, kvr_build_id, pooled pending FIFOs
                                   (pending_ring may be as large as the trace);
                                8: KVR_ROUTE_CACHE_AWARE + kvr_policy.ca_* (160-B policy),
                                   tracker_lag up to KVR_MAX_TRACKER_LAG at any capacity,
                                   phase ledger (kvr_trace_build_phases, kvr_sim_run_ledger) */
#define KVR_MAX_TRACKER_LAG 32u

typedef int32_t kvr_status;
enum {
  KVR_OK = 0,
  KVR_ERR_INVALID_ARG = 1,        /* bad pointer / size / parameter / malformed trace */
  KVR_ERR_CAPACITY = 2,           /* some n_in+n_out > B: premise beta*L_max <= B (beta=1) */
  KVR_ERR_UNSUPPORTED = 3,        /* W > 32, B > 65536, no state tier fits, or a trace of
                                     >= 2^32 - 1 blocks (per-worker counters are 32-bit) */
  KVR_ERR_HASH_COLLISION = 4,     /* kvr_trace_check_collisions found two prefixes with one
                                     identity: reload the trace with another hash_salt */
  KVR_ERR_WORKSPACE_TOO_SMALL = 5,
  KVR_ERR_CUDA = 6                /* a CUDA runtime call failed (message in kvr_last_error) */
};

/* per-trial status (kvr_trial_result.status) */
enum {
  KVR_TRIAL_OK = 0,
  KVR_TRIAL_RING_OVERFLOW = 1,    /* a worker's pending-completion FIFO exceeded pending_ring:
                                     the trial stops before the overflowing query's cache update */
  KVR_TRIAL_VICTIM_LOG_FULL = 2,  /* recorded trial produced more victims than its log share */
  KVR_TRIAL_BAD_POLICY = 3,       /* per-trial policy out of range (trial not run): an enum out
                                     of range, rho not in (0,1], delta_t <= 0, a non-finite
                                     parameter (delta_t = +inf allowed), NLMS mu not in [0,2)
                                     (A8), RLS mu not in (0,1] or rls_p0 not finite > 0 */
  KVR_TRIAL_ADMISSION = 4,        /* batching engine: full cache and every leaf in flight
                                     (SPEC S:137); impossible when beta*L_max <= B, which
                                     kvr_sim_run enforces.  Counters of a trial with a nonzero
                                     status are unspecified in the batching engine. */
  KVR_TRIAL_BAD_TRACE = 5         /* kvr_sim_run_multi: d_trial_trace[t] >= n_traces (trial not run) */
};

const char* kvr_last_error(void);
uint32_t kvr_abi_version(void);
/* Hex SHA-256 prefix of the sources this library was compiled from (build provenance:
 * paper_2601_18999_b200/build.py recompiles whenever it differs from the tree's). */
const char* kvr_build_id(void);

/* ------------------------------------------------------------------ trace */
/* Raw trace: block-hashed queries.  Gamma_j = n_in_j input blocks followed by
 * n_out_j output blocks (complete token path; reading A2); a block is
 * block_tokens tokens (A1) so |q_j| = block_tokens*n_in_j.  Block content
 * keys are arbitrary u64; the loader chains them into prefix identities
 *   S_{j,d} = sum_{e<=d} fmix64(c_{j,e} ^ (e+1)*0x9E3779B97F4A7C15 ^ salt),
 *   H_{j,d} = fmix64(S_{j,d})                     (reading A26)
 * so that equal identities <=> equal prefixes (up to 2^-64 collisions). */
typedef struct {
  uint32_t n_queries;             /* N >= 0 */
  uint32_t block_tokens;          /* >= 1 (16 in every config) */
  uint64_t hash_salt;
  uint64_t n_blocks_total;        /* host copy of block_offsets[N] */
  const double*   arrival_ms;     /* DEVICE [N]  finite, >= 0, nondecreasing (A22) */
  const uint32_t* n_in_blocks;    /* DEVICE [N]  >= 1 */
  const uint32_t* n_out_blocks;   /* DEVICE [N]  >= 0 */
  const uint32_t* out_tokens;     /* DEVICE [N]  |a_j| for O_ij = o*|a_j| (A13) */
  const uint64_t* block_offsets;  /* DEVICE [N+1] CSR, offsets[0]=0, offsets[j+1]-offsets[j] = n_in+n_out */
  const uint64_t* block_keys;     /* DEVICE [n_blocks_total] content keys */
} kvr_trace_desc;

typedef struct kvr_trace kvr_trace;

/* Bytes of the packed-trace buffer and of the loader's scratch for `desc`. */
kvr_status kvr_trace_packed_bytes(const kvr_trace_desc* desc, size_t* packed_bytes,
                                  size_t* scratch_bytes);
/* Validate and pack the raw trace into d_packed (16-B aligned DEVICE buffer of
 * at least packed_bytes): per-query 32-B headers, block offsets and the chained
 * identities (one warp per query, warp-scan of the associative chain).
 * SYNCHRONOUS on `stream` (reads back the validation word and max path
 * length).  Returns KVR_ERR_INVALID_ARG for a malformed trace.  The returned
 * handle borrows d_packed, which must outlive it. */
kvr_status kvr_trace_load(const kvr_trace_desc* desc, void* d_packed, size_t packed_bytes,
                          void* d_scratch, size_t scratch_bytes, void* stream, kvr_trace** out);
/* Query counts of a loaded trace (host values). */
kvr_status kvr_trace_info(const kvr_trace* tr, uint32_t* n_queries, uint32_t* max_path_blocks,
                          uint64_t* n_blocks_total);
/* DEVICE pointer to the chained identities H (CSR order, [n_blocks_total]). */
kvr_status kvr_trace_chained_hashes(const kvr_trace* tr, const uint64_t** d_hashes);
kvr_status kvr_trace_destroy(kvr_trace* tr);

/* Optional identity collision check (the chain of reading A26 is a
 * 64-bit hash, so two different prefixes could share an identity with probability
 * ~ n^2 / 2^65).  A block's identity is legitimately determined by (depth, parent
 * identity, content key); the check sorts (identity, occurrence) pairs on the
 * device and counts adjacent occurrences with equal identity but a different
 * tuple -- by induction over depth, zero certifies that every identity names one
 * prefix.  d_block_keys: DEVICE, the raw keys the trace was loaded from
 * ([n_blocks_total], CSR order); d_scratch: DEVICE, caller-owned, >=
 * kvr_trace_collision_bytes.  SYNCHRONOUS on `stream`.  Returns KVR_OK (zero
 * collisions) or KVR_ERR_HASH_COLLISION with *n_collisions = the number of such
 * adjacent pairs (the caller re-salts and reloads); INVALID_ARG / UNSUPPORTED
 * (>= 2^31 blocks) / WORKSPACE_TOO_SMALL as usual. */
kvr_status kvr_trace_collision_bytes(const kvr_trace* tr, size_t* scratch_bytes);
kvr_status kvr_trace_check_collisions(const kvr_trace* tr, const uint64_t* d_block_keys,
                                      void* d_scratch, size_t scratch_bytes, void* stream,
                                      uint64_t* n_collisions);

/* Next-use index for the offline Belady OPT analysis (KVR_EVICT_OPT; P:170,
 * SURVEY §8f #1): nu[o] = index of the next query after the one holding block
 * occurrence o (CSR order) whose path contains the same identity, 0xFFFFFFFF if
 * none.  Built on the device (stable radix sort of (identity, occurrence) pairs,
 * then one pass); asynchronous on `stream`.  d_nu: DEVICE [n_blocks_total] u32,
 * caller-owned; d_scratch: DEVICE, caller-owned, only used during the call.
 * Returns a NEW handle that borrows tr's packed buffer and d_nu (both must
 * outlive it); tr itself is unchanged.  INVALID_ARG for null buffers,
 * WORKSPACE_TOO_SMALL for short ones, UNSUPPORTED for >= 2^31 blocks. */
kvr_status kvr_trace_next_use_bytes(const kvr_trace* tr, size_t* nu_bytes, size_t* scratch_bytes);
kvr_status kvr_trace_build_next_use(const kvr_trace* tr, uint32_t* d_nu, size_t nu_bytes,
                                    void* d_scratch, size_t scratch_bytes, void* stream,
                                    kvr_trace** out);

/* Phase index for the phase-ledger analysis ("we partition Q~ into
 * disjoint phases, where each phase contains exactly B_i distinct tokens"; SURVEY
 * §8f #1; reading A39): the flattened block-access sequence (Gamma_1 || Gamma_2 ...)
 * is cut greedily into phases of exactly B distinct identities (the last possibly
 * fewer).  d_phase (DEVICE, caller-owned, >= phase_bytes) receives
 *   u32 ph[n_blocks_total]  phase of occurrence o | 0x80000000 if o is the first
 *                           appearance of its identity in that phase ("new" token)
 *   u32 nx[n_blocks_total]  index of the identity's next occurrence, 0xFFFFFFFF if none
 *   u32 distinct[n_phases]  distinct identities per phase
 * and *n_phases (host, written before return: SYNCHRONOUS on `stream`) the phase count.
 * d_scratch (DEVICE, caller-owned) is only used during the call.  Returns a NEW handle
 * that borrows tr's packed buffer, tr's next-use index (if any) and d_phase; tr is
 * unchanged.  INVALID_ARG for B = 0 / null buffers, WORKSPACE_TOO_SMALL,
 * UNSUPPORTED for >= 2^31 blocks. */
kvr_status kvr_trace_phase_bytes(const kvr_trace* tr, size_t* phase_bytes, size_t* scratch_bytes);
kvr_status kvr_trace_build_phases(const kvr_trace* tr, uint32_t B, uint32_t* d_phase,
                                  size_t phase_bytes, void* d_scratch, size_t scratch_bytes,
                                  void* stream, uint32_t* n_phases, kvr_trace** out);

/* --------------------------------------------------------------- policies */
/* KVR_EVICT_OPT: offline Belady for competitive ratios: evict the leaf
 * != parent(t) whose next use is furthest; leaves never used again first (lowest
 * slot among them), equal next use -> the deeper one.  Needs W = 1 and a trace
 * with a next-use index (kvr_trace_build_next_use); a per-trial OPT policy
 * without them gets KVR_TRIAL_BAD_POLICY, a default one is refused at
 * kvr_sim_create (W) / kvr_sim_run (index). */
typedef enum { KVR_EVICT_LRU = 0, KVR_EVICT_RLT = 1, KVR_EVICT_OPT = 2 } kvr_eviction;
/* Alg. 1 leaves U = {} undefined (reading A5): */
typedef enum { KVR_RLT_EARLY_RESET = 0,   /* T <- {t}, then uniform over leaves != parent(t) */
               KVR_RLT_UNIFORM_LEAF = 1,  /* uniform over leaves != parent(t), no reset */
               KVR_RLT_LRU_MARKED = 2     /* Leaf-LRU over leaves != parent(t), no draw */
} kvr_rlt_fallback;
typedef enum { KVR_ROUTE_LBGR = 0,           /* Alg. 2 / Eq. 4-6 */
               KVR_ROUTE_STATIC_LINEAR = 1,  /* w_load*pending - w_hit*h/|q| (A17) */
               KVR_ROUTE_THRESHOLD = 2,      /* cache-aware: balance if max>tau*max(1,min) (A16) */
               KVR_ROUTE_ROUND_ROBIN = 3,    /* j mod W */
               KVR_ROUTE_RANDOM = 4,         /* Philox(K,(j,0xFFFFFFFF,2)) */
               KVR_ROUTE_LBGR_RLS = 5,       /* LBGR with the RLS reading of "learning rate
                                                0.992" (reading A8b): exponentially
                                                weighted least squares, forgetting factor mu,
                                                P(0) = rls_p0 * I */
               KVR_ROUTE_CACHE_AWARE = 6     /* SGLang-style cache-aware rule ("switches
                                                between the highest-hit-rate and the least-loaded
                                                routing based on a predefined heuristic load-balance
                                                threshold"; reading A38): pending
                                                loads imbalanced iff max-min > ca_balance_abs AND
                                                max > ca_balance_rel*min -> least loaded; else the
                                                highest match h~ if h~/|q| > ca_cache_threshold,
                                                else the worker with the fewest cached blocks.
                                                Lowest index on ties (A15). */
} kvr_router;

/* Eq. 1 ground truth: Cost = aC*h + aM*(|q|-h) + o*|a| (A13, A14) */
typedef struct { double alpha_cached_ms, alpha_miss_ms, out_ms_per_token; } kvr_service_model;

/* one replay's policy (host struct for the default, DEVICE array for per-trial overrides) */
typedef struct {
  uint32_t eviction, rlt_fallback, router, _pad;
  double est_alpha_cached_ms, est_alpha_miss_ms;  /* Eq. 5 estimator (App. A: 0, 1 ms/token) */
  double rho, delta_t_ms, mu, theta0[4];          /* decay rho in (0,1], dt > 0 (inf = none),
                                                     NLMS step mu (A8), initial theta */
  double tau;                                     /* THRESHOLD */
  double w_hit, w_load;                           /* STATIC_LINEAR */
  double rls_p0;                                  /* LBGR_RLS: initial covariance scale (> 0) */
  uint32_t tracker_lag;    /* App. E ("staleness ... caused by concurrent updates") /
                              reading A29: k in 0..KVR_MAX_TRACKER_LAG; the router's hit
                              estimate h~ for query j is matched on the caches as they were
                              after query j-1-k (the last k cache updates are not yet seen) */
  uint32_t tracker_grain;  /* A29: the router sees grain*floor(m/grain) matched blocks (>= 1);
                              service times (Eq. 1) always use the true h */
  double ca_balance_abs;   /* KVR_ROUTE_CACHE_AWARE (A38): absolute pending-load gap */
  double ca_balance_rel;   /*   relative pending-load ratio */
  double ca_cache_threshold; /* minimum match rate h~/|q| for the highest-match branch */
  uint64_t _pad2;
} kvr_policy;

typedef struct {
  uint32_t W;                      /* workers, 1..32 */
  uint32_t capacity_blocks;        /* B per worker, 1..65536 */
  kvr_service_model truth;
  kvr_policy default_policy;
  uint32_t pending_ring;           /* per-worker cap on pending completions (>= 1; a worker that
                                      would exceed it stops the trial, KVR_TRIAL_RING_OVERFLOW).
                                      beta = 1 engine: the FIFOs of a trial's W workers share one
                                      pool of min(N, W*pending_ring) records in 32-record chunks,
                                      so pending_ring >= N (the trace length) never overflows at a
                                      workspace of ~64 B x N per resident CTA */
  uint32_t record_trials;          /* the first R trials emit per-query records + victim logs */
  uint32_t latency_hist_bins;      /* 0, or 1..256 log-bucket bins (4 per octave, bin 0 = <1 ms) */
  uint32_t force_tier;             /* 0 auto, 1 shared-memory tables, 2 global-memory tables,
                                      3 split (W >= 2: identities + tables in global memory,
                                      tree arrays / bitmaps / stamps in shared memory, two
                                      workers per warp; beta = 1 engine only) */
  uint32_t extended_policies;      /* 1: per-trial policies may use OPT / LBGR_RLS / tracker bias
                                      (runs the kernel instantiation that carries them; implied
                                      when default_policy uses one).  0: such a per-trial policy
                                      gets KVR_TRIAL_BAD_POLICY; the lean instantiation runs. */
  uint32_t batch_slots;            /* 0: the beta = 1 model (update at assignment, single-server
                                      FIFO; readings A3, A12).  1..64: continuous batching with
                                      beta = batch_slots concurrent queries per worker (P:195-208,
                                      Thm 2; readings A30-A36): FIFO wait for a slot, UpdateCache
                                      at dequeue, in-flight paths pinned.  Runs kvr_batch.cu;
                                      policies: LRU/RLT with every router (OPT and tracker bias
                                      -> INVALID_ARG / KVR_TRIAL_BAD_POLICY); premise
                                      beta * L_max <= B checked by kvr_sim_run (KVR_ERR_CAPACITY).
                                      A recorded trial's victim share is split evenly over the
                                      W workers, each logging its victims in dequeue order. */
} kvr_sim_config;

typedef struct kvr_sim kvr_sim;
kvr_status kvr_sim_create(const kvr_sim_config* cfg, kvr_sim** out);
kvr_status kvr_sim_destroy(kvr_sim* sim);

/* per-trial outputs */
typedef struct {
  uint64_t queries, hit_tokens, input_tokens, probes, inserted_blocks, evictions,
           rlt_draws, rlt_resets, rlt_fallbacks, max_pending, decision_digest;
  double   sum_latency_ms, sum_ttft_ms, max_latency_ms,
           makespan_ms,          /* max_i P_i^(N) (A21) */
           last_completion_ms,   /* max_i F_i */
           sum_load_ms;          /* sum_i P_i */
  int32_t  status; uint32_t _pad;
} kvr_trial_result;

/* per-query record of a recorded trial (score = router score of i*: LBGR
 * E^_{i*j}, STATIC s_{i*}, 0 otherwise; victim_offset indexes the trial's
 * victim-log share) */
typedef struct { uint32_t worker, hit_tokens, n_victims, _pad; double ttft_ms, latency_ms, score;
                 uint64_t victim_offset; } kvr_query_record;

/* Tier and launch shape chosen for (sim, trace): tier 1 = per-worker tables in
 * shared memory, 2 = in global memory (L2-resident), 3 = split (identities + tables
 * global, the rest shared; chosen automatically for W > 16 when tier 1 does not fit);
 * dynamic smem per CTA. */
kvr_status kvr_sim_plan(const kvr_sim* sim, uint32_t max_path_blocks, uint32_t* tier,
                        size_t* smem_bytes, uint32_t* ctas_per_sm);
/* Workspace bytes for a run of n_trials whose longest path is max_path_blocks. */
kvr_status kvr_sim_workspace_bytes(const kvr_sim* sim, const kvr_trace* trace,
                                   uint32_t n_trials, size_t* bytes);

/* Run n_trials independent replays of `trace`.
 *   d_philox_keys [n_trials] DEVICE   Philox4x32-10 key of each trial (RLT draws, RANDOM router)
 *   d_policies    [n_trials] DEVICE or NULL (-> default_policy)
 *   d_results     [n_trials] DEVICE   written for every trial
 *   d_latency_hist [n_trials*bins] DEVICE or NULL
 *   d_records     [record_trials*N] DEVICE or NULL
 *   d_victims     [victims_cap] DEVICE or NULL: recorded trial r owns entries
 *                 [r*victims_cap/record_trials, (r+1)*victims_cap/record_trials)
 *   d_workspace   DEVICE, >= kvr_sim_workspace_bytes(...)
 * Asynchronous on `stream`. */
kvr_status kvr_sim_run(kvr_sim* sim, const kvr_trace* trace, uint32_t n_trials,
                       const uint64_t* d_philox_keys, const kvr_policy* d_policies,
                       kvr_trial_result* d_results, uint32_t* d_latency_hist,
                       kvr_query_record* d_records, uint64_t* d_victims, uint64_t victims_cap,
                       void* d_workspace, size_t workspace_bytes, void* stream);

/* Same, for trials spread over several traces in ONE launch (keeps every SM
 * busy across small cells): trial t replays traces[d_trial_trace[t]].
 * Records use a stride of max_j N_j per recorded trial. */
kvr_status kvr_sim_workspace_bytes_multi(const kvr_sim* sim, uint32_t n_traces,
                                         const kvr_trace* const* traces, uint32_t n_trials,
                                         size_t* bytes);
kvr_status kvr_sim_run_multi(kvr_sim* sim, uint32_t n_traces, const kvr_trace* const* traces,
                             const uint32_t* d_trial_trace, uint32_t n_trials,
                             const uint64_t* d_philox_keys, const kvr_policy* d_policies,
                             kvr_trial_result* d_results, uint32_t* d_latency_hist,
                             kvr_query_record* d_records, uint64_t* d_victims,
                             uint64_t victims_cap, void* d_workspace, size_t workspace_bytes,
                             void* stream);

/* Phase-ledger run (Lemmas 1-3, Thm 3): the same replay as
 * kvr_sim_run on a trace from kvr_trace_build_phases (built for this sim's B), W = 1
 * only (the single-cache analysis of §3.2), every trial counting per phase v:
 *   d_ledger[t*4*n_phases + 4v + 0]  distinct identities of the phase
 *                             + 1    misses
 *                             + 2    misses at first appearances ("new" tokens; the
 *                                    misses on "old" tokens are [1] - [2])
 *                             + 3    clean tokens: first appearances of identities that
 *                                    were not in this trial's cache at the end of phase
 *                                    v-1 (reading A39)
 * d_ledger: DEVICE u32 [n_trials * 4 * n_phases].  Records / histograms / victims are
 * not produced.  INVALID_ARG for W != 1, a trace without a phase index or one built
 * for another B, or batch_slots > 0.  Asynchronous on `stream`. */
kvr_status kvr_sim_run_ledger(kvr_sim* sim, const kvr_trace* trace, uint32_t n_trials,
                              const uint64_t* d_philox_keys, const kvr_policy* d_policies,
                              kvr_trial_result* d_results, uint32_t* d_ledger,
                              void* d_workspace, size_t workspace_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* KVR_H */
