// kvr_internal.h — layouts shared by the host API (kvr_api.cu) and the kernels
// (kvr_pack.cu, kvr_kernel.cu, kvr_batch.cu, kvr_nextuse.cu).  Not part of the public ABI (include/kvr.h).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <algorithm>
#include <stdint.h>

#include "kvr.h"

namespace kvr {

constexpr uint32_t kNumStages = 4;      // query staging ring depth (bulk-async copies)
constexpr uint32_t kAhead = 2;          // queries staged ahead; a buffer lives 2 barriers
                                        // after its query for the deferred apply
constexpr uint32_t kMaxTraces = 64;     // traces per multi-trace launch
constexpr uint32_t kFifoRecBytes = 64;  // one pending completion {c,a,E^,phi0..2,C^,k_a}
constexpr uint32_t kFifoChunk = 32;     // records per chunk of a CTA's pending-FIFO pool
constexpr uint32_t kMaxHistBins = 256;
constexpr uint32_t kMaxW = 32;
constexpr uint32_t kMaxLag = KVR_MAX_TRACKER_LAG;   // stale-tracker lag k (A29)
constexpr uint32_t kLagRing = kMaxLag + 2;          // per-CTA ring of the last updates

// Packed trace, per query: a 32-byte header, bulk-copied with the query's hashes.
struct __align__(16) QueryHdr {
  double arrival_ms;
  uint64_t block_off;   // offset of the query's first identity in the hash array
  uint32_t n_in, n_out, out_tokens, _pad;
};
static_assert(sizeof(QueryHdr) == 32, "header is 32 B");

struct TraceDev {
  const QueryHdr* hdr;  // [N]
  const uint64_t* hash; // [total] chained identities, CSR order
  const uint32_t* nu;   // [total] next-use index (offline OPT) or null
  const uint32_t* ph;   // [total] phase | first-appearance bit (phase ledger) or null
  const uint32_t* nx;   // [total] next occurrence of the identity (phase ledger)
  const uint32_t* distinct;   // [n_phases] distinct identities per phase
  uint32_t N, max_n, block_tokens, n_phases;
};

// packed buffer = [QueryHdr x N][pad to 16][u64 hash x total]
inline size_t packed_hash_offset(uint32_t N) { return ((size_t)N * sizeof(QueryHdr) + 15) & ~(size_t)15; }
inline size_t packed_bytes(uint32_t N, uint64_t total) { return packed_hash_offset(N) + total * 8 + 16; }

__host__ __device__ constexpr size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }

// Per-trial policy checks applied on the device to every per-trial policy (the host
// checks the default one with messages in kvr_api.cu): enums in range, rho in (0, 1],
// delta_t > 0 (+inf = no decay), every other parameter finite (x - x == 0 iff finite),
// NLMS step 0 <= mu < 2 (reading A8), RLS forgetting factor in (0, 1] (A8b).
__host__ __device__ inline bool policy_valid(const kvr_policy& p) {
  auto fin = [](double v) { return (v - v) == 0.0; };
  if (p.eviction > KVR_EVICT_OPT || p.rlt_fallback > KVR_RLT_LRU_MARKED ||
      p.router > KVR_ROUTE_CACHE_AWARE || p.tracker_lag > kMaxLag || p.tracker_grain < 1)
    return false;
  if (!(p.rho > 0.0 && p.rho <= 1.0) || !(p.delta_t_ms > 0.0)) return false;
  if (!fin(p.est_alpha_cached_ms) || !fin(p.est_alpha_miss_ms) || !fin(p.mu) ||
      !fin(p.theta0[0]) || !fin(p.theta0[1]) || !fin(p.theta0[2]) || !fin(p.theta0[3]) ||
      !fin(p.tau) || !fin(p.w_hit) || !fin(p.w_load) || !fin(p.ca_balance_abs) ||
      !fin(p.ca_balance_rel) || !fin(p.ca_cache_threshold))
    return false;
  if (p.router == KVR_ROUTE_LBGR && !(p.mu >= 0.0 && p.mu < 2.0)) return false;
  if (p.router == KVR_ROUTE_LBGR_RLS &&
      !(p.mu > 0.0 && p.mu <= 1.0 && p.rls_p0 > 0.0 && fin(p.rls_p0)))
    return false;
  return true;
}

// Per-worker cache state (one worker = one warp), latency-critical part, held in
// shared memory (tier 1, u16 slot ids) or global memory (tier 2, u32 slot ids):
// slot arrays of the prefix tree (identity, parent slot, child count), an
// open-addressed linear-probing table identity -> slot with tombstones, and the
// LEAF / MARK bitmaps (RLT's marking set T is exactly the MARK bits, T in S).
struct WorkerLayout {
  uint32_t B, T, nwords, idx_bytes;
  uint32_t rebuild_at, _pad;   // rebuild the table when live + tombstones exceed this
  size_t off_key, off_parent, off_nchild, off_table, off_leaf, off_mark, off_stamp, bytes;
  // split layout (kernel tier 4): identities + table in global memory (gbytes per worker,
  // offsets from the global base), tree arrays / bitmaps / stamps in shared memory
  // (sbytes per worker, offsets from the shared base); unsplit: gbytes = sbytes = bytes
  size_t gbytes, sbytes;
};

inline WorkerLayout make_layout(uint32_t B, uint32_t idx_bytes, bool split = false) {
  WorkerLayout L{};
  L.B = B;
  uint32_t T = 4;
  while (T < 4 * B) T <<= 1;     // live load <= 1/4; rebuilt when live + tombstones > 1/2
  L.T = T;
  L.nwords = (B + 31) / 32;
  L.idx_bytes = idx_bytes;
  L.rebuild_at = T >> 1;
  if (split) {
    // (measured: the table on chip at half the size, T = 2B rebuilt at 3T/4, costs more
    // in longer probe chains against the L2-resident identities than it saves: 10.5 ->
    // 8.1 M query-replays/s at W = 32, so it stays in global memory at T = 4B)
    size_t g = 0, o = 0;
    L.off_key = g;    g = align16(g + (size_t)B * 8);
    L.off_table = g;  g = align16(g + (size_t)T * idx_bytes);
    L.off_parent = o; o = align16(o + (size_t)B * idx_bytes);
    L.off_nchild = o; o = align16(o + (size_t)B * idx_bytes);
    L.off_leaf = o;   o = align16(o + (size_t)L.nwords * 4);
    L.off_mark = o;   o = align16(o + (size_t)L.nwords * 4);
    L.off_stamp = o;  o = align16(o + (size_t)B * 2);
    L.gbytes = g;
    L.sbytes = o;
    L.bytes = g + o;
    return L;
  }
  size_t o = 0;
  L.off_key = o;    o = align16(o + (size_t)B * 8);
  L.off_parent = o; o = align16(o + (size_t)B * idx_bytes);
  L.off_nchild = o; o = align16(o + (size_t)B * idx_bytes);
  L.off_table = o;  o = align16(o + (size_t)T * idx_bytes);
  L.off_leaf = o;   o = align16(o + (size_t)L.nwords * 4);
  L.off_mark = o;   o = align16(o + (size_t)L.nwords * 4);
  L.off_stamp = o;  o = align16(o + (size_t)B * 2);     // Leaf-LRU recency stamps (u16)
  L.bytes = o;
  L.gbytes = o;
  L.sbytes = o;
  return L;
}

// Per-worker auxiliary state in global memory (L2-resident): the Leaf-LRU recency
// log (append-only ring of (stamp, slot), compacted when full; validated by the
// per-slot stamps of the worker state), the LBGR_RLS matrix, and for the extended
// policies the stale tracker's mirror of the worker's cache (identity per slot and a
// table identity -> slot, reading A29) and the per-slot last access (phase ledger).
struct AuxLayout {
  uint32_t log_cap, T;
  size_t off_log, off_rls, off_mkey, off_mtab, off_last, bytes;
};

inline AuxLayout make_aux(uint32_t B, uint32_t max_n, uint32_t T, bool ext) {
  AuxLayout A{};
  // live entries after a compaction <= B; 4x headroom keeps the amortised compaction
  // cost at ~1.25 entries read per entry appended and the log L2-resident
  uint32_t C = 64;
  while (C < 4 * (B + max_n + 32)) C <<= 1;
  A.log_cap = C;
  A.T = T;
  size_t o = 0;
  // u32 entries (stamp << 16 | slot); OPT reuses the region for its u64 per-slot keys
  A.off_log = o;   o = align16(o + std::max((size_t)C * 4, (size_t)B * 8));
  A.off_rls = o;   o = align16(o + 16 * 8);
  A.off_mkey = o;  o = align16(o + (ext ? (size_t)B * 8 : 0));
  A.off_mtab = o;  o = align16(o + (ext ? (size_t)T * 4 : 0));
  A.off_last = o;  o = align16(o + (ext ? (size_t)B * 4 : 0));
  A.bytes = (o + 127) & ~(size_t)127;
  return A;
}

// Per-CTA ring of the last kLagRing cache updates of the trial (stale tracker, A29):
// entry = header, then the update's per-miss slots (slot | evicted << 31).
struct __align__(16) LagHdr {
  uint64_t block_off;     // the query's first identity in the trace
  uint32_t j, worker, kf, M;
  uint32_t _pad[2];
};
static_assert(sizeof(LagHdr) == 32, "lag header is 32 B");
inline size_t lag_entry_bytes(uint32_t max_n) { return align16(sizeof(LagHdr) + 4 * (size_t)max_n); }

// Pending-completion FIFOs of one CTA's trial: every worker's FIFO is a linked list
// of 32-record chunks from one per-CTA pool (link words, then the chunks).  Chunks a
// worker empties go to that worker's free list and are reused first (LIFO, so the
// few chunks in use stay in L2); new ones come from a bump counter.  A worker holds
// at most ceil(pending/32) + 1 chunks, so ceil(N/32) + 2W chunks never run out, and
// W (ceil(ring/32) + 2) bound it when the per-worker cap `ring` is smaller.
struct FifoLayout {
  uint32_t chunks;
  size_t off_rec, bytes;
};

inline FifoLayout make_fifo(uint32_t W, uint32_t ring, uint32_t max_N) {
  FifoLayout F{};
  const uint64_t by_trace = ((uint64_t)max_N + kFifoChunk - 1) / kFifoChunk + 2ull * W;
  const uint64_t by_ring = (uint64_t)W * (((uint64_t)ring + kFifoChunk - 1) / kFifoChunk + 2);
  F.chunks = (uint32_t)(by_trace < by_ring ? by_trace : by_ring);
  F.off_rec = ((size_t)F.chunks * 4 + 127) & ~(size_t)127;
  F.bytes = F.off_rec + (size_t)F.chunks * kFifoChunk * kFifoRecBytes;
  return F;
}

// Control block at the start of dynamic shared memory.
struct __align__(16) Ctrl {
  unsigned long long mbar[kNumStages];
  double score[2][kMaxW];
  uint32_t mhit[2][kMaxW];
  uint32_t npend[2][kMaxW];
  uint32_t csize[2][kMaxW];    // cached blocks per worker (CACHE_AWARE router, A38)
  // (each worker's final Eq. 2 load P and last completion F go to score[0] / score[1] at
  // the end of a trial, when the scores are dead: 512 B of shared memory less)
  double sum_lat, sum_ttft, max_lat;
  unsigned long long digest, dkey, vcursor;
  unsigned long long cnt[10];   // probes, inserted, evictions, draws, resets, fallbacks, hit, in, queries, maxpend
  kvr_policy pol;                      // this trial's policy
  uint32_t trial, status, abortf[2];   // abort flag double-buffered by query parity
  uint32_t fifo_bump, _pad_f[3];       // next never-used chunk of the CTA's FIFO pool
  uint32_t* led;                       // phase ledger of this trial (extended policies) or null
  const uint32_t* lph;                 // its trace's phase index (ph, nx)
  const uint32_t* lnx;
};

inline size_t ctrl_bytes() { return align16(sizeof(Ctrl)); }
inline size_t stage_bytes(uint32_t max_n) { return align16(sizeof(QueryHdr) + 8 * ((size_t)max_n + 2)); }
// Per-warp (worker) scalar and sequential state of one trial.
struct WorkerRegs {
  uint32_t size, cntT, used, wq, lhead, ltail;
  uint64_t e;                      // RLT draw counter e_i
  uint32_t c_ins, c_evict, c_draws, c_resets, c_fb;
};

// Per-warp shared-memory block: the pending (deferred) apply of this worker's
// last update, its per-miss slots (Leaf-LRU takes its victims in place), the overlay victim bitmap
// staging area, and the worker's trial counters.
struct __align__(16) WarpSm {
  double ttft, lat, score;
  unsigned long long vc;           // victim-log offset of the pending update
  unsigned long long c_probes, c_hit, c_in;
  uint32_t active, j, buf, n, kf, M, m, nev, h, ltail0, wq, p0;
  uint32_t c_q, c_maxp;
  uint32_t ftail, ffree;           // FIFO: next record index to write; free-chunk list head
  WorkerRegs x;                    // RLT decision state in/out, e_i and counters
  uint32_t x_ri;                   // next unused draw of x_rbuf
  uint32_t m_used, m_size, m_cur;  // stale-tracker mirror: table fill, slots, next ring entry
  unsigned long long x_rbuf[32];   // RLT: 32 counter-based draws, one per lane
};
inline size_t scratch_bytes(uint32_t) { return align16(sizeof(WarpSm)); }
// Per-miss slot buffers of an update ([max_n] slot | evicted << 31, then the [32] victim
// bitmap staging of the overlay): at most two updates are live at once (the one being
// decided, and the previous query's pending apply), so a CTA holds two, by query parity.
inline size_t slotbuf_bytes(uint32_t max_n) { return align16(4 * ((size_t)max_n + 32)); }

// Save area of one worker's query-loop scalars when a warp serves two workers (split
// tier): uniform doubles (P, F, P~, theta, front completion time), tick count, FIFO
// head / count, the front record (lanes 0..7) and the overlay victim bitmap (per lane).
struct __align__(16) WSave {
  double u[8];
  unsigned long long k;
  uint32_t fh, fn;
  double fr[8];
  uint32_t vb[32];
};

// ---- continuous batching (kvr_batch.cu; readings A30-A36) ----
// one assigned query: waiting in the FIFO ring, then in a batch slot (c set at dequeue)
struct __align__(16) BFlight {
  double c, a, Ehat, phi0, phi1, phi2, Chat;
  uint64_t ka;
  uint32_t j, _p;
};
static_assert(sizeof(BFlight) == 80, "flight record is 80 B");

// Per-worker state of the batching kernel: u16 (shared-memory tier) or u32
// (global tier) slot ids, all-ones = NONE,
// pin counts (u8, beta <= 64) per slot, LEAFU / MARK bitmaps, the table
// (T >= 2B, linear probing, backward-shift deletion), beta in-flight records,
// the LBGR_RLS matrix and the staged path of the query being dequeued.
struct BatchLayout {
  uint32_t B, T, beta, max_n, nwords, _pad;
  size_t off_key, off_stamp, off_parent, off_nchild, off_depth, off_table, off_pin, off_leafu,
      off_mark, off_fl, off_rls, off_gam, bytes;
};

__host__ __device__ constexpr BatchLayout make_batch_layout(uint32_t B, uint32_t beta, uint32_t max_n,
                                                        uint32_t idx_bytes) {
  BatchLayout L{};
  L.B = B;
  L.beta = beta;
  L.max_n = max_n;
  uint32_t T = 64;
  while (T < 2 * B) T <<= 1;
  L.T = T;
  size_t o = 0;
  L.off_key = o;    o = align16(o + (size_t)B * 8);
  L.off_stamp = o;  o = align16(o + (size_t)B * 4);
  L.off_parent = o; o = align16(o + (size_t)B * idx_bytes);
  L.off_nchild = o; o = align16(o + (size_t)B * idx_bytes);
  L.off_depth = o;  o = align16(o + (size_t)B * idx_bytes);
  L.off_table = o;  o = align16(o + (size_t)T * idx_bytes);
  L.nwords = (B + 31) / 32;
  L.off_pin = o;    o = align16(o + (size_t)B + 4);
  L.off_leafu = o;  o = align16(o + (size_t)L.nwords * 4);   // unpinned-leaf bitmap
  L.off_mark = o;   o = align16(o + (size_t)L.nwords * 4);   // RLT marking set T
  L.off_fl = o;     o = align16(o + (size_t)beta * sizeof(BFlight));
  L.off_rls = o;    o = align16(o + 16 * 8);
  L.off_gam = o;    o = align16(o + (size_t)max_n * 8);
  L.bytes = o;
  return L;
}

struct ReplayParams {
  TraceDev traces[kMaxTraces];
  const uint32_t* trial_trace;   // [n_trials] or null
  uint32_t n_traces, n_trials, W, B;
  uint32_t ring, record_trials, rec_stride, bins;
  uint32_t stage_bytes, scratch_bytes, slotbuf_bytes;
  uint32_t max_n, _pad1;
  WorkerLayout lay;
  AuxLayout aux;
  FifoLayout fifo;
  uint8_t* fifo_base;            // [grid][fifo.bytes] pending-FIFO pools (beta = 1 engine)
  uint8_t* lag_base;             // [grid][kLagRing][lag_entry] update rings (extended policies)
  uint32_t lag_entry, ledger_stride;   // bytes per ring entry; u32 per trial of the ledger
  uint32_t* ledger;              // phase ledger [n_trials][ledger_stride] or null
  double* divtab_base;           // [grid][max_n + 1] exact (bt * k) / 1000 per CTA (global, L1)
  kvr_service_model truth;
  kvr_policy defpol;
  const kvr_policy* policies;
  const uint64_t* keys;
  kvr_trial_result* results;
  uint32_t* hist;
  kvr_query_record* records;
  uint64_t* victims;
  uint64_t victims_per_trial;
  uint8_t* aux_base;             // [grid][W][aux.bytes]
  uint8_t* gstate;               // [grid][W][lay.bytes] (global tier) or null
  unsigned int* work_counter;
  // batching kernel only (kvr_batch.cu)
  uint32_t beta, bglobal;        // batch slots; per-worker state in gstate (1) or smem (0)
  BatchLayout blay;              // aux_base = [grid][W][ring] BFlight waiting FIFOs
  uint64_t* blog_base;           // [grid][W][blog_cap] Leaf-LRU recency logs (stamp << 32 | slot)
  uint32_t blog_cap, _pad3;
};

// exact table (bt * k) / 1000.0 for k = 0..max_n (the A9 feature scaling of integer token counts)
inline size_t divtab_bytes(uint32_t max_n) { return align16(8 * ((size_t)max_n + 1)); }

// Leaf-LRU recency log of the batching engine: one valid entry per cached node, 2x
// headroom (compacted in place when full)
inline uint32_t batch_log_cap(uint32_t B, uint32_t max_n) {
  uint32_t C = 64;
  while (C < 2 * (B + max_n + 32)) C <<= 1;
  return C;
}

inline size_t smem_base_bytes(uint32_t W, uint32_t max_n) {
  return ctrl_bytes() + kNumStages * stage_bytes(max_n) + (size_t)W * scratch_bytes(max_n) +
         2 * slotbuf_bytes(max_n);
}

// launchers (kvr_pack.cu / kvr_kernel.cu)
cudaError_t launch_pack(const kvr_trace_desc& d, QueryHdr* hdr, uint64_t* hash, uint32_t* scratch,
                        cudaStream_t s);
// tier 1 = tables in shared memory (u16 slot ids), 2 = tables in global memory (u32 slot ids),
// 3 = global memory with u16 ids (W > 16), 4 = split: identities + tables in global memory,
// tree arrays / bitmaps / stamps in shared memory (u16 ids, W > 16)
// ext: the instantiation with the extended policies (OPT, LBGR_RLS, tracker bias)
cudaError_t replay_attrs(uint32_t tier, size_t smem, int* ctas_per_sm, uint32_t W, bool ext);
cudaError_t launch_replay(uint32_t tier, const ReplayParams& p, uint32_t grid, size_t smem,
                          cudaStream_t s, bool ext);
// continuous-batching kernel (kvr_batch.cu)
size_t batch_ctrl_bytes();
cudaError_t batch_attrs(size_t smem, int* ctas_per_sm, uint32_t W, bool global, uint32_t B);
cudaError_t launch_batch(const ReplayParams& p, uint32_t grid, size_t smem, cudaStream_t s);
// next-use index for the offline OPT analysis (kvr_nextuse.cu)
cudaError_t next_use_scratch_bytes(uint64_t n_blocks, size_t* bytes);
cudaError_t build_next_use(const QueryHdr* hdr, uint32_t N, const uint64_t* hash, uint64_t n,
                           uint32_t* nu, void* scratch, size_t scratch_bytes, cudaStream_t s);
// identity collision check (kvr_nextuse.cu): adjacent equal identities with a
// different (depth, parent identity, content key) after the (identity, occurrence) sort
cudaError_t collision_scratch_bytes(uint64_t n_blocks, size_t* bytes);
cudaError_t count_collisions(const QueryHdr* hdr, uint32_t N, const uint64_t* hash,
                             const uint64_t* block_keys, uint64_t n, void* scratch,
                             size_t scratch_bytes, cudaStream_t s, unsigned long long* h_count);
// phase index of the phase ledger (kvr_nextuse.cu): out = [n] ph | [n] nx | [<= n] distinct
cudaError_t phase_scratch_bytes(uint64_t n_blocks, size_t* bytes);
cudaError_t build_phases(const uint64_t* hash, uint64_t n, uint32_t B, uint32_t* out, void* scratch,
                         size_t scratch_bytes, cudaStream_t s, uint32_t* h_n_phases);
// phase profiler (profiling build, -DKVR_PHASE_PROFILE); cudaErrorNotSupported otherwise
cudaError_t phase_cycles(unsigned long long* out16, int reset);
cudaError_t batch_phase_cycles(unsigned long long* out32, int reset);   // batching kernel

}  // namespace kvr
