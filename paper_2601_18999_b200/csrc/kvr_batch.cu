// kvr_batch.cu — the continuous-batching replay kernel (beta >= 1 concurrent
// queries per worker, readings A30-A36).
//
// Model ("the system handles beta distinct queries concurrently",
// Thm 2; the SPEC's event engine S:499-549): every worker has beta batch slots;
// an assigned query waits FIFO until a slot frees; UpdateCache (Eq. 3, Alg. 1 /
// Leaf-LRU) runs when it is DEQUEUED and yields the true h; its blocks stay
// pinned until its completion, so evictions pick unpinned leaves only.
//
// Execution: one CTA per trial (persistent over a work counter), one warp per
// worker.  Per query j: every warp catches its worker up to a_j (decay ticks,
// completions in time order, the dequeues they trigger — each warp mutates only
// its own cache, so the W catch-ups run in parallel), matches the query's
// prefix (lane-parallel probes + ballot) and scores; one __syncthreads; every
// warp takes the same argmin; the chosen warp enqueues the query (or starts it
// at once if a slot is free).  Scores, matches and the abort flag are
// double-buffered by query parity so one barrier per query suffices.
//
// Per-worker state (tree slots, open-addressed identity -> slot table with
// tombstones, pin counts, RLT marks, in-flight records, staged path) lives in shared
// memory when W of them fit, else in the workspace (L2-resident); the waiting FIFO is a
// ring in the workspace.  Victim selection: Leaf-LRU takes the first unpinned valid
// entries of a per-worker recency log, 32 per ballot; RLT (B <= 1024) keeps LEAFU, MARK
// and U = LEAFU & ~MARK in registers (lane l: word l) with U's prefix counts and selects
// each victim with two CREDUX reductions, fetching the victim's parent / child count /
// pin speculatively; its table erases, digest terms and the loaded slots' arrays are
// written in one lane-parallel pass after the decisions.  LEAFU is maintained
// incrementally: hits/loads pin (clear), unpins of a childless node and evictions that
// empty an unpinned parent set it.
#include <math.h>

#include "kvr_device.cuh"
#include "kvr_internal.h"

namespace kvr {

extern __shared__ __align__(16) uint8_t kvr_bsmem[];

#ifdef KVR_PHASE_PROFILE
// phase profiler of the batching kernel (profiling build only): cycles summed by lane 0
__device__ unsigned long long g_bphase[32];
#define BP_T0(v) unsigned long long v = clock64()
#define BP_ACC(ph, v)                                                        \
  do {                                                                       \
    const unsigned long long _n = clock64();                                 \
    if ((threadIdx.x & 31) == 0) atomicAdd(&g_bphase[ph], _n - (v));         \
    v = _n;                                                                  \
  } while (0)
#define BP_CNT(ph, cnt)                                                                 \
  do {                                                                                  \
    if ((threadIdx.x & 31) == 0) atomicAdd(&g_bphase[ph], (unsigned long long)(cnt));   \
  } while (0)
#else
#define BP_T0(v) (void)0
#define BP_ACC(ph, v) (void)0
#define BP_CNT(ph, cnt) (void)0
#endif

namespace {

constexpr uint32_t kNone = 0xffffffffu;
#ifndef KVR_BATCH_REBUILD_NUM
#define KVR_BATCH_REBUILD_NUM 6u   // rebuild the table when live + tombstones > (num / 8) T
#endif

// Idx = u16 (shared-memory tier) or u32 (global tier) slot ids; all-ones = NONE
template <typename Idx>
struct BView {
  static constexpr uint32_t NIL = (uint32_t)(Idx)~(Idx)0;
  static constexpr uint32_t TOMB = NIL - 1u;
  uint64_t* key;
  uint32_t* stamp;
  Idx *parent, *nchild, *depth, *table;
  uint8_t* pin;
  uint32_t *leafu, *markb;   // bitmaps: unpinned leaves (eviction candidates), RLT marks T
  BFlight* fl;
  double* rlsP;
  uint64_t* gam;
  uint32_t tmask;
};

// kFixedB > 0: the capacity is a compile-time constant (B = 512, every BASELINE config
// that replays W > 1 workers), so the offsets of the fixed-size arrays fold into the
// shared-memory instructions instead of being rematerialised from the parameters
template <typename Idx, int kFixedB>
__device__ __forceinline__ BView<Idx> bview(uint8_t* base, const BatchLayout& Lr) {
  constexpr BatchLayout LF = make_batch_layout(kFixedB > 0 ? kFixedB : 64, 1, 1, sizeof(Idx));
  const BatchLayout& L = Lr;
  if constexpr (kFixedB > 0) {
    BView<Idx> v;
    v.key = reinterpret_cast<uint64_t*>(base + LF.off_key);
    v.stamp = reinterpret_cast<uint32_t*>(base + LF.off_stamp);
    v.parent = reinterpret_cast<Idx*>(base + LF.off_parent);
    v.nchild = reinterpret_cast<Idx*>(base + LF.off_nchild);
    v.depth = reinterpret_cast<Idx*>(base + LF.off_depth);
    v.table = reinterpret_cast<Idx*>(base + LF.off_table);
    v.pin = base + LF.off_pin;
    v.leafu = reinterpret_cast<uint32_t*>(base + LF.off_leafu);
    v.markb = reinterpret_cast<uint32_t*>(base + LF.off_mark);
    v.fl = reinterpret_cast<BFlight*>(base + LF.off_fl);       // depends on B only
    v.rlsP = reinterpret_cast<double*>(base + L.off_rls);      // after the beta records
    v.gam = reinterpret_cast<uint64_t*>(base + L.off_gam);
    v.tmask = LF.T - 1;
    return v;
  }
  BView<Idx> v;
  v.key = reinterpret_cast<uint64_t*>(base + L.off_key);
  v.stamp = reinterpret_cast<uint32_t*>(base + L.off_stamp);
  v.parent = reinterpret_cast<Idx*>(base + L.off_parent);
  v.nchild = reinterpret_cast<Idx*>(base + L.off_nchild);
  v.depth = reinterpret_cast<Idx*>(base + L.off_depth);
  v.table = reinterpret_cast<Idx*>(base + L.off_table);
  v.pin = base + L.off_pin;
  v.leafu = reinterpret_cast<uint32_t*>(base + L.off_leafu);
  v.markb = reinterpret_cast<uint32_t*>(base + L.off_mark);
  v.fl = reinterpret_cast<BFlight*>(base + L.off_fl);
  v.rlsP = reinterpret_cast<double*>(base + L.off_rls);
  v.gam = reinterpret_cast<uint64_t*>(base + L.off_gam);
  v.tmask = L.T - 1;
  return v;
}

// ---- identity -> slot table: linear probing, tombstones ----
// An erased entry becomes a tombstone (probes continue past it, inserts reuse it), or
// EMPTY when its successor is EMPTY (no probe path can run through it).  Lanes may erase
// concurrently (distinct slots): an entry only turns EMPTY when its successor was EMPTY
// when read, and nothing turns an EMPTY entry back during an erase pass, so no live
// entry is ever cut off from its home.  live + tombstones is counted per worker (x.used)
// and the table is rebuilt without tombstones when it exceeds 3T/4 (KVR_BATCH_REBUILD_NUM).
template <typename Idx>
__device__ __forceinline__ uint32_t t_find(const BView<Idx>& S, uint64_t t) {
  uint32_t i = (uint32_t)t & S.tmask;
  for (;;) {
    const uint32_t s = S.table[i];
    if (s == BView<Idx>::NIL) return kNone;
    if (s != BView<Idx>::TOMB && S.key[s] == t) return s;
    i = (i + 1) & S.tmask;
  }
}
// One 32-block window of a prefix match (lane l: block base + l; blocks >= nq miss): the
// lanes step their probe chains together and the warp stops once the prefix is decided
// -- the first lane that is not a hit has finished with a miss -- instead of waiting for
// the window's longest chain.  Returns the hit ballot, exact up to its first zero bit;
// slot = the lane's slot when it is a known hit, else kNone.
template <typename Idx>
__device__ __forceinline__ uint32_t b_probe_window(const BView<Idx>& S, const uint64_t* H, uint32_t base,
                                                   uint32_t nq, uint32_t lane, uint32_t& slot) {
  const uint32_t d = base + lane;
  bool done = d >= nq, hit = false;
  const uint64_t t = done ? 0ull : H[d];
  uint32_t i = (uint32_t)t & S.tmask;
  slot = kNone;
  for (;;) {
    if (!done) {
      const uint32_t s = S.table[i];
      if (s == BView<Idx>::NIL) {
        done = true;
      } else if (s != BView<Idx>::TOMB && S.key[s] == t) {
        done = true;
        hit = true;
        slot = s;
      } else {
        i = (i + 1) & S.tmask;
      }
    }
    const uint32_t dn = __ballot_sync(kFull, done);
    const uint32_t hb = __ballot_sync(kFull, done && hit);
    if (hb == kFull || dn == kFull) return hb;
    const uint32_t k = __ffs(~hb) - 1;   // first lane not (yet) known to hit
    if ((dn >> k) & 1u) return hb;       // ... and it finished with a miss
  }
}

// warp-cooperative insert of (t, slot) for the active lanes, no atomics: each round every
// pending lane reads its probe position; among the lanes that found the same free entry
// (EMPTY or tombstone) the lowest one takes it, the others move on.  Returns the number of
// EMPTY entries used (warp-uniform).  (Measured faster than per-lane 32-bit CAS claims.)
template <typename Idx>
__device__ __forceinline__ uint32_t t_insert_warp(const BView<Idx>& S, bool act, uint64_t t, uint32_t slot,
                                                  uint32_t lane) {
  uint32_t pos = (uint32_t)t & S.tmask, fresh = 0;
  bool pending = act;
  while (__any_sync(kFull, pending)) {
    const uint32_t e = pending ? (uint32_t)S.table[pos] : 0u;
    const bool fr = pending && (e == BView<Idx>::NIL || e == BView<Idx>::TOMB);
    const uint32_t peers = __match_any_sync(kFull, fr ? pos : 0xffffffffu);
    const bool win = fr && (uint32_t)(__ffs(peers) - 1) == lane;
    __syncwarp();   // every read of this round precedes its writes
    if (win) {
      S.table[pos] = (Idx)slot;
      pending = false;
    } else if (pending && !fr) {
      pos = (pos + 1) & S.tmask;
    }
    fresh += __popc(__ballot_sync(kFull, win && e == BView<Idx>::NIL));
  }
  __syncwarp();
  return fresh;
}
// remove slot's entry (identity t, present); returns 1 if it became EMPTY
template <typename Idx>
__device__ __forceinline__ uint32_t t_erase(const BView<Idx>& S, uint64_t t, uint32_t slot) {
  uint32_t i = (uint32_t)t & S.tmask;
  while (S.table[i] != (Idx)slot) i = (i + 1) & S.tmask;   // present (caller's contract)
  const bool clear = S.table[(i + 1) & S.tmask] == BView<Idx>::NIL;
  S.table[i] = (Idx)(clear ? BView<Idx>::NIL : BView<Idx>::TOMB);
  return clear ? 1u : 0u;
}
// rebuild without tombstones (warp): slots [0, size) are the live nodes
template <typename Idx>
__device__ __forceinline__ void t_rebuild(const BView<Idx>& S, uint32_t size, uint32_t lane) {
  __syncwarp();
  for (uint32_t q = lane; q <= S.tmask; q += 32) S.table[q] = (Idx)BView<Idx>::NIL;
  __syncwarp();
  for (uint32_t b0 = 0; b0 < size; b0 += 32) {
    const uint32_t q = b0 + lane;
    t_insert_warp(S, q < size, q < size ? S.key[q] : 0ull, q, lane);
  }
}

__device__ __forceinline__ uint64_t warp_min_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const uint64_t u = __shfl_xor_sync(kFull, v, o);
    v = u < v ? u : v;
  }
  return v;
}

__device__ __forceinline__ uint32_t hist_bin_b(double lat, uint32_t bins) {
  if (!(lat >= 1.0)) return 0;
  int e;
  const double f = frexp(lat, &e);
  const uint32_t q = (uint32_t)((f * 2.0 - 1.0) * 4.0);
  const uint64_t b = 1 + 4 * (uint64_t)(e - 1) + q;
  return b >= bins ? bins - 1 : (uint32_t)b;
}

// Control block of one CTA (one trial).
struct __align__(16) BCtrl {
  double score[2][kMaxW];
  uint32_t mhit[2][kMaxW];
  uint32_t pend[2][kMaxW];
  uint32_t csize[2][kMaxW];   // cached blocks (CACHE_AWARE router, A38)
  uint32_t abortf[2];
  uint32_t trial, status;
  kvr_policy pol;
  // per-worker partials, combined in worker order at the end of the trial (A34)
  double P[kMaxW], F[kMaxW], slat[kMaxW], sttft[kMaxW], mlat[kMaxW];
  // per-worker counters, accumulated by lane 0 of the worker's warp: probes, inserted,
  // evictions, draws, resets, fallbacks, hit blocks, input blocks, queries, max pending,
  // digest sum, victim-log overflow
  unsigned long long cnt[kMaxW][12];
  unsigned long long vcur[kMaxW];   // next victim-log entry of the worker
  uint32_t hist[kMaxHistBins];
};

// Per-warp (worker) scalar state: warp-uniform registers.
struct BW {
  uint32_t size, cntT, nfl, wh, wn;
  uint32_t used;           // table entries that are live or tombstones
  uint32_t lhead, ltail;   // Leaf-LRU recency log cursors (first maybe-valid entry, end)
  uint64_t e, k;
  double Pt, th0, th1, th2, th3;
  bool dead;   // admission failure / violation: stop this worker
};
// (the Eq. 2 load, last completion, latency / TTFT partial sums, counters and the
// victim-log cursor live in the control block, updated by lane 0: fewer registers)

struct BTrial {
  const ReplayParams* p;
  TraceDev tr;
  const kvr_policy* pol;
  uint64_t K;
  uint32_t W, B, beta, i, lane, bt, nwords;
  bool rlt, lbgr, rls;
  kvr_query_record* rec;
  uint64_t* vlog;
  uint64_t vshare;
  BFlight* ring;
  uint32_t ringcap;
  BCtrl* ctrl;
  unsigned long long* cnt;   // ctrl->cnt[i]
  uint64_t* log;      // this worker's recency log (Leaf-LRU trials)
  uint32_t lmask;
};

// counter k of this worker += v (lane 0; call from warp-uniform code)
__device__ __forceinline__ void cadd(const BTrial& T, int k, uint64_t v) {
  if (T.lane == 0) T.cnt[k] += v;
}

// in-place order-preserving compaction of the recency log [head, tail): keeps the
// entries whose stamp is still the node's (pinned or not); returns the new tail
template <typename Idx>
__device__ __forceinline__ uint32_t blog_compact(const BTrial& T, const BView<Idx>& S, uint32_t head,
                                                 uint32_t tail) {
  uint32_t w = head;
  for (uint32_t r = head; r < tail; r += 32) {
    const uint32_t idx = r + T.lane;
    const uint64_t e = idx < tail ? T.log[idx & T.lmask] : 0ull;
    const bool v = idx < tail && S.stamp[(uint32_t)e] == (uint32_t)(e >> 32);
    const uint32_t bal = __ballot_sync(kFull, v);
    __syncwarp();   // every read of this window precedes the writes (they land below r + 32)
    if (v) T.log[(w + __popc(bal & ((1u << T.lane) - 1u))) & T.lmask] = e;
    w += __popc(bal);
    __syncwarp();
  }
  return w;
}

__device__ __forceinline__ bool bit_test(const uint32_t* bm, uint32_t s) {
  return (bm[s >> 5] >> (s & 31)) & 1u;
}

// |candidates|: unpinned leaves (LEAFU), without RLT marks if `unmarked`
template <typename Idx>
__device__ __forceinline__ uint32_t cand_count(const BView<Idx>& S, const BTrial& T, bool unmarked) {
  uint32_t c = 0;
  for (uint32_t w = T.lane; w < T.nwords; w += 32)
    c += __popc(S.leafu[w] & (unmarked ? ~S.markb[w] : ~0u));
  return __reduce_add_sync(kFull, c);
}

// slot of the idx-th candidate in physical-slot order (idx < count): one warp
// scan of the per-word counts per round of 32 words, then a bit select
template <typename Idx>
__device__ __forceinline__ uint32_t cand_select(const BView<Idx>& S, const BTrial& T, bool unmarked,
                                                uint32_t idx) {
  for (uint32_t w0 = 0; w0 < T.nwords; w0 += 32) {
    const uint32_t w = w0 + T.lane;
    const uint32_t word = w < T.nwords ? (S.leafu[w] & (unmarked ? ~S.markb[w] : ~0u)) : 0u;
    const uint32_t c = __popc(word);
    uint32_t inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(kFull, inc, o);
      if (T.lane >= (uint32_t)o) inc += u;
    }
    const uint32_t tot = __shfl_sync(kFull, inc, 31);
    if (idx < tot) {
      const uint32_t exc = inc - c;
      const bool mine = idx >= exc && idx < inc;
      const uint32_t owner = __ffs(__ballot_sync(kFull, mine)) - 1;
      const uint32_t pos = mine ? (w << 5) + select_bit(word, idx - exc) : 0u;
      return __shfl_sync(kFull, pos, owner);
    }
    idx -= tot;
  }
  return kNone;
}

// Register-resident candidate words (B <= 1024, lane l holds word l): inclusive prefix
// counts of the per-lane popcounts by six bit-sliced ballots; returns the total
__device__ __forceinline__ uint32_t words_count(uint32_t w, uint32_t lane, uint32_t& incl) {
  const uint32_t c = __popc(w);
  const uint32_t le = lane == 31 ? kFull : (2u << lane) - 1u;
  uint32_t tot = 0, inc = 0;
#pragma unroll
  for (int b = 0; b < 6; ++b) {
    const uint32_t bal = __ballot_sync(kFull, (c >> b) & 1u);
    tot += (uint32_t)__popc(bal) << b;
    inc += (uint32_t)__popc(bal & le) << b;
  }
  incl = inc;
  return tot;
}
// the idx-th set bit (slot order) of the words w, incl as from words_count
__device__ __forceinline__ uint32_t words_select(uint32_t w, uint32_t incl, uint32_t idx, uint32_t lane) {
  const uint32_t owner = __reduce_min_sync(kFull, incl > idx ? lane : 32u);
  const uint32_t ou = __shfl_sync(kFull, w, owner);
  const uint32_t rem = idx - (__shfl_sync(kFull, incl, owner) - (uint32_t)__popc(ou));
  const uint32_t lmle = lane == 31 ? kFull : (2u << lane) - 1u;
  const uint32_t bit = __reduce_min_sync(kFull, (uint32_t)__popc(ou & lmle) > rem ? lane : 32u);
  return owner * 32 + bit;
}

// RLT miss decisions of an update, blocks [d0, n) (all misses; Alg. 1 l.6-17 with
// pinning, A30-A33), B <= 1024.  LEAFU (lw), MARK (mw) and U = LEAFU & ~MARK (uw) are
// held in registers with U's prefix counts; a draw selects its victim by two CREDUX
// reductions, the victim's parent / child count / pin are fetched speculatively for
// the whole owner word while the bit is selected.  Everything the decisions do not
// read is deferred to one lane-parallel pass at the end: the victims' table erases,
// digest terms and victim-log entries (their identities are still in place), and the
// loaded slots' identities, parents, child counts, stamps, depths and pins.  gam[d]
// <- slot | evicted << 32.
template <typename Idx>
__device__ __forceinline__ bool b_rlt_misses(const BTrial& T, const BView<Idx>& S, BW& x, uint32_t j,
                                             uint32_t d0, uint32_t n, uint32_t prev0, const uint64_t* Hj,
                                             uint32_t* nvict, uint64_t* Vout) {
  const uint32_t lane = T.lane, B = T.B, nw = T.nwords;
  const uint32_t fallback = T.pol->rlt_fallback;
  uint32_t lw = lane < nw ? S.leafu[lane] : 0u;
  uint32_t mw = lane < nw ? S.markb[lane] : 0u;
  uint32_t uw = 0, incl = 0, total = 0;
  bool dirty = true;
  // loop state in plain registers (written back to x at the end)
  uint32_t cntT = x.cntT, size = x.size, nres = 0, nfb = 0;
  uint64_t e = x.e;
  const uint64_t e0 = x.e;
  // draws for counters rbase .. rbase+31, lane l holds counter rbase + l (ri = next unused)
  uint32_t rlo = 0, rhi = 0, ri = 32;
  uint64_t rbase = 0;
  const uint32_t lmle = lane == 31 ? kFull : (2u << lane) - 1u;
  uint32_t nv = 0;
  auto refill = [&]() {
    rbase = e;
    const uint64_t r = philox_r64(T.K, rbase + lane, T.i, 1);
    rlo = (uint32_t)r;
    rhi = (uint32_t)(r >> 32);
    ri = 0;
  };
  uint32_t d = d0;
  while (d < n) {
    // ---- fast segment: evictions from U with no mark reset, no refill, U != {} ----
    if (size == B && !dirty && total > 0 && ri < 32 && cntT < B) {
      const uint32_t lim = min(n, min(d + (B - cntT), d + (32u - ri)));
      const uint32_t d1 = d;
#pragma unroll 1
      for (; d < lim && total > 0; ++d) {
        const uint32_t dlo = __shfl_sync(kFull, rlo, ri), dhi = __shfl_sync(kFull, rhi, ri);
        ++ri;
        // floor(r64 * |U| / 2^64) (A6) with |U| < 2^32
        const uint32_t idx = (uint32_t)(((uint64_t)dhi * total + __umulhi(dlo, total)) >> 32);
        const uint32_t owner = __reduce_min_sync(kFull, incl > idx ? lane : 32u);
        // speculative: lane l fetches the parent of slot owner*32+l, its child count and pin
        uint32_t sp = (uint32_t)S.parent[owner * 32 + lane];
        const bool sok = sp < B;
        sp = sok ? sp : 0u;
        const uint32_t snc = (uint32_t)S.nchild[sp];
        const uint32_t spin = (uint32_t)S.pin[sp];
        const uint32_t smw = __shfl_sync(kFull, mw, sp >> 5);
        const uint32_t ou = __shfl_sync(kFull, uw, owner);
        const uint32_t rem = idx - (__shfl_sync(kFull, incl, owner) - (uint32_t)__popc(ou));
        const uint32_t bit = __reduce_min_sync(kFull, (uint32_t)__popc(ou & lmle) > rem ? lane : 32u);
        const uint32_t v = owner * 32 + bit;
        const uint32_t pa = __shfl_sync(kFull, sp, bit);
        const bool hasp = __shfl_sync(kFull, (uint32_t)sok, bit) != 0u;
        const uint32_t nc = __shfl_sync(kFull, snc, bit) - 1u;
        const uint32_t ppin = __shfl_sync(kFull, spin, bit);
        const uint32_t pmw = __shfl_sync(kFull, smw, bit);
        // U and LEAFU lose v (its slot is reloaded with t: pinned, marked); U gains pa iff
        // pa became an unpinned unmarked leaf
        if (lane == owner) {
          uw &= ~(1u << bit);
          lw &= ~(1u << bit);
          mw |= 1u << bit;
        }
        if (lane >= owner) --incl;
        --total;
        if (hasp) {
          S.nchild[pa] = (Idx)nc;   // uniform store (every lane read its value above)
          if (nc == 0 && ppin == 0) {
            const uint32_t pw = pa >> 5, pb = 1u << (pa & 31);
            if (lane == pw) lw |= pb;
            if (!(pmw & pb)) {   // pa != v (v is its child): the victim's MARK bit is irrelevant
              if (lane == pw) uw |= pb;
              if (lane >= pw) ++incl;
              ++total;
            }
          }
        }
        if (lane == 0) S.gam[d] = (uint64_t)v | (1ull << 32);
      }
      const uint32_t k = d - d1;
      cntT += k;   // t marked at each step, no reset inside the segment
      e += k;
      nv += k;
      continue;
    }
    // ---- general step: one block ----
    // Alg. 1 l.6-9: t is not cached, so not in T; the (B+1)-th distinct mark resets T
    if (cntT == B) {
      mw = 0u;
      cntT = 1;
      ++nres;
      dirty = true;
    } else {
      ++cntT;
    }
    uint32_t slot, ev = 0;
    if (size < B) {
      slot = size++;
    } else {
      if (dirty) {
        uw = lw & ~mw;
        total = words_count(uw, lane, incl);
        dirty = false;
      }
      uint32_t v;
      if (total == 0) {   // U = {} (A5)
        ++nfb;
        dirty = true;
        bool draw = true;
        if (fallback == KVR_RLT_EARLY_RESET) {
          mw = 0u;       // T <- {t}; t is loaded marked below
          cntT = 1;
          ++nres;
        } else if (fallback == KVR_RLT_LRU_MARKED) {   // least (stamp, -depth) unpinned leaf
          draw = false;
        }
        if (draw) {   // uniform over the unpinned leaves (marks cleared or ignored)
          uint32_t ci = 0;
          const uint32_t ct = words_count(lw, lane, ci);
          if (ct == 0) return false;   // every leaf is in flight
          if (ri == 32) refill();
          const uint32_t dlo = __shfl_sync(kFull, rlo, ri), dhi = __shfl_sync(kFull, rhi, ri);
          ++ri;
          ++e;
          v = words_select(lw, ci, (uint32_t)(((uint64_t)dhi * ct + __umulhi(dlo, ct)) >> 32), lane);
        } else {
          uint64_t best = ~0ull;
          uint32_t bits = lw;
          while (bits) {
            const uint32_t q = (lane << 5) + (__ffs(bits) - 1);
            bits &= bits - 1;
            const uint64_t key = ((uint64_t)S.stamp[q] << 32) |
                                 ((uint64_t)((0x10000u - S.depth[q]) & 0xffffu) << 16) | (uint64_t)q;
            best = key < best ? key : best;
          }
          best = warp_min_u64(best);
          if (best == ~0ull) return false;
          v = (uint32_t)(best & 0xffffu);
        }
        if ((__shfl_sync(kFull, mw, v >> 5) >> (v & 31)) & 1u) --cntT;   // a marked victim leaves T
        const uint32_t pa = S.parent[v];
        if (pa != BView<Idx>::NIL) {
          const uint32_t nc = S.nchild[pa] - 1u;
          __syncwarp();
          S.nchild[pa] = (Idx)nc;
          if (nc == 0 && S.pin[pa] == 0 && lane == (pa >> 5)) lw |= 1u << (pa & 31);
        }
      } else {
        // Alg. 1 l.14-16: uniform over U in slot order (A6), counter e_i
        if (ri == 32) refill();
        const uint32_t dlo = __shfl_sync(kFull, rlo, ri), dhi = __shfl_sync(kFull, rhi, ri);
        ++ri;
        ++e;
        const uint32_t idx = (uint32_t)(((uint64_t)dhi * total + __umulhi(dlo, total)) >> 32);
        v = words_select(uw, incl, idx, lane);
        const uint32_t pa = S.parent[v];
        if (lane == (v >> 5)) uw &= ~(1u << (v & 31));
        if (lane >= (v >> 5)) --incl;
        --total;
        if (pa != BView<Idx>::NIL) {
          const uint32_t nc = S.nchild[pa] - 1u;
          __syncwarp();
          S.nchild[pa] = (Idx)nc;
          if (nc == 0 && S.pin[pa] == 0) {
            const uint32_t pw = pa >> 5, pb = 1u << (pa & 31);
            if (lane == pw) lw |= pb;
            if (!((__shfl_sync(kFull, mw, pw) >> (pa & 31)) & 1u)) {   // joins U
              if (lane == pw) uw |= pb;
              if (lane >= pw) ++incl;
              ++total;
            }
          }
        }
      }
      // v leaves LEAFU; its MARK bit is replaced by t's (below)
      if (lane == (v >> 5)) lw &= ~(1u << (v & 31));
      slot = v;
      ev = 1;
      ++nv;
    }
    if (lane == (slot >> 5)) mw |= 1u << (slot & 31);   // t in T (Alg. 1 l.7)
    if (lane == 0) S.gam[d] = (uint64_t)slot | ((uint64_t)ev << 32);
    ++d;
  }
  if (lane < nw) {
    S.leafu[lane] = lw;
    S.markb[lane] = mw;
  }
  cadd(T, 1, n - d0);          // loads
  cadd(T, 2, nv);              // evictions
  cadd(T, 3, e - e0);          // draws
  cadd(T, 4, nres);
  cadd(T, 5, nfb);
  x.cntT = cntT;
  x.size = size;
  x.e = e;
  __syncwarp();
  // deferred, lane-parallel: victims' erases / digest terms / log entries (the k-th victim
  // of the update is the k-th evicting block), then the loads
  uint64_t V = 0;
  uint32_t k0 = 0, cleared = 0, prev_last = prev0, vfull = 0;
  const uint64_t vc0 = T.ctrl->vcur[T.i];
  for (uint32_t b0 = d0; b0 < n; b0 += 32) {
    const uint32_t q = b0 + lane;
    const bool act = q < n;
    const uint64_t g = act ? S.gam[q] : 0ull;
    const uint32_t slot = (uint32_t)g;
    const bool ev = act && (g >> 32) != 0;
    const uint32_t evb = __ballot_sync(kFull, ev);
    const uint32_t k = k0 + __popc(evb & ((1u << lane) - 1u));
    uint64_t hv = 0;
    if (ev) {
      hv = S.key[slot];
      cleared += t_erase(S, hv, slot);
      V ^= fmix64(hv ^ ((uint64_t)(k + 1) * kPosMul));
      if (T.vlog) {
        if (vc0 + k < T.vshare) T.vlog[(uint64_t)T.i * T.vshare + vc0 + k] = hv;
        else vfull = 1;
      }
    }
    k0 += __popc(evb);
    const uint32_t up = __shfl_up_sync(kFull, slot, 1);
    const uint32_t par = lane == 0 ? prev_last : up;
    const uint32_t last = min(31u, n - 1 - b0);
    __syncwarp();   // every victim identity is read before the slots are reloaded
    if (act) {
      S.key[slot] = Hj[q];
      S.parent[slot] = (Idx)par;   // kNone -> NIL (root child)
      S.nchild[slot] = (Idx)(q + 1 < n ? 1 : 0);
      S.stamp[slot] = j;
      S.depth[slot] = (Idx)(q + 1);
      S.pin[slot] = 1;
      S.gam[q] = slot;
    }
    prev_last = __shfl_sync(kFull, slot, last);
    __syncwarp();
  }
  if (prev0 != kNone && lane == 0) S.nchild[prev0] = (Idx)(S.nchild[prev0] + 1);   // prev0 is pinned
  x.used -= __reduce_add_sync(kFull, cleared);
  if (__any_sync(kFull, vfull != 0u) && lane == 0) T.cnt[11] = 1;
  V = warp_xor64(V);
  if (lane == 0) T.ctrl->vcur[T.i] = vc0 + nv;
  __syncwarp();
  *nvict += nv;
  *Vout ^= V;
  return true;
}

// UpdateCache(S_i, Gamma_j) at dequeue (Eq. 3 with Alg. 1 / Leaf-LRU, P:115-122,
// P:225-245), pinning every block as it is accessed (A30, A33).
// Returns the number of leading input hits m, or kNone on an admission failure.
template <typename Idx>
__device__ __forceinline__ uint32_t b_update(const BTrial& T, const BView<Idx>& S, BW& x, uint32_t j, uint32_t n,
                             uint32_t n_in, const uint64_t* Hj, uint32_t* nvict, uint64_t* Vout) {
  const uint32_t lane = T.lane, B = T.B;
  const kvr_policy& pol = *T.pol;
  uint32_t prev = kNone;
  uint32_t m = 0;
  bool hitrun = true;   // hits are a prefix of Gamma (prefix closure)
  uint32_t nv = 0;
  uint64_t V = 0;
  const bool lru = !T.rlt;
  if (lru && x.ltail - x.lhead + n > T.lmask + 1) x.ltail = blog_compact(T, S, x.lhead, x.ltail);
  // room for this update's n inserts with an EMPTY entry left (probes must terminate)
  if (x.used + n >= S.tmask) {
    t_rebuild(S, x.size, lane);
    x.used = x.size;
  }
  // Leaf-LRU victims (A33) = the unpinned nodes in recency-log order (stamp, -depth)
  // from the head: the minimum over the unpinned nodes is always a leaf, and the
  // nodes this update loads are pinned, so the e victims of a miss run are the e
  // first unpinned valid entries.  The head only moves past entries
  // that are no longer valid.
  uint32_t lpos = x.lhead, cm = 0;
  uint64_t le = 0;
  bool lwin = false, headfix = false;
  auto lru_take = [&]() -> uint32_t {
    for (;;) {
      if (cm == 0) {
        if (lwin) lpos += 32;
        if (lpos >= x.ltail) return kNone;
        const uint32_t idx = lpos + lane;
        le = idx < x.ltail ? T.log[idx & T.lmask] : 0ull;
        const uint32_t sl = (uint32_t)le;
        const bool valid = idx < x.ltail && S.stamp[sl] == (uint32_t)(le >> 32);
        const uint32_t vb = __ballot_sync(kFull, valid);
        cm = __ballot_sync(kFull, valid && S.pin[sl] == 0);
        if (!headfix) {
          if (vb) {
            x.lhead = lpos + (__ffs(vb) - 1);
            headfix = true;
          } else {
            x.lhead = min(lpos + 32, x.ltail);
          }
        }
        lwin = true;
        continue;
      }
      const uint32_t L = __ffs(cm) - 1;
      cm &= cm - 1;
      return __shfl_sync(kFull, (uint32_t)le, L);
    }
  };
  // the victims of the evicting lanes evb (the k-th set bit of evb takes the k-th victim),
  // 32 log entries per ballot; returns false if the log runs out (every node in flight)
  auto lru_take_batch = [&](uint32_t evb, uint32_t& v) -> bool {
    const uint32_t need = __popc(evb);
    const uint32_t rk = __popc(evb & ((1u << lane) - 1u));
    const bool evl = (evb >> lane) & 1u;
    uint32_t got = 0;
    while (got < need) {
      if (cm == 0) {
        if (lwin) lpos += 32;
        if (lpos >= x.ltail) return false;
        const uint32_t idx = lpos + lane;
        le = idx < x.ltail ? T.log[idx & T.lmask] : 0ull;
        const uint32_t sl = (uint32_t)le;
        const bool valid = idx < x.ltail && S.stamp[sl] == (uint32_t)(le >> 32);
        const uint32_t vb = __ballot_sync(kFull, valid);
        cm = __ballot_sync(kFull, valid && S.pin[sl] == 0);
        if (!headfix) {
          if (vb) {
            x.lhead = lpos + (__ffs(vb) - 1);
            headfix = true;
          } else {
            x.lhead = min(lpos + 32, x.ltail);
          }
        }
        lwin = true;
        continue;
      }
      const uint32_t c = __popc(cm);
      const uint32_t take = min(c, need - got);
      const bool mine = evl && rk >= got && rk < got + take;
      const uint32_t src = mine ? select_bit(cm, rk - got) : 0u;
      const uint32_t val = __shfl_sync(kFull, (uint32_t)le, src);
      if (mine) v = val;
      cm = take == c ? 0u : (cm & ~((2u << select_bit(cm, take - 1)) - 1u));
      got += take;
    }
    return true;
  };
  // Lane-parallel hit run: 32 blocks per step, each lane looks up its own block; the
  // leading hits are refreshed, pinned and (RLT) marked at once when no |T| = B+1
  // reset can fall inside the step, else the step is left to the serial loop below.
  uint32_t d = 0;
  BP_T0(tu);
  while (d < n) {
    const uint32_t q = d + lane;
    uint32_t sl;
    const uint32_t hb = b_probe_window(S, S.gam, d, n, lane, sl);
    const uint32_t hc = (~hb) ? (uint32_t)(__ffs(~hb) - 1) : 32u;   // leading hits of this step
    const bool hit = lane < hc;
    if (T.rlt) {
      const uint32_t nnew = __popc(__ballot_sync(kFull, hit && !bit_test(S.markb, sl)));
      if (x.cntT + nnew > B) break;                                  // a reset: serial path
      if (hit && !bit_test(S.markb, sl)) atomicOr(&S.markb[sl >> 5], 1u << (sl & 31));
      x.cntT += nnew;
    }
    if (hit) {
      S.stamp[sl] = j;
      S.gam[q] = sl;   // block q's slot (recency log)
      const uint32_t pv = S.pin[sl];
      S.pin[sl] = (uint8_t)(pv + 1);
      if (pv == 0) atomicAnd(&S.leafu[sl >> 5], ~(1u << (sl & 31)));
    }
    __syncwarp();
    if (hc > 0) {
      prev = __shfl_sync(kFull, sl, hc - 1);
      m = min(d + hc, n_in);
    }
    d += hc;
    if (hc < 32) {
      hitrun = false;   // the first miss: every later block of Gamma misses too
      break;
    }
  }
  // Serial part: the (rare) hit steps around a mark reset, then the misses.  Table
  // inserts of the loaded blocks are deferred to one lane-parallel pass after the
  // loop (no lookup happens inside a miss run); gam[d] then holds block d's slot.
  // RLT keeps |U| incrementally (a victim leaves U, its parent may join) and draws
  // from a batch of 32 consecutive Philox counters computed lane-parallel.
  BP_ACC(8, tu);   // hit run
  const uint32_t d_miss0 = hitrun ? n : d;   // first block known to miss (if any)
  uint32_t d_ins0 = n;                       // first block whose insert is deferred
  int32_t nU_known = -1;                     // |U| when known, -1 = recount
  // B <= 1024: U's words in registers (lane l: word l) with their inclusive prefix
  // counts, valid whenever nU_known >= 0 (reloaded at every recount)
  const bool regu = T.nwords <= 32;
  uint32_t uw = 0, uincl = 0;
  if (lru && !hitrun && d < n) {
    // Leaf-LRU miss run, 32 misses per step: the first B - size take free slots, the rest
    // the next unpinned entries of the recency log (in order, one per evicting lane);
    // victims' table entries are erased by lane 0 (backward shift is serial), every other
    // write is lane-parallel.  Leaf-LRU keeps no tree (parents, child counts and the
    // LEAFU / MARK bitmaps serve RLT only).
    const uint32_t M = n - d, nfree = min(M, B - x.size);
    d_ins0 = d;
    const uint64_t vc0 = T.ctrl->vcur[T.i];
    uint32_t vfull = 0;
    for (uint32_t cb = 0; cb < M; cb += 32) {
      const uint32_t q = cb + lane;
      const bool act = q < M;
      const bool ev = act && q >= nfree;
      const uint32_t evb = __ballot_sync(kFull, ev);
      uint32_t v = kNone;
      BP_T0(tl);
      if (!lru_take_batch(evb, v)) return kNone;   // every node is in flight
      BP_ACC(9, tl);
      const uint32_t slot = ev ? v : x.size + q;
      uint64_t hv = 0;
      if (ev) {
        hv = S.key[v];
        const uint64_t k = nv + (q - max(cb, nfree));   // index of this victim in the update
        V ^= fmix64(hv ^ ((k + 1) * kPosMul));
        if (T.vlog) {
          if (vc0 + k < T.vshare) T.vlog[(uint64_t)T.i * T.vshare + vc0 + k] = hv;
          else vfull = 1;
        }
      }
      __syncwarp();
      // victims leave the table first (their slots are reloaded just below), one lane each
      const uint32_t clr = ev ? t_erase(S, hv, v) : 0u;
      x.used -= __popc(__ballot_sync(kFull, clr != 0u));
      __syncwarp();
      BP_ACC(10, tl);
      if (act) {   // Load(S, t): pinned, stamped at j; the table insert is deferred
        const uint32_t dd = d + q;
        S.key[slot] = S.gam[dd];
        S.stamp[slot] = j;
        S.depth[slot] = (Idx)(dd + 1);
        S.pin[slot] = 1;
        S.gam[dd] = slot;
      }
      const uint32_t ne = __popc(evb);
      nv += ne;
      __syncwarp();
    }
    if (__any_sync(kFull, vfull != 0u) && lane == 0) T.cnt[11] = 1;
    cadd(T, 1, M);
    cadd(T, 2, nv);
    if (lane == 0) T.ctrl->vcur[T.i] = vc0 + nv;
    __syncwarp();
    x.size += nfree;
    V = warp_xor64(V);
    d = n;   // the serial loop below has nothing left
  }
  BP_ACC(11, tu);   // Leaf-LRU miss run (incl. take / erase)
  uint64_t rbatch = 0, rbase = 0;            // draws for counters rbase .. rbase+31
  bool rvalid = false;
  for (; d < n; ++d) {
    const uint64_t t = S.gam[d];
    uint32_t s = (hitrun && d < d_miss0) ? t_find(S, t) : kNone;
    if (s == kNone) hitrun = false;
    if (s == kNone && T.rlt && regu) break;   // every later block misses too: fast path below
    // Alg. 1 l.6-9: mark t; the (B+1)-th distinct mark resets T to {t}
    if (T.rlt) {
      const bool marked = s != kNone && bit_test(S.markb, s);
      if (!marked) {
        if (x.cntT + 1 == B + 1) {
          for (uint32_t w = lane; w < T.nwords; w += 32) S.markb[w] = 0;
          __syncwarp();
          x.cntT = 1;
          cadd(T, 4, 1);
          nU_known = -1;
        } else {
          x.cntT++;
        }
        if (s != kNone && lane == 0) S.markb[s >> 5] |= 1u << (s & 31);
        __syncwarp();
      }
    }
    if (s != kNone) {   // hit (Alg. 1 l.10-11): refresh, pin (an unpinned leaf stops being a candidate)
      __syncwarp();
      if (lane == 0) {
        S.stamp[s] = j;
        S.gam[d] = s;
        const uint32_t pv = S.pin[s];
        S.pin[s] = (uint8_t)(pv + 1);
        if (pv == 0) S.leafu[s >> 5] &= ~(1u << (s & 31));
      }
      __syncwarp();
      if (d < n_in) m = d + 1;
      prev = s;
      continue;
    }
    if (d_ins0 == n) d_ins0 = d;
    uint32_t slot;
    if (x.size == B) {
      // choose the victim among unpinned leaves (A30, A33): LEAFU bitmap
      uint32_t v = kNone;
      bool use_lru = false;    // the LRU_MARKED fallback of RLT (A5): least unpinned leaf
      bool via_u = false;      // v drawn from U = LEAFU \ T (the incremental count applies)
      if (lru) v = lru_take();
      if (T.rlt) {
        bool mark_ok = true;
        uint32_t nU;
        if (nU_known >= 0) {
          nU = (uint32_t)nU_known;
        } else if (regu) {   // (re)load U = LEAFU & ~MARK into registers, word l on lane l
          uw = lane < T.nwords ? (S.leafu[lane] & ~S.markb[lane]) : 0u;
          const uint32_t c = __popc(uw);
          const uint32_t le = lane == 31 ? kFull : (2u << lane) - 1u;
          uint32_t tot = 0, inc = 0;
#pragma unroll
          for (int b = 0; b < 6; ++b) {   // bit-sliced prefix sums of the per-lane counts
            const uint32_t bal = __ballot_sync(kFull, (c >> b) & 1u);
            tot += (uint32_t)__popc(bal) << b;
            inc += (uint32_t)__popc(bal & le) << b;
          }
          uincl = inc;
          nU = tot;
        } else {
          nU = cand_count(S, T, true);
        }
        if (nU == 0) {   // A5: U empty
          cadd(T, 5, 1);
          mark_ok = false;
          nU_known = -1;
          if (pol.rlt_fallback == KVR_RLT_EARLY_RESET) {
            for (uint32_t w = lane; w < T.nwords; w += 32) S.markb[w] = 0;
            __syncwarp();
            x.cntT = 1;    // T <- {t}; t is loaded marked below
            cadd(T, 4, 1);
          } else if (pol.rlt_fallback == KVR_RLT_LRU_MARKED) {
            use_lru = true;
          }
          if (!use_lru) nU = cand_count(S, T, false);
        }
        if (!use_lru && nU > 0) {
          // Alg. 1 l.15: uniform over U in physical-slot order (A6); counter x.e
          if (!rvalid || x.e - rbase >= 32) {
            rvalid = true;
            rbase = x.e;
            rbatch = philox_r64(T.K, rbase + lane, T.i, 1);
          }
          const uint64_t r = __shfl_sync(kFull, rbatch, (int)(x.e - rbase));
          x.e++;
          cadd(T, 3, 1);
          const uint32_t idx = (uint32_t)pick_index(r, nU);
          if (mark_ok && regu) {
            // owner word: first lane whose inclusive count exceeds idx; the bit inside
            // it: the first lane l with popc(word & lanes <= l) > rem
            const uint32_t owner = __reduce_min_sync(kFull, uincl > idx ? lane : 32u);
            const uint32_t ou = __shfl_sync(kFull, uw, owner);
            const uint32_t rem = idx - (__shfl_sync(kFull, uincl, owner) - (uint32_t)__popc(ou));
            const uint32_t lmle = lane == 31 ? kFull : (2u << lane) - 1u;
            const uint32_t bit = __reduce_min_sync(kFull, (uint32_t)__popc(ou & lmle) > rem ? lane : 32u);
            v = owner * 32 + bit;
          } else {
            v = cand_select(S, T, mark_ok, idx);
          }
          via_u = mark_ok;
          if (mark_ok) nU_known = (int32_t)nU;
        }
      }
      if (use_lru) {   // least (stamp, -depth) among unpinned leaves
        uint64_t best = ~0ull;
        for (uint32_t w = lane; w < T.nwords; w += 32) {
          uint32_t bits = S.leafu[w];
          while (bits) {
            const uint32_t q = (w << 5) + (__ffs(bits) - 1);
            bits &= bits - 1;
            const uint64_t key = ((uint64_t)S.stamp[q] << 32) |
                                 ((uint64_t)((0x10000u - S.depth[q]) & 0xffffu) << 16) | (uint64_t)q;
            best = key < best ? key : best;
          }
        }
        best = warp_min_u64(best);
        if (best != ~0ull) v = (uint32_t)(best & 0xffffu);   // B <= 65536: slot fits 16 bits
      }
      if (v == kNone) return kNone;   // every leaf is in flight
      // Evict(S, v): table delete, parent child count (+ LEAFU), T \ {v}
      const uint64_t hv = S.key[v];
      if (bit_test(S.markb, v)) x.cntT--;
      const uint32_t pa = S.parent[v];
      const bool has_pa = pa != BView<Idx>::NIL;
      const uint32_t nc = has_pa ? S.nchild[pa] - 1u : 1u;
      const bool pa_leafu = has_pa && nc == 0 && S.pin[pa] == 0;   // parent joins LEAFU
      if (via_u) {
        const bool join = pa_leafu && !bit_test(S.markb, pa);   // the parent joins U
        nU_known = nU_known - 1 + (join ? 1 : 0);
        if (regu) {   // U loses v, maybe gains pa
          const uint32_t vw = v >> 5;
          if (lane == vw) uw &= ~(1u << (v & 31));
          if (lane >= vw) --uincl;
          if (join) {
            const uint32_t pw = pa >> 5;
            if (lane == pw) uw |= 1u << (pa & 31);
            if (lane >= pw) ++uincl;
          }
        }
      }
      __syncwarp();
      uint32_t clr = 0;
      if (lane == 0) {
        clr = t_erase(S, hv, v);
        if (has_pa) {
          S.nchild[pa] = (Idx)nc;
          if (pa_leafu) S.leafu[pa >> 5] |= 1u << (pa & 31);
        }
        S.markb[v >> 5] &= ~(1u << (v & 31));
        S.leafu[v >> 5] &= ~(1u << (v & 31));
      }
      x.used -= __shfl_sync(kFull, clr, 0);
      __syncwarp();
      cadd(T, 2, 1);
      V ^= fmix64(hv ^ ((uint64_t)(nv + 1) * kPosMul));
      if (lane == 0) {
        const uint64_t vc = T.ctrl->vcur[T.i];
        if (T.vlog) {
          if (vc < T.vshare) T.vlog[(uint64_t)T.i * T.vshare + vc] = hv;
          else T.cnt[11] = 1;
        }
        T.ctrl->vcur[T.i] = vc + 1;
      }
      __syncwarp();
      nv++;
      slot = v;
    } else {
      slot = x.size++;
    }
    // Load(S, t): pinned (not in LEAFU), stamped, marked under RLT (t in T after
    // l.6-9); the table insert is deferred (gam[d] <- slot)
    if (lane == 0) {
      S.key[slot] = t;
      S.parent[slot] = (Idx)prev;           // kNone -> NIL (root child)
      S.nchild[slot] = 0;
      S.stamp[slot] = j;
      S.depth[slot] = (Idx)(d + 1);
      S.pin[slot] = 1;
      if (T.rlt) S.markb[slot >> 5] |= 1u << (slot & 31);
      S.gam[d] = slot;
      if (prev != kNone) S.nchild[prev] = (Idx)(S.nchild[prev] + 1);   // prev is pinned: never in LEAFU
    }
    __syncwarp();
    cadd(T, 1, 1);
    prev = slot;
  }
  if (d < n) {   // RLT misses with register-resident LEAFU / MARK words (B <= 1024)
    d_ins0 = d;
    if (!b_rlt_misses(T, S, x, j, d, n, prev, Hj, &nv, &V)) return kNone;
    d = n;
  }
  BP_ACC(12, tu);   // serial loop (RLT misses, hit steps around a reset)
  // deferred table inserts, lane-parallel (linear probing, CAS-claimed entries)
  for (uint32_t b0 = d_ins0; b0 < n; b0 += 32) {
    const uint32_t q = b0 + lane;
    const uint32_t slot = q < n ? (uint32_t)S.gam[q] : 0u;
    x.used += t_insert_warp(S, q < n, q < n ? S.key[slot] : 0ull, slot, lane);
  }
  BP_ACC(17, tu);   // deferred inserts
  if (x.used > KVR_BATCH_REBUILD_NUM * (S.tmask + 1u) / 8u) {   // too many tombstones: rebuild
    t_rebuild(S, x.size, lane);
    x.used = x.size;
    BP_CNT(23, 1);
  }
  BP_ACC(18, tu);   // rebuilds
  if (lru) {   // the path, deepest first, at stamp j (it was compacted to fit)
    for (uint32_t q = lane; q < n; q += 32)
      T.log[(x.ltail + (n - 1 - q)) & T.lmask] = ((uint64_t)j << 32) | (uint32_t)S.gam[q];
    x.ltail += n;
    __syncwarp();
  }
  BP_ACC(13, tu);   // log append append
  *nvict = nv;
  *Vout = V;
  return m;
}

// Dequeue r on worker T.i at time s (A30): stage Gamma_j, UpdateCache with
// pinning, true h, Eq. 1 truth, record/digest/histogram, into a batch slot.
template <typename Idx>
__device__ __forceinline__ bool b_dequeue(const BTrial& T, const BView<Idx>& S, BW& x, const BFlight& r, double s) {
  const uint32_t j = r.j, lane = T.lane;
  const QueryHdr& h = T.tr.hdr[j];
  const uint32_t n_in = h.n_in, n = h.n_in + h.n_out;
  const uint64_t* Hj = T.tr.hash + h.block_off;
  BP_T0(td);
  for (uint32_t d = lane; d < n; d += 32) S.gam[d] = Hj[d];
  __syncwarp();
  BP_ACC(14, td);   // dequeue: header + path staging
  BP_CNT(20, 1);
  uint32_t nv = 0;
  uint64_t V = 0;
  const uint32_t m = b_update(T, S, x, j, n, n_in, Hj, &nv, &V);
  if (m == kNone) return false;
  BP_T0(ta);
  const kvr_service_model& tm = T.p->truth;
  const uint32_t q = T.bt * n_in;
  const uint32_t hh = T.bt * m;
  const double xh = (double)hh, yh = (double)(q - hh);
  const double pre = (tm.alpha_cached_ms * xh) + (tm.alpha_miss_ms * yh);   // Eq. 1
  const double O = tm.out_ms_per_token * (double)h.out_tokens;
  const double cost = pre + O;
  const double ttft = (s + pre) - r.a;                                        // A20
  const double comp = s + cost;
  const double lat = comp - r.a;
  if (lane == 0) {
    BFlight f = r;
    f.c = comp;
    S.fl[x.nfl] = f;
  }
  __syncwarp();
  x.nfl++;
  if (lane == 0) {
    BCtrl* c = T.ctrl;
    const uint32_t i = T.i;
    if (comp > c->F[i]) c->F[i] = comp;
    c->P[i] = c->P[i] + cost;                                                 // Eq. 2
    c->slat[i] = c->slat[i] + lat;
    c->sttft[i] = c->sttft[i] + ttft;
    if (lat > c->mlat[i]) c->mlat[i] = lat;
    T.cnt[6] += m;      // hit blocks   (x bt at the end)
    T.cnt[7] += n_in;   // input blocks (x bt at the end)
    T.cnt[8] += 1;
  }
  uint64_t Tj = fmix64(T.K ^ (uint64_t)j);
  Tj = fmix64(Tj ^ (uint64_t)T.i);
  Tj = fmix64(Tj ^ (uint64_t)m);
  Tj = fmix64(Tj ^ (uint64_t)nv);
  Tj = fmix64(Tj ^ V);
  if (lane == 0) T.cnt[10] += Tj;
  if (lane == 0) {
    if (T.rec) {
      kvr_query_record& R = T.rec[j];
      R.worker = T.i;
      R.hit_tokens = hh;
      R.n_victims = nv;
      R._pad = 0;
      R.ttft_ms = ttft;
      R.latency_ms = lat;
      R.victim_offset = (uint64_t)T.i * T.vshare + (T.ctrl->vcur[T.i] - nv);
    }
    if (T.p->bins) atomicAdd(&T.ctrl->hist[hist_bin_b(lat, T.p->bins)], 1u);
  }
  BP_ACC(15, ta);   // dequeue accounting
  return true;
}

// Completion of the earliest in-flight query (ties: lower j, A31): LBGR
// OnlineUpdate (NLMS A8 / RLS A8b) and ReleaseLoad (A10) as in the beta = 1
// model, unpin Gamma_j, then start the head of the waiting FIFO at c.
template <typename Idx>
__device__ __forceinline__ bool b_complete(const BTrial& T, const BView<Idx>& S, BW& x, uint32_t b) {
  const uint32_t lane = T.lane;
  const BFlight r = S.fl[b];
  __syncwarp();
  if (lane == 0) S.fl[b] = S.fl[x.nfl - 1];
  __syncwarp();
  x.nfl--;
  const kvr_policy& pol = *T.pol;
  if (T.lbgr) {
    const double res = (r.c - r.a) - r.Ehat;
    if (T.rls) {
      // one exponentially weighted RLS step in the oracle's literal order (rls_step)
      const double lam = pol.mu;
      const double phi[4] = {r.phi0, r.phi1, r.phi2, 1.0};
      double* Pm = S.rlsP;
      double pi[4];
      for (int a = 0; a < 4; ++a) {
        double t = Pm[4 * a] * phi[0];
        t = t + Pm[4 * a + 1] * phi[1];
        t = t + Pm[4 * a + 2] * phi[2];
        t = t + Pm[4 * a + 3] * phi[3];
        pi[a] = t;
      }
      double g = phi[0] * pi[0];
      g = g + phi[1] * pi[1];
      g = g + phi[2] * pi[2];
      g = g + phi[3] * pi[3];
      const double gamma = lam + g;
      double kv[4];
      for (int a = 0; a < 4; ++a) kv[a] = pi[a] / gamma;
      x.th0 = x.th0 + kv[0] * res;
      x.th1 = x.th1 + kv[1] * res;
      x.th2 = x.th2 + kv[2] * res;
      x.th3 = x.th3 + kv[3] * res;
      double nP = 0.0;
      if (lane < 16) nP = (Pm[lane] - kv[lane >> 2] * pi[lane & 3]) / lam;
      __syncwarp();
      if (lane < 16) Pm[lane] = nP;
      __syncwarp();
    } else {
      const double phi3 = 1.0;
      double s2 = r.phi0 * r.phi0;
      s2 = s2 + r.phi1 * r.phi1;
      s2 = s2 + r.phi2 * r.phi2;
      s2 = s2 + phi3 * phi3;
      const double gs = (pol.mu * res) / (1.0 + s2);
      x.th0 = x.th0 + gs * r.phi0;
      x.th1 = x.th1 + gs * r.phi1;
      x.th2 = x.th2 + gs * r.phi2;
      x.th3 = x.th3 + gs * phi3;
    }
    uint64_t kap = x.k - r.ka;
    double pw = 1.0, bb = pol.rho;
    while (kap) {
      if (kap & 1) pw = pw * bb;
      bb = bb * bb;
      kap >>= 1;
    }
    x.Pt = x.Pt - r.Chat * pw;
    if (x.Pt < 0.0) x.Pt = 0.0;
  }
  // release_path: lane-parallel lookups, distinct slots
  BP_T0(tr_);
  BP_CNT(21, 1);
  const QueryHdr& h = T.tr.hdr[r.j];
  const uint32_t n = h.n_in + h.n_out;
  const uint64_t* Hj = T.tr.hash + h.block_off;
  bool bad = false;
  for (uint32_t d = lane; d < n; d += 32) {
    const uint32_t s = t_find(S, Hj[d]);
    if (s == kNone || S.pin[s] == 0) {
      bad = true;
    } else {
      const uint32_t pv = S.pin[s] - 1u;
      S.pin[s] = (uint8_t)pv;
      if (pv == 0 && S.nchild[s] == 0) atomicOr(&S.leafu[s >> 5], 1u << (s & 31));
    }
  }
  if (__any_sync(kFull, bad)) return false;
  __syncwarp();
  BP_ACC(16, tr_);   // release path (unpin)
  if (x.wn > 0) {
    const BFlight hq = T.ring[(size_t)T.i * T.ringcap + x.wh];
    x.wh = x.wh + 1 == T.ringcap ? 0 : x.wh + 1;
    x.wn--;
    return b_dequeue(T, S, x, hq, r.c);
  }
  return true;
}

template <typename Idx>
__device__ __forceinline__ uint32_t b_next(const BView<Idx>& S, const BW& x, double* c) {
  uint32_t b = kNone;
  double bc = INFINITY;
  uint32_t bj = 0;
  for (uint32_t u = 0; u < x.nfl; ++u) {
    const double cu = S.fl[u].c;
    const uint32_t ju = S.fl[u].j;
    if (b == kNone || cu < bc || (cu == bc && ju < bj)) {
      b = u;
      bc = cu;
      bj = ju;
    }
  }
  *c = bc;
  return b;
}

// register cap: 128 per thread up to 512 threads (2 CTAs of 8 warps per SM when
// their state fits the shared memory), 64 at 1024 threads
template <int kMaxThreads>
struct BMinBlocks { static constexpr int value = kMaxThreads <= 128 ? 4 : (kMaxThreads <= 256 ? 2 : 1); };

template <typename Idx, int kMaxThreads, int kFixedB>
__global__ void __launch_bounds__(kMaxThreads, BMinBlocks<kMaxThreads>::value)
    batch_kernel(const __grid_constant__ ReplayParams p) {
  uint8_t* smem = kvr_bsmem;
  const uint32_t tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t W = p.W, B = p.B;
  const BatchLayout& L = p.blay;
  BCtrl* ctrl = reinterpret_cast<BCtrl*>(smem);
  uint8_t* sbase = smem + align16(sizeof(BCtrl));
  // tier 1 (u16 ids) keeps the state in shared memory, tier 2 (u32) in the workspace;
  // deciding it at compile time lets the compiler use 32-bit shared addressing (LDS/STS)
  uint8_t* wbase;
  if constexpr (sizeof(Idx) == 4) wbase = p.gstate + ((size_t)blockIdx.x * W + w) * L.bytes;
  else wbase = sbase + (size_t)w * L.bytes;
  const BView<Idx> S = bview<Idx, kFixedB>(wbase, L);

#pragma unroll 1
  for (;;) {
    if (tid == 0) {
      const uint32_t tt = atomicAdd(p.work_counter, 1u);
      ctrl->trial = tt;
      if (tt < p.n_trials) ctrl->pol = p.policies ? p.policies[tt] : p.defpol;
      ctrl->abortf[0] = 0;
      ctrl->abortf[1] = 0;
      ctrl->status = 0;
    }
    for (uint32_t b = tid; b < p.bins; b += blockDim.x) ctrl->hist[b] = 0;
    __syncthreads();
    const uint32_t trial = ctrl->trial;
    if (trial >= p.n_trials) break;
    const kvr_policy& pol = ctrl->pol;
    BTrial T;
    T.p = &p;
    const uint32_t tix = p.trial_trace ? p.trial_trace[trial] : 0u;
    const bool tr_ok = tix < p.n_traces;   // else KVR_TRIAL_BAD_TRACE, trial not run
    T.tr = p.traces[tr_ok ? tix : 0u];
    T.pol = &pol;
    T.K = p.keys[trial];
    T.W = W;
    T.B = B;
    T.beta = p.beta;
    T.i = w;
    T.lane = lane;
    T.bt = T.tr.block_tokens;
    T.nwords = L.nwords;
    T.rlt = pol.eviction == KVR_EVICT_RLT;
    T.rls = pol.router == KVR_ROUTE_LBGR_RLS;
    T.lbgr = pol.router == KVR_ROUTE_LBGR || T.rls;
    const bool recorded = trial < p.record_trials;
    T.rec = recorded ? p.records + (size_t)trial * p.rec_stride : nullptr;
    T.vlog = (recorded && p.victims) ? p.victims + (size_t)trial * p.victims_per_trial : nullptr;
    T.vshare = T.vlog ? p.victims_per_trial / W : 0;
    T.ringcap = p.ring;
    T.ring = reinterpret_cast<BFlight*>(p.aux_base) + (size_t)blockIdx.x * W * p.ring;
    T.ctrl = ctrl;
    T.log = p.blog_base + ((size_t)blockIdx.x * W + w) * p.blog_cap;
    T.lmask = p.blog_cap - 1;
    const uint32_t N = T.tr.N;

    // a per-trial policy from device memory is validated here (A36)
    const bool pol_ok = policy_valid(pol) && pol.eviction <= KVR_EVICT_RLT &&
                        pol.tracker_lag == 0 && pol.tracker_grain == 1;
    // ---- per-trial init: empty caches, P = 0 ----
    for (uint32_t q = lane; q < L.T; q += 32) S.table[q] = (Idx)BView<Idx>::NIL;
    for (uint32_t q = lane; q < B; q += 32) S.pin[q] = 0;
    for (uint32_t q = lane; q < L.nwords; q += 32) {
      S.leafu[q] = 0;
      S.markb[q] = 0;
    }
    if (T.rls && lane < 16) S.rlsP[lane] = (lane % 5 == 0) ? pol.rls_p0 : 0.0;
    __syncwarp();
    BW x;
    x.size = 0; x.cntT = 0; x.nfl = 0; x.wh = 0; x.wn = 0; x.used = 0;
    x.lhead = 0; x.ltail = 0;
    x.e = 0; x.k = 0;
    x.Pt = 0.0;
    x.th0 = pol.theta0[0]; x.th1 = pol.theta0[1]; x.th2 = pol.theta0[2]; x.th3 = pol.theta0[3];
    x.dead = false;
    if (lane == 0) {
      for (int c = 0; c < 12; ++c) ctrl->cnt[w][c] = 0;
      ctrl->P[w] = 0.0;
      ctrl->F[w] = 0.0;
      ctrl->slat[w] = 0.0;
      ctrl->sttft[w] = 0.0;
      ctrl->mlat[w] = 0.0;
      ctrl->vcur[w] = 0;
    }
    T.cnt = ctrl->cnt[w];
    if (!pol_ok && tid == 0) ctrl->status = KVR_TRIAL_BAD_POLICY;
    if (!tr_ok && tid == 0) ctrl->status = KVR_TRIAL_BAD_TRACE;
    const uint32_t Nrun = (pol_ok && tr_ok) ? N : 0;
    const double rho = pol.rho, dt = pol.delta_t_ms;
    bool aborted = false;
    // Ehat / C^ / phi of this worker for the current query (used if it is chosen)
    double myE = 0.0, myC = 0.0, f0 = 0.0, f1 = 0.0, f2 = 0.0;

#pragma unroll 1
    for (uint32_t j = 0; j < Nrun; ++j) {
      const uint32_t par = j & 1;
      BP_T0(tp);
      const QueryHdr& hq = T.tr.hdr[j];
      const double t = hq.arrival_ms;
      const uint32_t n_in = hq.n_in;
      const uint32_t q = T.bt * n_in;
      // 1. catch-up: ticks, completions and the dequeues they start, in time order (A31)
      if (!x.dead) {
        for (;;) {
          double c;
          const uint32_t b = b_next(S, x, &c);
          if (T.lbgr) {   // every tick up to min(a_j, next completion): tick first on ties
            const double lim = c < t ? c : t;
            while ((double)(x.k + 1) * dt <= lim) {
              x.Pt = rho * x.Pt;
              x.k++;
            }
          }
          if (b != kNone && c <= t) {
            if (!b_complete(T, S, x, b)) {
              x.dead = true;
              break;
            }
                  continue;
          }
          break;
        }
        if (x.dead && lane == 0) {
          atomicCAS(&ctrl->status, 0u, (uint32_t)KVR_TRIAL_ADMISSION);
          ctrl->abortf[par] = 1;
        }
      }
      BP_ACC(0, tp);   // header + catch-up (completions, dequeues)
      // 2. longest cached prefix at a_j (A32): lane-parallel probes, first miss by ballot
      const uint64_t* Hj = T.tr.hash + hq.block_off;
      uint32_t m = 0;
      for (uint32_t b0 = 0; b0 < n_in; b0 += 32) {
        uint32_t sl;
        const uint32_t bal = b_probe_window(S, Hj, b0, n_in, lane, sl);
        if (bal != kFull) {
          m = b0 + __ffs(~bal) - 1;
          break;
        }
        m = b0 + 32;
      }
      if (m > n_in) m = n_in;
      cadd(T, 0, (m + 1 < n_in) ? m + 1 : n_in);
      const uint32_t pend = x.nfl + x.wn;
      double sc = 0.0;
      if (T.lbgr) {
        const double xx = (double)(T.bt * m), yy = (double)(q - T.bt * m);
        const double C = (pol.est_alpha_cached_ms * xx) + (pol.est_alpha_miss_ms * yy);   // Eq. 5
        f0 = xx / 1000.0;
        f1 = yy / 1000.0;
        f2 = x.Pt / 1000.0;
        double d = x.th0 * f0;
        d = d + x.th1 * f1;
        d = d + x.th2 * f2;
        d = d + x.th3 * 1.0;
        myE = (C + x.Pt) + d;                                                            // Eq. 4
        myC = C;
        sc = myE;
      } else if (pol.router == KVR_ROUTE_STATIC_LINEAR) {
        const double xx = (double)(T.bt * m);
        sc = (pol.w_load * (double)pend) - (pol.w_hit * (xx / (double)q));                // A17
      }
      if (lane == 0) {
        ctrl->score[par][w] = sc;
        ctrl->mhit[par][w] = m;
        ctrl->pend[par][w] = pend;
        ctrl->csize[par][w] = x.size;
      }
      BP_ACC(1, tp);   // match + score
      __syncthreads();
      BP_ACC(2, tp);   // barrier
      if (ctrl->abortf[par]) {
        aborted = true;
        break;
      }
      // 3. argmin (lowest index on ties, A15), identical in every warp
      uint32_t best = 0;
      const uint32_t router = pol.router;
      if (T.lbgr || router == KVR_ROUTE_STATIC_LINEAR) {   // NaN ranks last (A37)
        for (uint32_t i = 1; i < W; ++i) {
          const double si = ctrl->score[par][i], sb = ctrl->score[par][best];
          if (!isnan(si) && (isnan(sb) || si < sb)) best = i;
        }
      } else if (router == KVR_ROUTE_THRESHOLD) {   // A16 on pending = waiting + in flight
        uint32_t mx = ctrl->pend[par][0], mn = mx;
        for (uint32_t i = 1; i < W; ++i) {
          mx = max(mx, ctrl->pend[par][i]);
          mn = min(mn, ctrl->pend[par][i]);
        }
        if ((double)mx > pol.tau * (double)max(1u, mn)) {
          for (uint32_t i = 1; i < W; ++i)
            if (ctrl->pend[par][i] < ctrl->pend[par][best]) best = i;
        } else {
          for (uint32_t i = 1; i < W; ++i)
            if (ctrl->mhit[par][i] > ctrl->mhit[par][best]) best = i;
        }
      } else if (router == KVR_ROUTE_CACHE_AWARE) {   // A38 on pending = waiting + in flight
        uint32_t mx = ctrl->pend[par][0], mn = mx;
        for (uint32_t i = 1; i < W; ++i) {
          mx = max(mx, ctrl->pend[par][i]);
          mn = min(mn, ctrl->pend[par][i]);
        }
        if (((double)(mx - mn) > pol.ca_balance_abs) && ((double)mx > pol.ca_balance_rel * (double)mn)) {
          for (uint32_t i = 1; i < W; ++i)
            if (ctrl->pend[par][i] < ctrl->pend[par][best]) best = i;
        } else {
          for (uint32_t i = 1; i < W; ++i)
            if (ctrl->mhit[par][i] > ctrl->mhit[par][best]) best = i;
          if (!((double)(T.bt * ctrl->mhit[par][best]) / (double)q > pol.ca_cache_threshold)) {
            best = 0;
            for (uint32_t i = 1; i < W; ++i)
              if (ctrl->csize[par][i] < ctrl->csize[par][best]) best = i;
          }
        }
      } else if (router == KVR_ROUTE_ROUND_ROBIN) {
        best = j % W;
      } else {
        best = (uint32_t)pick_index(philox_r64(T.K, j, 0xFFFFFFFFu, 2), W);
      }
      BP_ACC(3, tp);   // argmin
      // 4. assignment on the chosen worker (Eq. 6 at assignment, A32)
      if (w == best) {
        BP_CNT(22, 1);
        const uint32_t np = par ^ 1;   // flags written now are read after the next barrier
        if (x.wn >= p.ring) {
          if (lane == 0) {
            atomicCAS(&ctrl->status, 0u, (uint32_t)KVR_TRIAL_RING_OVERFLOW);
            ctrl->abortf[np] = 1;
          }
          x.dead = true;
        } else if (!x.dead) {
          BFlight r;
          r.j = j;
          r._p = 0;
          r.a = t;
          r.c = 0.0;
          r.Ehat = T.lbgr ? myE : 0.0;
          r.phi0 = T.lbgr ? f0 : 0.0;
          r.phi1 = T.lbgr ? f1 : 0.0;
          r.phi2 = T.lbgr ? f2 : 0.0;
          r.Chat = T.lbgr ? myC : 0.0;
          r.ka = x.k;
          if (T.lbgr) x.Pt = x.Pt + myC;
          if (T.rec && lane == 0) T.rec[j].score = ctrl->score[par][best];
          if (x.nfl < T.beta) {
            if (!b_dequeue(T, S, x, r, t)) {
              x.dead = true;
              if (lane == 0) {
                atomicCAS(&ctrl->status, 0u, (uint32_t)KVR_TRIAL_ADMISSION);
                ctrl->abortf[np] = 1;
              }
            }
          } else {
            if (lane == 0) {
              uint32_t slot = x.wh + x.wn;
              if (slot >= T.ringcap) slot -= T.ringcap;
              T.ring[(size_t)T.i * T.ringcap + slot] = r;
            }
            __syncwarp();
            x.wn++;
          }
          const uint32_t pe = x.nfl + x.wn;
          if (lane == 0 && pe > ctrl->cnt[w][9]) ctrl->cnt[w][9] = pe;
        }
        BP_ACC(4, tp);   // assignment (incl. a dequeue into a free slot)
      }
    }
    if (!aborted) {
      __syncthreads();   // flags of the last query's assignment
      if (ctrl->abortf[Nrun & 1]) aborted = true;
    }
    // 5. drain (A35): remaining completions and dequeues, per worker, no ticks
    if (!aborted && !x.dead) {
      for (;;) {
        double c;
        const uint32_t b = b_next(S, x, &c);
        if (b == kNone) break;
        if (!b_complete(T, S, x, b)) {
          x.dead = true;
          if (lane == 0) atomicCAS(&ctrl->status, 0u, (uint32_t)KVR_TRIAL_ADMISSION);
          break;
        }
      }
    }
    if (lane == 0) {
      ctrl->cnt[w][6] *= T.bt;     // hit / input blocks -> tokens
      ctrl->cnt[w][7] *= T.bt;
    }
    __syncthreads();
    if (tid == 0) {
      kvr_trial_result Rr;
      unsigned long long s[12] = {0};
      unsigned long long mp = 0, vfull = 0;
      double mk = 0.0, lc = 0.0, sl = 0.0, slat = 0.0, sttft = 0.0, ml = 0.0;
      for (uint32_t i = 0; i < W; ++i) {   // worker-index order (A34)
        for (int c = 0; c < 12; ++c) s[c] += ctrl->cnt[i][c];
        if (ctrl->cnt[i][9] > mp) mp = ctrl->cnt[i][9];
        vfull |= ctrl->cnt[i][11];
        if (ctrl->P[i] > mk) mk = ctrl->P[i];
        if (ctrl->F[i] > lc) lc = ctrl->F[i];
        sl = sl + ctrl->P[i];
        slat = slat + ctrl->slat[i];
        sttft = sttft + ctrl->sttft[i];
        if (ctrl->mlat[i] > ml) ml = ctrl->mlat[i];
      }
      Rr.probes = s[0];
      Rr.inserted_blocks = s[1];
      Rr.evictions = s[2];
      Rr.rlt_draws = s[3];
      Rr.rlt_resets = s[4];
      Rr.rlt_fallbacks = s[5];
      Rr.hit_tokens = s[6];
      Rr.input_tokens = s[7];
      Rr.queries = s[8];
      Rr.max_pending = mp;
      Rr.decision_digest = T.K + s[10];
      Rr.sum_latency_ms = slat;
      Rr.sum_ttft_ms = sttft;
      Rr.max_latency_ms = ml;
      Rr.makespan_ms = mk;
      Rr.last_completion_ms = lc;
      Rr.sum_load_ms = sl;
      uint32_t st = ctrl->status;
      if (st == 0 && vfull) st = KVR_TRIAL_VICTIM_LOG_FULL;
      Rr.status = (int32_t)st;
      Rr._pad = 0;
      p.results[trial] = Rr;
    }
    if (p.hist)
      for (uint32_t b = tid; b < p.bins; b += blockDim.x)
        p.hist[(size_t)trial * p.bins + b] = ctrl->hist[b];
    __syncthreads();
  }
}

}  // namespace

size_t batch_ctrl_bytes() { return align16(sizeof(BCtrl)); }

cudaError_t batch_phase_cycles(unsigned long long* out32, int reset) {
#ifdef KVR_PHASE_PROFILE
  cudaError_t e = cudaMemcpyFromSymbol(out32, g_bphase, 32 * sizeof(unsigned long long));
  if (e == cudaSuccess && reset) {
    unsigned long long z[32] = {0};
    e = cudaMemcpyToSymbol(g_bphase, z, sizeof(z));
  }
  return e;
#else
  (void)out32;
  (void)reset;
  return cudaErrorNotSupported;
#endif
}

template <typename Idx, int kFixedB>
static const void* batch_kernel_t(uint32_t W) {
  if (W <= 4) return (const void*)batch_kernel<Idx, 128, kFixedB>;
  if (W <= 8) return (const void*)batch_kernel<Idx, 256, kFixedB>;
  if (W <= 16) return (const void*)batch_kernel<Idx, 512, kFixedB>;
  return (const void*)batch_kernel<Idx, 1024, kFixedB>;
}

// tier 1: per-worker state in shared memory, u16 slot ids (B = 512 with compile-time
// offsets); tier 2: workspace, u32
static const void* batch_kernel_for(uint32_t W, bool global, uint32_t B) {
  if (global) return batch_kernel_t<uint32_t, 0>(W);
  return B == 512 ? batch_kernel_t<uint16_t, 512>(W) : batch_kernel_t<uint16_t, 0>(W);
}

cudaError_t batch_attrs(size_t smem, int* ctas_per_sm, uint32_t W, bool global, uint32_t B) {
  const void* k = batch_kernel_for(W, global, B);
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(ctas_per_sm, k, 32 * W, smem);
}

cudaError_t launch_batch(const ReplayParams& p, uint32_t grid, size_t smem, cudaStream_t s) {
  void* args[] = {const_cast<ReplayParams*>(&p)};
  return cudaLaunchKernel(batch_kernel_for(p.W, p.bglobal != 0, p.B), dim3(grid), dim3(32 * p.W), args, smem, s);
}

}  // namespace kvr
