// kvr_kernel.cu — the replay kernel: one CTA per trial (persistent over a work
// counter), one warp per worker.  Per query j (trace order, t = a_j):
//   1. catch-up   (each warp, its worker): decay ticks merged with FIFO
//                 completions -> NLMS OnlineUpdate + ReleaseLoad
//                 (Alg. 2 l.11-17; readings A8, A10, A11)
//   2. match      (each warp: 32 lanes probe 32 blocks, ballot -> first miss):
//                 longest cached prefix m_ij of the query
//   3. score      LBGR Eq. 4-5 / STATIC / THRESHOLD / RR / RANDOM
//   -- one __syncthreads per query --
//   4. argmin     (every warp, shuffle reduction; lowest index on ties, A15)
//   5. update     (warp i* only), split in two:
//      decide     UpdateCache (Eq. 3) decisions and every piece of
//                 state the next decision needs: hit marks with the |T|=B+1
//                 reset located by a ballot prefix count (Alg. 1 l.6-9);
//                 RLT victims (Alg. 1 l.12-17) as the only serial chain —
//                 register-resident LEAF/MARK words, incrementally patched
//                 prefix counts of U, counter-based Philox draws (32 per lane
//                 batch); Leaf-LRU victims = the first e valid
//                 entries of the recency log; then Eq. 1-2 / Eq. 6 accounting
//                 and the FIFO push (A12-A14, A20)
//      apply      table deletes (tombstones) / inserts (CAS), slot arrays,
//                 log append, digest, records — deferred until after the next
//                 barrier, so it overlaps the other workers' next decisions.
//                 Until then this warp matches through an overlay: the old
//                 table minus this update's victims plus the query's own path.
// Query headers and identities are staged in shared memory by 1-D bulk-async
// copies (TMA engine: cp.async.bulk + mbarrier) two queries ahead.
//
// Scalar per-worker state is warp-uniform: every lane holds the same value and
// executes the same fp64 operation; fp64 follows the oracle's written
// operation order, compiled with -fmad=false and IEEE division.
#include <math.h>

#include "kvr_device.cuh"
#include "kvr_internal.h"

namespace kvr {

#ifdef KVR_WHO_LAST
// experiment build: which warp arrives last at the per-query barrier, by role
// (0: updated the previous query's chosen worker, 1: ran a deferred apply after the
// previous barrier, 2: scoring only); [4..6] the last arrival's lead over the second last
__device__ unsigned long long g_who[16];   // [8..12] apply phases: erase, arrays, inserts, rebuild, tail
#define KVR_WT(v) long long v = clock64()
#define KVR_WA(i, v)                                                              \
  do {                                                                            \
    const long long _n = clock64();                                               \
    if (lane == 0) atomicAdd(&g_who[i], (unsigned long long)(_n - (v)));          \
    v = _n;                                                                       \
  } while (0)
__shared__ uint32_t s_arrive[32], s_role[32];
#else
#define KVR_WT(v) (void)0
#define KVR_WA(i, v) (void)0
#endif
#ifdef KVR_PHASE_PROFILE
// Phase profiler (profiling build only): cycles per phase summed over warps.
__device__ unsigned long long g_phase_cycles[32];
__device__ unsigned long long g_trial_cycles[4096];   // per trial: kernel cycles of its CTA
#define KVR_T0(v) unsigned long long v = clock64()
#define KVR_ACC(ph, v)                                                     \
  do {                                                                     \
    unsigned long long _n = clock64();                                     \
    if (lane == 0) atomicAdd(&g_phase_cycles[ph], _n - (v));               \
    v = _n;                                                                \
  } while (0)
#define KVR_CNT(ph, x)                                                     \
  do {                                                                     \
    if (lane == 0) atomicAdd(&g_phase_cycles[ph], (unsigned long long)(x)); \
  } while (0)
#define KVR_RESET(v) v = clock64()
#else
#define KVR_RESET(v) (void)0
#define KVR_T0(v) (void)0
#define KVR_ACC(ph, v) (void)0
#define KVR_CNT(ph, x) (void)0
#endif

// Dynamic shared memory of the replay kernel.  Every function derives its
// shared-memory pointers from this array (never from pointer arguments) so the
// compiler emits shared-space LDS/STS instead of generic LD/ST.
extern __shared__ __align__(128) uint8_t kvr_dsmem[];

template <typename Idx>
struct Nil {
  static constexpr Idx empty = (Idx)~(Idx)0;
  static constexpr Idx tomb = (Idx)(~(Idx)0 - 1);
};

template <typename Idx>
struct WorkerView {
  uint64_t* key;
  Idx* parent;
  Idx* nchild;
  Idx* table;
  uint32_t* leaf;
  uint32_t* mark;
};

// gbase: identities + table; sbase: tree arrays, bitmaps (and stamps) -- the same base
// except in the split tier (kMem == 2)
template <typename Idx>
__device__ __forceinline__ WorkerView<Idx> make_view(uint8_t* gbase, uint8_t* sbase,
                                                     const WorkerLayout& L) {
  WorkerView<Idx> v;
  v.key = reinterpret_cast<uint64_t*>(gbase + L.off_key);
  v.parent = reinterpret_cast<Idx*>(sbase + L.off_parent);
  v.nchild = reinterpret_cast<Idx*>(sbase + L.off_nchild);
  v.table = reinterpret_cast<Idx*>(gbase + L.off_table);
  v.leaf = reinterpret_cast<uint32_t*>(sbase + L.off_leaf);
  v.mark = reinterpret_cast<uint32_t*>(sbase + L.off_mark);
  return v;
}

// dynamic shared memory map: [Ctrl][stages][WarpSm x W][slot buffers x 2][workers x W] (tier 1)
__device__ __forceinline__ size_t stage_off() { return align16(sizeof(Ctrl)); }
__device__ __forceinline__ size_t warps_off(const ReplayParams& p) {
  return stage_off() + (size_t)kNumStages * p.stage_bytes;
}
__device__ __forceinline__ size_t slotbuf_off(const ReplayParams& p) {
  return warps_off(p) + (size_t)p.W * p.scratch_bytes;
}
__device__ __forceinline__ size_t workers_off(const ReplayParams& p) {
  return slotbuf_off(p) + 2 * (size_t)p.slotbuf_bytes;
}
// the per-miss slots (and, after max_n of them, the overlay bitmap staging) of the update
// of query j: buffer j mod 2
__device__ __forceinline__ uint32_t* slot_buf(const ReplayParams& p, uint32_t j) {
  return reinterpret_cast<uint32_t*>(kvr_dsmem + slotbuf_off(p) + (size_t)(j & 1) * p.slotbuf_bytes);
}
// kMem: 0 = worker state in shared memory, 1 = in global memory, 2 = split (identities and
// tables global, the rest shared), 3 = shared memory like 0; kMem >= 2 runs two workers
// per warp (W > 16)
template <int kMem>
__device__ __forceinline__ uint8_t* worker_gbase(const ReplayParams& p, uint32_t w) {
  if constexpr (kMem == 1 || kMem == 2) return p.gstate + ((size_t)blockIdx.x * p.W + w) * p.lay.gbytes;
  else return kvr_dsmem + workers_off(p) + (size_t)w * p.lay.bytes;
}
template <int kMem>
__device__ __forceinline__ uint8_t* worker_sbase(const ReplayParams& p, uint32_t w) {
  if constexpr (kMem == 2) return kvr_dsmem + workers_off(p) + (size_t)w * p.lay.sbytes;
  else return worker_gbase<kMem>(p, w);
}
__device__ __forceinline__ WarpSm* warp_sm(const ReplayParams& p, uint32_t w) {
  return reinterpret_cast<WarpSm*>(kvr_dsmem + warps_off(p) + (size_t)w * p.scratch_bytes);
}

__device__ __forceinline__ uint32_t lanemask_lt(uint32_t lane) { return (1u << lane) - 1u; }

// ---------------------------------------------------------------- hash table
template <typename Idx>
__device__ __forceinline__ Idx tbl_find(const WorkerView<Idx>& S, uint32_t mask, uint64_t h) {
  uint32_t pos = (uint32_t)h & mask;
#pragma unroll 1
  for (;;) {
    const Idx e = S.table[pos];
    if (e == Nil<Idx>::empty) return Nil<Idx>::empty;
    if (e != Nil<Idx>::tomb && S.key[e] == h) return e;
    pos = (pos + 1) & mask;
  }
}

// remove the entry of `slot` (identity h); lanes may run this concurrently.  The
// entry becomes EMPTY when the next one is EMPTY (no probe path can run through
// it: linear-probing clusters are contiguous), else a tombstone.  A lane that reads
// its neighbour before a concurrent erase of it lands just writes a tombstone.
// Returns 1 when no tombstone was left.
template <typename Idx>
__device__ __forceinline__ uint32_t tbl_erase(const WorkerView<Idx>& S, uint32_t mask, uint64_t h,
                                              Idx slot) {
  uint32_t pos = (uint32_t)h & mask;
#pragma unroll 1
  while (S.table[pos] != slot) pos = (pos + 1) & mask;
  const bool clear = S.table[(pos + 1) & mask] == Nil<Idx>::empty;
  S.table[pos] = clear ? Nil<Idx>::empty : Nil<Idx>::tomb;
  return clear ? 1u : 0u;
}

// claim position pos if it is EMPTY or TOMB (CAS); returns 1 if it was EMPTY.  (Starting
// the CAS from a guessed all-EMPTY word instead of a load measured 3 % slower at W = 32.)
__device__ __forceinline__ uint32_t tbl_claim_at(uint16_t* table, uint32_t pos, uint16_t slot,
                                                 bool* ok) {
  uint32_t* w32 = reinterpret_cast<uint32_t*>(table) + (pos >> 1);
  const uint32_t sh = (pos & 1u) * 16u;
  uint32_t cur = *reinterpret_cast<volatile uint32_t*>(w32);
#pragma unroll 1
  for (;;) {
    const uint32_t e = (cur >> sh) & 0xffffu;
    if (e != 0xffffu && e != 0xfffeu) { *ok = false; return 0; }
    const uint32_t nw = (cur & ~(0xffffu << sh)) | ((uint32_t)slot << sh);
    const uint32_t old = atomicCAS(w32, cur, nw);
    if (old == cur) { *ok = true; return e == 0xffffu ? 1u : 0u; }
    cur = old;
  }
}
__device__ __forceinline__ uint32_t tbl_claim_at(uint32_t* table, uint32_t pos, uint32_t slot,
                                                 bool* ok) {
  uint32_t cur = *reinterpret_cast<volatile uint32_t*>(table + pos);
#pragma unroll 1
  for (;;) {
    if (cur != 0xffffffffu && cur != 0xfffffffeu) { *ok = false; return 0; }
    const uint32_t old = atomicCAS(table + pos, cur, slot);
    if (old == cur) { *ok = true; return cur == 0xffffffffu ? 1u : 0u; }
    cur = old;
  }
}
template <typename Idx>
__device__ __forceinline__ uint32_t tbl_insert(const WorkerView<Idx>& S, uint32_t mask, uint64_t h,
                                               Idx slot) {
  uint32_t pos = (uint32_t)h & mask;
#pragma unroll 1
  for (;;) {
    bool ok;
    const uint32_t was_empty = tbl_claim_at(S.table, pos, slot, &ok);
    if (ok) return was_empty;
    pos = (pos + 1) & mask;
  }
}

// rebuild without tombstones (warp): clear, then re-insert every live slot
template <typename Idx>
__device__ __forceinline__ void tbl_rebuild(const WorkerView<Idx>& S, uint32_t T, uint32_t size,
                                         uint32_t lane) {
  __syncwarp();
  uint4* t4 = reinterpret_cast<uint4*>(S.table);   // 16-B stores (T * sizeof(Idx) % 16 == 0)
  const uint32_t n4 = (uint32_t)(T * sizeof(Idx) / 16);
  for (uint32_t i = lane; i < n4; i += 32) t4[i] = make_uint4(~0u, ~0u, ~0u, ~0u);
  __syncwarp();
  for (uint32_t s = lane; s < size; s += 32) tbl_insert<Idx>(S, T - 1, S.key[s], (Idx)s);
  __syncwarp();
}

// One 32-block window of a longest-cached-prefix match: lane l looks up block base + l
// (blocks >= nq count as misses).  Membership = on the path Hp[0..npp) at the same depth,
// or in the table and, with ovl, not among the pending update's victims (bitmap vbits,
// lane l: word l).  The lanes step their probe chains together and the warp stops as soon
// as the prefix is decided -- the first lane that is not a hit has finished with a miss --
// instead of waiting for the longest chain of the window (most workers miss the first
// block).  Returns the hit ballot, exact up to its first zero bit.
template <typename Idx>
__device__ __forceinline__ uint32_t probe_window(const WorkerView<Idx>& S, uint32_t mask, const uint64_t* Hq,
                                                 uint32_t base, uint32_t nq, const uint64_t* Hp,
                                                 uint32_t npp, bool ovl, uint32_t vbits, uint32_t lane) {
  const uint32_t d = base + lane;
  bool done = true, hit = false;
  uint64_t hh = 0;
  uint32_t pos = 0;
  if (d < nq) {
    hh = Hq[d];
    if (d < npp && Hp[d] == hh) {
      hit = true;
    } else {
      done = false;
      pos = (uint32_t)hh & mask;
    }
  }
#pragma unroll 1
  for (;;) {
    bool fin = false;
    uint32_t sidx = 0;
    if (!done) {
      const Idx e = S.table[pos];
      if (e == Nil<Idx>::empty) {
        done = true;
      } else if (e != Nil<Idx>::tomb && S.key[e] == hh) {
        done = true;
        fin = true;
        hit = true;
        sidx = (uint32_t)e;
      } else {
        pos = (pos + 1) & mask;
      }
    }
    if (ovl) {   // found in the old table but evicted by the pending update?
      const uint32_t vw = __shfl_sync(kFull, vbits, fin ? (sidx >> 5) : 0u);
      if (fin && ((vw >> (sidx & 31)) & 1u)) hit = false;
    }
    const uint32_t dn = __ballot_sync(kFull, done);
    const uint32_t hb = __ballot_sync(kFull, done && hit);
    if (hb == kFull || dn == kFull) return hb;
    const uint32_t k = __ffs(~hb) - 1;   // first lane not (yet) known to hit
    if ((dn >> k) & 1u) return hb;       // ... and it finished with a miss
  }
}

__device__ __forceinline__ uint32_t hist_bin(double lat, uint32_t bins) {
  if (!(lat >= 1.0)) return 0;
  int e;
  const double f = frexp(lat, &e);
  const uint32_t q = (uint32_t)((f * 2.0 - 1.0) * 4.0);
  const uint64_t b = 1 + 4 * (uint64_t)(e - 1) + q;
  return b >= bins ? bins - 1 : (uint32_t)b;
}

// ------------------------------------------------------- Leaf-LRU recency log
// entry = stamp << 32 | slot; valid iff stamp[slot] == entry stamp (mod 2^16: a
// stale entry never survives one compaction period, < 2^16 worker queries).  The first
// e valid entries from the head are the e least-recently-used nodes in
// (stamp, -depth) order because each query appends its path deepest first.
constexpr int kLogDepth = 4;   // log windows (32 entries each) kept in flight

struct RecencyLog {
  uint32_t* log;     // entries stamp << 16 | slot (u16 stamps, slots < 65536)
  uint16_t* stamp;   // per slot, in the worker state (shared memory in tier 1)
  uint32_t cap_mask;
};

// take the first `need` valid entries in [head, tail) as victims -> out[0..need);
// returns the new head (just past the last victim)
// the first kLogDepth windows from `head` (entries are validated against the stamps
// at take time)
__device__ __forceinline__ void log_preload(const RecencyLog& R, uint32_t head, uint32_t tail,
                                            uint32_t lane, uint32_t (&e)[kLogDepth]) {
#pragma unroll
  for (int i = 0; i < kLogDepth; ++i) {
    const uint32_t idx = head + 32u * i + lane;
    e[i] = idx < tail ? R.log[idx & R.cap_mask] : 0u;
  }
}

// e: log_preload(R, head, tail, ...) (the log between head and tail unchanged since)
__device__ __forceinline__ uint32_t log_take(const RecencyLog& R, uint32_t head, uint32_t tail,
                                          uint32_t need, uint32_t* out, uint32_t lane,
                                          uint32_t (&e)[kLogDepth]) {
  uint32_t k = 0, pos = head;
  // software pipeline: kLogDepth windows of entries are in flight while one is filtered
#pragma unroll 1
  for (;;) {
#pragma unroll
    for (int i = 0; i < kLogDepth; ++i) {
      if (k >= need || pos >= tail) {
        __syncwarp();
        return pos;
      }
      const bool act = pos + lane < tail;
      const uint32_t slot = e[i] & 0xffffu;
      const bool valid = act && R.stamp[slot] == (uint16_t)(e[i] >> 16);
      const uint32_t bal = __ballot_sync(kFull, valid);
      const uint32_t take = min((uint32_t)__popc(bal), need - k);
      const uint32_t rank = __popc(bal & lanemask_lt(lane));
      if (valid && rank < take) out[k + rank] = slot;
      k += take;
      if (take > 0 && k == need) {
        pos += select_bit(bal, take - 1) + 1u;   // through the last victim
      } else {
        const uint32_t idx = pos + 32u * kLogDepth + lane;
        e[i] = idx < tail ? R.log[idx & R.cap_mask] : 0u;
        pos += 32u;
      }
    }
  }
}

// first valid entry from head (LRU over leaves != parent(t), fallback A5)
__device__ __forceinline__ uint32_t log_first_valid(const RecencyLog& R, uint32_t head, uint32_t tail,
                                                 uint32_t lane) {
#pragma unroll 1
  for (;; head += 32) {
    const uint32_t idx = head + lane;
    const bool act = idx < tail;
    const uint32_t ent = act ? R.log[idx & R.cap_mask] : 0u;
    const bool valid = act && R.stamp[ent & 0xffffu] == (uint16_t)(ent >> 16);
    const uint32_t bal = __ballot_sync(kFull, valid);
    if (bal) return __shfl_sync(kFull, ent, __ffs(bal) - 1) & 0xffffu;
  }
}

// in-place order-preserving compaction of [head, tail): returns the new tail
__device__ __forceinline__ uint32_t log_compact(const RecencyLog& R, uint32_t head, uint32_t tail,
                                             uint32_t lane) {
  // kLogDepth windows per step: all loads and stamp gathers are independent, only
  // the write cursor is serial.  Writes land below r + 32*kLogDepth (already read),
  // so the in-place order-preserving copy never clobbers an unread entry.
  uint32_t w = head;
#pragma unroll 1
  for (uint32_t r = head; r < tail; r += 32u * kLogDepth) {
    uint32_t e[kLogDepth];
    bool v[kLogDepth];
#pragma unroll
    for (int i = 0; i < kLogDepth; ++i) {
      const uint32_t idx = r + 32u * i + lane;
      e[i] = idx < tail ? R.log[idx & R.cap_mask] : 0u;
    }
#pragma unroll
    for (int i = 0; i < kLogDepth; ++i)
      v[i] = (r + 32u * i + lane < tail) && R.stamp[e[i] & 0xffffu] == (uint16_t)(e[i] >> 16);
    __syncwarp();
#pragma unroll
    for (int i = 0; i < kLogDepth; ++i) {
      const uint32_t bal = __ballot_sync(kFull, v[i]);
      if (v[i]) R.log[(w + __popc(bal & lanemask_lt(lane))) & R.cap_mask] = e[i];
      w += __popc(bal);
    }
    __syncwarp();
  }
  return w;
}

// -------------------------------------------------------------- bitmaps (RLT)
// Register-resident LEAF / MARK words: lane l holds word l (B <= 1024).
struct RegBits {
  uint32_t lw, mw;
  __device__ __forceinline__ void load(const uint32_t* leaf, const uint32_t* mark, uint32_t nw,
                                       uint32_t lane) {
    lw = lane < nw ? leaf[lane] : 0u;
    mw = lane < nw ? mark[lane] : 0u;
  }
  __device__ __forceinline__ void store(uint32_t* leaf, uint32_t* mark, uint32_t nw, uint32_t lane) {
    if (lane < nw) {
      leaf[lane] = lw;
      mark[lane] = mw;
    }
  }
  __device__ __forceinline__ void leaf_set(uint32_t s, uint32_t lane) { if (lane == (s >> 5)) lw |= 1u << (s & 31); }
  __device__ __forceinline__ void leaf_clr(uint32_t s, uint32_t lane) { if (lane == (s >> 5)) lw &= ~(1u << (s & 31)); }
  __device__ __forceinline__ void mark_set(uint32_t s, uint32_t lane) { if (lane == (s >> 5)) mw |= 1u << (s & 31); }
  __device__ __forceinline__ void mark_clr(uint32_t s, uint32_t lane) { if (lane == (s >> 5)) mw &= ~(1u << (s & 31)); }
  __device__ __forceinline__ bool mark_test(uint32_t s) const {
    return (__shfl_sync(kFull, mw, s >> 5) >> (s & 31)) & 1u;
  }
  __device__ __forceinline__ void mark_clear_all_w(uint32_t) { mw = 0u; }
  // |U| for U = LEAF (& ~MARK) minus bit p.  The per-lane popcounts (0..32) are
  // prefix-summed bit-sliced: six independent ballots, then popcounts under the
  // lane mask — no dependent shuffle chain.
  __device__ __forceinline__ uint32_t count(uint32_t p, bool use_mark, uint32_t lane, uint32_t& c,
                                            uint32_t& incl) const {
    uint32_t u = use_mark ? (lw & ~mw) : lw;
    if (lane == (p >> 5)) u &= ~(1u << (p & 31));
    c = __popc(u);
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
  // idx-th element of U in slot order; bit 31 of the result = MARK bit of that slot
  __device__ __forceinline__ uint32_t select(uint32_t p, bool use_mark, uint32_t lane, uint32_t c,
                                             uint32_t incl, uint32_t idx) const {
    const uint32_t owner = __ffs(__ballot_sync(kFull, incl > idx)) - 1;
    uint32_t u = use_mark ? (lw & ~mw) : lw;
    if (lane == (p >> 5)) u &= ~(1u << (p & 31));
    const uint32_t bit = select_bit(u, idx - (incl - c));
    const uint32_t packed = (lane * 32 + bit) | (((mw >> bit) & 1u) << 31);
    return __shfl_sync(kFull, packed, owner);
  }
};

// Memory-resident bitmaps (B > 1024): every lane scans a contiguous chunk of words.
struct MemBits {
  uint32_t* leaf;
  uint32_t* mark;
  uint32_t nw;
  __device__ __forceinline__ void upd(uint32_t* a, uint32_t s, bool set, uint32_t lane) {
    __syncwarp();
    if (lane == 0) {
      if (set) atomicOr(a + (s >> 5), 1u << (s & 31));
      else atomicAnd(a + (s >> 5), ~(1u << (s & 31)));
    }
    __syncwarp();
  }
  __device__ __forceinline__ void leaf_set(uint32_t s, uint32_t lane) { upd(leaf, s, true, lane); }
  __device__ __forceinline__ void leaf_clr(uint32_t s, uint32_t lane) { upd(leaf, s, false, lane); }
  __device__ __forceinline__ void mark_set(uint32_t s, uint32_t lane) { upd(mark, s, true, lane); }
  __device__ __forceinline__ void mark_clr(uint32_t s, uint32_t lane) { upd(mark, s, false, lane); }
  __device__ __forceinline__ bool mark_test(uint32_t s) const { return (mark[s >> 5] >> (s & 31)) & 1u; }
  __device__ __forceinline__ void mark_clear_all_w(uint32_t lane) {
    __syncwarp();
    for (uint32_t i = lane; i < nw; i += 32) mark[i] = 0u;
    __syncwarp();
  }
  __device__ __forceinline__ uint32_t word(uint32_t wi, uint32_t p, bool use_mark) const {
    uint32_t u = leaf[wi];
    if (use_mark) u &= ~mark[wi];
    if (wi == (p >> 5)) u &= ~(1u << (p & 31));
    return u;
  }
  __device__ __forceinline__ uint32_t count(uint32_t p, bool use_mark, uint32_t lane, uint32_t& c,
                                            uint32_t& incl) const {
    const uint32_t wpl = (nw + 31) >> 5;
    const uint32_t w0 = lane * wpl, w1 = min(nw, w0 + wpl);
    uint32_t cc = 0;
    for (uint32_t wi = w0; wi < w1; ++wi) cc += __popc(word(wi, p, use_mark));
    uint32_t v = cc;
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, v, s);
      if (lane >= (uint32_t)s) v += y;
    }
    c = cc;
    incl = v;
    return __shfl_sync(kFull, v, 31);
  }
  __device__ __forceinline__ uint32_t select(uint32_t p, bool use_mark, uint32_t lane, uint32_t c,
                                             uint32_t incl, uint32_t idx) const {
    const uint32_t owner = __ffs(__ballot_sync(kFull, incl > idx)) - 1;
    uint32_t slot = 0;
    if (lane == owner) {
      const uint32_t wpl = (nw + 31) >> 5;
      uint32_t rem = idx - (incl - c);
      for (uint32_t wi = lane * wpl;; ++wi) {
        const uint32_t u = word(wi, p, use_mark);
        const uint32_t pc = __popc(u);
        if (rem < pc) {
          const uint32_t bit = select_bit(u, rem);
          slot = (wi * 32 + bit) | (((mark[wi] >> bit) & 1u) << 31);
          break;
        }
        rem -= pc;
      }
    }
    return __shfl_sync(kFull, slot, owner);
  }
};

// one RLT draw per lane (counter n = e + lane); out of line: runs once per 32 draws
__device__ __noinline__ uint64_t philox_refill(uint64_t K, uint64_t n, uint32_t worker) {
  return philox_r64(K, n, worker, 1u);
}


// RLT decisions for misses [cb, cb+cnt), generic bitmaps (B > 1024).  Serial.
template <typename Bits, typename Idx>
__device__ __forceinline__ void rlt_chunk(Bits& bits, const WorkerView<Idx>& S, const RecencyLog& R,
                                          WorkerRegs& wr, uint32_t B, uint32_t cnt, uint32_t cb,
                                          Idx p0, uint32_t& pslot, uint32_t fallback,
                                          bool use_list, uint64_t K, uint32_t worker,
                                          uint64_t& rbuf, uint32_t& ri, uint32_t lane,
                                          uint32_t* slots, uint32_t& vbits) {
  const Idx NIL = Nil<Idx>::empty;
#pragma unroll 1
  for (uint32_t r = 0; r < cnt; ++r) {
    const uint32_t q = cb + r;
    if (wr.cntT == B) {   // Alg. 1 l.8-9 at the mark of t (t is not cached, not in T)
      bits.mark_clear_all_w(lane);
      wr.cntT = 1;
      ++wr.c_resets;
    } else {
      ++wr.cntT;
    }
    uint32_t slot, ev = 0;
    if (wr.size < B) {
      slot = wr.size++;
    } else {
      uint32_t c, incl;
      bool use_mark = true, draw = true;
      uint32_t total = bits.count(pslot, true, lane, c, incl);
      uint32_t v = 0;
      bool vmarked = false;
      if (total == 0) {   // U = {} (A5)
        ++wr.c_fb;
        if (fallback == KVR_RLT_EARLY_RESET) {
          bits.mark_clear_all_w(lane);
          wr.cntT = 1;
          ++wr.c_resets;
        } else if (fallback == KVR_RLT_UNIFORM_LEAF) {
          use_mark = false;
        } else {
          draw = false;
          v = log_first_valid(R, wr.lhead, wr.ltail, lane);
          vmarked = bits.mark_test(v);
        }
        if (draw) total = bits.count(pslot, use_mark, lane, c, incl);
      }
      if (draw) {
        if (ri == 32) {
          rbuf = philox_refill(K, wr.e + lane, worker);
          ri = 0;
        }
        const uint64_t rr = __shfl_sync(kFull, rbuf, ri);
        ++ri;
        ++wr.e;
        ++wr.c_draws;
        const uint32_t sel = bits.select(pslot, use_mark, lane, c, incl,
                                         (uint32_t)pick_index(rr, total));
        v = sel & 0x7fffffffu;
        vmarked = (sel >> 31) != 0;
      }
      const Idx pv = S.parent[v];
      if (pv != NIL) {
        const Idx nc = (Idx)(S.nchild[pv] - 1);
        __syncwarp();
        S.nchild[pv] = nc;
        if (nc == 0) bits.leaf_set(pv, lane);
      }
      bits.leaf_clr(v, lane);
      if (vmarked) {
        bits.mark_clr(v, lane);
        --wr.cntT;
      }
      ++wr.c_evict;
      slot = v;
      ev = 1;
    }
    bits.leaf_set(slot, lane);
    bits.mark_set(slot, lane);
    if (q == 0) {
      if (p0 != NIL) {
        const Idx nc = S.nchild[p0];
        __syncwarp();
        S.nchild[p0] = (Idx)(nc + 1);
        if (nc == 0) bits.leaf_clr(p0, lane);
      }
    } else {
      bits.leaf_clr(pslot, lane);
    }
    if (use_list) R.stamp[slot] = wr.wq;
    slots[q] = slot | (ev << 31);
    if (ev && lane == (slot >> 5)) vbits |= 1u << (slot & 31);
    pslot = slot;
  }
}

// floor(r64 * t / 2^64) for r64 = hi:lo and t < 2^32 (== __umul64hi(r64, t); A6)
__device__ __forceinline__ uint32_t pick32(uint32_t lo, uint32_t hi, uint32_t t) {
  return (uint32_t)(((uint64_t)hi * t + __umulhi(lo, t)) >> 32);
}

// All RLT miss decisions of one query (Alg. 1 l.6-17 in path order), register
// bitmaps (B <= 1024).  Out of line so the serial chain gets its own register
// allocation; state is copied in and out once per query.  Per lane l:
//   lw, mw  LEAF / MARK word l;   uw  word l of U = LEAF & ~MARK & ~{p};
//   incl    inclusive prefix count of U over words 0..l;   total = |U|.
// The common eviction step is a handful of dependent instructions: the owner
// word is popc(ballot(incl <= idx)), the bit inside it popc(ballot(rank_le <=
// rem)); U loses the victim (its slot is refilled by the new, marked leaf) and
// gains the victim's parent iff that became an unmarked leaf.  Resets and the
// U = {} fallbacks (A5) recount from lw/mw.
template <typename Idx, int kMem, int kTag>
__device__ __noinline__ void rlt_decide_reg(const ReplayParams& p_, uint32_t M, Idx p0,
                                            uint32_t fallback, uint64_t K, uint32_t worker,
                                            uint32_t lane, bool use_list, uint32_t jq) {
  const Idx NIL = Nil<Idx>::empty;
  const uint32_t B = p_.B, nwords = p_.lay.nwords;
  uint8_t* wb = worker_gbase<kMem>(p_, worker);
  uint8_t* sb = worker_sbase<kMem>(p_, worker);
  const WorkerView<Idx> S = make_view<Idx>(wb, sb, p_.lay);
  RecencyLog R;
  R.log = reinterpret_cast<uint32_t*>(p_.aux_base + ((size_t)blockIdx.x * p_.W + worker) * p_.aux.bytes +
                                      p_.aux.off_log);
  R.stamp = reinterpret_cast<uint16_t*>(sb + p_.lay.off_stamp);
  R.cap_mask = p_.aux.log_cap - 1;
  // state in and out through the warp's shared-memory block (no by-reference
  // arguments: they would put the caller's registers in local memory)
  WarpSm* ws = warp_sm(p_, worker);
  uint32_t* slots = slot_buf(p_, jq);
  uint32_t* vmap = slots + p_.max_n;
  // registers: size, |T| and e_i only; counters are bumped in shared memory (draws
  // = the change of e_i, evictions are counted by the caller), the log cursors and
  // recency stamp are read there on the rare paths that need them
  struct {
    uint32_t size, cntT;
    uint64_t e;
  } wr;
  wr.size = ws->x.size;
  wr.cntT = ws->x.cntT;
  wr.e = ws->x.e;
  const uint32_t wq = use_list ? ws->x.wq : 0u;
  const uint64_t rb_in = ws->x_rbuf[lane];
  uint32_t rlo = (uint32_t)rb_in, rhi = (uint32_t)(rb_in >> 32);
  uint32_t ri = ws->x_ri, vbits = 0, p = (uint32_t)p0;
  // The next batch of 32 draws (counters base + 32 + lane), computed at entry where the
  // Philox rounds overlap the bitmap loads and the first recount, when this update may
  // run past the current batch (at most M draws); a batch exhausted in the fast segment
  // is then replaced without leaving it.  (ri == 32: no current batch; it is computed
  // the same way.)  The counters are those a refill would use, so results are unchanged.
  uint32_t nlo = 0, nhi = 0;
  bool nready = false;
  if (wr.size + M > B && M > 32u - ri) {
    const uint64_t r = philox_r64(K, (wr.e - (ri == 32 ? 0u : ri)) + (ri == 32 ? 0u : 32u) + lane, worker, 1u);
    if (ri == 32) {
      rlo = (uint32_t)r;
      rhi = (uint32_t)(r >> 32);
      ri = 0;
    } else {
      nlo = (uint32_t)r;
      nhi = (uint32_t)(r >> 32);
      nready = true;
    }
  }
  RegBits rb;
  rb.load(S.leaf, S.mark, nwords, lane);
  const uint32_t lmle = lane == 31 ? kFull : (2u << lane) - 1u;   // lanes <= lane
  uint32_t uw = 0, incl = 0, total = 0;
  bool dirty = true;
  uint32_t q = 0;
#pragma unroll 1
  for (; q < M; ++q) {
    // ---- fast segment: evictions with no mark reset, no refill, U != {}, q > 0 ----
    // (victims are old nodes, so their parents are never the excluded p; the new
    // node's parent p is the previous new node, marked, hence outside U)
    if (q > 0 && wr.size == B && !dirty && wr.cntT < B && total > 0 && ri < 32) {
      const uint32_t lim = min(M, min(q + (B - wr.cntT), q + (32u - ri) + (nready ? 32u : 0u)));
      KVR_T0(tfast);
      KVR_CNT(26, 0u - q);
      uint32_t dlo = __shfl_sync(kFull, rlo, ri), dhi = __shfl_sync(kFull, rhi, ri);
#pragma unroll 1
      for (; q < lim && total > 0; ++q) {
        ++wr.cntT;
        ++ri;
        const uint32_t idx = pick32(dlo, dhi, total);
        if (ri == 32 && nready) {   // the prefetched batch takes over
          rlo = nlo;
          rhi = nhi;
          ri = 0;
          nready = false;
        }
        // the next draw's broadcast is off the chain (lane 0 when this was the last)
        dlo = __shfl_sync(kFull, rlo, ri & 31);
        dhi = __shfl_sync(kFull, rhi, ri & 31);
        // first lane whose inclusive count exceeds idx (incl is nondecreasing over
        // lanes); CREDUX.MIN is ~2x faster than VOTE+POPC on the chain
        const uint32_t owner = __reduce_min_sync(kFull, incl > idx ? lane : 32u);
        // speculative, while the bit is selected: lane l fetches for slot owner*32+l
        // its parent, the parent's child count and the parent's MARK word, so the
        // chosen bit's values arrive by three independent shuffles
        uint32_t sp = (uint32_t)S.parent[owner * 32 + lane];
        const bool sok = sp < B;            // NIL (root child) or padding slot
        sp = sok ? sp : 0u;
        const uint32_t snc = (uint32_t)S.nchild[sp];
        const uint32_t smw = __shfl_sync(kFull, rb.mw, sp >> 5);
        const uint32_t ou = __shfl_sync(kFull, uw, owner);
        const uint32_t rem = idx - (__shfl_sync(kFull, incl, owner) - (uint32_t)__popc(ou));
        const uint32_t bit = __reduce_min_sync(kFull, (uint32_t)__popc(ou & lmle) > rem ? lane : 32u);
        const uint32_t v = owner * 32 + bit;
        const uint32_t vb = 1u << bit;
        const uint32_t pv = __shfl_sync(kFull, sp, bit);
        const bool hasp = __shfl_sync(kFull, (uint32_t)sok, bit) != 0u;
        const uint32_t nc = __shfl_sync(kFull, snc, bit) - 1u;
        const uint32_t pmw = __shfl_sync(kFull, smw, bit);
        if (lane == owner) {
          uw &= ~vb;
          rb.mw |= vb;
          vbits |= vb;
        }
        if (lane >= owner) --incl;
        --total;
        if (hasp) S.nchild[pv] = (Idx)nc;   // uniform store (every lane read its value above)
        const bool leafp = hasp && nc == 0;
        const uint32_t pw = pv >> 5, pb = 1u << (pv & 31);
        const bool add = leafp && !(pmw & pb);   // pv != v: the victim's MARK bit is irrelevant
        if (leafp && lane == pw) {
          rb.lw |= pb;
          if (add) uw |= pb;
        }
        if (add) {
          if (lane >= pw) ++incl;
          ++total;
        }
        if (lane == (p >> 5)) rb.lw &= ~(1u << (p & 31));   // previous new node gets a child
        if (use_list) R.stamp[v] = (uint16_t)wq;
        slots[q] = v | 0x80000000u;
        p = v;
        ++wr.e;
      }
      KVR_ACC(25, tfast);
      KVR_CNT(26, q);
      if (q >= M) break;
    }
    if (wr.cntT == B) {   // Alg. 1 l.8-9 at the mark of t (t is not cached: not in T)
      rb.mw = 0u;
      wr.cntT = 1;
      if (lane == 0) ++ws->x.c_resets;
      dirty = true;
    } else {
      ++wr.cntT;
    }
    uint32_t slot, ev = 0;
    if (wr.size < B) {
      slot = wr.size++;   // new marked leaf: not in U
      rb.leaf_set(slot, lane);
      rb.mark_set(slot, lane);
    } else {
      if (dirty) {
        uw = rb.lw & ~rb.mw;
        if (lane == (p >> 5)) uw &= ~(1u << (p & 31));
        uint32_t c;
        total = rb.count(p, true, lane, c, incl);
        dirty = false;
      }
      bool generic = false;
      if (total == 0) {   // U = {} (A5)
        if (lane == 0) ++ws->x.c_fb;
        if (fallback == KVR_RLT_EARLY_RESET) {
          rb.mw = 0u;
          wr.cntT = 1;
              if (lane == 0) ++ws->x.c_resets;
          uw = rb.lw;
          if (lane == (p >> 5)) uw &= ~(1u << (p & 31));
          uint32_t c;
          total = rb.count(p, true, lane, c, incl);
        } else {
          generic = true;
        }
      }
      uint32_t v;
      if (!generic) {
        if (ri == 32) {   // 32 counter-based draws e .. e+31, one per lane
          if (nready) {
            rlo = nlo;
            rhi = nhi;
            nready = false;
          } else {
            const uint64_t r = philox_refill(K, wr.e + lane, worker);
            rlo = (uint32_t)r;
            rhi = (uint32_t)(r >> 32);
          }
          ri = 0;
        }
        const uint32_t dlo = __shfl_sync(kFull, rlo, ri), dhi = __shfl_sync(kFull, rhi, ri);
        ++ri;
        ++wr.e;
        const uint32_t idx = pick32(dlo, dhi, total);
        const uint32_t owner = __popc(__ballot_sync(kFull, incl <= idx));
        const uint32_t ou = __shfl_sync(kFull, uw, owner);
        const uint32_t rem = idx - (__shfl_sync(kFull, incl, owner) - (uint32_t)__popc(ou));
        const uint32_t bit = __popc(__ballot_sync(kFull, (uint32_t)__popc(ou & lmle) <= rem));
        v = owner * 32 + bit;
        // Evict(S, v) + Load(S, t) into slot v: LEAF stays, MARK set, U loses v
        if (lane == owner) {
          uw &= ~(1u << bit);
          rb.mw |= 1u << bit;
        }
        if (lane >= owner) --incl;
        --total;
        const Idx pv = S.parent[v];
        if (pv != NIL) {
          const Idx nc = (Idx)(S.nchild[pv] - 1);
          __syncwarp();
          S.nchild[pv] = nc;   // uniform store
          if (nc == 0) {       // pv became a leaf; joins U iff unmarked and != p
            const uint32_t pw = (uint32_t)pv >> 5, pb = 1u << ((uint32_t)pv & 31);
            const bool add = __ballot_sync(kFull, lane == pw && !(rb.mw & pb)) != 0u &&
                             (uint32_t)pv != p;
            if (lane == pw) {
              rb.lw |= pb;
              if (add) uw |= pb;
            }
            if (add) {
              if (lane >= pw) ++incl;
              ++total;
            }
          }
        }
      } else {
        bool vmarked;
        if (fallback == KVR_RLT_UNIFORM_LEAF) {   // uniform over leaves != p, marks ignored
          if (ri == 32) {
            if (nready) {
              rlo = nlo;
              rhi = nhi;
              nready = false;
            } else {
              const uint64_t r = philox_refill(K, wr.e + lane, worker);
              rlo = (uint32_t)r;
              rhi = (uint32_t)(r >> 32);
            }
            ri = 0;
          }
          const uint32_t dlo = __shfl_sync(kFull, rlo, ri), dhi = __shfl_sync(kFull, rhi, ri);
          ++ri;
          ++wr.e;
          uint32_t c, inc2;
          const uint32_t tot = rb.count(p, false, lane, c, inc2);
          const uint32_t sel = rb.select(p, false, lane, c, inc2, pick32(dlo, dhi, tot));
          v = sel & 0x7fffffffu;
          vmarked = (sel >> 31) != 0;
        } else {   // LRU_MARKED: least recently used leaf != p, no draw
          v = log_first_valid(R, ws->x.lhead, ws->x.ltail, lane);
          vmarked = rb.mark_test(v);
        }
        rb.leaf_clr(v, lane);
        if (vmarked) {
          rb.mark_clr(v, lane);
          --wr.cntT;
        }
        const Idx pv = S.parent[v];
        if (pv != NIL) {
          const Idx nc = (Idx)(S.nchild[pv] - 1);
          __syncwarp();
          S.nchild[pv] = nc;
          if (nc == 0) rb.leaf_set(pv, lane);
        }
        rb.leaf_set(v, lane);
        rb.mark_set(v, lane);
        dirty = true;
      }
      slot = v;
      ev = 1;
      if (lane == (v >> 5)) vbits |= 1u << (v & 31);
    }
    // the new node's parent stops being a leaf (excluded as p, or marked: U unchanged)
    if (q == 0) {
      if (p0 != NIL) {
        const Idx nc = S.nchild[p0];
        __syncwarp();
        S.nchild[p0] = (Idx)(nc + 1);
        if (nc == 0) rb.leaf_clr(p0, lane);
      }
    } else {
      rb.leaf_clr(p, lane);
    }
    if (use_list) R.stamp[slot] = (uint16_t)wq;   // LRU_MARKED fallback reads the log
    slots[q] = slot | (ev << 31);
    p = slot;
  }
  rb.store(S.leaf, S.mark, nwords, lane);
  __syncwarp();
  if (lane == 0) {
    ws->x.c_draws += (uint32_t)(wr.e - ws->x.e);   // one draw per e_i step
    ws->x.size = wr.size;
    ws->x.cntT = wr.cntT;
    ws->x.e = wr.e;
    ws->x_ri = ri;
  }
  ws->x_rbuf[lane] = ((uint64_t)rhi << 32) | rlo;
  vmap[lane] = vbits;   // victims of this update -> overlay bitmap (read back by the caller)
  __syncwarp();
}

// LBGR_RLS residual model (reading A8b of "learning rate 0.992"; squared
// loss): P (4x4, fp64) lives in the worker's aux region (global, L2).
__device__ __forceinline__ double* rls_region(const ReplayParams& p, uint32_t w) {
  return reinterpret_cast<double*>(p.aux_base + ((size_t)blockIdx.x * p.W + w) * p.aux.bytes +
                                   p.aux.off_rls);
}

// Offline Belady OPT (the W = 1 analysis of SURVEY §8f #1).  Per miss in
// path order: evict the leaf != parent(t) with the largest key (next use, depth) --
// leaves never used again rank highest, the lowest slot first -- found by a warp
// max over the per-slot keys of the current leaves.  A node's key is set whenever
// the current query touches it (hit or insert), so it is always its next use after
// the current query.  Keys live in the worker's aux region (the recency log's
// space, unused by OPT); LEAF bits and child counts are kept in place as for RLT.
__device__ __forceinline__ uint64_t opt_key(uint32_t nu, uint32_t depth, uint32_t slot) {
  return nu == 0xFFFFFFFFu ? (0xFFFFFFFF00000000ull | (0xFFFFu - slot))
                           : (((uint64_t)nu << 32) | depth);
}

__device__ __forceinline__ uint64_t* opt_keys(const ReplayParams& p, uint32_t w) {
  return reinterpret_cast<uint64_t*>(p.aux_base + ((size_t)blockIdx.x * p.W + w) * p.aux.bytes +
                                     p.aux.off_log);
}

template <typename Idx, int kMem, int kTag>
__device__ __noinline__ void opt_decide(const ReplayParams& p_, uint32_t M, uint32_t kf, Idx p0,
                                        const uint32_t* nu_q, uint32_t worker, uint32_t lane,
                                        uint32_t jq) {
  const Idx NIL = Nil<Idx>::empty;
  const uint32_t B = p_.B;
  uint8_t* wb = worker_gbase<kMem>(p_, worker);
  uint8_t* sb = worker_sbase<kMem>(p_, worker);
  const WorkerView<Idx> S = make_view<Idx>(wb, sb, p_.lay);
  uint64_t* okey = opt_keys(p_, worker);
  WarpSm* ws = warp_sm(p_, worker);
  uint32_t* slots = slot_buf(p_, jq);
  MemBits mb;
  mb.leaf = S.leaf;
  mb.mark = S.mark;
  mb.nw = p_.lay.nwords;
  uint32_t size = ws->x.size;
  uint32_t vbits = 0, p = (uint32_t)p0;
#pragma unroll 1
  for (uint32_t q = 0; q < M; ++q) {
    uint32_t slot, ev = 0;
    if (size < B) {
      slot = size++;
      mb.leaf_set(slot, lane);
    } else {
      uint64_t best = 0;
      uint32_t bs = 0;
#pragma unroll 4
      for (uint32_t base = 0; base < B; base += 32) {
        const uint32_t sl = base + lane;
        uint64_t k = 0;
        if (sl < B && sl != p && ((S.leaf[sl >> 5] >> (sl & 31)) & 1u)) k = okey[sl];
        if (k > best) {
          best = k;
          bs = sl;
        }
      }
      const uint32_t hi = (uint32_t)(best >> 32), lo = (uint32_t)best;
      const uint32_t mh = __reduce_max_sync(kFull, hi);
      const uint32_t ml = __reduce_max_sync(kFull, hi == mh ? lo : 0u);
      const uint32_t wl = __reduce_min_sync(kFull, (hi == mh && lo == ml) ? lane : 31u);
      const uint32_t v = __shfl_sync(kFull, bs, wl);
      // Evict(S, v): its parent loses a child and becomes a leaf without children
      const Idx pv = S.parent[v];
      if (pv != NIL) {
        const Idx nc = (Idx)(S.nchild[pv] - 1);
        __syncwarp();
        if (lane == 0) S.nchild[pv] = nc;
        if (nc == 0) mb.leaf_set((uint32_t)pv, lane);
      }
      slot = v;
      ev = 1;
      if (lane == (v >> 5)) vbits |= 1u << (v & 31);
    }
    // Load(S, t): the new leaf's key; its parent gets a child (stops being a leaf)
    const uint32_t d = kf + q;
    const uint64_t nk = opt_key(nu_q[d], d + 1, slot);
    if (lane == 0) okey[slot] = nk;
    if (q == 0) {
      if (p0 != NIL) {
        const Idx nc = S.nchild[p0];
        __syncwarp();
        if (lane == 0) S.nchild[p0] = (Idx)(nc + 1);
        if (nc == 0) mb.leaf_clr((uint32_t)p0, lane);
      }
    } else {
      mb.leaf_clr(p, lane);
    }
    if (lane == 0) slots[q] = slot | (ev << 31);
    p = slot;
    __syncwarp();
  }
  if (lane == 0) ws->x.size = size;
  (slots + p_.max_n)[lane] = vbits;   // victims -> overlay bitmap (read back by the caller)
  __syncwarp();
}

// ---------------------------------------------- stale global tracker (reading A29)
// The router's view of worker i under a lag of k events is the worker's cache as it
// was after query j-1-k: a mirror (identity per slot + table identity -> slot, in the
// worker's aux region) that replays the worker's own updates k queries late from
// the per-CTA ring of the trial's last kLagRing updates (header + per-miss slots).
template <typename Idx>
__device__ __forceinline__ WorkerView<Idx> mirror_view(const ReplayParams& p, uint32_t w) {
  uint8_t* a = p.aux_base + ((size_t)blockIdx.x * p.W + w) * p.aux.bytes;
  WorkerView<Idx> v{};
  v.key = reinterpret_cast<uint64_t*>(a + p.aux.off_mkey);
  v.table = reinterpret_cast<Idx*>(a + p.aux.off_mtab);
  return v;
}
__device__ __forceinline__ LagHdr* lag_entry(const ReplayParams& p, uint32_t j) {
  return reinterpret_cast<LagHdr*>(p.lag_base +
                                   ((size_t)blockIdx.x * kLagRing + j % kLagRing) * p.lag_entry);
}
__device__ __forceinline__ uint32_t* last_access(const ReplayParams& p, uint32_t w) {
  return reinterpret_cast<uint32_t*>(p.aux_base + ((size_t)blockIdx.x * p.W + w) * p.aux.bytes +
                                     p.aux.off_last);
}

// apply ring entry jj (an update of this warp's worker) to the worker's mirror: the
// same table deletes / slot overwrites / inserts as apply_update, nothing else
template <typename Idx, int kTag>
__device__ __noinline__ void mirror_apply(const ReplayParams& p, const uint64_t* hash, uint32_t w,
                                          uint32_t lane, uint32_t jj) {
  const LagHdr* e = lag_entry(p, jj);
  const uint32_t M = e->M, kf = e->kf;
  const uint64_t off = e->block_off;
  const uint32_t* sl = reinterpret_cast<const uint32_t*>(e + 1);
  const WorkerView<Idx> V = mirror_view<Idx>(p, w);
  const uint32_t tmask = p.lay.T - 1;
  WarpSm* ws = warp_sm(p, w);
  uint32_t add = 0, sub = 0, fresh = 0;
#pragma unroll 1
  for (uint32_t cb = 0; cb < M; cb += 32) {
    const uint32_t q = cb + lane;
    const bool act = q < M;
    const uint32_t sv = act ? sl[q] : 0u;
    const uint32_t slot = sv & 0x7fffffffu;
    const bool ev = (sv >> 31) != 0;
    const uint64_t t = act ? hash[off + kf + q] : 0ull;
    uint32_t cleared = 0;
    if (act && ev) cleared = tbl_erase<Idx>(V, tmask, V.key[slot], (Idx)slot);
    __syncwarp();
    if (act) V.key[slot] = t;
    __syncwarp();
    const uint32_t claimed = act ? tbl_insert<Idx>(V, tmask, t, (Idx)slot) : 0u;
    add += __popc(__ballot_sync(kFull, claimed != 0));
    sub += __popc(__ballot_sync(kFull, cleared != 0));
    fresh += __popc(__ballot_sync(kFull, act && !ev));
    __syncwarp();
  }
  uint32_t used = ws->m_used + add - sub;
  const uint32_t size = ws->m_size + fresh;
  if (used > p.lay.rebuild_at) {
    tbl_rebuild<Idx>(V, p.lay.T, size, lane);
    used = size;
  }
  __syncwarp();
  if (lane == 0) {
    ws->m_used = used;
    ws->m_size = size;
  }
  __syncwarp();
}

// Deferred apply of one update: table deletes/inserts, slot arrays, log entries,
// victim digest term and the query record (trial sums are added in query order
// by the accounting step).
template <typename Idx, int kMem, int kTag, bool kExt>
__device__ __noinline__ void apply_update(const ReplayParams& p, uint32_t lane, uint32_t w, bool tree,
                                          bool use_list, bool lbgr_or_static, kvr_query_record* rec,
                                          uint64_t* vlog) {
  Ctrl* ctrl = reinterpret_cast<Ctrl*>(kvr_dsmem);
  WarpSm* ws = warp_sm(p, w);
  const uint8_t* stage = kvr_dsmem + stage_off();
  uint8_t* wb = worker_gbase<kMem>(p, w);
  uint8_t* sb = worker_sbase<kMem>(p, w);
  const WorkerView<Idx> S = make_view<Idx>(wb, sb, p.lay);
  RecencyLog R;
  R.log = reinterpret_cast<uint32_t*>(p.aux_base + ((size_t)blockIdx.x * p.W + w) * p.aux.bytes +
                                      p.aux.off_log);
  R.stamp = reinterpret_cast<uint16_t*>(sb + p.lay.off_stamp);
  R.cap_mask = p.aux.log_cap - 1;
  const uint32_t tmask = p.lay.T - 1;
  const uint64_t* H = reinterpret_cast<const uint64_t*>(stage + (size_t)ws->buf * p.stage_bytes + 32);
  const uint64_t boff = reinterpret_cast<const QueryHdr*>(stage + (size_t)ws->buf * p.stage_bytes)->block_off;
  H += (boff & 1);
  // phase ledger of this trial (extended instantiation only; pointers in the control block)
  uint32_t* led = kExt ? ctrl->led : nullptr;
  const uint32_t* ph = kExt ? ctrl->lph : nullptr;
  const uint32_t* nx = kExt ? ctrl->lnx : nullptr;
  uint32_t* lastacc = led ? last_access(p, w) : nullptr;
  const uint32_t n = ws->n, kf = ws->kf, M = ws->M, nev = ws->nev, wq = ws->wq, ltail0 = ws->ltail0;
  const uint32_t* wslots = slot_buf(p, ws->j);
  const uint32_t nfree = M - nev;
  const uint64_t vc = ws->vc;
  uint64_t V = 0;
  uint32_t used_add = 0, used_sub = 0, prev_last = ws->p0;
  KVR_T0(t_ap);
  KVR_WT(tw);
#pragma unroll 1
  for (uint32_t cb = 0; cb < M; cb += 32) {
    const uint32_t cnt = min(32u, M - cb);
    const uint32_t qq = cb + lane;
    const bool act = lane < cnt;
    const uint32_t sv = act ? wslots[qq] : 0u;
    const uint32_t my_slot = sv & 0x7fffffffu;
    const bool my_ev = (sv >> 31) != 0;
    const uint64_t t = act ? H[kf + qq] : 0ull;
    uint32_t cleared = 0;
    if (led && act) {
      // phase ledger (A39): this miss, and whether the victim was cached when
      // this phase began and is first requested again in it (not clean then)
      const uint64_t o = boff + kf + qq;
      const uint32_t pw = ph[o], v = pw & 0x7fffffffu;
      atomicAdd(&led[4 * v + 1], 1u);
      if (pw >> 31) atomicAdd(&led[4 * v + 2], 1u);
      if (my_ev) {
        const uint32_t nxo = nx[lastacc[my_slot]];
        if (nxo != 0xFFFFFFFFu) {
          const uint32_t pn = ph[nxo];
          if ((pn >> 31) && (pn & 0x7fffffffu) == v) atomicAdd(&led[4 * v + 3], 1u);
        }
      }
      lastacc[my_slot] = (uint32_t)o;
    }
    if (act && my_ev) {
      const uint64_t vkey = S.key[my_slot];
      cleared = tbl_erase<Idx>(S, tmask, vkey, (Idx)my_slot);
      V ^= fmix64(vkey ^ ((uint64_t)(qq - nfree + 1) * kPosMul));
      if (vlog) {
        const uint64_t vi = vc + (qq - nfree);
        if (vi < p.victims_per_trial) vlog[vi] = vkey;
      }
    }
    KVR_ACC(29, t_ap);   // erase (victims) incl. slot/identity loads
    KVR_WA(8, tw);
    const uint32_t up = __shfl_up_sync(kFull, my_slot, 1);
    const uint32_t par_slot = lane == 0 ? prev_last : up;
    __syncwarp();
    if (act) {
      S.key[my_slot] = t;
      if (tree) {   // RLT and OPT keep the prefix tree (parents, child counts)
        S.parent[my_slot] = (Idx)par_slot;
        S.nchild[my_slot] = (Idx)(qq + 1 < M ? 1 : 0);
      }
      if (use_list) {
        if (!tree) R.stamp[my_slot] = wq;
        R.log[(ltail0 + (n - 1 - (kf + qq))) & R.cap_mask] = (wq << 16) | my_slot;
      }
    }
    __syncwarp();
    KVR_ACC(30, t_ap);   // slot arrays, stamps, log entries
    KVR_WA(9, tw);
    const uint32_t claimed = act ? tbl_insert<Idx>(S, tmask, t, (Idx)my_slot) : 0u;
    used_add += __popc(__ballot_sync(kFull, claimed != 0));
    used_sub += __popc(__ballot_sync(kFull, cleared != 0));
    prev_last = __shfl_sync(kFull, my_slot, cnt - 1);
    __syncwarp();
    KVR_ACC(31, t_ap);   // table inserts
    KVR_WA(10, tw);
  }
  uint32_t used = ws->x.used + used_add - used_sub;   // live + tombstone table entries
  if (used > p.lay.rebuild_at) {
    tbl_rebuild<Idx>(S, p.lay.T, ws->x.size, lane);
    used = ws->x.size;
  }
  KVR_ACC(24, t_ap);   // rebuilds
  KVR_WA(11, tw);
  V = warp_xor64(V);
  // (two workers per warp: another warp may be waiting to score this worker; every lane's
  // table / slot writes are made visible before lane 0 clears `active`.  With one worker
  // per warp only the worker's own warp ever reads them.)
  if constexpr (kMem >= 2) __threadfence_block();
  __syncwarp();   // every lane's reads of ws->x.used / ws->active precede lane 0's writes
  if (lane == 0) {
    // decision digest: D += T_j, order-independent across queries
    uint64_t T = fmix64(ctrl->dkey ^ (uint64_t)ws->j);
    T = fmix64(T ^ (uint64_t)w);
    T = fmix64(T ^ (uint64_t)ws->m);
    T = fmix64(T ^ (uint64_t)nev);
    T = fmix64(T ^ V);
    atomicAdd(&ctrl->digest, T);
    const double lat = ws->lat, ttft = ws->ttft;
    if (rec) {
      kvr_query_record Rq;
      Rq.worker = w;
      Rq.hit_tokens = ws->h;
      Rq.n_victims = nev;
      Rq._pad = 0;
      Rq.ttft_ms = ttft;
      Rq.latency_ms = lat;
      Rq.score = lbgr_or_static ? ws->score : 0.0;
      Rq.victim_offset = vc;
      rec[ws->j] = Rq;
    }
    ws->active = 0;
    ws->x.used = used;
  }
  __syncwarp();
  KVR_ACC(23, t_ap);   // digest term, record
  KVR_WA(12, tw);
}

// Scalar state of one worker in the query loop (see the kernel): FIFO head / count,
// Eq. 2 load P, last completion F, LBGR's decayed load P~ and theta, the tick count,
// the FIFO front record (lane f < 8 holds field f; fr_c uniform) and the overlay victim
// bitmap of a pending update (lane l: word l).
struct WSt {
  double P, F, Pt, th0, th1, th2, th3, fr, fr_c;
  uint64_t k;
  uint32_t fh, fn, vbits;
};
// its shared-memory save area (split tier: two workers per warp), after the workers
__device__ __forceinline__ WSave* wsave(const ReplayParams& p, uint32_t v) {
  return reinterpret_cast<WSave*>(kvr_dsmem + workers_off(p) + (size_t)p.W * p.lay.sbytes) + v;
}

// occupancy targets (shared memory allows ~4 CTAs/SM at W<=4 and 2 at W<=8):
// 128 threads -> 4 CTAs/SM (128 regs), 256 -> 2 (128 regs), else 1
template <int kMaxThreads>
struct MinBlocks { static constexpr int value = kMaxThreads <= 128 ? 4 : (kMaxThreads <= 256 ? 2 : 1); };

// kExt: the extended policies (offline OPT, LBGR_RLS, tracker bias) are
// compiled in.  The lean instantiation runs the paper's default policies without
// paying for them in registers and code layout (measured 2.6 %).
template <typename Idx, int kMem, int kMaxThreads, bool kExt>
__global__ void __launch_bounds__(kMaxThreads, MinBlocks<kMaxThreads>::value)
    replay_kernel(const __grid_constant__ ReplayParams p) {
  uint8_t* smem = kvr_dsmem;
  const Idx NIL = Nil<Idx>::empty;
  // workers per warp: the split tier (W > 16) runs W/2 warps of two workers each, so that
  // every thread keeps 128 registers (1,024 threads would cap them at 64 and spill)
  constexpr uint32_t kV = kMem >= 2 ? 2u : 1u;
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nwarps = blockDim.x >> 5;
  const uint32_t W = p.W, B = p.B;
  const WorkerLayout& L = p.lay;
  const uint32_t tmask = L.T - 1, nwords = L.nwords;

  Ctrl* ctrl = reinterpret_cast<Ctrl*>(smem);
  uint8_t* stage = smem + align16(sizeof(Ctrl));
  // exact (bt*k)/1000 for k = 0..max_n (A9), per CTA in global memory (L1-resident)
  double* divtab = p.divtab_base + (size_t)blockIdx.x * (p.max_n + 1);
  // this CTA's pending-FIFO pool: chunk links, then 32-record chunks (FifoLayout)
  uint32_t* flink = reinterpret_cast<uint32_t*>(p.fifo_base + (size_t)blockIdx.x * p.fifo.bytes);
  double* fifo = reinterpret_cast<double*>(p.fifo_base + (size_t)blockIdx.x * p.fifo.bytes +
                                           p.fifo.off_rec);
  const bool regbits = nwords <= 32;
  // per-worker scalar state of the query loop: registers (kV == 1) or, with two workers
  // per warp, saved in shared memory between uses (only one set live at a time)
  WSt st0{};
  auto st_load = [&](uint32_t v) -> WSt {
    const WSave* sv = wsave(p, v);
    WSt X;
    X.P = sv->u[0]; X.F = sv->u[1]; X.Pt = sv->u[2]; X.th0 = sv->u[3]; X.th1 = sv->u[4];
    X.th2 = sv->u[5]; X.th3 = sv->u[6]; X.fr_c = sv->u[7]; X.k = sv->k; X.fh = sv->fh; X.fn = sv->fn;
    X.fr = lane < 8 ? sv->fr[lane] : 0.0;
    X.vbits = sv->vb[lane];
    return X;
  };
  auto st_store = [&](uint32_t v, const WSt& X) {
    WSave* sv = wsave(p, v);
    __syncwarp();
    if (lane == 0) {
      sv->u[0] = X.P; sv->u[1] = X.F; sv->u[2] = X.Pt; sv->u[3] = X.th0; sv->u[4] = X.th1;
      sv->u[5] = X.th2; sv->u[6] = X.th3; sv->u[7] = X.fr_c; sv->k = X.k; sv->fh = X.fh; sv->fn = X.fn;
    }
    if (lane < 8) sv->fr[lane] = X.fr;
    sv->vb[lane] = X.vbits;
    __syncwarp();
  };
// binds the worker-local names (w, ws, S, R and the scalar state) for worker `vv`
#define KVR_BIND_WORKER(vv)                                                          \
  const uint32_t w = (vv);                                                           \
  WSt Xl_;                                                                           \
  if constexpr (kV > 1) Xl_ = st_load(w);                                            \
  WSt& X_ = kV > 1 ? Xl_ : st0;                                                      \
  uint32_t& fh = X_.fh; uint32_t& fn = X_.fn; uint32_t& vbits = X_.vbits;            \
  double& P = X_.P; double& F = X_.F; double& Pt = X_.Pt; double& fr = X_.fr;        \
  double& fr_c = X_.fr_c; double& th0 = X_.th0; double& th1 = X_.th1;              \
  double& th2 = X_.th2; double& th3 = X_.th3; uint64_t& k = X_.k;                    \
  WarpSm* ws = warp_sm(p, w);                                                        \
  const WorkerView<Idx> S =                                                          \
      make_view<Idx>(worker_gbase<kMem>(p, w), worker_sbase<kMem>(p, w), L);         \
  RecencyLog R;                                                                      \
  R.log = reinterpret_cast<uint32_t*>(p.aux_base + ((size_t)blockIdx.x * W + w) *    \
                                      p.aux.bytes + p.aux.off_log);                  \
  R.stamp = reinterpret_cast<uint16_t*>(worker_sbase<kMem>(p, w) + L.off_stamp);     \
  R.cap_mask = p.aux.log_cap - 1;                                                    \
  (void)fh; (void)fn; (void)vbits; (void)P; (void)F; (void)Pt; (void)fr; (void)fr_c; \
  (void)th0; (void)th1; (void)th2; (void)th3; (void)k; (void)S; (void)R
#define KVR_SAVE_WORKER() \
  do {                    \
    if constexpr (kV > 1) st_store(w, X_); \
  } while (0)

  if (tid == 0) {
    for (uint32_t b = 0; b < kNumStages; ++b) mbar_init(&ctrl->mbar[b], 1);
    fence_mbar_init();
  }
  __syncthreads();

  uint64_t gq = 0;   // queries staged by this CTA so far (drives buffer index and parity)
#pragma unroll 1
  for (;;) {
    if (tid == 0) {
      const uint32_t tt = atomicAdd(p.work_counter, 1u);
      ctrl->trial = tt;
      if (tt < p.n_trials) ctrl->pol = p.policies ? p.policies[tt] : p.defpol;
    }
    __syncthreads();
    const uint32_t trial = ctrl->trial;
    if (trial >= p.n_trials) break;

    const uint32_t tix = p.trial_trace ? p.trial_trace[trial] : 0u;
    const bool tr_ok = tix < p.n_traces;   // else KVR_TRIAL_BAD_TRACE, trial not run
    const TraceDev tr = p.traces[tr_ok ? tix : 0u];
    const kvr_policy& pol = ctrl->pol;   // shared memory, read on demand
    const uint64_t K = p.keys[trial];
    const uint32_t N = tr.N, bt = tr.block_tokens;
    const bool rlt = pol.eviction == KVR_EVICT_RLT;
    const bool opt = kExt && pol.eviction == KVR_EVICT_OPT;   // offline Belady analysis (W = 1)
    const bool tree = rlt || opt;                     // parents / child counts / LEAF bits
    const bool use_list = pol.eviction == KVR_EVICT_LRU || (rlt && pol.rlt_fallback == KVR_RLT_LRU_MARKED);
    const bool rls = kExt && pol.router == KVR_ROUTE_LBGR_RLS;   // LBGR, RLS reading A8b
    const bool lbgr = pol.router == KVR_ROUTE_LBGR || rls;
    const uint32_t router = pol.router, fallback = pol.rlt_fallback;
    const bool lbgr_or_static = lbgr || router == KVR_ROUTE_STATIC_LINEAR;
    const bool recorded = trial < p.record_trials;
    kvr_query_record* rec = recorded ? p.records + (size_t)trial * p.rec_stride : nullptr;
    uint64_t* vlog = (recorded && p.victims) ? p.victims + (size_t)trial * p.victims_per_trial : nullptr;
    // deferred apply needs the overlay (register victim bitmap): B <= 1024
    const bool defer = regbits;
    const uint32_t lag = kExt ? pol.tracker_lag : 0u;   // stale tracker (A29): k events
    uint32_t* led = (kExt && p.ledger) ? p.ledger + (size_t)trial * p.ledger_stride : nullptr;

#ifdef KVR_PHASE_PROFILE
    const unsigned long long t_trial0 = clock64();
#endif
    // ---- per-trial init: empty caches S_i^(0), P_i^(0) = 0 ----
    if (led)
      for (uint32_t i = tid; i < p.ledger_stride; i += blockDim.x) led[i] = 0u;
#pragma unroll
    for (uint32_t vi = 0; vi < kV; ++vi) {
      if (kV > 1 && wid + vi * nwarps >= W) break;
      KVR_BIND_WORKER(wid + vi * nwarps);
      for (uint32_t i = lane; i < L.T; i += 32) S.table[i] = NIL;
      for (uint32_t i = lane; i < nwords; i += 32) {
        S.leaf[i] = 0;
        S.mark[i] = 0;
      }
      if (use_list)
        for (uint32_t i = lane; i < B; i += 32) R.stamp[i] = 0;
      if (lag) {   // the tracker's mirror starts empty too
        const WorkerView<Idx> MV = mirror_view<Idx>(p, w);
        for (uint32_t i = lane; i < L.T; i += 32) MV.table[i] = NIL;
      }
      // The worker's scalar cache state (size, |T|, log cursors, e_i, counters) lives in
      // its shared-memory block ws->x; the chosen warp works on a register copy for
      // the duration of its update (nothing of it stays live across the query loop).
      if (lane == 0) {
        WorkerRegs w0;
        w0.size = 0; w0.cntT = 0; w0.used = 0; w0.wq = 0; w0.lhead = 0; w0.ltail = 0; w0.e = 0;
        w0.c_ins = 0; w0.c_evict = 0; w0.c_draws = 0; w0.c_resets = 0; w0.c_fb = 0;
        ws->x = w0;
        ws->x_ri = 32;   // next unused draw of the batch (none yet)
        ws->m_used = 0;
        ws->m_size = 0;
        ws->m_cur = 0;
      }
      fh = 0;
      fn = 0;
      P = 0.0;
      F = 0.0;
      Pt = 0.0;
      th0 = pol.theta0[0];
      th1 = pol.theta0[1];
      th2 = pol.theta0[2];
      th3 = pol.theta0[3];
      k = 0;
      fr = 0.0;      // front record of the pending FIFO
      fr_c = 0.0;
      vbits = 0;     // victims of this worker's pending update
      if (rls && lane < 16) rls_region(p, w)[lane] = (lane % 5 == 0) ? pol.rls_p0 : 0.0;   // P = p0 I
      if (lane == 0) {
        ws->active = 0;
        ws->c_probes = 0; ws->c_hit = 0; ws->c_in = 0; ws->c_q = 0; ws->c_maxp = 0;
        ws->ftail = 0;        // record index of the next push (chunk boundary: allocate first)
        ws->ffree = ~0u;      // this worker's free-chunk list (empty)
      }
      KVR_SAVE_WORKER();
    }
    for (uint32_t i = tid; i < 2 * 32; i += blockDim.x)   // overlay staging of both slot buffers
      slot_buf(p, i >> 5)[p.max_n + (i & 31)] = 0u;
    if (tid == 0) {
      ctrl->sum_lat = 0.0;
      ctrl->sum_ttft = 0.0;
      ctrl->max_lat = 0.0;
      ctrl->digest = K;
      ctrl->dkey = K;
      ctrl->vcursor = 0;
      ctrl->abortf[0] = 0;
      ctrl->abortf[1] = 0;
      ctrl->status = 0;
      ctrl->fifo_bump = 0;
      for (int c = 0; c < 10; ++c) ctrl->cnt[c] = 0;
      if (kExt) {
        ctrl->led = led;
        ctrl->lph = tr.ph;
        ctrl->lnx = tr.nx;
      }
    }
    uint32_t* hist = p.hist ? p.hist + (size_t)trial * p.bins : nullptr;   // global, per trial
    if (hist)
      for (uint32_t b = tid; b < p.bins; b += blockDim.x) hist[b] = 0;
    // (bt*k)/1000.0 computed once per trial with the same IEEE division (A9)
    for (uint32_t kk = tid; kk <= p.max_n; kk += blockDim.x) divtab[kk] = (double)(bt * kk) / 1000.0;

    // a per-trial policy from device memory is validated here (host validated the default)
    const bool pol_ok = policy_valid(pol) &&
                        (!opt || (W == 1 && (tr.nu != nullptr || N == 0))) &&
                        (kExt ? (!p.ledger || (W == 1 && tr.ph != nullptr)) : p.ledger == nullptr) &&
                        (kExt || (pol.eviction <= KVR_EVICT_RLT && pol.router <= KVR_ROUTE_RANDOM &&
                                  pol.tracker_lag == 0 && pol.tracker_grain == 1));
    if (!pol_ok && tid == 0) ctrl->status = KVR_TRIAL_BAD_POLICY;
    if (!tr_ok && tid == 0) ctrl->status = KVR_TRIAL_BAD_TRACE;
    const uint32_t Nrun = (pol_ok && tr_ok) ? N : 0;

    // staging prologue: queries 0 .. kAhead-1
    uint32_t issued = min(Nrun, kAhead);
    uint64_t pf_off = 0;
    uint32_t pf_n = 0;
    if (tid == 0) {
      for (uint32_t q = 0; q < issued; ++q) {
        const QueryHdr* h = tr.hdr + q;
        const uint64_t off = h->block_off;
        const uint32_t n = h->n_in + h->n_out;
        const uint64_t b0 = (off * 8) & ~15ull, b1 = ((off + n) * 8 + 15) & ~15ull;
        const uint32_t buf = (uint32_t)((gq + q) % kNumStages);
        uint8_t* dst = stage + (size_t)buf * p.stage_bytes;
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&ctrl->mbar[buf], 32u + (uint32_t)(b1 - b0));
        bulk_g2s(dst, h, 32, &ctrl->mbar[buf]);
        bulk_g2s(dst + 32, reinterpret_cast<const uint8_t*>(tr.hash) + b0, (uint32_t)(b1 - b0),
                 &ctrl->mbar[buf]);
      }
      if (issued < Nrun) {
        pf_off = tr.hdr[issued].block_off;
        pf_n = tr.hdr[issued].n_in + tr.hdr[issued].n_out;
      }
    }
    __syncthreads();

    uint32_t consumed = 0;
    // two workers per warp: the warp that updated the previous query's chosen worker scores
    // only that worker for the next query; its other workers move to the following warps
    // (one each), so the chooser's critical path carries one worker's catch-up / match /
    // score, not two.  pb / pcw: the previous chosen worker and the warp that updated it
    // (identical in every warp)
    constexpr uint32_t kL = kV > 1 ? 3u : 1u;   // workers a warp may score in one query
    uint32_t pb = 0xffffffffu, pcw = 0xffffffffu;
#ifdef KVR_WHO_LAST
    uint32_t my_role = 2;
#endif

    const double pol_inv_dt = 1.0 / pol.delta_t_ms;
#pragma unroll 1
    for (uint32_t j = 0; j < Nrun; ++j) {
      const uint64_t g = gq + j;
      const uint32_t buf = (uint32_t)(g % kNumStages);
      const uint32_t par = j & 1;
      KVR_T0(tp);
      mbar_wait(&ctrl->mbar[buf], (uint32_t)((g / kNumStages) & 1));
      KVR_ACC(0, tp);
      consumed = j + 1;
      const uint8_t* st = stage + (size_t)buf * p.stage_bytes;
      const QueryHdr hd = *reinterpret_cast<const QueryHdr*>(st);
      const uint64_t* H = reinterpret_cast<const uint64_t*>(st + 32) + (hd.block_off & 1);
      const double a = hd.arrival_ms;
      const uint32_t n_in = hd.n_in, n = hd.n_in + hd.n_out;
      const uint32_t q = bt * n_in;

      // this query's workers of this warp (kV == 1: its own; kV == 2: see pb / pcw)
      uint32_t wl[kL];
      if constexpr (kV == 1) {
        wl[0] = wid;
      } else {
        const uint32_t NONE = 0xffffffffu;
#pragma unroll
        for (uint32_t li = 0; li < kL; ++li) wl[li] = NONE;
        if (pb == NONE) {
          wl[0] = wid;
          wl[1] = wid + nwarps < W ? wid + nwarps : NONE;
        } else if (wid == pcw) {
          wl[0] = pb;
        } else {
          const uint32_t o0 = wid, o1 = wid + nwarps;
          wl[0] = o0 == pb ? NONE : o0;
          wl[1] = (o1 >= W || o1 == pb) ? NONE : o1;
          // pcw's own workers other than pb, the k-th one to warp pcw + 1 + k
          uint32_t k = 0;
#pragma unroll
          for (uint32_t r = 0; r < 2; ++r) {
            const uint32_t x = pcw + r * nwarps;
            if (x < W && x != pb) {
              if ((pcw + 1 + k) % nwarps == wid) wl[2] = x;
              ++k;
            }
          }
        }
      }
      // steps 1-3 for each of those workers; the chooser reuses its worker's values
      uint32_t m_v[kL] = {}, mview_v[kL] = {};
      double score_v[kL] = {}, Chat_v[kL] = {}, f0_v[kL] = {}, f1_v[kL] = {}, f2_v[kL] = {};
#pragma unroll
      for (uint32_t vi = 0; vi < kL; ++vi) {
        if (kV > 1 && wl[vi] == 0xffffffffu) continue;
        KVR_BIND_WORKER(wl[vi]);
        // ---- steps 1-3 of one query for this warp's worker ----
        // Membership = the table, or the path Hp[0..np) (same position, same identity),
        // minus the pending update's victims (register bitmap vbits) if minus_victims.
        auto score_query = [&](const uint64_t* Hq, double aq, uint32_t nq_in, uint32_t qtok,
                               const uint64_t* Hp, uint32_t np, bool minus_victims, uint32_t& m_o,
                               uint32_t& mview_o,
                               double& score_o, double& Chat_o, double& f0_o, double& f1_o,
                               double& f2_o) {
          KVR_T0(tl);
          // 1. catch-up (A11: tick before completion before routing)
          {
            const double rho = pol.rho, dt = pol.delta_t_ms, inv_dt = pol_inv_dt;
    #pragma unroll 1
            for (;;) {
              if (lbgr) {
                // every tick k' with (double)k'*dt <= min(a, c) comes first (A11); (double)k'*dt
                // is monotone in k', so find the last such k' and apply the multiplications
                // one by one (same rounding sequence as a per-tick loop)
                const double lim = (fn == 0 || aq < fr_c) ? aq : fr_c;
                const double est = lim * inv_dt;   // a guess only: the loops below make it exact
                uint64_t kk = est < 1.8e19 ? (uint64_t)est : k;
                if (kk < k) kk = k;
                while ((double)(kk + 1) * dt <= lim) ++kk;
                while (kk > k && (double)kk * dt > lim) --kk;
                if (kk > k) {
                  if (Pt != 0.0) {
                    uint32_t nt = (uint32_t)(kk - k);
    #pragma unroll 1
                    for (; nt >= 4; nt -= 4) {
                      Pt = rho * Pt;
                      Pt = rho * Pt;
                      Pt = rho * Pt;
                      Pt = rho * Pt;
                    }
                    for (; nt; --nt) Pt = rho * Pt;
                  }
                  k = kk;
                }
              }
              if (fn != 0 && fr_c <= aq) {
                // pop the front record (its fields are in fr); an emptied chunk goes to this
                // worker's free list and the head follows the chunk link
                const uint32_t nh = fh + 1;
                --fn;
                if ((nh & (kFifoChunk - 1)) == 0) {
                  const uint32_t c0 = (nh - 1) / kFifoChunk;
                  const uint32_t nxt = fn ? flink[c0] : 0u;
                  __syncwarp();
                  if (lane == 0) {
                    flink[c0] = ws->ffree;
                    ws->ffree = c0;
                  }
                  fh = fn ? nxt * kFifoChunk : nh;
                } else {
                  fh = nh;
                }
                if (lbgr) {
                  const double fa = __shfl_sync(kFull, fr, 1), fE = __shfl_sync(kFull, fr, 2);
                  const double g0 = __shfl_sync(kFull, fr, 3), g1 = __shfl_sync(kFull, fr, 4);
                  const double g2 = __shfl_sync(kFull, fr, 5), fC = __shfl_sync(kFull, fr, 6);
                  const uint64_t ka = (uint64_t)__double_as_longlong(__shfl_sync(kFull, fr, 7));
                  const double E = fr_c - fa;
                  const double res = E - fE;
                  if (rls) {
                    // OnlineUpdate, RLS reading (A8b), one weighted least-squares step in
                    // the oracle's order (rls_step): lane 4a+b holds P[a][b]; every sum is
                    // gathered by shuffles left to right.  pi = P phi, gamma = lam + phi'pi,
                    // k = pi / gamma, theta += k e, P = (P - k pi') / lam.
                    const double lam = pol.mu;
                    double* Rg = rls_region(p, w);
                    const uint32_t ra = (lane >> 2) & 3u, rb = lane & 3u;
                    const double Pab = lane < 16 ? Rg[lane] : 0.0;
                    const double phb = rb == 0 ? g0 : (rb == 1 ? g1 : (rb == 2 ? g2 : 1.0));
                    const double prod = Pab * phb;
                    double pi = __shfl_sync(kFull, prod, 4 * ra);
                    pi = pi + __shfl_sync(kFull, prod, 4 * ra + 1);
                    pi = pi + __shfl_sync(kFull, prod, 4 * ra + 2);
                    pi = pi + __shfl_sync(kFull, prod, 4 * ra + 3);   // pi[a] in lanes 4a..4a+3
                    double gsum = g0 * __shfl_sync(kFull, pi, 0);
                    gsum = gsum + g1 * __shfl_sync(kFull, pi, 4);
                    gsum = gsum + g2 * __shfl_sync(kFull, pi, 8);
                    gsum = gsum + 1.0 * __shfl_sync(kFull, pi, 12);
                    const double gamma = lam + gsum;
                    const double kk = pi / gamma;                       // k[a]
                    const double pib = __shfl_sync(kFull, pi, 4 * rb);  // pi[b]
                    if (lane < 16) Rg[lane] = (Pab - kk * pib) / lam;
                    th0 = th0 + __shfl_sync(kFull, kk, 0) * res;
                    th1 = th1 + __shfl_sync(kFull, kk, 4) * res;
                    th2 = th2 + __shfl_sync(kFull, kk, 8) * res;
                    th3 = th3 + __shfl_sync(kFull, kk, 12) * res;
                  } else {     // OnlineUpdate (A8): NLMS on the squared residual
                    const double g3 = 1.0;
                    double s = g0 * g0;
                    s = s + g1 * g1;
                    s = s + g2 * g2;
                    s = s + g3 * g3;
                    const double gstep = (pol.mu * res) / (1.0 + s);
                    th0 = th0 + gstep * g0;
                    th1 = th1 + gstep * g1;
                    th2 = th2 + gstep * g2;
                    th3 = th3 + gstep * g3;
                  }
                  // ReleaseLoad (A10): P~ <- max(0, P~ - C^ rho^kappa)
                  uint64_t kap = k - ka;
                  double pw = 1.0, bb = rho;
    #pragma unroll 1
                  while (kap) {
                    if (kap & 1) pw = pw * bb;
                    bb = bb * bb;
                    kap >>= 1;
                  }
                  Pt = Pt - fC * pw;
                  if (Pt < 0.0) Pt = 0.0;
                }
                if (fn) {
                  if (lane < 8) fr = fifo[(size_t)fh * 8 + lane];
                  fr_c = __shfl_sync(kFull, fr, 0);
                }
                continue;
              }
              break;
            }
          }
          KVR_ACC(1, tl);

          // 2. longest cached prefix over the input (ballot of 32 probes) on the worker's
          // cache, and with the stale tracker (App. E, reading A29) the router's view: the
          // same match on the mirror of the cache after query j-1-k
          auto match_on = [&](const WorkerView<Idx> V, bool ovl, uint32_t npp) -> uint32_t {
            uint32_t mx = 0;
    #pragma unroll 1
            for (uint32_t base = 0; base < nq_in; base += 32) {
              const uint32_t bal = probe_window<Idx>(V, tmask, Hq, base, nq_in, Hp, npp, ovl, vbits, lane);
              if (bal == kFull) {
                mx = base + 32;
                continue;
              }
              mx = base + (__ffs(~bal) - 1);
              break;
            }
            return mx > nq_in ? nq_in : mx;
          };
          const uint32_t mm = match_on(S, minus_victims, np);
          uint32_t mv = mm;
          if (kExt && lag) mv = match_on(mirror_view<Idx>(p, w), false, 0u);
          if (kExt && pol.tracker_grain > 1) mv = pol.tracker_grain * (mv / pol.tracker_grain);
          KVR_ACC(2, tl);

          // 3. score (Eq. 4-5, A9) on the tracker's view h~ = bt*mv (= h by default)
          const double x = (double)(bt * mv), y = (double)(qtok - bt * mv);
          double sc = 0.0, Ch = 0.0, h0 = 0.0, h1 = 0.0, h2 = 0.0;
          if (lbgr) {
            Ch = (pol.est_alpha_cached_ms * x) + (pol.est_alpha_miss_ms * y);
            h0 = divtab[mv];            // == x / 1000.0 (x = bt*m~)
            h1 = divtab[nq_in - mv];    // == y / 1000.0 (y = bt*(n_in-m~))
            h2 = Pt / 1000.0;
            const double h3 = 1.0;
            double dd = th0 * h0;
            dd = dd + th1 * h1;
            dd = dd + th2 * h2;
            dd = dd + th3 * h3;
            sc = (Ch + Pt) + dd;
          } else if (router == KVR_ROUTE_STATIC_LINEAR) {
            sc = (pol.w_load * (double)fn) - (pol.w_hit * (x / (double)qtok));
          }
          KVR_ACC(3, tl);
          m_o = mm;
          mview_o = mv;
          score_o = sc;
          Chat_o = Ch;
          f0_o = h0;
          f1_o = h1;
          f2_o = h2;
        };
        if constexpr (kV > 1) {
          // two workers per warp: a worker whose last update was applied after the previous
          // barrier by another warp (it was updated while moved) may still be in that
          // apply -- wait for it to finish before reading its cache.  (pb, scored by the
          // warp that updated it, legitimately has its apply pending: overlay below.)
          if (w != pb) {
            if (lane == 0)
              while (*reinterpret_cast<volatile uint32_t*>(&ws->active)) {
              }
            __syncwarp();
            __threadfence_block();
          }
        }
        // with a pending deferred apply, membership = path of that query or the old
        // table minus that update's victims
        const bool overlay = defer && ws->active;
        const uint64_t* Hp = nullptr;
        uint32_t np = 0;
        if (overlay) {
          const uint8_t* sp = stage + (size_t)ws->buf * p.stage_bytes;
          Hp = reinterpret_cast<const uint64_t*>(sp + 32) +
               (reinterpret_cast<const QueryHdr*>(sp)->block_off & 1);
          np = ws->n;
        }
        if (kExt && lag && j >= lag) {
          // the tracker catches up to the caches after query j-1-k: this worker's updates
          // of queries < j-k, in query order (ring entries live kLagRing > k+1 queries)
          const uint32_t upto = j - lag;
          uint32_t cur = ws->m_cur;
#pragma unroll 1
          for (; cur < upto; ++cur)
            if (lag_entry(p, cur)->worker == w) mirror_apply<Idx, kMaxThreads>(p, tr.hash, w, lane, cur);
          __syncwarp();
          if (lane == 0) ws->m_cur = cur;
        }
        score_query(H, a, n_in, q, Hp, np, overlay, m_v[vi], mview_v[vi], score_v[vi], Chat_v[vi],
                    f0_v[vi], f1_v[vi], f2_v[vi]);
        if (lane == 0) {
          ctrl->score[par][w] = score_v[vi];
          ctrl->mhit[par][w] = mview_v[vi];   // the router's view (THRESHOLD)
          ctrl->npend[par][w] = fn;
          ctrl->csize[par][w] = ws->x.size;   // cached blocks (CACHE_AWARE, A38)
          ws->c_probes += min(m_v[vi] + 1, n_in);
        }
        KVR_SAVE_WORKER();
      }
      KVR_RESET(tp);
#ifdef KVR_WHO_LAST
      if (lane == 0) {
        s_arrive[wid] = (uint32_t)clock();
        s_role[wid] = my_role;
      }
      my_role = 2;
#endif
      __syncthreads();
#ifdef KVR_WHO_LAST
      if (tid == 0 && j > 2) {
        uint32_t best_w = 0, t1 = 0, t2 = 0;
        for (uint32_t w2 = 0; w2 < nwarps; ++w2) {
          const uint32_t t = s_arrive[w2] - s_arrive[0] + 0x40000000u;   // wrap-safe offsets
          if (t > t1) { t2 = t1; t1 = t; best_w = w2; } else if (t > t2) { t2 = t; }
        }
        atomicAdd(&g_who[s_role[best_w]], 1ull);
        atomicAdd(&g_who[4 + s_role[best_w]], (unsigned long long)(t1 - t2));
      }
#endif
      KVR_ACC(4, tp);
      if (ctrl->abortf[par]) break;   // set by i* of query j-1 (written to the other parity)
      if (issued < Nrun) {
        if (tid == 0) {
          const uint64_t b0 = (pf_off * 8) & ~15ull, b1 = ((pf_off + pf_n) * 8 + 15) & ~15ull;
          const uint32_t nb = (uint32_t)((gq + issued) % kNumStages);
          uint8_t* dst = stage + (size_t)nb * p.stage_bytes;
          fence_proxy_async_smem();
          mbar_arrive_expect_tx(&ctrl->mbar[nb], 32u + (uint32_t)(b1 - b0));
          bulk_g2s(dst, tr.hdr + issued, 32, &ctrl->mbar[nb]);
          bulk_g2s(dst + 32, reinterpret_cast<const uint8_t*>(tr.hash) + b0, (uint32_t)(b1 - b0),
                   &ctrl->mbar[nb]);
          if (issued + 1 < Nrun) {
            pf_off = tr.hdr[issued + 1].block_off;
            pf_n = tr.hdr[issued + 1].n_in + tr.hdr[issued + 1].n_out;
          }
        }
        ++issued;
      }

      // ---- 4. argmin over workers (every warp computes the same i*) ----
      uint32_t best = 0;
      if (lbgr || router == KVR_ROUTE_STATIC_LINEAR) {
        // first minimum = lowest lane holding the smallest order-preserving key of
        // the fp64 score (-0 folded into +0, which the fp compare treats as equal);
        // three uniform-datapath reductions instead of a 5-round shuffle tournament
        double v = lane < W ? ctrl->score[par][lane] : INFINITY;
        if (v == 0.0) v = 0.0;
        const uint64_t bits = (uint64_t)__double_as_longlong(v);
        // NaN ranks after every number (A37), padding lanes (+inf) after real workers
        const uint64_t key = isnan(v) ? 0xfffffffffffffffeull
                             : (lane >= W ? ~0ull
                                          : ((bits >> 63) ? ~bits : (bits | 0x8000000000000000ull)));
        const uint32_t khi = (uint32_t)(key >> 32), klo = (uint32_t)key;
        const uint32_t mhi = __reduce_min_sync(kFull, khi);
        const uint32_t mlo = __reduce_min_sync(kFull, khi == mhi ? klo : 0xffffffffu);
        best = __reduce_min_sync(kFull, (khi == mhi && klo == mlo) ? lane : 32u);
      } else if (router == KVR_ROUTE_THRESHOLD) {   // A16
        const uint32_t npd = lane < W ? ctrl->npend[par][lane] : 0xffffffffu;
        const uint32_t mh = lane < W ? ctrl->mhit[par][lane] : 0u;
        const uint32_t mx = __reduce_max_sync(kFull, lane < W ? npd : 0u);
        const uint32_t mn = __reduce_min_sync(kFull, npd);
        if ((double)mx > pol.tau * (double)max(1u, mn)) {
          best = __ffs(__ballot_sync(kFull, npd == mn)) - 1;
        } else {
          const uint32_t mmax = __reduce_max_sync(kFull, mh);
          best = __ffs(__ballot_sync(kFull, lane < W && mh == mmax)) - 1;
        }
      } else if (kExt && router == KVR_ROUTE_CACHE_AWARE) {   // A38
        const uint32_t npd = lane < W ? ctrl->npend[par][lane] : 0u;
        const uint32_t mx = __reduce_max_sync(kFull, npd);
        const uint32_t mn = __reduce_min_sync(kFull, lane < W ? npd : 0xffffffffu);
        if (((double)(mx - mn) > pol.ca_balance_abs) && ((double)mx > pol.ca_balance_rel * (double)mn)) {
          best = __ffs(__ballot_sync(kFull, lane < W && npd == mn)) - 1;
        } else {
          const uint32_t mh = lane < W ? ctrl->mhit[par][lane] : 0u;
          const uint32_t mmax = __reduce_max_sync(kFull, mh);
          best = __ffs(__ballot_sync(kFull, lane < W && mh == mmax)) - 1;
          if (!((double)(bt * mmax) / (double)q > pol.ca_cache_threshold)) {
            const uint32_t cs = lane < W ? ctrl->csize[par][lane] : 0xffffffffu;
            const uint32_t cmin = __reduce_min_sync(kFull, cs);
            best = __ffs(__ballot_sync(kFull, lane < W && cs == cmin)) - 1;
          }
        }
      } else if (router == KVR_ROUTE_ROUND_ROBIN) {
        best = j % W;
      } else {
        best = (uint32_t)pick_index(philox_r64(K, j, 0xffffffffu, 2u), W);
      }
      KVR_ACC(5, tp);

      // deferred apply of the previous update of a worker this warp scored (overlaps the
      // other warps' decisions)
#pragma unroll
      for (uint32_t vi = 0; vi < kL; ++vi) {
        if (kV > 1 && wl[vi] == 0xffffffffu) continue;
        const uint32_t w = wl[vi];
        WarpSm* ws = warp_sm(p, w);
        if (ws->active) {
#ifdef KVR_WHO_LAST
          const long long ta0 = clock64();
#endif
          apply_update<Idx, kMem, kMaxThreads, kExt>(p, lane, w, tree, use_list, lbgr_or_static, rec, vlog);
          if constexpr (kV > 1) wsave(p, w)->vb[lane] = 0u;
          else st0.vbits = 0;
#ifdef KVR_WHO_LAST
          my_role = 1;
          if (lane == 0) {
            atomicAdd(&g_who[3], (unsigned long long)(clock64() - ta0));
            atomicAdd(&g_who[7], 1ull);
          }
#endif
        }
      }
      uint32_t vib = 0xffffffffu;   // position of the chosen worker in this warp's list
#pragma unroll
      for (uint32_t vi = 0; vi < kL; ++vi)
        if (wl[vi] == best) vib = vi;
      if constexpr (kV > 1) {   // every warp tracks who updates the chosen worker
        uint32_t cw = 0xffffffffu;
        if (pb == 0xffffffffu) {
          cw = best % nwarps;
        } else if (best == pb) {
          cw = pcw;
        } else if (best % nwarps != pcw) {
          cw = best % nwarps;
        } else {   // a worker of pcw moved to the following warps
          uint32_t k = 0;
          for (uint32_t r = 0; r < 2; ++r) {
            const uint32_t x = pcw + r * nwarps;
            if (x < W && x != pb) {
              if (x == best) cw = (pcw + 1 + k) % nwarps;
              ++k;
            }
          }
        }
        pb = best;
        pcw = cw;
      }
#ifdef KVR_PHASE_PROFILE
      if (vib != 0xffffffffu && clock64() - tp > 200) {   // an apply on the critical path
        KVR_CNT(16, clock64() - tp);
        KVR_CNT(17, 1);
      }
#endif
      KVR_ACC(6, tp);

      if (vib == 0xffffffffu) continue;
#ifdef KVR_WHO_LAST
      my_role = 0;
#endif

      // ================= warp i* : UpdateCache decisions + accounting =================
      uint32_t m = m_v[0];
      double score = score_v[0], Chat = Chat_v[0], f0 = f0_v[0], f1 = f1_v[0], f2 = f2_v[0];
#pragma unroll
      for (uint32_t vi = 1; vi < kL; ++vi)
        if (vib == vi) {
          m = m_v[vi];
          score = score_v[vi];
          Chat = Chat_v[vi];
          f0 = f0_v[vi];
          f1 = f1_v[vi];
          f2 = f2_v[vi];
        }
#pragma unroll 1
      for (uint32_t once = 0; once < 1; ++once) {   // (break = leave the update early)
      KVR_BIND_WORKER(best);
      uint32_t* slots = slot_buf(p, j);        // [max_n] slot | evicted << 31 per miss
      uint32_t* vmap = slots + p.max_n;        // [32] victim bitmap staging (overlay)
      __syncwarp();
      // register copy of the scalars this update changes (written back at the end);
      // counters and e_i are bumped in shared memory
      struct {
        uint32_t size, cntT, wq, lhead, ltail;
      } wr;
      wr.size = ws->x.size;
      wr.cntT = ws->x.cntT;
      wr.wq = ws->x.wq;
      wr.lhead = ws->x.lhead;
      wr.ltail = ws->x.ltail;
      if (fn >= p.ring) {   // pending FIFO full -> trial status, stop (before Eq. 3)
        if (lane == 0) {
          ctrl->status = KVR_TRIAL_RING_OVERFLOW;
          ctrl->abortf[par ^ 1] = 1;
        }
        break;
      }
      // FIFO push position: the tail chunk's next record, or a new chunk (own free list
      // first, else the pool's bump counter) linked behind the tail
      uint32_t ftail = ws->ftail;
      if ((ftail & (kFifoChunk - 1)) == 0) {
        uint32_t c = ws->ffree;
        const bool reuse = c != ~0u;
        const uint32_t nf = reuse ? flink[c] : 0u;
        if (!reuse) c = ctrl->fifo_bump;
        if (c >= p.fifo.chunks) {   // cannot happen with the FifoLayout bound; fail safe
          if (lane == 0) {
            ctrl->status = KVR_TRIAL_RING_OVERFLOW;
            ctrl->abortf[par ^ 1] = 1;
          }
          break;
        }
        __syncwarp();
        if (lane == 0) {
          if (reuse) ws->ffree = nf;
          else ctrl->fifo_bump = c + 1;
          if (fn) flink[(ftail - 1) / kFifoChunk] = c;
        }
        ftail = c * kFifoChunk;
      }
      if (lane == 0) ws->ftail = ftail + 1;
      ++wr.wq;
      // log room for this query's n entries (Leaf-LRU order)
      if (use_list && wr.ltail - wr.lhead + n > p.aux.log_cap) {
        KVR_T0(tc);
        KVR_CNT(13, wr.ltail - wr.lhead);
        wr.ltail = log_compact(R, wr.lhead, wr.ltail, lane);
        KVR_ACC(10, tc);
        KVR_CNT(14, wr.ltail - wr.lhead);
        KVR_CNT(15, 1);
      }
      const uint32_t ltail0 = wr.ltail;

      KVR_T0(tk);
      // full-path cached prefix kf (hits of Gamma_j; m covers the input part)
      uint32_t kf = m;
      if (m == n_in) {
#pragma unroll 1
        for (uint32_t base = n_in; base < n; base += 32) {
          const uint32_t bal = probe_window<Idx>(S, tmask, H, base, n, nullptr, 0u, false, 0u, lane);
          if (bal == kFull) {
            kf = base + 32;
            continue;
          }
          kf = base + (__ffs(~bal) - 1);
          break;
        }
        if (kf > n) kf = n;
      }

      KVR_ACC(18, tk);
      // ---- hits: marks (Alg. 1 l.6-9), recency stamps, log entries ----
      Idx p0 = NIL;
#pragma unroll 1
      for (uint32_t base = 0; base < kf; base += 32) {
        const uint32_t d = base + lane;
        const bool act = d < kf;
        const Idx s = act ? tbl_find<Idx>(S, tmask, H[d]) : NIL;
        if (act && use_list) {
          R.stamp[s] = wr.wq;
          R.log[(ltail0 + (n - 1 - d)) & R.cap_mask] = ((wr.wq & 0xffffu) << 16) | (uint32_t)s;
        }
        if (opt && act) opt_keys(p, w)[s] = opt_key(tr.nu[hd.block_off + d], d + 1, (uint32_t)s);
        if (led && act) last_access(p, w)[s] = (uint32_t)(hd.block_off + d);   // phase ledger
        if (rlt) {
          const bool um = act && !((S.mark[(uint32_t)s >> 5] >> ((uint32_t)s & 31)) & 1u);
          const uint32_t u = __ballot_sync(kFull, um);
          const uint32_t need = B + 1 - wr.cntT;   // the need-th unmarked hit resets T
          const uint32_t nact = min(32u, kf - base);
          if ((uint32_t)__popc(u) >= need) {
            const uint32_t rr = select_bit(u, need - 1);
            __syncwarp();
            for (uint32_t i = lane; i < nwords; i += 32) S.mark[i] = 0u;
            __syncwarp();
            if (act && lane >= rr) atomicOr(&S.mark[(uint32_t)s >> 5], 1u << ((uint32_t)s & 31));
            wr.cntT = nact - rr;
            if (lane == 0) ++ws->x.c_resets;
          } else {
            if (um) atomicOr(&S.mark[(uint32_t)s >> 5], 1u << ((uint32_t)s & 31));
            wr.cntT += __popc(u);
          }
        }
        p0 = (Idx)__shfl_sync(kFull, (uint32_t)s, min(31u, kf - 1 - base));
      }
      __syncwarp();
      KVR_ACC(19, tk);
      KVR_ACC(7, tp);

      const uint32_t M = n - kf;
      const uint32_t size0 = wr.size;
      const uint32_t nfree = min(M, B - size0);
      const uint32_t nev = M - nfree;

      // ---- accounting: Eq. 1 truth, Eq. 2, FIFO single server (A12, A20) ----
      // (needs only the hits; done before the decisions so that the next query's
      // catch-up can run ahead of them)
      const uint32_t h = bt * m;
      const double hx = (double)h, hy = (double)(q - h);
      const double pre = (p.truth.alpha_cached_ms * hx) + (p.truth.alpha_miss_ms * hy);
      const double O = p.truth.out_ms_per_token * (double)hd.out_tokens;
      const double cost = pre + O;
      const double start = (a >= F) ? a : F;
      const double ttft = (start + pre) - a;
      const double comp = start + cost;
      const double lat = comp - a;
      F = comp;
      P = P + cost;
      KVR_T0(ta);
      {
        const uint32_t slotf = ftail;
        if (fn == 0) fh = ftail;
        const double rE = lbgr ? score : 0.0, r0 = lbgr ? f0 : 0.0, r1 = lbgr ? f1 : 0.0,
                     r2 = lbgr ? f2 : 0.0, rC = lbgr ? Chat : 0.0;
        double val = 0.0;
        switch (lane) {
          case 0: val = comp; break;
          case 1: val = a; break;
          case 2: val = rE; break;
          case 3: val = r0; break;
          case 4: val = r1; break;
          case 5: val = r2; break;
          case 6: val = rC; break;
          case 7: val = __longlong_as_double((long long)k); break;
          default: break;
        }
        if (lane < 8) fifo[(size_t)slotf * 8 + lane] = val;
        if (fn == 0) {
          fr = val;
          fr_c = comp;
        }
        ++fn;
      }
      if (lbgr) Pt = Pt + Chat;   // Eq. 6
      KVR_ACC(27, ta);
      // trial sums in query order, victim-log offsets (prefix sums of n_victims)
      uint64_t vc = 0;
      if (lane == 0) {
        ctrl->sum_lat = ctrl->sum_lat + lat;
        ctrl->sum_ttft = ctrl->sum_ttft + ttft;
        if (lat > ctrl->max_lat) ctrl->max_lat = lat;
        if (hist) atomicAdd(&hist[hist_bin(lat, p.bins)], 1u);
        if (fn > ws->c_maxp) ws->c_maxp = fn;   // before any catch-up for j+1
        vc = ctrl->vcursor;
        ctrl->vcursor = vc + nev;
        if (vlog && vc + nev > p.victims_per_trial)
          atomicCAS(&ctrl->status, 0u, (uint32_t)KVR_TRIAL_VICTIM_LOG_FULL);
      }
      KVR_ACC(28, ta);
      KVR_ACC(9, tp);

      // ---- misses: decisions (victims and slots) ----
      if (rlt) {
        uint32_t pslot = (uint32_t)p0;
        if (regbits) {
          if (M) {
            __syncwarp();
            if (lane == 0) {
              ws->x.size = wr.size;
              ws->x.cntT = wr.cntT;
              ws->x.wq = wr.wq;
              ws->x.lhead = wr.lhead;
              ws->x.ltail = wr.ltail;
            }
            __syncwarp();
            rlt_decide_reg<Idx, kMem, kMaxThreads>(p, M, p0, fallback, K, w, lane, use_list, j);
            wr.size = ws->x.size;
            wr.cntT = ws->x.cntT;
            if (lane == 0) ws->x.c_evict += nev;
          }
        } else {
          MemBits mb;
          mb.leaf = S.leaf;
          mb.mark = S.mark;
          mb.nw = nwords;
          __syncwarp();
          WorkerRegs xw = ws->x;
          xw.size = wr.size;
          xw.cntT = wr.cntT;
          xw.wq = wr.wq;
          xw.lhead = wr.lhead;
          xw.ltail = wr.ltail;
          uint64_t rbuf = ws->x_rbuf[lane];
          uint32_t ri = ws->x_ri;
#pragma unroll 1
          for (uint32_t cb = 0; cb < M; cb += 32)
            rlt_chunk<MemBits, Idx>(mb, S, R, xw, B, min(32u, M - cb), cb, p0, pslot, fallback,
                                    use_list, K, w, rbuf, ri, lane, slots, vbits);
          __syncwarp();
          if (lane == 0) {
            ws->x = xw;
            ws->x_ri = ri;
          }
          ws->x_rbuf[lane] = rbuf;
          wr.size = xw.size;
          wr.cntT = xw.cntT;
        }
      } else if (opt) {
        if (M) {
          __syncwarp();
          if (lane == 0) ws->x.size = wr.size;
          __syncwarp();
          opt_decide<Idx, kMem, kMaxThreads>(p, M, kf, p0, tr.nu + hd.block_off, w, lane, j);
          wr.size = ws->x.size;
          if (lane == 0) ws->x.c_evict += nev;
        }
      } else {
        // Leaf-LRU: the nev least recently used nodes, in order (batch == sequential)
        if (nev) {
          KVR_T0(tt);
#ifdef KVR_PHASE_PROFILE
          const uint32_t h0 = wr.lhead;
#endif
          // (loading the head windows earlier hides their latency but costs the
          // registers to hold them across the hits and accounting: slower overall)
          uint32_t lpre[kLogDepth];
          log_preload(R, wr.lhead, ltail0, lane, lpre);
          // the victims land in place, in slots[nfree .. M) (flagged below)
          wr.lhead = log_take(R, wr.lhead, ltail0, nev, slots + nfree, lane, lpre);
          KVR_ACC(11, tt);
          KVR_CNT(12, wr.lhead - h0);
        }
#pragma unroll 1
        for (uint32_t qq = lane; qq < M; qq += 32) {
          uint32_t sv;
          if (qq < nfree) {
            sv = size0 + qq;
          } else {
            const uint32_t v = slots[qq];
            sv = v | 0x80000000u;
            if (defer) atomicOr(&vmap[v >> 5], 1u << (v & 31));   // overlay bitmap
          }
          slots[qq] = sv;
        }
        wr.size = size0 + nfree;
        if (lane == 0) ws->x.c_evict += nev;
      }
      if (lane == 0) ws->x.c_ins += M;
      __syncwarp();
      if (kExt && lag) {   // this update, for the trackers of the next queries (A29)
        LagHdr* le = lag_entry(p, j);
        uint32_t* lsl = reinterpret_cast<uint32_t*>(le + 1);
        for (uint32_t qq = lane; qq < M; qq += 32) lsl[qq] = slots[qq];
        if (lane == 0) {
          le->block_off = hd.block_off;
          le->j = j;
          le->worker = w;
          le->kf = kf;
          le->M = M;
        }
      }
      KVR_ACC(8, tp);

      if (defer) {   // overlay bitmap of this update's victims -> registers
        vbits = vmap[lane];
        vmap[lane] = 0u;
      }
      if (lane == 0) {
        ws->j = j; ws->buf = buf; ws->n = n; ws->kf = kf; ws->M = M; ws->m = m; ws->nev = nev;
        ws->h = h; ws->ltail0 = ltail0; ws->wq = wr.wq; ws->p0 = (uint32_t)p0;
        ws->ttft = ttft; ws->lat = lat; ws->score = score; ws->vc = vc;
        ws->c_hit += h; ws->c_in += q; ws->c_q += 1;
        ws->active = 1;
      }
      if (use_list) wr.ltail = ltail0 + n;
      __syncwarp();
      if (lane == 0) {
        ws->x.size = wr.size;
        ws->x.cntT = wr.cntT;
        ws->x.wq = wr.wq;
        ws->x.lhead = wr.lhead;
        ws->x.ltail = wr.ltail;
      }
      __syncwarp();
      if (!defer) {
        apply_update<Idx, kMem, kMaxThreads, kExt>(p, lane, w, tree, use_list, lbgr_or_static, rec, vlog);
        vbits = 0;
      }
      KVR_SAVE_WORKER();
      }   // once
    }

    // ---- end of trial ----
    __syncthreads();   // all warps are past their last query before the final applies
#pragma unroll
    for (uint32_t vi = 0; vi < kV; ++vi) {
      if (kV > 1 && wid + vi * nwarps >= W) break;
      const uint32_t w = wid + vi * nwarps;
      WarpSm* ws = warp_sm(p, w);
      if (ws->active) {
        apply_update<Idx, kMem, kMaxThreads, kExt>(p, lane, w, tree, use_list, lbgr_or_static, rec, vlog);
        if constexpr (kV > 1) wsave(p, w)->vb[lane] = 0u;
        else st0.vbits = 0;
      }
    }
    __syncthreads();
    // drain staged-but-unconsumed queries (only after an abort)
    for (uint32_t qd = consumed; qd < issued; ++qd) {
      const uint64_t g = gq + qd;
      mbar_wait(&ctrl->mbar[g % kNumStages], (uint32_t)((g / kNumStages) & 1));
    }
    gq += issued;
#pragma unroll
    for (uint32_t vi = 0; vi < kV; ++vi) {
      if (kV > 1 && wid + vi * nwarps >= W) break;
      KVR_BIND_WORKER(wid + vi * nwarps);
    if (lane == 0) {
      atomicAdd(&ctrl->cnt[0], ws->c_probes);
      atomicAdd(&ctrl->cnt[1], (unsigned long long)ws->x.c_ins);
      atomicAdd(&ctrl->cnt[2], (unsigned long long)ws->x.c_evict);
      atomicAdd(&ctrl->cnt[3], (unsigned long long)ws->x.c_draws);
      atomicAdd(&ctrl->cnt[4], (unsigned long long)ws->x.c_resets);
      atomicAdd(&ctrl->cnt[5], (unsigned long long)ws->x.c_fb);
      atomicAdd(&ctrl->cnt[6], ws->c_hit);
      atomicAdd(&ctrl->cnt[7], ws->c_in);
      atomicAdd(&ctrl->cnt[8], (unsigned long long)ws->c_q);
      atomicMax(&ctrl->cnt[9], (unsigned long long)ws->c_maxp);
      ctrl->score[0][w] = P;   // (the scores are dead after the last query's barrier)
      ctrl->score[1][w] = F;
    }
    }
    __syncthreads();
    if (tid == 0) {
      kvr_trial_result Rr;
      Rr.probes = ctrl->cnt[0];
      Rr.inserted_blocks = ctrl->cnt[1];
      Rr.evictions = ctrl->cnt[2];
      Rr.rlt_draws = ctrl->cnt[3];
      Rr.rlt_resets = ctrl->cnt[4];
      Rr.rlt_fallbacks = ctrl->cnt[5];
      Rr.hit_tokens = ctrl->cnt[6];
      Rr.input_tokens = ctrl->cnt[7];
      Rr.queries = ctrl->cnt[8];
      Rr.max_pending = ctrl->cnt[9];
      Rr.decision_digest = ctrl->digest;
      Rr.sum_latency_ms = ctrl->sum_lat;
      Rr.sum_ttft_ms = ctrl->sum_ttft;
      Rr.max_latency_ms = ctrl->max_lat;
      double mk = 0.0, lc = 0.0, sl = 0.0;
      for (uint32_t i = 0; i < W; ++i) {   // makespan max_i P_i, in worker order
        const double Pi = ctrl->score[0][i], Fi = ctrl->score[1][i];
        if (Pi > mk) mk = Pi;
        if (Fi > lc) lc = Fi;
        sl = sl + Pi;
      }
      Rr.makespan_ms = mk;
      Rr.last_completion_ms = lc;
      Rr.sum_load_ms = sl;
      Rr.status = (int32_t)ctrl->status;
      Rr._pad = 0;
      p.results[trial] = Rr;
#ifdef KVR_PHASE_PROFILE
      if (trial < 4096) g_trial_cycles[trial] = clock64() - t_trial0;
#endif
    }
    if (led && Nrun) {   // distinct per phase; clean = first-appearance misses - not clean
      __threadfence_block();
      for (uint32_t v = tid; v < tr.n_phases; v += blockDim.x) {
        led[4 * v] = tr.distinct[v];
        led[4 * v + 3] = led[4 * v + 2] - led[4 * v + 3];
      }
    }
    __syncthreads();
  }
}

template <bool kExt>
static const void* kernel_for_t(uint32_t tier, uint32_t W) {
  if (tier == 1) {
    if (W <= 4) return (const void*)replay_kernel<uint16_t, 0, 128, kExt>;
    if (W <= 8) return (const void*)replay_kernel<uint16_t, 0, 256, kExt>;
    if (W <= 16) return (const void*)replay_kernel<uint16_t, 0, 512, kExt>;
    return (const void*)replay_kernel<uint16_t, 3, 512, kExt>;   // W > 16: two workers per warp
  }
  if (tier == 4) return (const void*)replay_kernel<uint16_t, 2, 512, kExt>;   // W > 16, 2 per warp
  if (W <= 4) return (const void*)replay_kernel<uint32_t, 1, 128, kExt>;
  if (W <= 8) return (const void*)replay_kernel<uint32_t, 1, 256, kExt>;
  if (W <= 16) return (const void*)replay_kernel<uint32_t, 1, 512, kExt>;
  if (tier == 3) return (const void*)replay_kernel<uint16_t, 1, 1024, kExt>;
  return (const void*)replay_kernel<uint32_t, 1, 1024, kExt>;
}

static const void* kernel_for(uint32_t tier, uint32_t W, bool ext) {
  return ext ? kernel_for_t<true>(tier, W) : kernel_for_t<false>(tier, W);
}

// threads per CTA: one warp per worker, two workers per warp in the split tier
static uint32_t replay_threads(uint32_t tier, uint32_t W) {
  return (tier == 4 || (tier == 1 && W > 16)) ? 32 * ((W + 1) / 2) : 32 * W;
}

cudaError_t replay_attrs(uint32_t tier, size_t smem, int* ctas_per_sm, uint32_t W, bool ext) {
  const void* k = kernel_for(tier, W, ext);
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(ctas_per_sm, k, replay_threads(tier, W), smem);
}

cudaError_t launch_replay(uint32_t tier, const ReplayParams& p, uint32_t grid, size_t smem,
                          cudaStream_t s, bool ext) {
  void* args[] = {const_cast<ReplayParams*>(&p)};
  return cudaLaunchKernel(kernel_for(tier, p.W, ext), dim3(grid), dim3(replay_threads(tier, p.W)),
                          args, smem, s);
}

cudaError_t phase_cycles(unsigned long long* out16, int reset) {
#ifdef KVR_WHO_LAST
  if (reset >= 5) {   // who-arrives-last counters (reset 6: and clear)
    cudaError_t e = cudaMemcpyFromSymbol(out16, g_who, 16 * sizeof(unsigned long long));
    if (e == cudaSuccess && reset == 6) {
      unsigned long long z[16] = {0};
      e = cudaMemcpyToSymbol(g_who, z, sizeof(z));
    }
    return e;
  }
#endif
#ifdef KVR_PHASE_PROFILE
  if (reset == 2)   // per-trial cycles (4096 entries)
    return cudaMemcpyFromSymbol(out16, g_trial_cycles, 4096 * sizeof(unsigned long long));
  cudaError_t e = cudaMemcpyFromSymbol(out16, g_phase_cycles, 32 * sizeof(unsigned long long));
  if (e == cudaSuccess && reset) {
    unsigned long long z[32] = {0};
    e = cudaMemcpyToSymbol(g_phase_cycles, z, sizeof(z));
  }
  return e;
#else
  (void)out16;
  (void)reset;
  return cudaErrorNotSupported;
#endif
}

}  // namespace kvr
