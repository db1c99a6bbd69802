// kvr_replay.cu — the replay kernel: one CTA per trial (persistent over a work
// counter), one warp per worker.  Per query j (trace order, t = a_j):
//   1. catch-up   (each warp, its worker): decay ticks merged with FIFO
//                 completions -> NLMS OnlineUpdate + ReleaseLoad
//                 (Alg. 2 l.11-17; readings A8, A10, A11)
//   2. match      (each warp, 32 lanes probe 32 blocks, ballot -> first miss):
//                 longest cached prefix m_ij of the query
//   3. score      LBGR Eq. 4-5 / STATIC / THRESHOLD / RR / RANDOM
//   -- one __syncthreads per query --
//   4. argmin     (every warp, shuffle reduction; lowest index on ties, A15)
//   5. update     (warp i* only): UpdateCache (Eq. 3) with RLT
//                 (Alg. 1; marking = MARK bitmap, uniform unmarked
//                 leaf by a warp popcount scan + Philox draw) or Leaf-LRU
//                 (O(1) intrusive list in (stamp,-depth) order)
//   6. accounting (warp i*): Eq. 1-2 truth, Eq. 6, FIFO latency / TTFT (A12-A14, A20)
// while the other warps already run steps 1-3 of query j+1.  Query headers and
// identities are staged in shared memory by 1-D bulk-async copies (TMA engine,
// cp.async.bulk + mbarrier) kNumStages-1 queries ahead.
//
// Scalar per-worker state (loads, theta, counters, list head) is warp-uniform:
// every lane holds the same value and performs the same fp64 operation, so
// no broadcast is needed; stores of shared scalars are made by all lanes
// with identical values.  fp64 follows the oracle's written operation order;
// the library is compiled with -fmad=false (no contraction) and IEEE division.
#include <math.h>

#include "kvr_device.cuh"
#include "kvr_internal.h"

namespace kvr {

template <typename Idx>
struct WorkerView {
  uint64_t* key;
  Idx* parent;
  Idx* nchild;
  Idx* prev;
  Idx* next;
  Idx* table;
  uint32_t* leaf;
  uint32_t* mark;
};

template <typename Idx>
__device__ __forceinline__ WorkerView<Idx> make_view(uint8_t* base, const WorkerLayout& L) {
  WorkerView<Idx> v;
  v.key = reinterpret_cast<uint64_t*>(base + L.off_key);
  v.parent = reinterpret_cast<Idx*>(base + L.off_parent);
  v.nchild = reinterpret_cast<Idx*>(base + L.off_nchild);
  v.prev = reinterpret_cast<Idx*>(base + L.off_prev);
  v.next = reinterpret_cast<Idx*>(base + L.off_next);
  v.table = reinterpret_cast<Idx*>(base + L.off_table);
  v.leaf = reinterpret_cast<uint32_t*>(base + L.off_leaf);
  v.mark = reinterpret_cast<uint32_t*>(base + L.off_mark);
  return v;
}

template <typename Idx>
__device__ __forceinline__ Idx table_lookup(const WorkerView<Idx>& S, uint32_t mask, uint64_t h) {
  const Idx NIL = (Idx)~(Idx)0;
  uint32_t pos = (uint32_t)h & mask;
  for (;;) {
    const Idx e = S.table[pos];
    if (e == NIL) return NIL;
    if (S.key[e] == h) return e;
    pos = (pos + 1) & mask;
  }
}

// linear probing insert: first empty position from home (table never full, T >= 2B)
template <typename Idx>
__device__ __forceinline__ void table_insert(const WorkerView<Idx>& S, uint32_t mask, uint64_t h,
                                             Idx slot, uint32_t lane) {
  const Idx NIL = (Idx)~(Idx)0;
  uint32_t pos = (uint32_t)h & mask;
  while (S.table[pos] != NIL) pos = (pos + 1) & mask;
  __syncwarp();
  if (lane == 0) S.table[pos] = slot;
  __syncwarp();
}

// backward-shift deletion of `slot` (identity h) keeps probe sequences intact
template <typename Idx>
__device__ __forceinline__ void table_delete(const WorkerView<Idx>& S, uint32_t mask, uint64_t h,
                                             Idx slot, uint32_t lane) {
  const Idx NIL = (Idx)~(Idx)0;
  uint32_t i = (uint32_t)h & mask;
  while (S.table[i] != slot) i = (i + 1) & mask;
  uint32_t j = (i + 1) & mask;
  for (;;) {
    const Idx e = S.table[j];
    if (e == NIL) break;
    const uint32_t home = (uint32_t)S.key[e] & mask;
    if (((j - home) & mask) >= ((j - i) & mask)) {
      __syncwarp();
      if (lane == 0) S.table[i] = e;
      __syncwarp();
      i = j;
    }
    j = (j + 1) & mask;
  }
  __syncwarp();
  if (lane == 0) S.table[i] = NIL;
  __syncwarp();
}

__device__ __forceinline__ void bit_set(uint32_t* w, uint32_t s, uint32_t lane) {
  const uint32_t v = w[s >> 5] | (1u << (s & 31));
  __syncwarp();
  if (lane == 0) w[s >> 5] = v;
  __syncwarp();
}
__device__ __forceinline__ void bit_clear(uint32_t* w, uint32_t s, uint32_t lane) {
  const uint32_t v = w[s >> 5] & ~(1u << (s & 31));
  __syncwarp();
  if (lane == 0) w[s >> 5] = v;
  __syncwarp();
}
__device__ __forceinline__ bool bit_test(const uint32_t* w, uint32_t s) {
  return (w[s >> 5] >> (s & 31)) & 1u;
}

// Uniform choice over U = LEAF (& ~MARK if use_mark) minus parent slot p, in
// physical-slot order (reading A6).  Returns |U| through *total; if idx_src is
// given it is the 64-bit random draw and the selected slot is returned.
__device__ __forceinline__ uint32_t rlt_count(const uint32_t* leaf, const uint32_t* mark,
                                              uint32_t nwords, uint32_t p, bool use_mark,
                                              uint32_t lane, uint32_t& lane_cnt,
                                              uint32_t& incl) {
  const uint32_t wpl = (nwords + 31) >> 5;
  const uint32_t w0 = lane * wpl, w1 = min(nwords, w0 + wpl);
  uint32_t c = 0;
  for (uint32_t wi = w0; wi < w1; ++wi) {
    uint32_t u = leaf[wi];
    if (use_mark) u &= ~mark[wi];
    if (wi == (p >> 5)) u &= ~(1u << (p & 31));
    c += __popc(u);
  }
  uint32_t v = c;
#pragma unroll
  for (int s = 1; s < 32; s <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, v, s);
    if (lane >= (uint32_t)s) v += y;
  }
  lane_cnt = c;
  incl = v;
  return __shfl_sync(kFull, v, 31);
}

__device__ __forceinline__ uint32_t rlt_select(const uint32_t* leaf, const uint32_t* mark,
                                               uint32_t nwords, uint32_t p, bool use_mark,
                                               uint32_t lane, uint32_t lane_cnt, uint32_t incl,
                                               uint32_t idx) {
  const uint32_t owner = __ffs(__ballot_sync(kFull, incl > idx)) - 1;
  uint32_t slot = 0;
  if (lane == owner) {
    const uint32_t wpl = (nwords + 31) >> 5;
    uint32_t rem = idx - (incl - lane_cnt);
    for (uint32_t wi = lane * wpl;; ++wi) {
      uint32_t u = leaf[wi];
      if (use_mark) u &= ~mark[wi];
      if (wi == (p >> 5)) u &= ~(1u << (p & 31));
      const uint32_t pc = __popc(u);
      if (rem < pc) {
        slot = wi * 32 + select_bit(u, rem);
        break;
      }
      rem -= pc;
    }
  }
  return __shfl_sync(kFull, slot, owner);
}

__device__ __forceinline__ uint32_t hist_bin(double lat, uint32_t bins) {
  if (!(lat >= 1.0)) return 0;
  int e;
  const double f = frexp(lat, &e);
  const uint32_t q = (uint32_t)((f * 2.0 - 1.0) * 4.0);
  const uint64_t b = 1 + 4 * (uint64_t)(e - 1) + q;
  return b >= bins ? bins - 1 : (uint32_t)b;
}

template <typename Idx>
__device__ __forceinline__ void list_unlink(const WorkerView<Idx>& S, Idx s, Idx& head, Idx& tail,
                                            uint32_t lane) {
  const Idx NIL = (Idx)~(Idx)0;
  const Idx pr = S.prev[s], nx = S.next[s];
  __syncwarp();
  if (lane == 0) {
    if (pr != NIL) S.next[pr] = nx;
    if (nx != NIL) S.prev[nx] = pr;
  }
  __syncwarp();
  if (pr == NIL) head = nx;
  if (nx == NIL) tail = pr;
}

// insert s at the start of the current query's segment (the segment holds the
// nodes touched by this query, deepest first, at the tail of the list)
template <typename Idx>
__device__ __forceinline__ void list_insert_seg(const WorkerView<Idx>& S, Idx s, Idx& head,
                                                Idx& tail, Idx& seg, uint32_t lane) {
  const Idx NIL = (Idx)~(Idx)0;
  if (seg == NIL) {
    const Idx t = tail;
    __syncwarp();
    if (lane == 0) {
      S.prev[s] = t;
      S.next[s] = NIL;
      if (t != NIL) S.next[t] = s;
    }
    __syncwarp();
    if (t == NIL) head = s;
    tail = s;
  } else {
    const Idx pr = S.prev[seg];
    __syncwarp();
    if (lane == 0) {
      S.prev[s] = pr;
      S.next[s] = seg;
      S.prev[seg] = s;
      if (pr != NIL) S.next[pr] = s;
    }
    __syncwarp();
    if (pr == NIL) head = s;
  }
  seg = s;
}

template <typename Idx, bool kGlobal, int kMaxThreads>
__global__ void __launch_bounds__(kMaxThreads, 1) replay_kernel(const __grid_constant__ ReplayParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  const Idx NIL = (Idx)~(Idx)0;
  const uint32_t tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t W = p.W, B = p.B;
  const WorkerLayout& L = p.lay;
  const uint32_t tmask = L.T - 1, nwords = L.nwords;

  Ctrl* ctrl = reinterpret_cast<Ctrl*>(smem);
  uint8_t* stage = smem + align16(sizeof(Ctrl));
  uint8_t* wbase = kGlobal ? p.gstate + ((size_t)blockIdx.x * W + w) * L.bytes
                           : stage + (size_t)kNumStages * p.stage_bytes + (size_t)w * L.bytes;
  const WorkerView<Idx> S = make_view<Idx>(wbase, L);
  double* fifo = reinterpret_cast<double*>(p.fifo + ((size_t)blockIdx.x * W + w) * p.ring * kFifoRecBytes);

  if (tid == 0) {
    for (uint32_t b = 0; b < kNumStages; ++b) mbar_init(&ctrl->mbar[b], 1);
    fence_mbar_init();
  }
  __syncthreads();

  uint64_t gq = 0;   // queries staged by this CTA so far (drives buffer index and parity)
  for (;;) {
    if (tid == 0) {
      const uint32_t tt = atomicAdd(p.work_counter, 1u);
      ctrl->trial = tt;
      if (tt < p.n_trials) ctrl->pol = p.policies ? p.policies[tt] : p.defpol;
    }
    __syncthreads();
    const uint32_t trial = ctrl->trial;
    if (trial >= p.n_trials) break;

    const TraceDev tr = p.traces[p.trial_trace ? p.trial_trace[trial] : 0];
    const kvr_policy& pol = ctrl->pol;   // shared memory, read on demand
    const uint64_t K = p.keys[trial];
    const uint32_t N = tr.N, bt = tr.block_tokens;
    const bool rlt = pol.eviction == KVR_EVICT_RLT;
    const bool use_list = !rlt || pol.rlt_fallback == KVR_RLT_LRU_MARKED;
    const bool lbgr = pol.router == KVR_ROUTE_LBGR;
    const bool recorded = trial < p.record_trials;
    kvr_query_record* rec = recorded ? p.records + (size_t)trial * p.rec_stride : nullptr;
    uint64_t* vlog = (recorded && p.victims) ? p.victims + (size_t)trial * p.victims_per_trial : nullptr;

    // ---- per-trial init: empty caches S_i^(0), P_i^(0) = 0 ----
    for (uint32_t i = lane; i < L.T; i += 32) S.table[i] = NIL;
    for (uint32_t i = lane; i < nwords; i += 32) {
      S.leaf[i] = 0;
      S.mark[i] = 0;
    }
    uint32_t size = 0, cntT = 0, fh = 0, fn = 0;
    Idx head = NIL, tail = NIL;
    double P = 0.0, F = 0.0, Pt = 0.0, front_c = 0.0;
    double th0 = pol.theta0[0], th1 = pol.theta0[1], th2 = pol.theta0[2], th3 = pol.theta0[3];
    uint64_t k = 0, e = 0;
    uint64_t c_probes = 0, c_ins = 0, c_evict = 0, c_draws = 0, c_resets = 0, c_fb = 0;
    uint64_t c_hit = 0, c_in = 0, c_q = 0, c_maxp = 0;
    if (tid == 0) {
      ctrl->sum_lat = 0.0;
      ctrl->sum_ttft = 0.0;
      ctrl->max_lat = 0.0;
      ctrl->digest = K;
      ctrl->vcursor = 0;
      ctrl->abortf[0] = 0;
      ctrl->abortf[1] = 0;
      ctrl->status = 0;
      for (int c = 0; c < 10; ++c) ctrl->cnt[c] = 0;
    }
    for (uint32_t b = tid; b < p.bins; b += blockDim.x) ctrl->hist[b] = 0;

    // a per-trial policy from device memory is validated here (host validated the default)
    const bool pol_ok = pol.eviction <= KVR_EVICT_RLT && pol.rlt_fallback <= KVR_RLT_LRU_MARKED &&
                        pol.router <= KVR_ROUTE_RANDOM && pol.rho > 0.0 && pol.rho <= 1.0 &&
                        pol.delta_t_ms > 0.0;
    if (!pol_ok && tid == 0) ctrl->status = KVR_TRIAL_BAD_POLICY;

    // staging prologue: queries 0 .. kNumStages-2
    const uint32_t Nrun = pol_ok ? N : 0;
    uint32_t issued = min(Nrun, kNumStages - 1);
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
    for (uint32_t j = 0; j < Nrun; ++j) {
      const uint64_t g = gq + j;
      const uint32_t buf = (uint32_t)(g % kNumStages);
      mbar_wait(&ctrl->mbar[buf], (uint32_t)((g / kNumStages) & 1));
      consumed = j + 1;
      const uint8_t* st = stage + (size_t)buf * p.stage_bytes;
      const QueryHdr hd = *reinterpret_cast<const QueryHdr*>(st);
      const uint64_t* H = reinterpret_cast<const uint64_t*>(st + 32) + (hd.block_off & 1);
      const double a = hd.arrival_ms;
      const uint32_t n_in = hd.n_in, n = hd.n_in + hd.n_out;
      const uint32_t q = bt * n_in;

      // ---- 1. catch-up (A11: tick before completion before routing) ----
      for (;;) {
        if (lbgr) {
          const double tau = (double)(k + 1) * pol.delta_t_ms;
          if (tau <= a && (fn == 0 || tau <= front_c)) {
            Pt = pol.rho * Pt;
            ++k;
            continue;
          }
        }
        if (fn != 0 && front_c <= a) {
          const double* r = fifo + (size_t)fh * 8;
          fh = (fh + 1 == p.ring) ? 0 : fh + 1;
          --fn;
          if (lbgr) {
            const double rc = r[0], ra = r[1], rE = r[2], f0 = r[3], f1 = r[4], f2 = r[5], rC = r[6];
            const uint64_t ka = __double_as_longlong(r[7]);
            // OnlineUpdate (A8): NLMS on the squared residual
            const double E = rc - ra;
            const double res = E - rE;
            const double f3 = 1.0;
            double s = f0 * f0;
            s = s + f1 * f1;
            s = s + f2 * f2;
            s = s + f3 * f3;
            const double gstep = (pol.mu * res) / (1.0 + s);
            th0 = th0 + gstep * f0;
            th1 = th1 + gstep * f1;
            th2 = th2 + gstep * f2;
            th3 = th3 + gstep * f3;
            // ReleaseLoad (A10): P~ <- max(0, P~ - C^ rho^kappa)
            uint64_t kap = k - ka;
            double pw = 1.0, bb = pol.rho;
            while (kap) {
              if (kap & 1) pw = pw * bb;
              bb = bb * bb;
              kap >>= 1;
            }
            Pt = Pt - rC * pw;
            if (Pt < 0.0) Pt = 0.0;
          }
          if (fn) front_c = fifo[(size_t)fh * 8];
          continue;
        }
        break;
      }

      // ---- 2. longest cached prefix over the input (ballot of 32 probes) ----
      uint32_t m = 0;
      for (uint32_t base = 0; base < n_in; base += 32) {
        const uint32_t d = base + lane;
        bool hit = false;
        if (d < n_in) hit = table_lookup<Idx>(S, tmask, H[d]) != NIL;
        const uint32_t bal = __ballot_sync(kFull, hit);
        if (bal == kFull) {
          m = base + 32;
          continue;
        }
        m = base + (__ffs(~bal) - 1);
        break;
      }
      if (m > n_in) m = n_in;
      c_probes += min(m + 1, n_in);

      // ---- 3. score (Eq. 4-5, A9) ----
      const double x = (double)(bt * m), y = (double)(q - bt * m);
      double score = 0.0, Chat = 0.0, f0 = 0.0, f1 = 0.0, f2 = 0.0;
      if (lbgr) {
        Chat = (pol.est_alpha_cached_ms * x) + (pol.est_alpha_miss_ms * y);
        f0 = x / 1000.0;
        f1 = y / 1000.0;
        f2 = Pt / 1000.0;
        const double f3 = 1.0;
        double dd = th0 * f0;
        dd = dd + th1 * f1;
        dd = dd + th2 * f2;
        dd = dd + th3 * f3;
        score = (Chat + Pt) + dd;
      } else if (pol.router == KVR_ROUTE_STATIC_LINEAR) {
        score = (pol.w_load * (double)fn) - (pol.w_hit * (x / (double)q));
      }
      const uint32_t par = j & 1;
      if (lane == 0) {
        ctrl->score[par][w] = score;
        ctrl->mhit[par][w] = m;
        ctrl->npend[par][w] = fn;
      }
      __syncthreads();
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
      if (pol.router == KVR_ROUTE_LBGR || pol.router == KVR_ROUTE_STATIC_LINEAR) {
        double v = lane < W ? ctrl->score[par][lane] : INFINITY;
        uint32_t bi = lane;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          const double v2 = __shfl_xor_sync(kFull, v, o);
          const uint32_t b2 = __shfl_xor_sync(kFull, bi, o);
          if (v2 < v || (v2 == v && b2 < bi)) {
            v = v2;
            bi = b2;
          }
        }
        best = bi;
      } else if (pol.router == KVR_ROUTE_THRESHOLD) {   // A16
        const uint32_t np = lane < W ? ctrl->npend[par][lane] : 0xffffffffu;
        const uint32_t mh = lane < W ? ctrl->mhit[par][lane] : 0u;
        const uint32_t mx = __reduce_max_sync(kFull, lane < W ? np : 0u);
        const uint32_t mn = __reduce_min_sync(kFull, np);
        if ((double)mx > pol.tau * (double)max(1u, mn)) {
          best = __ffs(__ballot_sync(kFull, np == mn)) - 1;
        } else {
          const uint32_t mmax = __reduce_max_sync(kFull, mh);
          best = __ffs(__ballot_sync(kFull, lane < W && mh == mmax)) - 1;
        }
      } else if (pol.router == KVR_ROUTE_ROUND_ROBIN) {
        best = j % W;
      } else {
        best = (uint32_t)pick_index(philox_r64(K, j, 0xffffffffu, 2u), W);
      }

      if (w != best) continue;

      // ================= warp i* : UpdateCache + accounting =================
      if (fn >= p.ring) {   // pending FIFO full -> trial status, stop (before Eq. 3)
        if (lane == 0) {
          ctrl->status = KVR_TRIAL_RING_OVERFLOW;
          ctrl->abortf[par ^ 1] = 1;
        }
        continue;
      }
      uint64_t D = ctrl->digest;
      D = fmix64(D ^ (uint64_t)j);
      D = fmix64(D ^ (uint64_t)best);
      D = fmix64(D ^ (uint64_t)m);
      uint64_t vc = ctrl->vcursor;
      const uint64_t vc0 = vc;
      uint32_t nv = 0;

      // full-path cached prefix kf (hits of Gamma_j; m covers the input part)
      uint32_t kf = m;
      if (m == n_in) {
        for (uint32_t base = n_in; base < n; base += 32) {
          const uint32_t d = base + lane;
          bool hit = false;
          if (d < n) hit = table_lookup<Idx>(S, tmask, H[d]) != NIL;
          const uint32_t bal = __ballot_sync(kFull, hit);
          if (bal == kFull) {
            kf = base + 32;
            continue;
          }
          kf = base + (__ffs(~bal) - 1);
          break;
        }
        if (kf > n) kf = n;
      }

      Idx seg = NIL;
      Idx pslot = NIL;
      for (uint32_t base = 0; base < n; base += 32) {
        const uint32_t d0 = base + lane;
        Idx myslot = NIL;
        if (d0 < kf) myslot = table_lookup<Idx>(S, tmask, H[d0]);
        const uint32_t cnt = min(32u, n - base);
        for (uint32_t l = 0; l < cnt; ++l) {
          const uint32_t d = base + l;
          if (d < kf) {
            // ---- hit (Alg. 1 l.10-11): mark, refresh recency ----
            const Idx s = (Idx)__shfl_sync(kFull, (uint32_t)myslot, l);
            if (rlt && !bit_test(S.mark, s)) {
              if (cntT == B) {   // |T|+1 = B+1 -> T = {t} (Alg. 1 l.8-9)
                __syncwarp();
                for (uint32_t i = lane; i < nwords; i += 32) S.mark[i] = 0;
                __syncwarp();
                cntT = 1;
                ++c_resets;
              } else {
                ++cntT;
              }
              bit_set(S.mark, s, lane);
            }
            if (use_list) {
              list_unlink<Idx>(S, s, head, tail, lane);
              list_insert_seg<Idx>(S, s, head, tail, seg, lane);
            }
            pslot = s;
            continue;
          }
          // ---- miss: mark t, evict if full, load t ----
          const uint64_t t = H[d];
          if (rlt) {
            if (cntT == B) {
              __syncwarp();
              for (uint32_t i = lane; i < nwords; i += 32) S.mark[i] = 0;
              __syncwarp();
              cntT = 1;
              ++c_resets;
            } else {
              ++cntT;
            }
          }
          Idx slot;
          if (size == B) {
            Idx v;
            if (!rlt) {
              v = head;   // Leaf-LRU: least recent (stamp, -depth) is the list head (A7)
            } else {
              uint32_t lc, inc;
              bool use_mark = true;
              uint32_t total = rlt_count(S.leaf, S.mark, nwords, (uint32_t)pslot, true, lane, lc, inc);
              bool draw = true;
              if (total == 0) {   // U empty (A5)
                ++c_fb;
                if (pol.rlt_fallback == KVR_RLT_EARLY_RESET) {
                  __syncwarp();
                  for (uint32_t i = lane; i < nwords; i += 32) S.mark[i] = 0;
                  __syncwarp();
                  cntT = 1;
                  ++c_resets;
                } else if (pol.rlt_fallback == KVR_RLT_UNIFORM_LEAF) {
                  use_mark = false;
                } else {
                  draw = false;
                }
                if (draw)
                  total = rlt_count(S.leaf, S.mark, nwords, (uint32_t)pslot, use_mark, lane, lc, inc);
              }
              if (draw) {
                const uint64_t r = philox_r64(K, e, best, 1u);
                ++e;
                ++c_draws;
                const uint32_t idx = (uint32_t)pick_index(r, total);
                v = (Idx)rlt_select(S.leaf, S.mark, nwords, (uint32_t)pslot, use_mark, lane, lc, inc, idx);
              } else {
                v = head;   // LRU over leaves != parent(t) = list head
              }
            }
            // ---- Evict(S, v) ----
            const uint64_t vkey = S.key[v];
            table_delete<Idx>(S, tmask, vkey, v, lane);
            if (use_list) list_unlink<Idx>(S, v, head, tail, lane);
            const Idx pv = S.parent[v];
            if (pv != NIL) {
              const Idx nc = (Idx)(S.nchild[pv] - 1);
              __syncwarp();
              if (lane == 0) S.nchild[pv] = nc;
              __syncwarp();
              if (nc == 0) bit_set(S.leaf, pv, lane);
            }
            bit_clear(S.leaf, v, lane);
            if (rlt && bit_test(S.mark, v)) {
              bit_clear(S.mark, v, lane);
              --cntT;
            }
            ++c_evict;
            D = fmix64(D ^ vkey);
            if (vlog) {
              if (vc < p.victims_per_trial) {
                if (lane == 0) vlog[vc] = vkey;
              } else if (lane == 0) {
                atomicCAS(&ctrl->status, 0u, (uint32_t)KVR_TRIAL_VICTIM_LOG_FULL);
              }
            }
            ++vc;
            ++nv;
            slot = v;
          } else {
            slot = (Idx)size;
            ++size;
          }
          // ---- Load(S, t) ----
          __syncwarp();
          if (lane == 0) {
            S.key[slot] = t;
            S.parent[slot] = pslot;
            S.nchild[slot] = 0;
          }
          __syncwarp();
          bit_set(S.leaf, slot, lane);
          if (pslot != NIL) {
            const Idx nc = S.nchild[pslot];
            __syncwarp();
            if (lane == 0) S.nchild[pslot] = (Idx)(nc + 1);
            __syncwarp();
            if (nc == 0) bit_clear(S.leaf, pslot, lane);
          }
          if (rlt) bit_set(S.mark, slot, lane);
          table_insert<Idx>(S, tmask, t, slot, lane);
          if (use_list) list_insert_seg<Idx>(S, slot, head, tail, seg, lane);
          ++c_ins;
          pslot = slot;
        }
      }

      // ---- accounting: Eq. 1 truth, Eq. 2, FIFO single server (A12, A20) ----
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
      {
        const uint32_t slotf = (fh + fn >= p.ring) ? fh + fn - p.ring : fh + fn;
        double* r = fifo + (size_t)slotf * 8;
        double val = 0.0;
        switch (lane) {
          case 0: val = comp; break;
          case 1: val = a; break;
          case 2: val = lbgr ? score : 0.0; break;
          case 3: val = lbgr ? f0 : 0.0; break;
          case 4: val = lbgr ? f1 : 0.0; break;
          case 5: val = lbgr ? f2 : 0.0; break;
          case 6: val = lbgr ? Chat : 0.0; break;
          case 7: val = __longlong_as_double((long long)k); break;
          default: break;
        }
        if (lane < 8) r[lane] = val;
        if (fn == 0) front_c = comp;
        ++fn;
        if (fn > c_maxp) c_maxp = fn;
      }
      if (lbgr) Pt = Pt + Chat;   // Eq. 6
      c_hit += h;
      c_in += q;
      ++c_q;
      D = fmix64(D ^ (uint64_t)nv);
      if (lane == 0) {
        ctrl->sum_lat = ctrl->sum_lat + lat;
        ctrl->sum_ttft = ctrl->sum_ttft + ttft;
        if (lat > ctrl->max_lat) ctrl->max_lat = lat;
        ctrl->digest = D;
        ctrl->vcursor = vc;
        if (rec) {
          kvr_query_record R;
          R.worker = best;
          R.hit_tokens = h;
          R.n_victims = nv;
          R._pad = 0;
          R.ttft_ms = ttft;
          R.latency_ms = lat;
          R.score = (lbgr || pol.router == KVR_ROUTE_STATIC_LINEAR) ? score : 0.0;
          R.victim_offset = vc0;
          rec[j] = R;
        }
        if (p.bins) ctrl->hist[hist_bin(lat, p.bins)] += 1;
      }
      __syncwarp();
    }

    // ---- end of trial ----
    __syncthreads();
    // drain staged-but-unconsumed queries (only after an abort)
    for (uint32_t qd = consumed; qd < issued; ++qd) {
      const uint64_t g = gq + qd;
      mbar_wait(&ctrl->mbar[g % kNumStages], (uint32_t)((g / kNumStages) & 1));
    }
    gq += issued;
    if (lane == 0) {
      atomicAdd(&ctrl->cnt[0], (unsigned long long)c_probes);
      atomicAdd(&ctrl->cnt[1], (unsigned long long)c_ins);
      atomicAdd(&ctrl->cnt[2], (unsigned long long)c_evict);
      atomicAdd(&ctrl->cnt[3], (unsigned long long)c_draws);
      atomicAdd(&ctrl->cnt[4], (unsigned long long)c_resets);
      atomicAdd(&ctrl->cnt[5], (unsigned long long)c_fb);
      atomicAdd(&ctrl->cnt[6], (unsigned long long)c_hit);
      atomicAdd(&ctrl->cnt[7], (unsigned long long)c_in);
      atomicAdd(&ctrl->cnt[8], (unsigned long long)c_q);
      atomicMax(&ctrl->cnt[9], (unsigned long long)c_maxp);
      ctrl->P[w] = P;
      ctrl->F[w] = F;
    }
    __syncthreads();
    if (tid == 0) {
      kvr_trial_result R;
      R.probes = ctrl->cnt[0];
      R.inserted_blocks = ctrl->cnt[1];
      R.evictions = ctrl->cnt[2];
      R.rlt_draws = ctrl->cnt[3];
      R.rlt_resets = ctrl->cnt[4];
      R.rlt_fallbacks = ctrl->cnt[5];
      R.hit_tokens = ctrl->cnt[6];
      R.input_tokens = ctrl->cnt[7];
      R.queries = ctrl->cnt[8];
      R.max_pending = ctrl->cnt[9];
      R.decision_digest = ctrl->digest;
      R.sum_latency_ms = ctrl->sum_lat;
      R.sum_ttft_ms = ctrl->sum_ttft;
      R.max_latency_ms = ctrl->max_lat;
      double mk = 0.0, lc = 0.0, sl = 0.0;
      for (uint32_t i = 0; i < W; ++i) {   // makespan max_i P_i, in worker order
        if (ctrl->P[i] > mk) mk = ctrl->P[i];
        if (ctrl->F[i] > lc) lc = ctrl->F[i];
        sl = sl + ctrl->P[i];
      }
      R.makespan_ms = mk;
      R.last_completion_ms = lc;
      R.sum_load_ms = sl;
      R.status = (int32_t)ctrl->status;
      R._pad = 0;
      p.results[trial] = R;
    }
    if (p.hist)
      for (uint32_t b = tid; b < p.bins; b += blockDim.x)
        p.hist[(size_t)trial * p.bins + b] = ctrl->hist[b];
    __syncthreads();
  }
}

static const void* kernel_for(uint32_t tier, uint32_t W) {
  if (tier == 1) {
    if (W <= 8) return (const void*)replay_kernel<uint16_t, false, 256>;
    if (W <= 16) return (const void*)replay_kernel<uint16_t, false, 512>;
    return (const void*)replay_kernel<uint16_t, false, 1024>;
  }
  if (W <= 8) return (const void*)replay_kernel<uint32_t, true, 256>;
  if (W <= 16) return (const void*)replay_kernel<uint32_t, true, 512>;
  return (const void*)replay_kernel<uint32_t, true, 1024>;
}

cudaError_t replay_attrs(uint32_t tier, size_t smem, int* ctas_per_sm, uint32_t W) {
  const void* k = kernel_for(tier, W);
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(ctas_per_sm, k, 32 * W, smem);
}

cudaError_t launch_replay(uint32_t tier, const ReplayParams& p, uint32_t grid, size_t smem,
                          cudaStream_t s) {
  void* args[] = {const_cast<ReplayParams*>(&p)};
  return cudaLaunchKernel(kernel_for(tier, p.W), dim3(grid), dim3(32 * p.W), args, smem, s);
}

}  // namespace kvr
