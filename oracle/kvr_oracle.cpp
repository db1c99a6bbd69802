// kvr_oracle.cpp — plain CPU oracle (TEST INFRASTRUCTURE; see kvr_oracle.h).
//
// Written from PAPER.md (arxiv 2601.18999) and the readings recorded in
// DESIGN.md §3 ("Readings of the paper", ids A1..A27 follow SURVEY §8(c)).
// Deliberately plain: std::unordered_map keyed by the chained block identity,
// one node per cached block, a linear scan over every cached node for each
// victim choice, std::deque FIFOs, fp64 arithmetic in the literal operation
// order (built with -ffp-contract=off -fno-fast-math).  Nothing here is
// shared with the CUDA path.
#include "kvr_oracle.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <deque>
#include <functional>
#include <map>
#include <unordered_map>
#include <unordered_set>
#include <utility>
#include <vector>

namespace {

// ---------------------------------------------------------------------------
// Block identity (A1, A26; SURVEY §8(c) "Definitions").  The paper keys its
// radix tree by token position along the path; a block's
// identity must therefore encode its whole prefix.  S_d = sum_{e<=d}
// fmix64(c_e ^ (e+1)*K ^ salt) mod 2^64, H_d = fmix64(S_d).
// ---------------------------------------------------------------------------
const uint64_t K_POS = 0x9E3779B97F4A7C15ULL;

uint64_t fmix64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return x;
}

// Philox4x32-10 (Salmon et al. 2011, Random123; constants as in curand's
// curand_philox4x32_x.h).  Counter-based: the RLT draw of worker i uses
// counter (e_i, i, tag 1), the RANDOM router counter (j, 0xFFFFFFFF, tag 2).
void philox(const uint32_t cin[4], const uint32_t kin[2], uint32_t out[4]) {
  uint32_t c0 = cin[0], c1 = cin[1], c2 = cin[2], c3 = cin[3];
  uint32_t k0 = kin[0], k1 = kin[1];
  for (int r = 0; r < 10; ++r) {
    if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

uint64_t philox_r64(uint64_t key, uint64_t n, uint32_t stream, uint32_t tag) {
  uint32_t c[4] = {(uint32_t)n, (uint32_t)(n >> 32), stream, tag};
  uint32_t k[2] = {(uint32_t)key, (uint32_t)(key >> 32)};
  uint32_t o[4];
  philox(c, k, o);
  return (uint64_t)o[0] | ((uint64_t)o[1] << 32);
}

// uniform index in [0, m): floor(r * m / 2^64)  (A6)
uint64_t pick(uint64_t r, uint64_t m) {
  return (uint64_t)(((unsigned __int128)r * (unsigned __int128)m) >> 64);
}

// i* = argmin over the scores, first index on ties (A15).  A NaN score (possible only
// through fp overflow, e.g. inf - inf in theta' phi) ranks after every number; all NaN
// -> worker 0 (reading A37).
uint32_t first_min(const std::vector<double>& s, uint32_t W) {
  uint32_t best = 0;
  for (uint32_t i = 1; i < W; ++i)
    if (!std::isnan(s[i]) && (std::isnan(s[best]) || s[i] < s[best])) best = i;
  return best;
}

// Cache-aware routing as SGLang's router does it ("switches between the
// highest-hit-rate and the least-loaded routing based on a predefined heuristic
// load-balance threshold"; reading A38): the load is imbalanced iff
// max - min > abs AND max > rel * min (pending queries); then the least loaded
// worker; else the highest match (router's view h~) if its rate h~/|q| exceeds the
// cache threshold, else the worker holding the fewest cached blocks (the most free
// capacity).  Lowest index on every tie (A15).
uint32_t cache_aware_choice(const kvro_policy* pol, const std::vector<uint64_t>& pending,
                            const std::vector<uint32_t>& mview, const std::vector<uint64_t>& size,
                            uint32_t W, uint32_t block_tokens, uint32_t q) {
  uint64_t mx = pending[0], mn = pending[0];
  for (uint32_t i = 1; i < W; ++i) {
    mx = std::max(mx, pending[i]);
    mn = std::min(mn, pending[i]);
  }
  const bool imbalanced = ((double)(mx - mn) > pol->ca_balance_abs) &&
                          ((double)mx > pol->ca_balance_rel * (double)mn);
  uint32_t best = 0;
  if (imbalanced) {
    for (uint32_t i = 1; i < W; ++i)
      if (pending[i] < pending[best]) best = i;
    return best;
  }
  for (uint32_t i = 1; i < W; ++i)
    if (mview[i] > mview[best]) best = i;
  const double rate = (double)(block_tokens * mview[best]) / (double)q;
  if (rate > pol->ca_cache_threshold) return best;
  best = 0;
  for (uint32_t i = 1; i < W; ++i)
    if (size[i] < size[best]) best = i;
  return best;
}

// per-trial policy checks shared by both engines (A8: NLMS needs 0 <= mu < 2;
// every parameter finite except delta_t_ms = +inf, which means no decay)
bool policy_valid(const kvro_policy* p) {
  if (p->eviction > KVRO_EVICT_OPT || p->rlt_fallback > KVRO_RLT_LRU_MARKED ||
      p->router > KVRO_ROUTE_CACHE_AWARE)
    return false;
  if (p->tracker_lag > KVRO_MAX_TRACKER_LAG || p->tracker_grain < 1) return false;
  if (!(p->rho > 0.0 && p->rho <= 1.0) || !(p->delta_t_ms > 0.0)) return false;
  const double fin[] = {p->est_alpha_cached_ms, p->est_alpha_miss_ms, p->mu, p->theta0[0],
                        p->theta0[1], p->theta0[2], p->theta0[3], p->tau, p->w_hit, p->w_load,
                        p->ca_balance_abs, p->ca_balance_rel, p->ca_cache_threshold};
  for (double v : fin)
    if (!std::isfinite(v)) return false;
  if (p->router == KVRO_ROUTE_LBGR && !(p->mu >= 0.0 && p->mu < 2.0)) return false;
  if (p->router == KVRO_ROUTE_LBGR_RLS &&
      (!(p->mu > 0.0 && p->mu <= 1.0) || !(p->rls_p0 > 0.0) || !std::isfinite(p->rls_p0)))
    return false;
  return true;
}

int validate_trace(const kvro_trace* tr) {
  if (!tr || tr->block_tokens == 0) return 1;
  if (tr->n_queries && (!tr->arrival_ms || !tr->n_in_blocks || !tr->n_out_blocks ||
                        !tr->out_tokens || !tr->block_offsets || !tr->block_keys))
    return 1;
  if (tr->n_queries && !tr->block_offsets) return 1;
  if (tr->block_offsets && tr->block_offsets[0] != 0) return 1;
  double prev = 0.0;
  for (uint32_t j = 0; j < tr->n_queries; ++j) {
    if (tr->n_in_blocks[j] < 1) return 1;
    uint64_t n = (uint64_t)tr->n_in_blocks[j] + tr->n_out_blocks[j];
    if (tr->block_offsets[j + 1] - tr->block_offsets[j] != n) return 1;
    double a = tr->arrival_ms[j];
    if (!std::isfinite(a) || a < 0.0 || a < prev) return 1;
    prev = a;
  }
  return 0;
}

std::vector<uint64_t> chain_all(const kvro_trace* tr) {
  uint64_t total = tr->n_queries ? tr->block_offsets[tr->n_queries] : 0;
  std::vector<uint64_t> H(total);
  for (uint32_t j = 0; j < tr->n_queries; ++j) {
    uint64_t S = 0;
    uint64_t o = tr->block_offsets[j];
    uint64_t n = tr->block_offsets[j + 1] - o;
    for (uint64_t d = 0; d < n; ++d) {
      S += fmix64(tr->block_keys[o + d] ^ ((d + 1) * K_POS) ^ tr->hash_salt);
      H[o + d] = fmix64(S);
    }
  }
  return H;
}

// ---------------------------------------------------------------------------
// One worker's cache S_i (Eq. 3): a prefix tree of blocks.
// ---------------------------------------------------------------------------
struct Node {
  uint64_t parent;     // identity of the parent block (valid iff has_parent)
  bool has_parent;     // false: child of the root
  uint32_t nchild;     // number of cached children
  uint32_t slot;       // physical slot (A6 slot rule)
  uint64_t stamp;      // index j of the last query that touched it (A7)
  uint32_t depth;      // position along the path, 1-based
  uint32_t pin = 0;    // in-flight paths holding it (continuous batching, A30)
};

struct Cache {
  uint32_t B = 0;
  std::unordered_map<uint64_t, Node> S;   // cache state S_i
  std::unordered_set<uint64_t> T;         // RLT marking set (Alg. 1 l.1)
};

struct UpdateCtx {
  uint32_t eviction = KVRO_EVICT_LRU;
  uint32_t fallback = KVRO_RLT_EARLY_RESET;
  uint64_t j = 0;                                      // stamp of this query
  std::function<uint64_t(uint64_t)> choose;            // uniform index in [0, n)
  std::function<std::pair<uint64_t, uint32_t>(uint64_t)> next_use;  // OPT only
  uint64_t hits = 0, inserted = 0, evictions = 0, draws = 0, resets = 0, fallbacks = 0;
  std::vector<uint64_t> victims;
  std::vector<uint8_t>* miss_flags = nullptr;
  bool invariant_violation = false;
  // continuous batching (A30): the path is pinned block by block as it is
  // accessed, and only unpinned leaves are eviction candidates
  bool pinning = false;
  bool admission_fail = false;  // full cache and no unpinned leaf
  // phase ledger (kvro_phase_ledger): called with the cache as it stands before the
  // d-th block access of the path is processed
  std::function<void(const Cache&, uint32_t)> before_access;
};

// (stamp, -depth) order of Leaf-LRU (A7): true if a is less recently used.
bool lru_less(const Node& a, const Node& b) {
  if (a.stamp != b.stamp) return a.stamp < b.stamp;
  return a.depth > b.depth;
}

// UpdateCache(S_i, Gamma_j, B_i) — Eq. 3 with Alg. 1 (RLT) or
// Leaf-LRU, block by block in path order.
void update_cache(Cache& C, const uint64_t* H, uint32_t n, UpdateCtx& x) {
  for (uint32_t d = 0; d < n; ++d) {
    if (x.before_access) x.before_access(C, d);
    const uint64_t t = H[d];
    const bool has_p = d > 0;
    const uint64_t p = has_p ? H[d - 1] : 0;
    // Alg. 1 l.6-9: mark t; the (B+1)-th distinct marked token resets T to {t}.
    if (x.eviction == KVRO_EVICT_RLT) {
      if (!C.T.count(t)) {
        if (C.T.size() + 1 == (size_t)C.B + 1) {
          C.T.clear();
          C.T.insert(t);
          x.resets++;
        } else {
          C.T.insert(t);
        }
      }
    }
    // Alg. 1 l.10-11: hit
    auto it = C.S.find(t);
    if (it != C.S.end()) {
      it->second.stamp = x.j;
      if (x.pinning) it->second.pin++;
      x.hits++;
      if (x.miss_flags) x.miss_flags->push_back(0);
      continue;
    }
    if (x.miss_flags) x.miss_flags->push_back(1);
    uint32_t slot;
    if (C.S.size() == C.B) {
      // Alg. 1 l.13-16 / Leaf-LRU: choose the victim v
      uint64_t v = 0;
      bool found = false;
      if (x.eviction == KVRO_EVICT_LRU) {
        // least recently used node among those not touched by this query;
        // always a leaf and never on Gamma_j (A7).
        const Node* best = nullptr;
        for (auto& kv : C.S) {
          if (x.pinning) {
            // A30/A33: least recently used UNPINNED leaf (the current path is pinned)
            if (kv.second.pin != 0 || kv.second.nchild != 0) continue;
          } else if (kv.second.stamp >= x.j) {
            continue;
          }
          if (!best || lru_less(kv.second, *best)) { best = &kv.second; v = kv.first; found = true; }
        }
        if (found && C.S[v].nchild != 0) x.invariant_violation = true;
        if (found && x.pinning) {
          // under pinning the minimum over ALL unpinned nodes is that leaf too (a
          // child's stamp never exceeds its parent's; an unpinned node's children
          // are unpinned) -- the basis of a one-selection Leaf-LRU
          for (auto& kv : C.S)
            if (kv.second.pin == 0 && lru_less(kv.second, C.S[v])) x.invariant_violation = true;
        }
      } else if (x.eviction == KVRO_EVICT_RLT) {
        // U = leaf tokens \ T, excluding parent(t) (A4)
        std::vector<std::pair<uint32_t, uint64_t>> U;  // (slot, id)
        for (auto& kv : C.S) {
          if (kv.second.nchild != 0) continue;
          if (has_p && kv.first == p) continue;
          if (kv.second.pin != 0) continue;          // A30: in-flight blocks stay
          if (C.T.count(kv.first)) continue;
          U.push_back({kv.second.slot, kv.first});
        }
        bool no_draw = false;
        if (U.empty()) {
          // A5: Alg. 1 leaves U = {} undefined
          x.fallbacks++;
          if (x.fallback == KVRO_RLT_EARLY_RESET) {
            C.T.clear();
            C.T.insert(t);
            x.resets++;
          }
          if (x.fallback == KVRO_RLT_LRU_MARKED) {
            const Node* best = nullptr;
            for (auto& kv : C.S) {
              if (kv.second.nchild != 0) continue;
              if (has_p && kv.first == p) continue;
              if (kv.second.pin != 0) continue;
              if (!best || lru_less(kv.second, *best)) { best = &kv.second; v = kv.first; found = true; }
            }
            no_draw = true;
          } else {
            for (auto& kv : C.S) {
              if (kv.second.nchild != 0) continue;
              if (has_p && kv.first == p) continue;
              if (kv.second.pin != 0) continue;
              U.push_back({kv.second.slot, kv.first});
            }
          }
        }
        if (!no_draw) {
          // Alg. 1 l.15: uniform over U, U ordered by physical slot (A6)
          std::sort(U.begin(), U.end());
          if (!U.empty()) {
            uint64_t idx = x.choose(U.size());
            if (idx >= U.size()) idx = U.size() - 1;
            v = U[idx].second;
            found = true;
            x.draws++;
          }
        }
      } else {  // OPT (Belady on leaves): furthest next use; ties -> lowest slot
        const Node* best = nullptr;
        std::pair<uint64_t, uint32_t> bnu{0, 0};
        for (auto& kv : C.S) {
          if (kv.second.nchild != 0) continue;
          if (has_p && kv.first == p) continue;
          auto nu = x.next_use(kv.first);
          bool better;
          if (!best) better = true;
          else if (nu.first != bnu.first) better = nu.first > bnu.first;
          else if (nu.first == UINT64_MAX) better = kv.second.slot < best->slot;
          else better = nu.second > bnu.second;
          if (better) { best = &kv.second; bnu = nu; v = kv.first; found = true; }
        }
      }
      if (!found) {
        if (x.pinning) x.admission_fail = true;   // every leaf is in flight
        else x.invariant_violation = true;
        return;
      }
      // Evict(S, v)
      Node nv = C.S[v];
      if (nv.nchild != 0) x.invariant_violation = true;
      slot = nv.slot;
      if (nv.has_parent) C.S[nv.parent].nchild--;
      C.T.erase(v);
      C.S.erase(v);
      x.victims.push_back(v);
      x.evictions++;
    } else {
      slot = (uint32_t)C.S.size();
    }
    // Load(S, t)
    Node nn;
    nn.parent = p; nn.has_parent = has_p; nn.nchild = 0; nn.slot = slot;
    nn.stamp = x.j; nn.depth = d + 1;
    nn.pin = x.pinning ? 1 : 0;
    C.S[t] = nn;
    if (has_p) C.S[p].nchild++;
    x.inserted++;
  }
}

// longest m <= n_in with H[0..m-1] all in S
uint32_t match_prefix(const Cache& C, const uint64_t* H, uint32_t n_in) {
  uint32_t m = 0;
  while (m < n_in && C.S.count(H[m])) ++m;
  return m;
}

bool check_cache(const Cache& C) {
  if (C.S.size() > C.B) return false;
  if (C.T.size() > C.B) return false;
  std::unordered_map<uint64_t, uint32_t> kids;
  std::vector<int> slot_used(C.B, 0);
  for (auto& kv : C.S) {
    if (kv.second.slot >= C.B) return false;
    if (slot_used[kv.second.slot]++) return false;
    if (kv.second.has_parent) {
      auto it = C.S.find(kv.second.parent);
      if (it == C.S.end()) return false;                       // prefix closure
      if (it->second.depth + 1 != kv.second.depth) return false;
      kids[kv.second.parent]++;
    } else if (kv.second.depth != 1) {
      return false;
    }
  }
  for (auto& kv : C.S)
    if (kv.second.nchild != kids[kv.first]) return false;
  for (uint64_t t : C.T)
    if (!C.S.count(t)) return false;                           // T subset of S
  return true;
}

uint64_t cache_fingerprint(const Cache& C) {
  uint64_t f = C.S.size() * 0x100000001B3ULL;
  for (auto& kv : C.S) f += fmix64(kv.first ^ ((uint64_t)kv.second.slot << 1) ^ (kv.second.stamp * 31));
  for (uint64_t t : C.T) f += fmix64(t + 7);
  return f;
}

// log-bucket histogram bin (exact bit rule, 4 bins per octave): 0 for lat < 1 ms
uint32_t hist_bin(double lat, uint32_t bins) {
  if (!(lat >= 1.0)) return 0;
  int e;
  double f = std::frexp(lat, &e);   // lat = f * 2^e, f in [0.5, 1)
  uint32_t q = (uint32_t)((f * 2.0 - 1.0) * 4.0);
  uint64_t b = 1 + 4 * (uint64_t)(e - 1) + q;
  return b >= bins ? bins - 1 : (uint32_t)b;
}

struct Rec {  // one pending completion (A12)
  double c, a, Ehat, phi0, phi1, phi2, Chat;
  uint64_t ka;
};

// One step of exponentially weighted recursive least squares (forgetting factor
// lam): pi = P phi, gamma = lam + phi' pi, k = pi / gamma, theta += k e,
// P = (P - k pi') / lam; every sum and loop in ascending index order.
void rls_step(double Pm[4][4], double th[4], const double phi[4], double e, double lam) {
  double pi[4];
  for (int a = 0; a < 4; ++a) {
    double t = Pm[a][0] * phi[0];
    t = t + Pm[a][1] * phi[1];
    t = t + Pm[a][2] * phi[2];
    t = t + Pm[a][3] * phi[3];
    pi[a] = t;
  }
  double g = phi[0] * pi[0];
  g = g + phi[1] * pi[1];
  g = g + phi[2] * pi[2];
  g = g + phi[3] * pi[3];
  const double gamma = lam + g;
  double kv[4];
  for (int a = 0; a < 4; ++a) kv[a] = pi[a] / gamma;
  for (int a = 0; a < 4; ++a) th[a] = th[a] + kv[a] * e;
  for (int a = 0; a < 4; ++a)
    for (int b = 0; b < 4; ++b) Pm[a][b] = (Pm[a][b] - kv[a] * pi[b]) / lam;
}

struct Worker {
  Cache cache;
  double P = 0.0, F = 0.0, Pt = 0.0;
  double th[4] = {0, 0, 0, 0};
  double Pm[4][4] = {};          // LBGR_RLS inverse-correlation matrix
  std::deque<Rec> fifo;
  uint64_t k = 0, e = 0;
};


// ---------------------------------------------------------------------------
// Continuous batching, beta >= 1 ("the system handles beta distinct
// queries concurrently"; SPEC simulator S:499-549; readings A30-A35 in DESIGN.md).
// Per worker: beta batch slots; assigned queries wait FIFO until a slot frees;
// UpdateCache (Eq. 3) runs at DEQUEUE and gives the true h; in-flight paths are
// pinned (SPEC access_path S:133-141) until their completion.
// ---------------------------------------------------------------------------
struct BRec {            // one assigned query (waiting, then in flight)
  uint32_t j;
  double a, Ehat, phi0, phi1, phi2, Chat;
  uint64_t ka;
  double c;              // completion time, set at dequeue
};

struct BWorker {
  Cache cache;
  double P = 0.0, F = 0.0, Pt = 0.0;
  double th[4] = {0, 0, 0, 0};
  double Pm[4][4] = {};
  std::deque<BRec> waiting;     // FIFO (A30)
  std::vector<BRec> inflight;   // <= beta
  uint64_t k = 0, e = 0;
  uint64_t vcur = 0;                       // per-worker victim-log cursor (A34)
};

int run_batched(const kvro_config* cfg, const kvro_trace* tr, const kvro_policy* pol,
                uint64_t K, const std::vector<uint64_t>& H, kvro_result* out,
                kvro_query_record* records, uint64_t* victims, uint64_t victims_cap,
                uint32_t* hist, int check_invariants) {
  const uint32_t W = cfg->W, B = cfg->capacity_blocks, beta = cfg->batch_slots;
  std::vector<BWorker> w(W);
  const bool rls = pol->router == KVRO_ROUTE_LBGR_RLS;
  const bool lbgr = pol->router == KVRO_ROUTE_LBGR || rls;
  for (auto& x : w) {
    x.cache.B = B;
    for (int k = 0; k < 4; ++k) x.th[k] = pol->theta0[k];
    if (rls)
      for (int k = 0; k < 4; ++k) x.Pm[k][k] = pol->rls_p0;
  }
  const double rho = pol->rho, dt = pol->delta_t_ms, mu = pol->mu;
  const uint64_t vshare = (victims && W) ? victims_cap / W : 0;   // A34: per-worker sub-share
  uint64_t D = K;
  bool vlog_full = false, admission = false, violation = false;
  // latency / TTFT of every dequeued query, summed in query order at the end (the plain
  // definition of the trial sums; reading A34)
  std::vector<double> lat_q(tr->n_queries, 0.0), ttft_q(tr->n_queries, 0.0);
  std::vector<uint8_t> done_q(tr->n_queries, 0);

  // Dequeue r on worker i at time s: UpdateCache with pinning, true h, Eq. 1 truth.
  auto dequeue = [&](uint32_t i, BRec r, double s) {
    BWorker& x = w[i];
    const uint32_t j = r.j;
    const uint32_t n_in = tr->n_in_blocks[j], n_out = tr->n_out_blocks[j];
    const uint32_t q = tr->block_tokens * n_in;
    const uint64_t* Hj = H.data() + tr->block_offsets[j];
    const uint32_t m = match_prefix(x.cache, Hj, n_in);      // true h at dequeue (A30)
    UpdateCtx ux;
    ux.eviction = pol->eviction;
    ux.fallback = pol->rlt_fallback;
    ux.j = j;                                                // A33: per-worker dequeue order
    ux.pinning = true;
    ux.choose = [&](uint64_t nU) -> uint64_t {
      uint64_t rr = philox_r64(K, x.e, i, 1);
      x.e++;
      return pick(rr, nU);
    };
    update_cache(x.cache, Hj, n_in + n_out, ux);
    if (ux.invariant_violation) { violation = true; return; }
    if (ux.admission_fail) { admission = true; return; }
    out->inserted_blocks += ux.inserted;
    out->evictions += ux.evictions;
    out->rlt_draws += ux.draws;
    out->rlt_resets += ux.resets;
    out->rlt_fallbacks += ux.fallbacks;
    const uint32_t h = tr->block_tokens * m;
    const double xh = (double)h, yh = (double)(q - h);
    const double pre = (cfg->alpha_cached_ms * xh) + (cfg->alpha_miss_ms * yh);   // Eq. 1
    const double O = cfg->out_ms_per_token * (double)tr->out_tokens[j];
    const double cost = pre + O;
    const double ttft = (s + pre) - r.a;                    // A20 (prefill done - arrival)
    const double comp = s + cost;
    const double lat = comp - r.a;
    r.c = comp;
    x.inflight.push_back(r);
    if (comp > x.F) x.F = comp;
    x.P = x.P + cost;                                        // Eq. 2
    out->hit_tokens += h;
    out->input_tokens += q;
    lat_q[j] = lat;
    ttft_q[j] = ttft;
    done_q[j] = 1;
    if (lat > out->max_latency_ms) out->max_latency_ms = lat;
    out->queries++;
    uint64_t V = 0;
    for (size_t k = 0; k < ux.victims.size(); ++k)
      V ^= fmix64(ux.victims[k] ^ ((uint64_t)(k + 1) * K_POS));
    uint64_t T = fmix64(K ^ (uint64_t)j);
    T = fmix64(T ^ (uint64_t)i);
    T = fmix64(T ^ (uint64_t)m);
    T = fmix64(T ^ (uint64_t)ux.victims.size());
    T = fmix64(T ^ V);
    D += T;
    if (records) {
      kvro_query_record& R = records[j];
      R.worker = i; R.hit_tokens = h; R.n_victims = (uint32_t)ux.victims.size(); R._pad = 0;
      R.ttft_ms = ttft; R.latency_ms = lat;
      R.victim_offset = (uint64_t)i * vshare + x.vcur;
      for (uint64_t v : ux.victims) {
        if (victims && x.vcur < vshare) victims[(uint64_t)i * vshare + x.vcur] = v;
        else if (victims) vlog_full = true;
        x.vcur++;
      }
    }
    if (hist && cfg->latency_hist_bins) hist[hist_bin(lat, cfg->latency_hist_bins)]++;
  };

  // Completion of the earliest in-flight query (ties: lower j, A31): LBGR
  // OnlineUpdate + ReleaseLoad exactly as in the beta = 1 model, unpin Gamma_j,
  // free the slot and start the head of the waiting FIFO at the same instant.
  auto complete_next = [&](uint32_t i) {
    BWorker& x = w[i];
    size_t b = 0;
    for (size_t u = 1; u < x.inflight.size(); ++u)
      if (x.inflight[u].c < x.inflight[b].c ||
          (x.inflight[u].c == x.inflight[b].c && x.inflight[u].j < x.inflight[b].j))
        b = u;
    BRec r = x.inflight[b];
    x.inflight.erase(x.inflight.begin() + (long)b);
    if (lbgr && !rls) {
      double E = r.c - r.a;
      double res = E - r.Ehat;
      double phi3 = 1.0;
      double s2 = r.phi0 * r.phi0;
      s2 = s2 + r.phi1 * r.phi1;
      s2 = s2 + r.phi2 * r.phi2;
      s2 = s2 + phi3 * phi3;
      double g = (mu * res) / (1.0 + s2);
      x.th[0] = x.th[0] + g * r.phi0;
      x.th[1] = x.th[1] + g * r.phi1;
      x.th[2] = x.th[2] + g * r.phi2;
      x.th[3] = x.th[3] + g * phi3;
    } else if (rls) {
      const double phi[4] = {r.phi0, r.phi1, r.phi2, 1.0};
      rls_step(x.Pm, x.th, phi, (r.c - r.a) - r.Ehat, mu);
    }
    if (lbgr) {
      uint64_t kap = x.k - r.ka;
      double pw = 1.0, bb = rho;
      while (kap) {
        if (kap & 1) pw = pw * bb;
        bb = bb * bb;
        kap >>= 1;
      }
      x.Pt = x.Pt - r.Chat * pw;
      if (x.Pt < 0.0) x.Pt = 0.0;
    }
    const uint64_t* Hj = H.data() + tr->block_offsets[r.j];
    const uint32_t n = tr->n_in_blocks[r.j] + tr->n_out_blocks[r.j];
    for (uint32_t d = 0; d < n; ++d) {                       // release_path
      auto it = x.cache.S.find(Hj[d]);
      if (it == x.cache.S.end() || it->second.pin == 0) { violation = true; return; }
      it->second.pin--;
    }
    while (x.inflight.size() < beta && !x.waiting.empty() && !admission && !violation) {
      BRec h = x.waiting.front();
      x.waiting.pop_front();
      dequeue(i, h, r.c);
    }
  };

  auto next_completion = [&](const BWorker& x) -> double {
    double c = INFINITY;
    for (const BRec& r : x.inflight) if (r.c < c) c = r.c;
    return c;
  };

  std::vector<uint32_t> m(W);
  std::vector<double> Ehat(W), Chat(W), phi0(W), phi1(W), phi2(W);
  for (uint32_t j = 0; j < tr->n_queries && !admission && !violation; ++j) {
    const double t = tr->arrival_ms[j];
    const uint32_t n_in = tr->n_in_blocks[j];
    const uint32_t q = tr->block_tokens * n_in;
    const uint64_t* Hj = H.data() + tr->block_offsets[j];

    // 1. catch-up per worker: ticks, completions (and the dequeues they
    //    trigger) in time order; tick < completion at equal times (A31)
    for (uint32_t i = 0; i < W && !admission && !violation; ++i) {
      BWorker& x = w[i];
      for (;;) {
        const double c = next_completion(x);
        if (lbgr) {
          double tau = (double)(x.k + 1) * dt;
          if (tau <= t && tau <= c) {
            x.Pt = rho * x.Pt;
            x.k++;
            continue;
          }
        }
        if (c <= t) {
          complete_next(i);
          if (admission || violation) break;
          continue;
        }
        break;
      }
    }
    if (admission || violation) break;

    // 2. match on the cache as it stands at a_j (A32)
    for (uint32_t i = 0; i < W; ++i) {
      m[i] = match_prefix(w[i].cache, Hj, n_in);
      out->probes += std::min<uint64_t>(m[i] + 1, n_in);
    }
    auto pending = [&](uint32_t i) -> size_t { return w[i].waiting.size() + w[i].inflight.size(); };

    // 3. score + argmin (lowest index on ties, A15); pending = waiting + in flight (A32)
    uint32_t best = 0;
    double score_best = 0.0;
    if (lbgr) {
      for (uint32_t i = 0; i < W; ++i) {
        double x = (double)(tr->block_tokens * m[i]);
        double y = (double)(q - tr->block_tokens * m[i]);
        double C = (pol->est_alpha_cached_ms * x) + (pol->est_alpha_miss_ms * y);   // Eq. 5
        double f0 = x / 1000.0, f1 = y / 1000.0, f2 = w[i].Pt / 1000.0, f3 = 1.0;  // A9
        double d = w[i].th[0] * f0;
        d = d + w[i].th[1] * f1;
        d = d + w[i].th[2] * f2;
        d = d + w[i].th[3] * f3;
        Ehat[i] = (C + w[i].Pt) + d;                                               // Eq. 4
        Chat[i] = C; phi0[i] = f0; phi1[i] = f1; phi2[i] = f2;
      }
      best = first_min(Ehat, W);
      score_best = Ehat[best];
    } else if (pol->router == KVRO_ROUTE_STATIC_LINEAR) {
      std::vector<double> s(W);
      for (uint32_t i = 0; i < W; ++i) {
        double x = (double)(tr->block_tokens * m[i]);
        s[i] = (pol->w_load * (double)pending(i)) - (pol->w_hit * (x / (double)q));
      }
      best = first_min(s, W);
      score_best = s[best];
    } else if (pol->router == KVRO_ROUTE_THRESHOLD) {
      size_t mx = pending(0), mn = pending(0);
      for (uint32_t i = 1; i < W; ++i) {
        mx = std::max(mx, pending(i));
        mn = std::min(mn, pending(i));
      }
      if ((double)mx > pol->tau * (double)std::max<size_t>(1, mn)) {
        for (uint32_t i = 1; i < W; ++i)
          if (pending(i) < pending(best)) best = i;
      } else {
        for (uint32_t i = 1; i < W; ++i)
          if (m[i] > m[best]) best = i;
      }
    } else if (pol->router == KVRO_ROUTE_CACHE_AWARE) {   // A38; pending = waiting + in flight
      std::vector<uint64_t> pend(W), size(W);
      for (uint32_t i = 0; i < W; ++i) {
        pend[i] = pending(i);
        size[i] = w[i].cache.S.size();
      }
      best = cache_aware_choice(pol, pend, m, size, W, tr->block_tokens, q);
    } else if (pol->router == KVRO_ROUTE_ROUND_ROBIN) {
      best = j % W;
    } else {
      best = (uint32_t)pick(philox_r64(K, j, 0xFFFFFFFFu, 2), W);
    }
    BWorker& xs = w[best];
    if (cfg->pending_ring && xs.waiting.size() >= cfg->pending_ring) {
      out->status = KVRO_TRIAL_RING_OVERFLOW;
      break;
    }

    // 4. assignment: Eq. 6 at assignment, enqueue, start now if a slot is free
    BRec r;
    r.j = j; r.a = t; r.c = 0.0;
    r.Ehat = lbgr ? Ehat[best] : 0.0;
    r.phi0 = lbgr ? phi0[best] : 0.0;
    r.phi1 = lbgr ? phi1[best] : 0.0;
    r.phi2 = lbgr ? phi2[best] : 0.0;
    r.Chat = lbgr ? Chat[best] : 0.0;
    r.ka = xs.k;
    if (lbgr) xs.Pt = xs.Pt + Chat[best];
    if (records) records[j].score = score_best;
    if (xs.inflight.size() < beta) dequeue(best, r, t);   // the FIFO is empty here (A30)
    else xs.waiting.push_back(r);
    if (pending(best) > out->max_pending) out->max_pending = pending(best);

    if (check_invariants && !admission && !violation) {
      for (uint32_t i = 0; i < W; ++i) {
        const BWorker& x = w[i];
        if (!check_cache(x.cache) || x.inflight.size() > beta) return 9;
        if (!x.waiting.empty() && x.inflight.size() < beta) return 9;
        // pin count of every block = number of in-flight paths through it
        std::unordered_map<uint64_t, uint32_t> pins;
        for (const BRec& f : x.inflight) {
          const uint64_t* Hf = H.data() + tr->block_offsets[f.j];
          const uint32_t n = tr->n_in_blocks[f.j] + tr->n_out_blocks[f.j];
          for (uint32_t d = 0; d < n; ++d) pins[Hf[d]]++;
        }
        for (auto& kv : x.cache.S) {
          auto it = pins.find(kv.first);
          if (kv.second.pin != (it == pins.end() ? 0u : it->second)) return 9;
        }
        if (x.Pt < 0.0) return 9;
      }
    }
  }
  // 5. drain (A35): every remaining completion and dequeue, in time order per
  //    worker; decay ticks can no longer change any output and are not run
  if (out->status == 0)
    for (uint32_t i = 0; i < W && !admission && !violation; ++i)
      while (!w[i].inflight.empty() && !admission && !violation) complete_next(i);
  if (violation) return 9;
  if (admission && out->status == 0) out->status = KVRO_TRIAL_ADMISSION;

  for (uint32_t j = 0; j < tr->n_queries; ++j)        // query order
    if (done_q[j]) {
      out->sum_latency_ms = out->sum_latency_ms + lat_q[j];
      out->sum_ttft_ms = out->sum_ttft_ms + ttft_q[j];
    }
  for (uint32_t i = 0; i < W; ++i) {
    if (w[i].P > out->makespan_ms) out->makespan_ms = w[i].P;
    if (w[i].F > out->last_completion_ms) out->last_completion_ms = w[i].F;
    out->sum_load_ms = out->sum_load_ms + w[i].P;
  }
  out->decision_digest = D;
  if (out->status == 0 && vlog_full) out->status = KVRO_TRIAL_VICTIM_LOG_FULL;
  return 0;
}

}  // namespace

extern "C" {

uint32_t kvro_version(void) { return 1; }
void kvro_rls_step(double P[16], double theta[4], const double phi[4], double e, double lam) {
  rls_step(reinterpret_cast<double(*)[4]>(P), theta, phi, e, lam);
}
uint64_t kvro_fmix64(uint64_t x) { return fmix64(x); }
void kvro_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) { philox(ctr, key, out); }

int kvro_chain(const kvro_trace* tr, uint64_t* out) {
  if (validate_trace(tr) || !out) return 1;
  std::vector<uint64_t> H = chain_all(tr);
  if (!H.empty()) std::memcpy(out, H.data(), H.size() * sizeof(uint64_t));
  return 0;
}

// Identity collisions (SURVEY §8a a0 "optional collision check"): list every block
// occurrence as (identity, occurrence index), sort, and count adjacent pairs with
// the same identity but a different (depth, parent identity, content key).
int kvro_count_collisions(const kvro_trace* tr, uint64_t* count) {
  if (validate_trace(tr) || !count) return 1;
  const std::vector<uint64_t> H = chain_all(tr);
  std::vector<std::pair<uint64_t, uint64_t>> occ;
  std::vector<uint64_t> depth(H.size()), parent(H.size());
  for (uint32_t j = 0; j < tr->n_queries; ++j)
    for (uint64_t o = tr->block_offsets[j]; o < tr->block_offsets[j + 1]; ++o) {
      depth[o] = o - tr->block_offsets[j];
      parent[o] = depth[o] ? H[o - 1] : 0;
      occ.push_back({H[o], o});
    }
  std::sort(occ.begin(), occ.end());
  uint64_t c = 0;
  for (size_t i = 1; i < occ.size(); ++i) {
    if (occ[i].first != occ[i - 1].first) continue;
    const uint64_t a = occ[i - 1].second, b = occ[i].second;
    if (depth[a] != depth[b] || parent[a] != parent[b] || tr->block_keys[a] != tr->block_keys[b]) c++;
  }
  *count = c;
  return 0;
}

int kvro_run(const kvro_config* cfg, const kvro_trace* tr, const kvro_policy* pol,
             uint64_t K, kvro_result* out, kvro_query_record* records,
             uint64_t* victims, uint64_t victims_cap, uint32_t* hist, int check_invariants) {
  if (!cfg || !pol || !out) return 1;
  if (validate_trace(tr)) return 1;
  const uint32_t W = cfg->W, B = cfg->capacity_blocks;
  if (W < 1 || W > 32 || B < 1 || B > 65536) return 1;
  if (!policy_valid(pol)) return 1;
  // Belady OPT is defined for one cache: the offline analysis runs it at W = 1
  if (pol->eviction == KVRO_EVICT_OPT && W != 1) return 1;
  // beta * L_max <= B (beta = 1 in the default model)
  const uint64_t beta = cfg->batch_slots > 0 ? cfg->batch_slots : 1;
  if (cfg->batch_slots > 64) return 1;
  if (cfg->batch_slots > 0 &&
      (pol->eviction == KVRO_EVICT_OPT || pol->tracker_lag != 0 || pol->tracker_grain != 1))
    return 1;   // the batched engine (A30) carries neither OPT nor tracker bias
  for (uint32_t j = 0; j < tr->n_queries; ++j)
    if (beta * ((uint64_t)tr->n_in_blocks[j] + tr->n_out_blocks[j]) > B) return 2;

  std::memset(out, 0, sizeof(*out));
  if (hist) std::memset(hist, 0, sizeof(uint32_t) * cfg->latency_hist_bins);
  const std::vector<uint64_t> H = chain_all(tr);
  if (cfg->batch_slots > 0)
    return run_batched(cfg, tr, pol, K, H, out, records, victims, victims_cap, hist,
                       check_invariants);
  // OPT: identity -> ascending query indices containing it, and its path depth
  std::unordered_map<uint64_t, std::vector<uint64_t>> occ;
  std::unordered_map<uint64_t, uint32_t> depth_of;
  if (pol->eviction == KVRO_EVICT_OPT)
    for (uint32_t j = 0; j < tr->n_queries; ++j)
      for (uint64_t o = tr->block_offsets[j]; o < tr->block_offsets[j + 1]; ++o) {
        occ[H[o]].push_back(j);
        depth_of[H[o]] = (uint32_t)(o - tr->block_offsets[j]) + 1;
      }
  std::vector<Worker> w(W);
  const bool rls = pol->router == KVRO_ROUTE_LBGR_RLS;
  for (auto& x : w) {
    x.cache.B = B;
    for (int k = 0; k < 4; ++k) x.th[k] = pol->theta0[k];
    if (rls)
      for (int k = 0; k < 4; ++k) x.Pm[k][k] = pol->rls_p0;
  }
  // LBGR_RLS is LBGR (Eq. 4-6, Alg. 2) with the other reading of the update (A8b)
  const bool lbgr = pol->router == KVRO_ROUTE_LBGR || rls;
  const double rho = pol->rho, dt = pol->delta_t_ms, mu = pol->mu;
  uint64_t D = K;
  uint64_t vcursor = 0;
  bool vlog_full = false;
  std::vector<uint32_t> m(W), mt(W);   // true match, and the tracker's view of it (A29)
  // global tracker lag (A29): the caches of the last k choosers as they were before
  // their updates, oldest first; the router's view of worker i is the oldest copy of
  // i in the window (the cache after query j-1-k), else its current cache
  std::deque<std::pair<uint32_t, Cache>> lagged;
  std::vector<double> Ehat(W), Chat(W), phi0(W), phi1(W), phi2(W);

  for (uint32_t j = 0; j < tr->n_queries; ++j) {
    const double t = tr->arrival_ms[j];
    const uint32_t n_in = tr->n_in_blocks[j], n_out = tr->n_out_blocks[j];
    const uint32_t q = tr->block_tokens * n_in;                   // |q_j| (A1)
    const uint64_t* Hj = H.data() + tr->block_offsets[j];

    // 1. catch-up: decay ticks (Alg. 2 l.17) merged with completions
    //    (Alg. 2 l.11-14); tick before completion before routing (A11)
    for (uint32_t i = 0; i < W; ++i) {
      Worker& x = w[i];
      for (;;) {
        if (lbgr) {
          double tau = (double)(x.k + 1) * dt;
          bool has = !x.fifo.empty();
          if (tau <= t && (!has || tau <= x.fifo.front().c)) {
            x.Pt = rho * x.Pt;
            x.k++;
            continue;
          }
        }
        if (!x.fifo.empty() && x.fifo.front().c <= t) {
          Rec r = x.fifo.front();
          x.fifo.pop_front();
          if (lbgr && !rls) {
            // OnlineUpdate: NLMS step on the squared residual (A8)
            double E = r.c - r.a;
            double res = E - r.Ehat;
            double phi3 = 1.0;
            double s = r.phi0 * r.phi0;
            s = s + r.phi1 * r.phi1;
            s = s + r.phi2 * r.phi2;
            s = s + phi3 * phi3;
            double g = (mu * res) / (1.0 + s);
            x.th[0] = x.th[0] + g * r.phi0;
            x.th[1] = x.th[1] + g * r.phi1;
            x.th[2] = x.th[2] + g * r.phi2;
            x.th[3] = x.th[3] + g * phi3;
          } else if (rls) {
            // OnlineUpdate, RLS reading (A8b) on the same residual e = E - E^
            const double phi[4] = {r.phi0, r.phi1, r.phi2, 1.0};
            rls_step(x.Pm, x.th, phi, (r.c - r.a) - r.Ehat, mu);
          }
          if (lbgr) {
            // ReleaseLoad: remove the decayed remainder rho^kappa * Chat (A10)
            uint64_t kap = x.k - r.ka;
            double pw = 1.0, b = rho;
            while (kap) {
              if (kap & 1) pw = pw * b;
              b = b * b;
              kap >>= 1;
            }
            x.Pt = x.Pt - r.Chat * pw;
            if (x.Pt < 0.0) x.Pt = 0.0;
          }
          continue;
        }
        break;
      }
    }

    // 2. longest cached prefix on every worker (h_ij)
    for (uint32_t i = 0; i < W; ++i) {
      m[i] = match_prefix(w[i].cache, Hj, n_in);
      out->probes += std::min<uint64_t>(m[i] + 1, n_in);
      // global tracker (App. E; reading A29): the router's estimate h~
      // lags the previous query's update and is coarsened to whole grains
      const Cache* view = &w[i].cache;
      for (auto it = lagged.rbegin(); it != lagged.rend(); ++it)
        if (it->first == i) view = &it->second;   // ends at the oldest copy of worker i
      uint32_t v = view == &w[i].cache ? m[i] : match_prefix(*view, Hj, n_in);
      mt[i] = pol->tracker_grain * (v / pol->tracker_grain);
    }

    // 3. score + argmin (lowest index on ties, A15)
    uint32_t best = 0;
    double score_best = 0.0;
    if (lbgr) {
      for (uint32_t i = 0; i < W; ++i) {
        double x = (double)(tr->block_tokens * mt[i]);          // h~ (A29; = h by default)
        double y = (double)(q - tr->block_tokens * mt[i]);
        double C = (pol->est_alpha_cached_ms * x) + (pol->est_alpha_miss_ms * y);   // Eq. 5
        double f0 = x / 1000.0, f1 = y / 1000.0, f2 = w[i].Pt / 1000.0, f3 = 1.0;  // A9
        double d = w[i].th[0] * f0;
        d = d + w[i].th[1] * f1;
        d = d + w[i].th[2] * f2;
        d = d + w[i].th[3] * f3;
        Ehat[i] = (C + w[i].Pt) + d;                                               // Eq. 4
        Chat[i] = C; phi0[i] = f0; phi1[i] = f1; phi2[i] = f2;
      }
      best = first_min(Ehat, W);
      score_best = Ehat[best];
    } else if (pol->router == KVRO_ROUTE_STATIC_LINEAR) {   // A17
      std::vector<double> s(W);
      for (uint32_t i = 0; i < W; ++i) {
        double x = (double)(tr->block_tokens * mt[i]);
        s[i] = (pol->w_load * (double)w[i].fifo.size()) - (pol->w_hit * (x / (double)q));
      }
      best = first_min(s, W);
      score_best = s[best];
    } else if (pol->router == KVRO_ROUTE_THRESHOLD) {       // A16
      size_t mx = w[0].fifo.size(), mn = w[0].fifo.size();
      for (uint32_t i = 1; i < W; ++i) {
        mx = std::max(mx, w[i].fifo.size());
        mn = std::min(mn, w[i].fifo.size());
      }
      if ((double)mx > pol->tau * (double)std::max<size_t>(1, mn)) {
        for (uint32_t i = 1; i < W; ++i)
          if (w[i].fifo.size() < w[best].fifo.size()) best = i;
      } else {
        for (uint32_t i = 1; i < W; ++i)
          if (mt[i] > mt[best]) best = i;
      }
    } else if (pol->router == KVRO_ROUTE_CACHE_AWARE) {     // A38
      std::vector<uint64_t> pend(W), size(W);
      for (uint32_t i = 0; i < W; ++i) {
        pend[i] = w[i].fifo.size();
        size[i] = w[i].cache.S.size();
      }
      best = cache_aware_choice(pol, pend, mt, size, W, tr->block_tokens, q);
    } else if (pol->router == KVRO_ROUTE_ROUND_ROBIN) {
      best = j % W;
    } else {  // RANDOM
      best = (uint32_t)pick(philox_r64(K, j, 0xFFFFFFFFu, 2), W);
    }
    Worker& xs = w[best];

    if (cfg->pending_ring && xs.fifo.size() >= cfg->pending_ring) {
      out->status = KVRO_TRIAL_RING_OVERFLOW;
      break;
    }
    uint64_t fp_before = 0;
    if (check_invariants)
      for (uint32_t i = 0; i < W; ++i)
        if (i != best) fp_before += cache_fingerprint(w[i].cache) * (i + 1);

    // 4. UpdateCache on i* only (Eq. 3)
    UpdateCtx ux;
    ux.eviction = pol->eviction;
    ux.fallback = pol->rlt_fallback;
    ux.j = j;
    ux.choose = [&](uint64_t nU) -> uint64_t {
      uint64_t r = philox_r64(K, xs.e, best, 1);
      xs.e++;
      return pick(r, nU);
    };
    const uint64_t jj = j;
    ux.next_use = [&](uint64_t id) -> std::pair<uint64_t, uint32_t> {   // OPT only
      const std::vector<uint64_t>& v = occ[id];
      auto it = std::upper_bound(v.begin(), v.end(), jj);
      if (it == v.end()) return {UINT64_MAX, 0};
      return {*it, depth_of[id]};
    };
    if (pol->tracker_lag) {   // the tracker still sees this cache for the next k queries
      lagged.emplace_back(best, xs.cache);
      if (lagged.size() > pol->tracker_lag) lagged.pop_front();
    }
    update_cache(xs.cache, Hj, n_in + n_out, ux);
    if (ux.invariant_violation) return 9;
    out->inserted_blocks += ux.inserted;
    out->evictions += ux.evictions;
    out->rlt_draws += ux.draws;
    out->rlt_resets += ux.resets;
    out->rlt_fallbacks += ux.fallbacks;

    // 5. accounting: Eq. 1-2 truth, FIFO single server (A12-A14, A20)
    const uint32_t h = tr->block_tokens * m[best];
    const double x = (double)h, y = (double)(q - h);
    const double pre = (cfg->alpha_cached_ms * x) + (cfg->alpha_miss_ms * y);
    const double O = cfg->out_ms_per_token * (double)tr->out_tokens[j];
    const double cost = pre + O;
    const double start = (t >= xs.F) ? t : xs.F;
    const double ttft = (start + pre) - t;
    const double comp = start + cost;
    const double lat = comp - t;
    xs.F = comp;
    xs.P = xs.P + cost;
    Rec r;
    r.c = comp; r.a = t;
    r.Ehat = lbgr ? Ehat[best] : 0.0;
    r.phi0 = lbgr ? phi0[best] : 0.0;
    r.phi1 = lbgr ? phi1[best] : 0.0;
    r.phi2 = lbgr ? phi2[best] : 0.0;
    r.Chat = lbgr ? Chat[best] : 0.0;
    r.ka = xs.k;
    xs.fifo.push_back(r);
    if (xs.fifo.size() > out->max_pending) out->max_pending = xs.fifo.size();
    if (lbgr) xs.Pt = xs.Pt + Chat[best];                                     // Eq. 6
    out->hit_tokens += h;
    out->input_tokens += q;
    out->sum_latency_ms = out->sum_latency_ms + lat;
    out->sum_ttft_ms = out->sum_ttft_ms + ttft;
    if (lat > out->max_latency_ms) out->max_latency_ms = lat;
    out->queries++;

    // 6. decision digest (DESIGN.md §3 "decision digest"): per query a tuple hash
    //    T_j of the index, the chosen worker, its hit blocks, the victim count and an
    //    order-sensitive combination of the victims, V = XOR_k fmix64(H_{v_k} ^ (k+1)*K);
    //    D = K + sum_j T_j mod 2^64 (order-independent across queries; K = trial key).
    uint64_t V = 0;
    for (size_t k = 0; k < ux.victims.size(); ++k)
      V ^= fmix64(ux.victims[k] ^ ((uint64_t)(k + 1) * K_POS));
    uint64_t T = fmix64(K ^ (uint64_t)j);
    T = fmix64(T ^ (uint64_t)best);
    T = fmix64(T ^ (uint64_t)m[best]);
    T = fmix64(T ^ (uint64_t)ux.victims.size());
    T = fmix64(T ^ V);
    D += T;

    if (records) {
      kvro_query_record& R = records[j];
      R.worker = best; R.hit_tokens = h; R.n_victims = (uint32_t)ux.victims.size(); R._pad = 0;
      R.ttft_ms = ttft; R.latency_ms = lat; R.score = score_best; R.victim_offset = vcursor;
      for (uint64_t v : ux.victims) {
        if (victims && vcursor < victims_cap) victims[vcursor] = v;
        else if (victims) vlog_full = true;
        vcursor++;
      }
    }
    if (hist && cfg->latency_hist_bins) hist[hist_bin(lat, cfg->latency_hist_bins)]++;

    if (check_invariants) {
      for (uint32_t i = 0; i < W; ++i)
        if (!check_cache(w[i].cache)) return 9;
      uint64_t fp_after = 0;
      for (uint32_t i = 0; i < W; ++i)
        if (i != best) fp_after += cache_fingerprint(w[i].cache) * (i + 1);
      if (fp_after != fp_before) return 9;                // Eq. 3: others unchanged
      if (m[best] > n_in || ux.hits + ux.inserted != (uint64_t)n_in + n_out) return 9;
      for (uint32_t i = 0; i < W; ++i)
        if (w[i].Pt < 0.0) return 9;
      if (ttft > lat && cfg->out_ms_per_token >= 0.0) return 9;
    }
  }

  // end of trial: makespan max_i P_i (A21), last completion, sum of loads
  for (uint32_t i = 0; i < W; ++i) {
    if (w[i].P > out->makespan_ms) out->makespan_ms = w[i].P;
    if (w[i].F > out->last_completion_ms) out->last_completion_ms = w[i].F;
    out->sum_load_ms = out->sum_load_ms + w[i].P;
  }
  out->decision_digest = D;
  if (out->status == 0 && vlog_full) out->status = KVRO_TRIAL_VICTIM_LOG_FULL;
  return 0;
}

// ---------------------------------------------------------------------------
// Single-cache analysis tools (W = 1; §3.2, App. C).  Arrivals and costs are
// ignored: only the eviction process over the flattened block sequence.
// ---------------------------------------------------------------------------
int kvro_single_replay(const kvro_trace* tr, uint32_t B, uint32_t eviction, uint32_t fallback,
                       uint64_t K, uint8_t* miss_flags, uint64_t* total_misses,
                       const uint32_t* choices, uint32_t* arity, uint32_t max_draws,
                       uint32_t* n_draws) {
  if (validate_trace(tr) || B < 1 || eviction > KVRO_EVICT_OPT || fallback > KVRO_RLT_LRU_MARKED)
    return 1;
  for (uint32_t j = 0; j < tr->n_queries; ++j)
    if ((uint64_t)tr->n_in_blocks[j] + tr->n_out_blocks[j] > B) return 2;
  const std::vector<uint64_t> H = chain_all(tr);
  // next-use index for OPT: identity -> ascending list of query indices
  std::unordered_map<uint64_t, std::vector<uint64_t>> occ;
  std::unordered_map<uint64_t, uint32_t> depth_of;
  if (eviction == KVRO_EVICT_OPT) {
    for (uint32_t j = 0; j < tr->n_queries; ++j)
      for (uint64_t o = tr->block_offsets[j]; o < tr->block_offsets[j + 1]; ++o) {
        occ[H[o]].push_back(j);
        depth_of[H[o]] = (uint32_t)(o - tr->block_offsets[j]) + 1;
      }
  }
  Cache C;
  C.B = B;
  std::vector<uint8_t> flags;
  uint64_t e = 0, misses = 0;
  uint32_t draw_idx = 0;
  bool overflow = false;
  for (uint32_t j = 0; j < tr->n_queries; ++j) {
    UpdateCtx ux;
    ux.eviction = eviction;
    ux.fallback = fallback;
    ux.j = j;
    ux.miss_flags = &flags;
    ux.choose = [&](uint64_t nU) -> uint64_t {
      uint64_t idx;
      if (choices) {
        idx = draw_idx < max_draws ? choices[draw_idx] : 0;
        if (idx >= nU) idx = nU - 1;
      } else {
        idx = pick(philox_r64(K, e, 0, 1), nU);
      }
      if (arity) {
        if (draw_idx < max_draws) arity[draw_idx] = (uint32_t)nU;
        else overflow = true;
      }
      draw_idx++;
      e++;
      return idx;
    };
    const uint64_t jj = j;
    ux.next_use = [&](uint64_t id) -> std::pair<uint64_t, uint32_t> {
      const std::vector<uint64_t>& v = occ[id];
      auto it = std::upper_bound(v.begin(), v.end(), jj);
      if (it == v.end()) return {UINT64_MAX, 0};
      return {*it, depth_of[id]};
    };
    uint64_t n = tr->block_offsets[j + 1] - tr->block_offsets[j];
    update_cache(C, H.data() + tr->block_offsets[j], (uint32_t)n, ux);
    if (ux.invariant_violation) return 9;
    misses += ux.inserted;
  }
  if (miss_flags && !flags.empty()) std::memcpy(miss_flags, flags.data(), flags.size());
  if (total_misses) *total_misses = misses;
  if (n_draws) *n_draws = draw_idx;
  return overflow ? 4 : 0;
}

namespace {
struct BF {
  uint32_t B;
  std::vector<uint64_t> acc;      // flattened accesses
  std::vector<uint64_t> par;      // parent identity of each access (0 + flag)
  std::vector<uint8_t> has_par;
  std::unordered_map<uint64_t, uint64_t> parent_of;
  std::map<std::pair<size_t, std::vector<uint64_t>>, uint64_t> memo;

  uint64_t solve(size_t pos, std::vector<uint64_t>& cached) {   // cached kept sorted
    if (pos == acc.size()) return 0;
    auto key = std::make_pair(pos, cached);
    auto it = memo.find(key);
    if (it != memo.end()) return it->second;
    const uint64_t t = acc[pos];
    uint64_t res;
    if (std::binary_search(cached.begin(), cached.end(), t)) {
      res = solve(pos + 1, cached);
    } else if (cached.size() < B) {
      std::vector<uint64_t> nx = cached;
      nx.insert(std::upper_bound(nx.begin(), nx.end(), t), t);
      res = 1 + solve(pos + 1, nx);
    } else {
      res = UINT64_MAX;
      for (uint64_t u : cached) {
        if (has_par[pos] && u == par[pos]) continue;
        bool leaf = true;   // no cached child
        for (uint64_t c : cached) {
          auto pi = parent_of.find(c);
          if (pi != parent_of.end() && pi->second == u) { leaf = false; break; }
        }
        if (!leaf) continue;
        std::vector<uint64_t> nx;
        for (uint64_t c : cached) if (c != u) nx.push_back(c);
        nx.insert(std::upper_bound(nx.begin(), nx.end(), t), t);
        uint64_t r = solve(pos + 1, nx);
        if (r != UINT64_MAX && 1 + r < res) res = 1 + r;
      }
    }
    memo[key] = res;
    return res;
  }
};
}  // namespace

// Phase ledger (reading A39): phases of exactly B distinct blocks over the
// flattened access sequence, and per phase the misses of one single-cache replay and
// the clean tokens relative to that replay's own cache at the end of the previous phase.
int kvro_phase_ledger(const kvro_trace* tr, uint32_t B, uint32_t eviction, uint32_t fallback,
                      uint64_t K, uint32_t* ledger, uint32_t max_phases, uint32_t* n_phases) {
  if (validate_trace(tr) || B < 1 || eviction > KVRO_EVICT_OPT || fallback > KVRO_RLT_LRU_MARKED ||
      !n_phases)
    return 1;
  for (uint32_t j = 0; j < tr->n_queries; ++j)
    if ((uint64_t)tr->n_in_blocks[j] + tr->n_out_blocks[j] > B) return 2;
  const std::vector<uint64_t> H = chain_all(tr);
  const uint64_t total = H.size();
  // 1. greedy phases over the access sequence: a phase ends just before the access
  //    that would be its (B+1)-th distinct block
  std::vector<uint32_t> phase_of(total);
  std::vector<uint8_t> first(total);
  std::vector<uint64_t> start;   // first access of every phase
  {
    std::unordered_set<uint64_t> seen;
    for (uint64_t o = 0; o < total; ++o) {
      if (!seen.count(H[o])) {
        if (seen.size() == B || start.empty()) {
          start.push_back(o);
          seen.clear();
        }
        seen.insert(H[o]);
        first[o] = 1;
      }
      phase_of[o] = (uint32_t)start.size() - 1;
    }
  }
  *n_phases = (uint32_t)start.size();
  if (start.size() > max_phases) return 3;
  if (!ledger) return 1;
  std::memset(ledger, 0, sizeof(uint32_t) * 4 * start.size());
  // 2. the single-cache replay; the cache is copied at every phase start
  std::unordered_map<uint64_t, std::vector<uint64_t>> occ;
  std::unordered_map<uint64_t, uint32_t> depth_of;
  if (eviction == KVRO_EVICT_OPT)
    for (uint32_t j = 0; j < tr->n_queries; ++j)
      for (uint64_t o = tr->block_offsets[j]; o < tr->block_offsets[j + 1]; ++o) {
        occ[H[o]].push_back(j);
        depth_of[H[o]] = (uint32_t)(o - tr->block_offsets[j]) + 1;
      }
  Cache C;
  C.B = B;
  std::vector<uint8_t> flags;
  std::unordered_set<uint64_t> at_start;   // cache content at the start of the current phase
  uint64_t e = 0;
  for (uint32_t j = 0; j < tr->n_queries; ++j) {
    const uint64_t off = tr->block_offsets[j];
    UpdateCtx ux;
    ux.eviction = eviction;
    ux.fallback = fallback;
    ux.j = j;
    ux.miss_flags = &flags;
    ux.choose = [&](uint64_t nU) -> uint64_t { return pick(philox_r64(K, e++, 0, 1), nU); };
    const uint64_t jj = j;
    ux.next_use = [&](uint64_t id) -> std::pair<uint64_t, uint32_t> {
      const std::vector<uint64_t>& v = occ[id];
      auto it = std::upper_bound(v.begin(), v.end(), jj);
      if (it == v.end()) return {UINT64_MAX, 0};
      return {*it, depth_of[id]};
    };
    ux.before_access = [&](const Cache& c, uint32_t d) {
      const uint64_t o = off + d;
      if (o == start[phase_of[o]]) {   // the end of phase v-1: remember the cache
        at_start.clear();
        for (auto& kv : c.S) at_start.insert(kv.first);
      }
      uint32_t* L = ledger + 4 * (size_t)phase_of[o];
      if (first[o]) {
        L[0] += 1;
        if (!at_start.count(H[o])) L[3] += 1;   // clean: not cached when the phase began
      }
    };
    const uint32_t n = (uint32_t)(tr->block_offsets[j + 1] - off);
    update_cache(C, H.data() + off, n, ux);
    if (ux.invariant_violation) return 9;
    for (uint32_t d = 0; d < n; ++d)
      if (flags[off + d]) {
        uint32_t* L = ledger + 4 * (size_t)phase_of[off + d];
        L[1] += 1;
        if (first[off + d]) L[2] += 1;
      }
  }
  return 0;
}

int kvro_bruteforce_min_misses(const kvro_trace* tr, uint32_t B, uint64_t* min_misses) {
  if (validate_trace(tr) || B < 1 || !min_misses) return 1;
  uint64_t total = tr->n_queries ? tr->block_offsets[tr->n_queries] : 0;
  if (B > 6 || total > 48) return 3;
  for (uint32_t j = 0; j < tr->n_queries; ++j)
    if ((uint64_t)tr->n_in_blocks[j] + tr->n_out_blocks[j] > B) return 2;
  const std::vector<uint64_t> H = chain_all(tr);
  BF bf;
  bf.B = B;
  for (uint32_t j = 0; j < tr->n_queries; ++j)
    for (uint64_t o = tr->block_offsets[j]; o < tr->block_offsets[j + 1]; ++o) {
      bool hp = o > tr->block_offsets[j];
      bf.acc.push_back(H[o]);
      bf.has_par.push_back(hp);
      bf.par.push_back(hp ? H[o - 1] : 0);
      if (hp) bf.parent_of[H[o]] = H[o - 1];
    }
  std::vector<uint64_t> empty;
  *min_misses = bf.solve(0, empty);
  return 0;
}

int kvro_rlt_exact_expectation(const kvro_trace* tr, uint32_t B, uint32_t fallback,
                               double* mean, double* second_moment, uint64_t* leaves) {
  if (!mean || !second_moment) return 1;
  const uint32_t MAXD = 4096;
  std::vector<uint32_t> choice(MAXD, 0), arity(MAXD, 0);
  double m1 = 0.0, m2 = 0.0;
  uint64_t nleaves = 0;
  for (;;) {
    uint64_t misses = 0;
    uint32_t nd = 0;
    int rc = kvro_single_replay(tr, B, KVRO_EVICT_RLT, fallback, 0, nullptr, &misses,
                                choice.data(), arity.data(), MAXD, &nd);
    if (rc) return rc;
    double p = 1.0;
    for (uint32_t k = 0; k < nd; ++k) p = p / (double)arity[k];
    m1 += p * (double)misses;
    m2 += p * (double)misses * (double)misses;
    if (++nleaves > 20000000ULL) return 3;
    // odometer over the decision tree (later arities depend on earlier choices)
    int k = (int)nd - 1;
    while (k >= 0 && choice[k] + 1 >= arity[k]) --k;
    if (k < 0) break;
    choice[k]++;
    for (uint32_t r = k + 1; r < MAXD; ++r) choice[r] = 0;
  }
  *mean = m1;
  *second_moment = m2;
  if (leaves) *leaves = nleaves;
  return 0;
}

}  // extern "C"
