// kvr_api.cu — host side of the C ABI declared in include/kvr.h: argument
// validation, handles, state-tier selection, workspace sizing and launches.
// No device memory is allocated here; every buffer belongs to the caller.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "kvr_internal.h"

struct kvr_trace {
  uint32_t N, block_tokens, max_n;
  uint64_t total, salt;
  kvr::QueryHdr* hdr;
  uint64_t* hash;
  const uint32_t* nu = nullptr;   // next-use index (offline OPT), borrowed
  const uint32_t* ph = nullptr;   // phase index (phase ledger), borrowed: ph, nx, distinct
  uint32_t n_phases = 0, phase_B = 0;
};

struct kvr_sim {
  kvr_sim_config cfg;
};

namespace {

thread_local std::string g_err;

kvr_status fail(kvr_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

kvr_status cuda_fail(cudaError_t e, const char* what) {
  return fail(KVR_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

// policies that need the extended kernel instantiation
bool policy_extended(const kvr_policy& p) {
  return p.eviction == KVR_EVICT_OPT || p.router == KVR_ROUTE_LBGR_RLS ||
         p.router == KVR_ROUTE_CACHE_AWARE || p.tracker_lag != 0 || p.tracker_grain != 1;
}

bool sim_extended(const kvr_sim_config& c) {
  return c.extended_policies != 0 || policy_extended(c.default_policy);
}

bool policy_ok(const kvr_policy& p, std::string* why) {
  char b[256];
  auto bad = [&](const char* s) { snprintf(b, sizeof b, "policy: %s", s); *why = b; return false; };
  if (p.eviction > KVR_EVICT_OPT) return bad("eviction must be LRU(0), RLT(1) or OPT(2)");
  if (p.rlt_fallback > KVR_RLT_LRU_MARKED) return bad("rlt_fallback must be 0..2");
  if (p.router > KVR_ROUTE_CACHE_AWARE) return bad("router must be 0..6");
  if (p.tracker_lag > kvr::kMaxLag) return bad("tracker_lag must be in 0..32");
  if (p.tracker_grain < 1) return bad("tracker_grain must be >= 1");
  if (p.router == KVR_ROUTE_LBGR_RLS && !(p.mu > 0.0 && p.mu <= 1.0))
    return bad("LBGR_RLS forgetting factor mu must be in (0, 1]");
  if (p.router == KVR_ROUTE_LBGR_RLS && !(p.rls_p0 > 0.0 && std::isfinite(p.rls_p0)))
    return bad("LBGR_RLS rls_p0 must be finite and > 0");
  if (!(p.rho > 0.0 && p.rho <= 1.0)) return bad("rho must be in (0, 1]");
  if (!(p.delta_t_ms > 0.0)) return bad("delta_t_ms must be > 0 (inf allowed)");
  const double fin[] = {p.est_alpha_cached_ms, p.est_alpha_miss_ms, p.mu, p.theta0[0], p.theta0[1],
                        p.theta0[2], p.theta0[3], p.tau, p.w_hit, p.w_load,
                        p.ca_balance_abs, p.ca_balance_rel, p.ca_cache_threshold};
  for (double v : fin)
    if (!std::isfinite(v)) return bad("parameters must be finite");
  if (p.router == KVR_ROUTE_LBGR && !(p.mu >= 0.0 && p.mu < 2.0))
    return bad("LBGR NLMS step mu must be in [0, 2) (reading A8)");
  return kvr::policy_valid(p) ? true : bad("invalid policy");
}

int num_sms() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
  return n;
}

int smem_optin() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) return 0;
  return n;
}

struct Plan {
  uint32_t tier, ktier;   // tier reported (1 shared, 2 global); kernel tier (3 = global, u16 ids)
  size_t smem;
  int ctas_per_sm;
  uint32_t grid;
  kvr::WorkerLayout lay;
  kvr::AuxLayout aux;
  kvr::FifoLayout fifo;
  kvr::BatchLayout blay;
  size_t ws_aux, ws_fifo, ws_lag, ws_div, ws_state, ws_total;
};

// continuous batching (kvr_batch.cu): per-worker state in shared memory when W
// of them fit next to the control block (tier 1), else in the workspace (tier 2)
kvr_status make_batch_plan(const kvr_sim* sim, uint32_t max_n, uint32_t n_trials, int optin,
                           Plan* pl) {
  const kvr_sim_config& c = sim->cfg;
  const uint32_t mx = std::max<uint32_t>(max_n, 1);
  const kvr::BatchLayout l16 = kvr::make_batch_layout(c.capacity_blocks, c.batch_slots, mx, 2);
  const kvr::BatchLayout l32 = kvr::make_batch_layout(c.capacity_blocks, c.batch_slots, mx, 4);
  const size_t ctrl = kvr::batch_ctrl_bytes();
  const size_t smem1 = ctrl + (size_t)c.W * l16.bytes;
  const bool fit1 = c.capacity_blocks <= 65535 && smem1 <= (size_t)optin;   // 0xFFFF = NONE
  const uint32_t tier = c.force_tier ? c.force_tier : (fit1 ? 1u : 2u);
  if (tier == 3) return fail(KVR_ERR_UNSUPPORTED, "batching: no split tier (force_tier 0..2)");
  if (tier == 1 && !fit1)
    return fail(KVR_ERR_UNSUPPORTED, "batching: shared-memory tier needs %zu B > %d B", smem1, optin);
  pl->tier = tier;
  pl->ktier = tier;
  pl->blay = tier == 1 ? l16 : l32;
  pl->smem = tier == 1 ? smem1 : ctrl;
  cudaError_t e = kvr::batch_attrs(pl->smem, &pl->ctas_per_sm, c.W, tier == 2, c.capacity_blocks);
  if (e != cudaSuccess) return cuda_fail(e, "occupancy query (batching kernel)");
  if (pl->ctas_per_sm < 1) return fail(KVR_ERR_UNSUPPORTED, "batching kernel cannot be resident");
  const uint64_t slots = (uint64_t)pl->ctas_per_sm * (uint64_t)num_sms();
  pl->grid = (uint32_t)std::min<uint64_t>(std::max<uint32_t>(n_trials, 1), slots);
  pl->ws_aux = kvr::align16((size_t)pl->grid * c.W * c.pending_ring * sizeof(kvr::BFlight));
  // + the Leaf-LRU recency logs (after the FIFO rings)
  pl->ws_aux += kvr::align16((size_t)pl->grid * c.W * kvr::batch_log_cap(c.capacity_blocks, mx) * 8);
  pl->ws_fifo = 0;
  pl->ws_lag = 0;
  pl->ws_div = 0;
  pl->ws_state = tier == 2 ? (size_t)pl->grid * c.W * pl->blay.bytes : 0;
  pl->ws_total = 256 + pl->ws_aux + pl->ws_state;
  return KVR_OK;
}

kvr_status make_plan(const kvr_sim* sim, uint32_t max_n, uint32_t max_N, uint32_t n_trials, Plan* pl) {
  const kvr_sim_config& c = sim->cfg;
  const int optin = smem_optin();
  if (optin <= 0) return fail(KVR_ERR_CUDA, "no CUDA device available");
  if (c.batch_slots > 0) return make_batch_plan(sim, max_n, n_trials, optin, pl);
  const size_t base = kvr::smem_base_bytes(c.W, max_n);
  const kvr::WorkerLayout l16 = kvr::make_layout(c.capacity_blocks, 2);
  const kvr::WorkerLayout l32 = kvr::make_layout(c.capacity_blocks, 4);
  const kvr::WorkerLayout lsp = kvr::make_layout(c.capacity_blocks, 2, true);
  // W > 16 runs two workers per warp, whose idle one's scalars wait in a save area
  const size_t wsv = c.W > 16 ? sizeof(kvr::WSave) : 0;
  const size_t smem1 = base + (size_t)c.W * (l16.bytes + wsv);
  const size_t smem3 = base + (size_t)c.W * (lsp.sbytes + sizeof(kvr::WSave));
  const bool fit1 = c.capacity_blocks <= 65533 && smem1 <= (size_t)optin;   // 0xFFFE/F = tomb/empty
  // split tier (identities + tables global, tree arrays / bitmaps / stamps shared): W > 16
  const bool fit3 = c.W >= 2 && c.capacity_blocks <= 65533 && smem3 <= (size_t)optin;
  uint32_t tier = c.force_tier ? c.force_tier : (fit1 ? 1u : ((fit3 && c.W > 16) ? 3u : 2u));
  if (tier == 1 && !fit1)
    return fail(KVR_ERR_UNSUPPORTED, "shared-memory tier needs %zu B > %d B (W=%u, B=%u)", smem1,
                optin, c.W, c.capacity_blocks);
  if (tier == 3 && !fit3)
    return fail(KVR_ERR_UNSUPPORTED, "split tier needs W >= 2 and %zu B <= %d B of shared memory",
                smem3, optin);
  if (tier == 2 && base > (size_t)optin)
    return fail(KVR_ERR_UNSUPPORTED, "query staging needs %zu B of shared memory", base);
  pl->tier = tier;
  // kernel tier: 1 shared, 2 global (u32 ids), 3 global with u16 ids (W > 16: halves the
  // L1/L2 footprint of the tables), 4 split
  pl->ktier = tier == 3 ? 4u : ((tier == 2 && c.W > 16 && c.capacity_blocks <= 65533) ? 3u : tier);
  pl->lay = tier == 3 ? lsp : ((tier == 1 || pl->ktier == 3) ? l16 : l32);
  pl->smem = tier == 1 ? smem1 : (tier == 3 ? smem3 : base);
  cudaError_t e = kvr::replay_attrs(pl->ktier, pl->smem, &pl->ctas_per_sm, c.W, sim_extended(c));
  if (e != cudaSuccess) return cuda_fail(e, "occupancy query");
  if (pl->ctas_per_sm < 1) return fail(KVR_ERR_UNSUPPORTED, "replay kernel cannot be resident");
  // experiment knob (scripts only): cap the resident trials per SM
  if (const char* cap = getenv("KVR_MAX_CTAS_PER_SM"))
    if (atoi(cap) > 0) pl->ctas_per_sm = std::min(pl->ctas_per_sm, atoi(cap));
  const uint64_t slots = (uint64_t)pl->ctas_per_sm * (uint64_t)num_sms();
  pl->grid = (uint32_t)std::min<uint64_t>(std::max<uint32_t>(n_trials, 1), slots);
  const bool ext = sim_extended(c);
  pl->aux = kvr::make_aux(c.capacity_blocks, max_n, pl->lay.T, ext);
  pl->ws_aux = (size_t)pl->grid * c.W * pl->aux.bytes;
  pl->fifo = kvr::make_fifo(c.W, c.pending_ring, max_N);
  pl->ws_fifo = (size_t)pl->grid * pl->fifo.bytes;
  pl->ws_lag = ext ? (size_t)pl->grid * kvr::kLagRing * kvr::lag_entry_bytes(max_n) : 0;
  pl->ws_div = kvr::align16((size_t)pl->grid * 8 * ((size_t)max_n + 1));
  pl->ws_state = tier >= 2 ? (size_t)pl->grid * c.W * pl->lay.gbytes : 0;
  pl->ws_total = 256 + pl->ws_aux + pl->ws_fifo + pl->ws_lag + pl->ws_div + pl->ws_state;
  return KVR_OK;
}

}  // namespace

extern "C" {

const char* kvr_last_error(void) { return g_err.c_str(); }

#ifndef KVR_BUILD_ID
#define KVR_BUILD_ID "unknown"
#endif
// the marker makes the id readable from the file without loading it (build.py)
static const char kBuildIdMarked[] = "KVR_BUILD_ID=" KVR_BUILD_ID;
const char* kvr_build_id(void) { return kBuildIdMarked + 13; }
uint32_t kvr_abi_version(void) { return KVR_ABI_VERSION; }

kvr_status kvr_trace_packed_bytes(const kvr_trace_desc* d, size_t* packed, size_t* scratch) {
  if (!d || !packed || !scratch) return fail(KVR_ERR_INVALID_ARG, "null argument");
  *packed = kvr::packed_bytes(d->n_queries, d->n_blocks_total);
  *scratch = 256;
  return KVR_OK;
}

kvr_status kvr_trace_load(const kvr_trace_desc* d, void* d_packed, size_t packed_bytes,
                          void* d_scratch, size_t scratch_bytes, void* stream, kvr_trace** out) {
  if (!d || !out) return fail(KVR_ERR_INVALID_ARG, "null argument");
  *out = nullptr;
  if (d->block_tokens == 0) return fail(KVR_ERR_INVALID_ARG, "block_tokens must be >= 1");
  if (!d_packed || !d_scratch) return fail(KVR_ERR_INVALID_ARG, "null packed/scratch buffer");
  if (((uintptr_t)d_packed & 15) != 0) return fail(KVR_ERR_INVALID_ARG, "d_packed must be 16-B aligned");
  if (packed_bytes < kvr::packed_bytes(d->n_queries, d->n_blocks_total))
    return fail(KVR_ERR_WORKSPACE_TOO_SMALL, "packed buffer too small");
  if (scratch_bytes < 16) return fail(KVR_ERR_WORKSPACE_TOO_SMALL, "scratch too small");
  if (d->n_queries && (!d->arrival_ms || !d->n_in_blocks || !d->n_out_blocks || !d->out_tokens ||
                       !d->block_offsets || (d->n_blocks_total && !d->block_keys)))
    return fail(KVR_ERR_INVALID_ARG, "null trace array");
  cudaStream_t s = (cudaStream_t)stream;
  kvr::QueryHdr* hdr = (kvr::QueryHdr*)d_packed;
  uint64_t* hash = (uint64_t*)((uint8_t*)d_packed + kvr::packed_hash_offset(d->n_queries));
  cudaError_t e = kvr::launch_pack(*d, hdr, hash, (uint32_t*)d_scratch, s);
  if (e != cudaSuccess) return cuda_fail(e, "pack kernel");
  uint32_t h_scr[4] = {0, 0, 0, 0};
  e = cudaMemcpyAsync(h_scr, d_scratch, 16, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "trace validation readback");
  if (h_scr[0]) {
    return fail(KVR_ERR_INVALID_ARG, "malformed trace (flags 0x%x:%s%s%s)", h_scr[0],
                (h_scr[0] & 1) ? " n_in<1 or offsets/length mismatch" : "",
                (h_scr[0] & 2) ? " arrivals not finite/nonnegative/nondecreasing" : "",
                (h_scr[0] & 4) ? " block_offsets[0]!=0 or [N]!=n_blocks_total" : "");
  }
  kvr_trace* t = new kvr_trace;
  t->N = d->n_queries;
  t->block_tokens = d->block_tokens;
  t->max_n = h_scr[1];
  t->total = d->n_blocks_total;
  t->salt = d->hash_salt;
  t->hdr = hdr;
  t->hash = hash;
  *out = t;
  return KVR_OK;
}

kvr_status kvr_trace_info(const kvr_trace* tr, uint32_t* n_queries, uint32_t* max_path_blocks,
                          uint64_t* n_blocks_total) {
  if (!tr) return fail(KVR_ERR_INVALID_ARG, "null trace");
  if (n_queries) *n_queries = tr->N;
  if (max_path_blocks) *max_path_blocks = tr->max_n;
  if (n_blocks_total) *n_blocks_total = tr->total;
  return KVR_OK;
}

kvr_status kvr_trace_chained_hashes(const kvr_trace* tr, const uint64_t** d_hashes) {
  if (!tr || !d_hashes) return fail(KVR_ERR_INVALID_ARG, "null argument");
  *d_hashes = tr->hash;
  return KVR_OK;
}

kvr_status kvr_trace_next_use_bytes(const kvr_trace* tr, size_t* nu_bytes, size_t* scratch_bytes) {
  if (!tr || !nu_bytes || !scratch_bytes) return fail(KVR_ERR_INVALID_ARG, "null argument");
  if (tr->total >= 0x7fffffffull) return fail(KVR_ERR_UNSUPPORTED, "next-use index needs < 2^31 blocks");
  *nu_bytes = (size_t)tr->total * 4;
  cudaError_t e = kvr::next_use_scratch_bytes(tr->total, scratch_bytes);
  if (e != cudaSuccess) return cuda_fail(e, "next-use scratch size");
  return KVR_OK;
}

kvr_status kvr_trace_build_next_use(const kvr_trace* tr, uint32_t* d_nu, size_t nu_bytes,
                                    void* d_scratch, size_t scratch_bytes, void* stream,
                                    kvr_trace** out) {
  if (!tr || !out) return fail(KVR_ERR_INVALID_ARG, "null argument");
  *out = nullptr;
  size_t need_nu = 0, need_scr = 0;
  kvr_status st = kvr_trace_next_use_bytes(tr, &need_nu, &need_scr);
  if (st) return st;
  if (tr->total && (!d_nu || !d_scratch)) return fail(KVR_ERR_INVALID_ARG, "null next-use/scratch buffer");
  if (nu_bytes < need_nu || scratch_bytes < need_scr)
    return fail(KVR_ERR_WORKSPACE_TOO_SMALL, "next-use buffers too small (%zu/%zu < %zu/%zu)",
                nu_bytes, scratch_bytes, need_nu, need_scr);
  cudaError_t e = kvr::build_next_use(tr->hdr, tr->N, tr->hash, tr->total, d_nu, d_scratch,
                                      scratch_bytes, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "next-use index");
  kvr_trace* t = new kvr_trace(*tr);
  t->nu = d_nu;
  *out = t;
  return KVR_OK;
}

kvr_status kvr_trace_phase_bytes(const kvr_trace* tr, size_t* phase_bytes, size_t* scratch_bytes) {
  if (!tr || !phase_bytes || !scratch_bytes) return fail(KVR_ERR_INVALID_ARG, "null argument");
  if (tr->total >= 0x7fffffffull) return fail(KVR_ERR_UNSUPPORTED, "phase index needs < 2^31 blocks");
  *phase_bytes = (size_t)tr->total * 12 + 16;   // ph, nx, distinct (<= one phase per access)
  cudaError_t e = kvr::phase_scratch_bytes(tr->total, scratch_bytes);
  if (e != cudaSuccess) return cuda_fail(e, "phase scratch size");
  return KVR_OK;
}

kvr_status kvr_trace_build_phases(const kvr_trace* tr, uint32_t B, uint32_t* d_phase,
                                  size_t phase_bytes, void* d_scratch, size_t scratch_bytes,
                                  void* stream, uint32_t* n_phases, kvr_trace** out) {
  if (!tr || !out || !n_phases) return fail(KVR_ERR_INVALID_ARG, "null argument");
  *out = nullptr;
  *n_phases = 0;
  if (B == 0) return fail(KVR_ERR_INVALID_ARG, "B must be >= 1");
  size_t need_ph = 0, need_scr = 0;
  kvr_status st = kvr_trace_phase_bytes(tr, &need_ph, &need_scr);
  if (st) return st;
  if (tr->total && (!d_phase || !d_scratch)) return fail(KVR_ERR_INVALID_ARG, "null phase/scratch buffer");
  if (phase_bytes < need_ph || scratch_bytes < need_scr)
    return fail(KVR_ERR_WORKSPACE_TOO_SMALL, "phase buffers too small (%zu/%zu < %zu/%zu)", phase_bytes,
                scratch_bytes, need_ph, need_scr);
  cudaError_t e = kvr::build_phases(tr->hash, tr->total, B, d_phase, d_scratch, scratch_bytes,
                                    (cudaStream_t)stream, n_phases);
  if (e != cudaSuccess) return cuda_fail(e, "phase index");
  kvr_trace* t = new kvr_trace(*tr);
  t->ph = d_phase;
  t->n_phases = *n_phases;
  t->phase_B = B;
  *out = t;
  return KVR_OK;
}

kvr_status kvr_trace_collision_bytes(const kvr_trace* tr, size_t* scratch_bytes) {
  if (!tr || !scratch_bytes) return fail(KVR_ERR_INVALID_ARG, "null argument");
  if (tr->total >= 0x7fffffffull) return fail(KVR_ERR_UNSUPPORTED, "collision check needs < 2^31 blocks");
  cudaError_t e = kvr::collision_scratch_bytes(tr->total, scratch_bytes);
  if (e != cudaSuccess) return cuda_fail(e, "collision scratch size");
  return KVR_OK;
}

kvr_status kvr_trace_check_collisions(const kvr_trace* tr, const uint64_t* d_block_keys,
                                      void* d_scratch, size_t scratch_bytes, void* stream,
                                      uint64_t* n_collisions) {
  if (!tr || !n_collisions) return fail(KVR_ERR_INVALID_ARG, "null argument");
  *n_collisions = 0;
  size_t need = 0;
  kvr_status st = kvr_trace_collision_bytes(tr, &need);
  if (st) return st;
  if (tr->total && (!d_block_keys || !d_scratch))
    return fail(KVR_ERR_INVALID_ARG, "null block keys / scratch");
  if (scratch_bytes < need)
    return fail(KVR_ERR_WORKSPACE_TOO_SMALL, "collision scratch %zu < %zu bytes", scratch_bytes, need);
  unsigned long long c = 0;
  cudaError_t e = kvr::count_collisions(tr->hdr, tr->N, tr->hash, d_block_keys, tr->total, d_scratch,
                                        scratch_bytes, (cudaStream_t)stream, &c);
  if (e != cudaSuccess) return cuda_fail(e, "collision check");
  *n_collisions = c;
  if (c) return fail(KVR_ERR_HASH_COLLISION, "%llu colliding identity pairs: reload with another hash_salt", c);
  return KVR_OK;
}

kvr_status kvr_trace_destroy(kvr_trace* tr) {
  delete tr;
  return KVR_OK;
}

kvr_status kvr_sim_create(const kvr_sim_config* cfg, kvr_sim** out) {
  if (!cfg || !out) return fail(KVR_ERR_INVALID_ARG, "null argument");
  *out = nullptr;
  if (cfg->W < 1 || cfg->W > kvr::kMaxW) return fail(KVR_ERR_UNSUPPORTED, "W must be in 1..32");
  if (cfg->capacity_blocks < 1 || cfg->capacity_blocks > 65536)
    return fail(KVR_ERR_UNSUPPORTED, "capacity_blocks must be in 1..65536");
  if (cfg->pending_ring < 1) return fail(KVR_ERR_INVALID_ARG, "pending_ring must be >= 1");
  if (cfg->latency_hist_bins > kvr::kMaxHistBins)
    return fail(KVR_ERR_INVALID_ARG, "latency_hist_bins must be <= 256");
  if (cfg->force_tier > 3) return fail(KVR_ERR_INVALID_ARG, "force_tier must be 0, 1, 2 or 3");
  if (cfg->extended_policies > 1) return fail(KVR_ERR_INVALID_ARG, "extended_policies must be 0 or 1");
  const kvr_service_model& t = cfg->truth;
  if (!std::isfinite(t.alpha_cached_ms) || !std::isfinite(t.alpha_miss_ms) ||
      !std::isfinite(t.out_ms_per_token))
    return fail(KVR_ERR_INVALID_ARG, "service model must be finite");
  std::string why;
  if (!policy_ok(cfg->default_policy, &why)) return fail(KVR_ERR_INVALID_ARG, "%s", why.c_str());
  if (cfg->default_policy.eviction == KVR_EVICT_OPT && cfg->W != 1)
    return fail(KVR_ERR_INVALID_ARG, "policy: OPT (offline Belady) is defined for W = 1");
  if (cfg->batch_slots > 64) return fail(KVR_ERR_INVALID_ARG, "batch_slots must be in 0..64");
  if (cfg->batch_slots > 0 &&
      (cfg->default_policy.eviction == KVR_EVICT_OPT || cfg->default_policy.tracker_lag != 0 ||
       cfg->default_policy.tracker_grain != 1))
    return fail(KVR_ERR_INVALID_ARG,
                "policy: the batching engine (batch_slots > 0) carries neither OPT nor tracker bias (A36)");
  kvr_sim* s = new kvr_sim;
  s->cfg = *cfg;
  *out = s;
  return KVR_OK;
}

kvr_status kvr_sim_destroy(kvr_sim* sim) {
  delete sim;
  return KVR_OK;
}

kvr_status kvr_sim_plan(const kvr_sim* sim, uint32_t max_path_blocks, uint32_t* tier,
                        size_t* smem_bytes, uint32_t* ctas_per_sm) {
  if (!sim) return fail(KVR_ERR_INVALID_ARG, "null sim");
  Plan pl;
  kvr_status st = make_plan(sim, max_path_blocks, 0, 1u << 30, &pl);
  if (st) return st;
  if (tier) *tier = pl.tier;
  if (smem_bytes) *smem_bytes = pl.smem;
  if (ctas_per_sm) *ctas_per_sm = (uint32_t)pl.ctas_per_sm;
  return KVR_OK;
}

kvr_status kvr_sim_workspace_bytes_multi(const kvr_sim* sim, uint32_t n_traces,
                                         const kvr_trace* const* traces, uint32_t n_trials,
                                         size_t* bytes) {
  if (!sim || !traces || !bytes || n_traces == 0) return fail(KVR_ERR_INVALID_ARG, "null argument");
  uint32_t max_n = 1, max_N = 0;
  for (uint32_t i = 0; i < n_traces; ++i) {
    if (!traces[i]) return fail(KVR_ERR_INVALID_ARG, "null trace %u", i);
    max_n = std::max(max_n, traces[i]->max_n);
    max_N = std::max(max_N, traces[i]->N);
  }
  Plan pl;
  kvr_status st = make_plan(sim, max_n, max_N, n_trials, &pl);
  if (st) return st;
  *bytes = pl.ws_total;
  return KVR_OK;
}

kvr_status kvr_sim_workspace_bytes(const kvr_sim* sim, const kvr_trace* trace, uint32_t n_trials,
                                   size_t* bytes) {
  return kvr_sim_workspace_bytes_multi(sim, 1, &trace, n_trials, bytes);
}

}  // extern "C"

namespace {
kvr_status run_impl(kvr_sim* sim, uint32_t n_traces, const kvr_trace* const* traces,
                    const uint32_t* d_trial_trace, uint32_t n_trials, const uint64_t* d_keys,
                    const kvr_policy* d_policies, kvr_trial_result* d_results, uint32_t* d_hist,
                    kvr_query_record* d_records, uint64_t* d_victims, uint64_t victims_cap,
                    void* d_ws, size_t ws_bytes, void* stream, uint32_t* d_ledger) {
  if (!sim || !traces) return fail(KVR_ERR_INVALID_ARG, "null argument");
  if (n_traces == 0 || n_traces > kvr::kMaxTraces)
    return fail(KVR_ERR_UNSUPPORTED, "n_traces must be in 1..%u", kvr::kMaxTraces);
  if (n_traces > 1 && !d_trial_trace) return fail(KVR_ERR_INVALID_ARG, "d_trial_trace required");
  if (n_trials == 0) return KVR_OK;
  if (!d_keys || !d_results || !d_ws) return fail(KVR_ERR_INVALID_ARG, "null keys/results/workspace");
  const kvr_sim_config& c = sim->cfg;
  uint32_t max_n = 1, max_N = 0;
  for (uint32_t i = 0; i < n_traces; ++i) {
    const kvr_trace* t = traces[i];
    if (!t) return fail(KVR_ERR_INVALID_ARG, "null trace %u", i);
    const uint64_t beta = c.batch_slots > 0 ? c.batch_slots : 1;
    if (beta * t->max_n > c.capacity_blocks)
      return fail(KVR_ERR_CAPACITY,
                  "trace %u: beta*L_max = %u*%u blocks > capacity B=%u (premise beta*L_max<=B, P:197)",
                  i, (uint32_t)beta, t->max_n, c.capacity_blocks);
    // the replay kernel keeps per-worker insert/eviction/draw counts in u32 registers: a
    // worker's count is at most the trace's total blocks
    if (t->total >= 0xffffffffull)
      return fail(KVR_ERR_UNSUPPORTED, "trace %u has %llu blocks; at most 2^32 - 1 per trace", i,
                  (unsigned long long)t->total);
    max_n = std::max(max_n, t->max_n);
    max_N = std::max(max_N, t->N);
    if (!d_policies && c.default_policy.eviction == KVR_EVICT_OPT && !t->nu && t->total)
      return fail(KVR_ERR_INVALID_ARG, "OPT needs a next-use index (kvr_trace_build_next_use) on trace %u", i);
  }
  const uint32_t R = d_ledger ? 0u : std::min(c.record_trials, n_trials);   // ledger runs record nothing
  if (R && !d_records) return fail(KVR_ERR_INVALID_ARG, "record_trials > 0 needs d_records");
  Plan pl;
  kvr_status st = make_plan(sim, max_n, max_N, n_trials, &pl);
  if (st) return st;
  if (ws_bytes < pl.ws_total)
    return fail(KVR_ERR_WORKSPACE_TOO_SMALL, "workspace %zu < %zu bytes", ws_bytes, pl.ws_total);

  kvr::ReplayParams p;
  std::memset(&p, 0, sizeof(p));
  for (uint32_t i = 0; i < n_traces; ++i) {
    p.traces[i].hdr = traces[i]->hdr;
    p.traces[i].hash = traces[i]->hash;
    p.traces[i].nu = traces[i]->nu;
    p.traces[i].N = traces[i]->N;
    p.traces[i].max_n = traces[i]->max_n;
    p.traces[i].block_tokens = traces[i]->block_tokens;
    if (traces[i]->ph) {
      p.traces[i].ph = traces[i]->ph;
      p.traces[i].nx = traces[i]->ph + traces[i]->total;
      p.traces[i].distinct = traces[i]->ph + 2 * traces[i]->total;
      p.traces[i].n_phases = traces[i]->n_phases;
    }
  }
  p.trial_trace = n_traces > 1 ? d_trial_trace : nullptr;
  p.n_traces = n_traces;
  p.n_trials = n_trials;
  p.W = c.W;
  p.B = c.capacity_blocks;
  p.ring = c.pending_ring;
  p.record_trials = R;
  p.rec_stride = max_N;
  p.bins = d_hist ? c.latency_hist_bins : 0;
  p.stage_bytes = (uint32_t)kvr::stage_bytes(max_n);
  p.scratch_bytes = (uint32_t)kvr::scratch_bytes(max_n);
  p.slotbuf_bytes = (uint32_t)kvr::slotbuf_bytes(max_n);
  p.max_n = max_n;
  p.aux = pl.aux;
  p.fifo = pl.fifo;
  p.lay = pl.lay;
  p.truth = c.truth;
  p.defpol = c.default_policy;
  p.policies = d_policies;
  p.keys = d_keys;
  p.results = d_results;
  p.hist = p.bins ? d_hist : nullptr;
  p.records = R ? d_records : nullptr;
  p.victims = (R && d_victims && victims_cap) ? d_victims : nullptr;
  p.victims_per_trial = p.victims ? victims_cap / R : 0;
  uint8_t* ws = (uint8_t*)d_ws;
  p.work_counter = (unsigned int*)ws;
  p.aux_base = ws + 256;
  p.fifo_base = ws + 256 + pl.ws_aux;
  p.lag_base = pl.ws_lag ? ws + 256 + pl.ws_aux + pl.ws_fifo : nullptr;
  p.lag_entry = (uint32_t)kvr::lag_entry_bytes(max_n);
  p.divtab_base = reinterpret_cast<double*>(ws + 256 + pl.ws_aux + pl.ws_fifo + pl.ws_lag);
  p.gstate = pl.tier >= 2 ? ws + 256 + pl.ws_aux + pl.ws_fifo + pl.ws_lag + pl.ws_div : nullptr;
  if (d_ledger) {
    p.ledger = d_ledger;
    p.ledger_stride = 4 * traces[0]->n_phases;
  }

  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(ws, 0, 256, s);
  if (e != cudaSuccess) return cuda_fail(e, "workspace reset");
  if (c.batch_slots > 0) {
    p.beta = c.batch_slots;
    p.blay = pl.blay;
    p.bglobal = pl.tier == 2 ? 1u : 0u;
    p.blog_cap = kvr::batch_log_cap(c.capacity_blocks, std::max<uint32_t>(max_n, 1));
    p.blog_base = reinterpret_cast<uint64_t*>(
        ws + 256 + kvr::align16((size_t)pl.grid * c.W * c.pending_ring * sizeof(kvr::BFlight)));
    p.gstate = pl.tier == 2 ? ws + 256 + pl.ws_aux : nullptr;
    e = kvr::launch_batch(p, pl.grid, pl.smem, s);
    if (e != cudaSuccess) return cuda_fail(e, "batching replay launch");
    return KVR_OK;
  }
  e = kvr::launch_replay(pl.ktier, p, pl.grid, pl.smem, s, sim_extended(c));
  if (e != cudaSuccess) return cuda_fail(e, "replay launch");
  return KVR_OK;
}
}  // namespace

extern "C" {

kvr_status kvr_sim_run_multi(kvr_sim* sim, uint32_t n_traces, const kvr_trace* const* traces,
                             const uint32_t* d_trial_trace, uint32_t n_trials,
                             const uint64_t* d_keys, const kvr_policy* d_policies,
                             kvr_trial_result* d_results, uint32_t* d_hist,
                             kvr_query_record* d_records, uint64_t* d_victims, uint64_t victims_cap,
                             void* d_ws, size_t ws_bytes, void* stream) {
  return run_impl(sim, n_traces, traces, d_trial_trace, n_trials, d_keys, d_policies, d_results,
                  d_hist, d_records, d_victims, victims_cap, d_ws, ws_bytes, stream, nullptr);
}

kvr_status kvr_sim_run_ledger(kvr_sim* sim, const kvr_trace* trace, uint32_t n_trials,
                              const uint64_t* d_keys, const kvr_policy* d_policies,
                              kvr_trial_result* d_results, uint32_t* d_ledger, void* d_ws,
                              size_t ws_bytes, void* stream) {
  if (!sim || !trace) return fail(KVR_ERR_INVALID_ARG, "null argument");
  if (sim->cfg.W != 1) return fail(KVR_ERR_INVALID_ARG, "phase ledger: W must be 1 (single-cache analysis)");
  if (sim->cfg.batch_slots) return fail(KVR_ERR_INVALID_ARG, "phase ledger: beta = 1 model only");
  if (!sim_extended(sim->cfg))
    return fail(KVR_ERR_INVALID_ARG, "phase ledger: create the sim with extended_policies = 1");
  if (!trace->ph) return fail(KVR_ERR_INVALID_ARG, "phase ledger: trace has no phase index");
  if (trace->phase_B != sim->cfg.capacity_blocks)
    return fail(KVR_ERR_INVALID_ARG, "phase ledger: phases built for B=%u, sim has B=%u", trace->phase_B,
                sim->cfg.capacity_blocks);
  if (n_trials && trace->n_phases && !d_ledger) return fail(KVR_ERR_INVALID_ARG, "null ledger");
  return run_impl(sim, 1, &trace, nullptr, n_trials, d_keys, d_policies, d_results, nullptr,
                  nullptr, nullptr, 0, d_ws, ws_bytes, stream, d_ledger ? d_ledger : nullptr);
}


kvr_status kvr_sim_run(kvr_sim* sim, const kvr_trace* trace, uint32_t n_trials,
                       const uint64_t* d_keys, const kvr_policy* d_policies,
                       kvr_trial_result* d_results, uint32_t* d_hist, kvr_query_record* d_records,
                       uint64_t* d_victims, uint64_t victims_cap, void* d_ws, size_t ws_bytes,
                       void* stream) {
  return kvr_sim_run_multi(sim, 1, &trace, nullptr, n_trials, d_keys, d_policies, d_results, d_hist,
                           d_records, d_victims, victims_cap, d_ws, ws_bytes, stream);
}

/* profiling builds only (not declared in kvr.h): per-phase cycle sums */
kvr_status kvr_debug_phase_cycles(uint64_t* out32, int reset) {
  // reset 3 / 4: the batching kernel's counters (read / read and clear)
  cudaError_t e = (reset == 3 || reset == 4) ? kvr::batch_phase_cycles((unsigned long long*)out32, reset - 3)
                                             : kvr::phase_cycles((unsigned long long*)out32, reset);
  if (e != cudaSuccess) return cuda_fail(e, "phase profile");
  return KVR_OK;
}

}  // extern "C"
