// kvr_nextuse.cu — next-use index of a packed trace for the offline Belady OPT
// analysis (OPT = evict the leaf whose next use is furthest).
//
// nu[o] for block occurrence o (CSR order of the packed identities) is the index
// of the next query after o's query whose path contains the same identity, or
// 0xFFFFFFFF.  Identities inside one query are distinct (they encode the
// position), so that is the query of the next occurrence of the identity in
// CSR order: a stable radix sort of (identity, occurrence) pairs puts every
// identity's occurrences next to each other in trace order, and one pass over the
// sorted pairs writes the answer.  The sort is CUB's (CUDA toolkit) LSD radix
// sort; this is offline preprocessing, not the replay path.
#include <cub/device/device_radix_sort.cuh>

#include "kvr_internal.h"

namespace kvr {

namespace {

constexpr size_t kAlign = 256;
inline size_t align_up(size_t x) { return (x + kAlign - 1) & ~(kAlign - 1); }

// query index of every occurrence: one warp per query
__global__ void occurrence_query_kernel(const QueryHdr* hdr, uint32_t N, uint32_t* qidx) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t j = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (j >= N) return;
  const uint64_t off = hdr[j].block_off;
  const uint32_t n = hdr[j].n_in + hdr[j].n_out;
  for (uint32_t d = lane; d < n; d += 32) qidx[off + d] = j;
}

__global__ void iota_kernel(uint32_t* v, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    v[i] = (uint32_t)i;
}

// sorted[i] = (identity, occurrence) in (identity, occurrence) order
__global__ void next_use_kernel(const uint64_t* key_sorted, const uint32_t* occ_sorted,
                                const uint32_t* qidx, uint64_t n, uint32_t* nu) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t o = occ_sorted[i];
    uint32_t next = 0xFFFFFFFFu;
    if (i + 1 < n && key_sorted[i + 1] == key_sorted[i]) next = qidx[occ_sorted[i + 1]];
    nu[o] = next;
  }
}

struct ScratchLayout {
  size_t keys_out, occ_in, occ_out, qidx, cub, total;
};

cudaError_t layout(uint64_t n, ScratchLayout* L) {
  size_t cub_bytes = 0;
  cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, cub_bytes, (const uint64_t*)nullptr,
                                                  (uint64_t*)nullptr, (const uint32_t*)nullptr,
                                                  (uint32_t*)nullptr, (int)n);
  if (e != cudaSuccess) return e;
  size_t o = 0;
  L->keys_out = o; o = align_up(o + n * 8);
  L->occ_in = o;   o = align_up(o + n * 4);
  L->occ_out = o;  o = align_up(o + n * 4);
  L->qidx = o;     o = align_up(o + n * 4);
  L->cub = o;      o = align_up(o + cub_bytes);
  L->total = o;
  return cudaSuccess;
}

// Identity collision check: after the (identity, occurrence) sort,
// adjacent occurrences with equal identity must carry the same (depth, parent
// identity, content key) -- the tuple that legitimately determines the identity
// (reading A26).  Counts the adjacent pairs that do not.
__global__ void collision_kernel(const uint64_t* key_sorted, const uint32_t* occ_sorted,
                                 const uint32_t* qidx, const QueryHdr* hdr, const uint64_t* hash,
                                 const uint64_t* block_keys, uint64_t n,
                                 unsigned long long* count) {
  unsigned long long c = 0;
  for (uint64_t i = 1 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (key_sorted[i] != key_sorted[i - 1]) continue;
    const uint32_t a = occ_sorted[i - 1], b = occ_sorted[i];
    const uint64_t da = a - hdr[qidx[a]].block_off, db = b - hdr[qidx[b]].block_off;
    const uint64_t pa = da ? hash[a - 1] : 0, pb = db ? hash[b - 1] : 0;
    if (da != db || pa != pb || block_keys[a] != block_keys[b]) c++;
  }
  if (c) atomicAdd(count, c);
}

// Phase index (reading A39), step 1: the next and previous occurrence of
// every occurrence's identity from the (identity, occurrence) sort.
__global__ void adjacent_occurrence_kernel(const uint64_t* key_sorted, const uint32_t* occ_sorted,
                                           uint64_t n, uint32_t* nx, uint32_t* pv) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t o = occ_sorted[i];
    nx[o] = (i + 1 < n && key_sorted[i + 1] == key_sorted[i]) ? occ_sorted[i + 1] : 0xFFFFFFFFu;
    pv[o] = (i > 0 && key_sorted[i - 1] == key_sorted[i]) ? occ_sorted[i - 1] : 0xFFFFFFFFu;
  }
}

// step 2: the greedy partition, one warp walking the access sequence 32 occurrences at
// a time.  Occurrence o is a first appearance in the phase that starts at s iff its
// identity's previous occurrence lies before s (or does not exist); a phase ends just
// before the first appearance that would be its (B+1)-th.  When a window crosses a
// boundary the lanes after it are re-classified against the new start.
__global__ void phase_partition_kernel(const uint32_t* pv, uint64_t n, uint32_t B, uint32_t* ph,
                                       uint32_t* distinct, uint32_t* n_phases) {
  const uint32_t lane = threadIdx.x;
  uint64_t s = 0;          // start of the current phase
  uint32_t cnt = 0, v = 0;  // distinct identities in it, its index
  for (uint64_t base = 0; base < n; base += 32) {
    const uint64_t o = base + lane;
    const bool valid = o < n;
    const uint32_t prev = valid ? pv[o] : 0u;
    uint32_t cur = 0;   // first lane not yet assigned
    for (;;) {
      const bool isnew = valid && lane >= cur && (prev == 0xFFFFFFFFu || (uint64_t)prev < s);
      const uint32_t bal = __ballot_sync(0xFFFFFFFFu, isnew);
      const uint32_t c = (uint32_t)__popc(bal);
      if (cnt + c <= B) {
        if (valid && lane >= cur) ph[o] = v | (isnew ? 0x80000000u : 0u);
        cnt += c;
        break;
      }
      // the (B - cnt + 1)-th first appearance of this window opens phase v + 1
      uint32_t need = B - cnt, m = bal, L = 0;
      for (uint32_t k = 0; k <= need; ++k) {
        L = (uint32_t)__ffs(m) - 1;
        m &= m - 1;
      }
      if (valid && lane >= cur && lane < L) ph[o] = v | (isnew ? 0x80000000u : 0u);
      if (lane == 0) distinct[v] = B;
      ++v;
      s = base + L;
      cnt = 0;
      cur = L;
    }
  }
  if (lane == 0) {
    if (n) distinct[v] = cnt;
    *n_phases = n ? v + 1 : 0;
  }
}

}  // namespace

cudaError_t build_phases(const uint64_t* hash, uint64_t n, uint32_t B, uint32_t* out, void* scratch,
                         size_t scratch_bytes, cudaStream_t s, uint32_t* h_n_phases) {
  *h_n_phases = 0;
  if (n == 0) return cudaSuccess;
  ScratchLayout L;
  cudaError_t e = layout(n, &L);
  if (e != cudaSuccess) return e;
  if (scratch_bytes < L.total + kAlign) return cudaErrorInvalidValue;
  uint8_t* b = static_cast<uint8_t*>(scratch);
  uint64_t* keys_out = reinterpret_cast<uint64_t*>(b + L.keys_out);
  uint32_t* occ_in = reinterpret_cast<uint32_t*>(b + L.occ_in);
  uint32_t* occ_out = reinterpret_cast<uint32_t*>(b + L.occ_out);
  uint32_t* pv = reinterpret_cast<uint32_t*>(b + L.qidx);
  uint32_t* d_np = reinterpret_cast<uint32_t*>(b + L.total);
  const int threads = 256;
  const int grid = (int)std::min<uint64_t>((n + threads - 1) / threads, 148ull * 16);
  iota_kernel<<<grid, threads, 0, s>>>(occ_in, n);
  size_t cub_bytes = L.total - L.cub;
  e = cub::DeviceRadixSort::SortPairs(b + L.cub, cub_bytes, hash, keys_out, occ_in, occ_out, (int)n,
                                      0, 64, s);
  if (e != cudaSuccess) return e;
  uint32_t* ph = out;
  uint32_t* nx = out + n;
  uint32_t* distinct = out + 2 * n;
  adjacent_occurrence_kernel<<<grid, threads, 0, s>>>(keys_out, occ_out, n, nx, pv);
  phase_partition_kernel<<<1, 32, 0, s>>>(pv, n, B, ph, distinct, d_np);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  e = cudaMemcpyAsync(h_n_phases, d_np, 4, cudaMemcpyDeviceToHost, s);
  if (e != cudaSuccess) return e;
  return cudaStreamSynchronize(s);
}

cudaError_t phase_scratch_bytes(uint64_t n_blocks, size_t* bytes) {
  ScratchLayout L;
  cudaError_t e = layout(n_blocks, &L);
  if (e == cudaSuccess) *bytes = L.total + kAlign;   // + the phase counter
  return e;
}

cudaError_t collision_scratch_bytes(uint64_t n_blocks, size_t* bytes) {
  ScratchLayout L;
  cudaError_t e = layout(n_blocks, &L);
  if (e == cudaSuccess) *bytes = L.total + kAlign;   // + the counter
  return e;
}

cudaError_t count_collisions(const QueryHdr* hdr, uint32_t N, const uint64_t* hash,
                             const uint64_t* block_keys, uint64_t n, void* scratch,
                             size_t scratch_bytes, cudaStream_t s, unsigned long long* h_count) {
  *h_count = 0;
  if (n < 2) return cudaSuccess;
  ScratchLayout L;
  cudaError_t e = layout(n, &L);
  if (e != cudaSuccess) return e;
  if (scratch_bytes < L.total + kAlign) return cudaErrorInvalidValue;
  uint8_t* b = static_cast<uint8_t*>(scratch);
  uint64_t* keys_out = reinterpret_cast<uint64_t*>(b + L.keys_out);
  uint32_t* occ_in = reinterpret_cast<uint32_t*>(b + L.occ_in);
  uint32_t* occ_out = reinterpret_cast<uint32_t*>(b + L.occ_out);
  uint32_t* qidx = reinterpret_cast<uint32_t*>(b + L.qidx);
  unsigned long long* cnt = reinterpret_cast<unsigned long long*>(b + L.total);
  const int threads = 256;
  const int grid = (int)std::min<uint64_t>((n + threads - 1) / threads, 148ull * 16);
  e = cudaMemsetAsync(cnt, 0, 8, s);
  if (e != cudaSuccess) return e;
  occurrence_query_kernel<<<(N + 7) / 8, 256, 0, s>>>(hdr, N, qidx);
  iota_kernel<<<grid, threads, 0, s>>>(occ_in, n);
  size_t cub_bytes = L.total - L.cub;
  e = cub::DeviceRadixSort::SortPairs(b + L.cub, cub_bytes, hash, keys_out, occ_in, occ_out, (int)n,
                                      0, 64, s);
  if (e != cudaSuccess) return e;
  collision_kernel<<<grid, threads, 0, s>>>(keys_out, occ_out, qidx, hdr, hash, block_keys, n, cnt);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  e = cudaMemcpyAsync(h_count, cnt, 8, cudaMemcpyDeviceToHost, s);
  if (e != cudaSuccess) return e;
  return cudaStreamSynchronize(s);
}

cudaError_t next_use_scratch_bytes(uint64_t n_blocks, size_t* bytes) {
  ScratchLayout L;
  cudaError_t e = layout(n_blocks, &L);
  if (e == cudaSuccess) *bytes = L.total;
  return e;
}

cudaError_t build_next_use(const QueryHdr* hdr, uint32_t N, const uint64_t* hash, uint64_t n,
                           uint32_t* nu, void* scratch, size_t scratch_bytes, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  ScratchLayout L;
  cudaError_t e = layout(n, &L);
  if (e != cudaSuccess) return e;
  if (scratch_bytes < L.total) return cudaErrorInvalidValue;
  uint8_t* b = static_cast<uint8_t*>(scratch);
  uint64_t* keys_out = reinterpret_cast<uint64_t*>(b + L.keys_out);
  uint32_t* occ_in = reinterpret_cast<uint32_t*>(b + L.occ_in);
  uint32_t* occ_out = reinterpret_cast<uint32_t*>(b + L.occ_out);
  uint32_t* qidx = reinterpret_cast<uint32_t*>(b + L.qidx);
  const int threads = 256;
  const int grid = (int)std::min<uint64_t>((n + threads - 1) / threads, 148ull * 16);
  occurrence_query_kernel<<<(N + 7) / 8, 256, 0, s>>>(hdr, N, qidx);
  iota_kernel<<<grid, threads, 0, s>>>(occ_in, n);
  size_t cub_bytes = scratch_bytes - L.cub;
  e = cub::DeviceRadixSort::SortPairs(b + L.cub, cub_bytes, hash, keys_out, occ_in, occ_out, (int)n,
                                      0, 64, s);
  if (e != cudaSuccess) return e;
  next_use_kernel<<<grid, threads, 0, s>>>(keys_out, occ_out, qidx, n, nu);
  return cudaGetLastError();
}

}  // namespace kvr
