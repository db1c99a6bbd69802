// kvr_pack.cu — trace packer: validates a raw block-hashed
// trace and writes, per query, a 32-byte header plus the chained block
// identities H_{j,d} (reading A26):
//   S_{j,d} = sum_{e<=d} fmix64(c_{j,e} ^ (e+1)*K ^ salt)  (mod 2^64),  H = fmix64(S).
// The chain is an associative prefix sum, so one warp per query computes it
// 32 blocks at a time with a shuffle scan; loads/stores are coalesced 8-byte
// accesses.  HBM-bound: reads 8 B key + writes 8 B identity per block.
#include <math.h>

#include "kvr_device.cuh"
#include "kvr_internal.h"

namespace kvr {

enum : uint32_t { kErrLen = 1u, kErrArrival = 2u, kErrOffsets = 4u };

__global__ void __launch_bounds__(256) pack_kernel(kvr_trace_desc d, QueryHdr* __restrict__ hdr,
                                                   uint64_t* __restrict__ hash,
                                                   uint32_t* __restrict__ scratch) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
  uint32_t err = 0, maxn = 0;
  for (uint32_t j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < d.n_queries; j += warps) {
    const uint64_t o0 = d.block_offsets[j], o1 = d.block_offsets[j + 1];
    const uint32_t n_in = d.n_in_blocks[j], n_out = d.n_out_blocks[j];
    const uint64_t n = o1 - o0;
    if (lane == 0) {
      const double a = d.arrival_ms[j];
      if (n_in < 1 || o1 < o0 || n != (uint64_t)n_in + n_out || n > 0xffffffffull) err |= kErrLen;
      if (!isfinite(a) || a < 0.0 || (j > 0 && a < d.arrival_ms[j - 1])) err |= kErrArrival;
      if (j == 0 && o0 != 0) err |= kErrOffsets;
      if (j + 1 == d.n_queries && o1 != d.n_blocks_total) err |= kErrOffsets;
      if (o1 > d.n_blocks_total) err |= kErrOffsets;
      QueryHdr h;
      h.arrival_ms = a;
      h.block_off = o0;
      h.n_in = n_in;
      h.n_out = n_out;
      h.out_tokens = d.out_tokens[j];
      h._pad = 0;
      hdr[j] = h;
      maxn = max(maxn, n > 0xffffffffull ? 0xffffffffu : (uint32_t)n);
    }
    if (o1 < o0 || o1 > d.n_blocks_total) continue;
    uint64_t carry = 0;
    for (uint64_t base = 0; base < n; base += 32) {
      const uint64_t dd = base + lane;
      uint64_t v = 0;
      if (dd < n) v = fmix64(d.block_keys[o0 + dd] ^ ((dd + 1) * kPosMul) ^ d.hash_salt);
#pragma unroll
      for (int s = 1; s < 32; s <<= 1) {
        const uint64_t u = __shfl_up_sync(kFull, v, s);
        if (lane >= (uint32_t)s) v += u;
      }
      v += carry;
      if (dd < n) hash[o0 + dd] = fmix64(v);
      carry = __shfl_sync(kFull, v, 31);
    }
  }
  err = __reduce_or_sync(kFull, err);
  maxn = __reduce_max_sync(kFull, maxn);
  if (lane == 0) {
    if (err) atomicOr(&scratch[0], err);
    if (maxn) atomicMax(&scratch[1], maxn);
  }
}

cudaError_t launch_pack(const kvr_trace_desc& d, QueryHdr* hdr, uint64_t* hash, uint32_t* scratch,
                        cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(scratch, 0, 16, s);
  if (e != cudaSuccess) return e;
  if (d.n_queries == 0) return cudaSuccess;
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const uint32_t warps_needed = d.n_queries;
  uint32_t blocks = (warps_needed + 7) / 8;
  const uint32_t cap = (uint32_t)nsm * 8;   // 8 x 256-thread CTAs per SM, grid-stride beyond
  if (blocks > cap) blocks = cap;
  pack_kernel<<<blocks, 256, 0, s>>>(d, hdr, hash, scratch);
  return cudaGetLastError();
}

}  // namespace kvr
