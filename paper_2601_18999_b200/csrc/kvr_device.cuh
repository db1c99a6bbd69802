// kvr_device.cuh — sm_100a device primitives of the replay engine.
// Counter-based RNG, the 64-bit finalizer, bulk-async (TMA 1-D) staging with
// mbarriers, and warp collectives.  Independent of the CPU oracle.
#pragma once
#include <stdint.h>

namespace kvr {

constexpr uint32_t kFull = 0xffffffffu;

// MurmurHash3 fmix64 finalizer (a bijection on u64); block identity chain
// (reading A26) and the decision digest.
__device__ __forceinline__ uint64_t fmix64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return x;
}

constexpr uint64_t kPosMul = 0x9E3779B97F4A7C15ULL;

// Philox4x32-10 (Salmon et al., SC'11), counter (lo n, hi n, stream, tag),
// key (lo K, hi K); returns x0 | x1 << 32.
__device__ __forceinline__ uint64_t philox_r64(uint64_t key, uint64_t n, uint32_t stream,
                                               uint32_t tag) {
  uint32_t c0 = (uint32_t)n, c1 = (uint32_t)(n >> 32), c2 = stream, c3 = tag;
  uint32_t k0 = (uint32_t)key, k1 = (uint32_t)(key >> 32);
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  return (uint64_t)c0 | ((uint64_t)c1 << 32);
}

// uniform index in [0, m) from 64 random bits (reading A6)
__device__ __forceinline__ uint64_t pick_index(uint64_t r, uint64_t m) { return __umul64hi(r, m); }

// position of the rem-th (0-based) set bit of w; w must have > rem set bits
__device__ __forceinline__ uint32_t select_bit(uint32_t w, uint32_t rem) {
  uint32_t pos = 0, c;
  c = __popc(w & 0xffffu); if (rem >= c) { rem -= c; w >>= 16; pos += 16; }
  c = __popc(w & 0xffu);   if (rem >= c) { rem -= c; w >>= 8;  pos += 8; }
  c = __popc(w & 0xfu);    if (rem >= c) { rem -= c; w >>= 4;  pos += 4; }
  c = __popc(w & 0x3u);    if (rem >= c) { rem -= c; w >>= 2;  pos += 2; }
  c = w & 1u;              if (rem >= c) { pos += 1; }
  return pos;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// one-dimensional bulk copy global -> shared (TMA engine), completes on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "KVR_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra KVR_WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// XOR of a u64 over the warp: two uniform-datapath reductions (REDUX.XOR) instead of a
// ten-shuffle butterfly
__device__ __forceinline__ uint64_t warp_xor64(uint64_t v) {
  const uint32_t lo = __reduce_xor_sync(kFull, (uint32_t)v), hi = __reduce_xor_sync(kFull, (uint32_t)(v >> 32));
  return ((uint64_t)hi << 32) | lo;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

}  // namespace kvr
