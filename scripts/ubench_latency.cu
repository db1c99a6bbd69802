// Dependent-chain latency (cycles per op) of the warp-level primitives on the RLT
// eviction chain.  One warp, 4096 dependent ops per measurement.
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/ubl scripts/ubench_latency.cu
#include <cstdio>
#include <cstdint>

#define N 4096
__global__ void k(uint32_t* out, unsigned long long* cyc, uint32_t seed) {
  __shared__ uint32_t sm[1024];
  const uint32_t lane = threadIdx.x;
  for (int i = lane; i < 1024; i += 32) sm[i] = (i * 2654435761u) & 1023u;
  __syncwarp();
  uint32_t x = seed + lane;
  unsigned long long t0, t1;
  int m = 0;
#define MEAS(expr)                               \
  t0 = clock64();                                \
  _Pragma("unroll 16") for (int i = 0; i < N; ++i) { expr; } \
  t1 = clock64();                                \
  if (lane == 0) cyc[m] = t1 - t0;               \
  ++m;
  MEAS(x = __popc(x) + x)                                   // 0 POPC + IADD
  MEAS(x = x * 3u + 1u)                                     // 1 IMAD
  MEAS(x = __umulhi(x, 0x9e3779b9u) + x)                    // 2 IMAD.HI + IADD
  MEAS(x = __clz(x) + x)                                    // 3 FLO + IADD
  MEAS(x = __brev(x) + 1u)                                  // 4 BREV + IADD
  MEAS(x = __ballot_sync(0xffffffffu, x & 1u) + x)          // 5 VOTE + IADD
  MEAS(x = __shfl_sync(0xffffffffu, x, x & 31u) + 1u)       // 6 SHFL.IDX + IADD
  MEAS(x = sm[x & 1023u] + 1u)                              // 7 LDS + IADD
  MEAS(x = __fns(x | 1u, 0, 1) + x)                         // 8 FNS + IADD
  MEAS(x = __reduce_add_sync(0xffffffffu, x) + 1u)          // 9 REDUX.SUM + IADD
  MEAS(x = __popc(__ballot_sync(0xffffffffu, x & 1u)) + x)  // 10 VOTE+POPC+IADD
  MEAS(x = (__ffs(~__ballot_sync(0xffffffffu, x & 1u))) + x) // 11 VOTE+BREV/FLO
  MEAS(x = __reduce_min_sync(0xffffffffu, x) + 1u)          // 12 REDUX.MIN + IADD
  MEAS(x = (x >> 3) ^ x)                                    // 13 SHF + LOP3
  double d = 1.0 + lane * 1e-3;
  MEAS(d = d + 1e-9)                                        // 14 DADD
  MEAS(d = d * 1.0000001)                                   // 15 DMUL
  MEAS(d = __fma_rn(d, 1.0000001, 1e-9))                    // 16 DFMA
  MEAS(d = d / 1.0000001)                                   // 17 DDIV (IEEE)
  MEAS(d = (double)(uint32_t)(d) + 1.5)                     // 18 F2I + I2F + DADD
  MEAS(d = d < 2.0 ? d * 1.0000001 : d * 0.9999999)         // 19 DSETP + DMUL
  MEAS(d = (double)__double_as_longlong(d) * 1e-300)        // 20 I2F.F64 + DMUL
  float f = 1.0f + lane;
  MEAS(f = f * 1.0001f + 1e-7f)                             // 21 FFMA
  out[lane] = x + (uint32_t)d + (uint32_t)f;
}

int main() {
  uint32_t* o;
  unsigned long long* c;
  cudaMalloc(&o, 128);
  cudaMallocManaged(&c, 32 * 8);
  k<<<1, 32>>>(o, c, 7);
  k<<<1, 32>>>(o, c, 7);
  cudaDeviceSynchronize();
  const char* names[] = {"POPC+IADD", "IMAD", "IMAD.HI+IADD", "CLZ(FLO)+IADD", "BREV+IADD",
                         "VOTE+IADD", "SHFL.IDX+IADD", "LDS+IADD", "FNS+IADD", "REDUX.SUM+IADD",
                         "VOTE+POPC+IADD", "VOTE+FFS+IADD", "REDUX.MIN+IADD", "SHF+LOP3",
                         "DADD", "DMUL", "DFMA", "DDIV", "F2I+I2F+DADD", "DSETP+DMUL", "I2F64+DMUL",
                         "FFMA"};
  for (int i = 0; i < 22; ++i) printf("%-16s %6.1f cycles/iter\n", names[i], (double)c[i] / N);
  return 0;
}
