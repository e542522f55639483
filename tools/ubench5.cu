// L2-resident open-addressing hash table: random 64-bit CAS inserts and random probes from all SMs.
// usage: ubench5 <log2 slots> <load factor percent>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
  return x | 1ull;
}

__global__ void k_build(unsigned long long *tab, unsigned *cnt, uint32_t log2, uint64_t n, uint64_t seed) {
  const uint64_t msk = (1ull << log2) - 1;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k = mix(i + seed);
    uint64_t s = k >> (64 - log2);
    while (true) {
      const unsigned long long old = atomicCAS(tab + s, 0ull, (unsigned long long)k);
      if (old == 0ull || old == k) { atomicAdd(cnt + s, 1u); break; }
      s = (s + 1) & msk;
    }
  }
}

__global__ void k_probe(const unsigned long long *tab, const unsigned *cnt, uint32_t log2, uint64_t n, uint64_t seed,
                        unsigned long long *hits) {
  const uint64_t msk = (1ull << log2) - 1;
  unsigned long long h = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k = mix(i * 3 + seed);
    uint64_t s = k >> (64 - log2);
    while (true) {
      const unsigned long long v = __ldcg(tab + s);
      if (v == 0ull) break;
      if (v == k) { h += __ldcg(cnt + s); break; }
      s = (s + 1) & msk;
    }
  }
  if (h) atomicAdd(hits, h);
}

int main(int argc, char **argv) {
  const uint32_t log2 = argc > 1 ? atoi(argv[1]) : 22;
  const int lf = argc > 2 ? atoi(argv[2]) : 50;
  const uint64_t slots = 1ull << log2, n = slots * lf / 100;
  unsigned long long *tab, *hits;
  unsigned *cnt;
  cudaMalloc(&tab, 8 * slots); cudaMalloc(&cnt, 4 * slots); cudaMalloc(&hits, 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int blocks : {148 * 4, 148 * 8, 148 * 16}) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemset(tab, 0, 8 * slots); cudaMemset(cnt, 0, 4 * slots); cudaMemset(hits, 0, 8);
      cudaEventRecord(a);
      k_build<<<blocks, 512>>>(tab, cnt, log2, n, 12345 + rep);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float mb = 0; cudaEventElapsedTime(&mb, a, b);
      cudaEventRecord(a);
      k_probe<<<blocks, 512>>>(tab, cnt, log2, 4 * n, 999 + rep, hits);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float mp = 0; cudaEventElapsedTime(&mp, a, b);
      if (rep == 2)
        printf("log2 %u lf %d%% blocks %d: build %.1f M keys in %.3f ms = %.1f G inserts/s; probe %.1f M in %.3f ms = %.1f G probes/s\n",
               log2, lf, blocks, n / 1e6, mb, n / (mb * 1e6), 4 * n / 1e6, mp, 4 * n / (mp * 1e6));
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
