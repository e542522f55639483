// tools/ubench.cu -- microbenchmarks of the join primitives on B200 (not part of the product).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench tools/ubench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

// smem atomicAdd with returned value, NB counters, random bucket per key
template <int NB>
__global__ void k_smem_atomic(uint32_t iters, uint32_t *out) {
  __shared__ uint32_t cnt[NB];
  for (int i = threadIdx.x; i < NB; i += blockDim.x) cnt[i] = 0;
  __syncthreads();
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x, acc = 0;
  for (uint32_t i = 0; i < iters; ++i) {
    s = mix32(s + i);
    acc += atomicAdd(&cnt[s & (NB - 1)], 1u);
  }
  if (acc == 0xdeadbeef) out[0] = acc;
}

// smem store to a private slot + no atomic (baseline)
__global__ void k_smem_store(uint32_t iters, uint32_t *out) {
  __shared__ uint64_t buf[4096];
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  for (uint32_t i = 0; i < iters; ++i) {
    s = mix32(s + i);
    buf[(s & 4095)] = s;
  }
  __syncthreads();
  if (buf[threadIdx.x] == 0xdeadbeef) out[0] = 1;
}

// global atomicCAS into a table of `slots` u64 (random), ILP = 4 independent CAS per thread
__global__ void k_global_cas(unsigned long long *tab, uint32_t mask, uint32_t iters, uint32_t *out) {
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long acc = 0;
  for (uint32_t i = 0; i < iters; ++i) {
    uint32_t a0 = mix32(s + 4 * i), a1 = mix32(a0), a2 = mix32(a1), a3 = mix32(a2);
    acc += atomicCAS(tab + (a0 & mask), 0ull, a0 | 1ull);
    acc += atomicCAS(tab + (a1 & mask), 0ull, a1 | 1ull);
    acc += atomicCAS(tab + (a2 & mask), 0ull, a2 | 1ull);
    acc += atomicCAS(tab + (a3 & mask), 0ull, a3 | 1ull);
    s = a3;
  }
  if (acc == 0xdeadbeef) out[0] = 1;
}

// global random u64 loads, ILP 4
__global__ void k_global_load(const unsigned long long *tab, uint32_t mask, uint32_t iters, uint32_t *out) {
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long acc = 0;
  for (uint32_t i = 0; i < iters; ++i) {
    uint32_t a0 = mix32(s + 4 * i), a1 = mix32(a0), a2 = mix32(a1), a3 = mix32(a2);
    acc += tab[a0 & mask] + tab[a1 & mask] + tab[a2 & mask] + tab[a3 & mask];
    s = a3;
  }
  if (acc == 0xdeadbeef) out[0] = 1;
}

// global random u64 stores (scatter), ILP 4
__global__ void k_global_store(unsigned long long *tab, uint32_t mask, uint32_t iters) {
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  for (uint32_t i = 0; i < iters; ++i) {
    uint32_t a0 = mix32(s + 4 * i), a1 = mix32(a0), a2 = mix32(a1), a3 = mix32(a2);
    tab[a0 & mask] = a0; tab[a1 & mask] = a1; tab[a2 & mask] = a2; tab[a3 & mask] = a3;
    s = a3;
  }
}

// smem hash-table probe: 8192-slot u64 table, random probes (LDS.64)
__global__ void k_smem_probe(uint32_t iters, uint32_t *out) {
  __shared__ unsigned long long t[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) t[i] = mix32(i);
  __syncthreads();
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long acc = 0;
  for (uint32_t i = 0; i < iters; ++i) {
    s = mix32(s + i);
    acc += t[s & 4095];
  }
  if (acc == 0xdeadbeef) out[0] = 1;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t *out;
  cudaMalloc(&out, 64);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](const char *name, double ops, auto launch) {
    launch();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("%-40s %10.3f ms  %8.2f Gop/s  (%s)\n", name, best, ops / (best * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  };
  const int blocks = sms * 8, threads = 256;
  const uint32_t it = 4096;
  const double nthr = (double)blocks * threads;
  timeit("smem atomicAdd NB=256", nthr * it, [&] { k_smem_atomic<256><<<blocks, threads>>>(it, out); });
  timeit("smem atomicAdd NB=2048", nthr * it, [&] { k_smem_atomic<2048><<<blocks, threads>>>(it, out); });
  timeit("smem store u64 random", nthr * it, [&] { k_smem_store<<<blocks, threads>>>(it, out); });
  timeit("smem probe u64 random", nthr * it, [&] { k_smem_probe<<<blocks, threads>>>(it, out); });
  for (uint32_t slots_log2 : {20u, 23u, 26u, 28u}) {
    unsigned long long *tab;
    cudaMalloc(&tab, 8ull << slots_log2);
    cudaMemset(tab, 0, 8ull << slots_log2);
    const uint32_t mask = (1u << slots_log2) - 1;
    char nm[64];
    const uint32_t it2 = 256;
    snprintf(nm, sizeof nm, "global CAS u64 table 2^%u (%u MB)", slots_log2, 8u << slots_log2 >> 20);
    timeit(nm, nthr * it2 * 4, [&] { cudaMemset(tab, 0, 8ull << slots_log2); k_global_cas<<<blocks, threads>>>(tab, mask, it2, out); });
    snprintf(nm, sizeof nm, "global load u64 table 2^%u", slots_log2);
    timeit(nm, nthr * it2 * 4, [&] { k_global_load<<<blocks, threads>>>(tab, mask, it2, out); });
    snprintf(nm, sizeof nm, "global store u64 table 2^%u", slots_log2);
    timeit(nm, nthr * it2 * 4, [&] { k_global_store<<<blocks, threads>>>(tab, mask, it2); });
    cudaFree(tab);
  }
  return 0;
}
