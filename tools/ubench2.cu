// tools/ubench2.cu -- microbenchmarks for the join redesign (not part of the product).
//   fold variants of the FNV step, L2-resident random CAS / load / atomicOr throughput.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench2 tools/ubench2.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

// V0: current (LOP3, IMAD.WIDE, IMAD, LEA, IADD)
__device__ __forceinline__ void f0(uint32_t &lo, uint32_t &hi, uint32_t v) {
  const uint32_t x = lo ^ v;
  const uint64_t p = (uint64_t)x * 435u;
  hi = hi * 435u + (uint32_t)(p >> 32) + (x << 8);
  lo = (uint32_t)p;
}
// V1: IMAD.WIDE with 64-bit addend (0, t): 4 instructions if the compiler keeps a zero low half
__device__ __forceinline__ void f1(uint32_t &lo, uint32_t &hi, uint32_t v) {
  const uint32_t x = lo ^ v;
  const uint32_t t = hi * 435u + (x << 8);
  uint64_t p;
  asm("mad.wide.u32 %0, %1, 435, %2;" : "=l"(p) : "r"(x), "l"((uint64_t)t << 32));
  lo = (uint32_t)p; hi = (uint32_t)(p >> 32);
}
// V2: lo chain with mul.lo + mul.hi
__device__ __forceinline__ void f2(uint32_t &lo, uint32_t &hi, uint32_t v) {
  const uint32_t x = lo ^ v;
  hi = hi * 435u + __umulhi(x, 435u) + (x << 8);
  lo = x * 435u;
}
// V3: native 64-bit
__device__ __forceinline__ void f3(uint32_t &lo, uint32_t &hi, uint32_t v) {
  uint64_t h = ((uint64_t)hi << 32) | lo;
  h = (h ^ v) * 0x100000001B3ull;
  lo = (uint32_t)h; hi = (uint32_t)(h >> 32);
}

template <int V, int CH>
__global__ void __launch_bounds__(256) k_fold(uint32_t iters, uint32_t seed, uint32_t *sink) {
  uint32_t lo[CH], hi[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) { lo[c] = seed * (threadIdx.x + 1) + c; hi[c] = blockIdx.x ^ c; }
  uint32_t v = threadIdx.x;
  for (uint32_t i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const uint32_t vv = (v + c) & 0xFFFFu;
      if (V == 0) f0(lo[c], hi[c], vv);
      if (V == 1) f1(lo[c], hi[c], vv);
      if (V == 2) f2(lo[c], hi[c], vv);
      if (V == 3) f3(lo[c], hi[c], vv);
    }
    v += 0x9E37u;
  }
  uint32_t acc = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) acc ^= lo[c] ^ hi[c];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// random 64-bit CAS into an L2-resident table, U independent per thread per iteration
template <int U>
__global__ void k_cas(unsigned long long *tab, uint32_t mask, uint32_t iters, uint32_t *out) {
  uint32_t s = (blockIdx.x * blockDim.x + threadIdx.x) * 0x9E3779B9u;
  unsigned long long acc = 0;
  for (uint32_t i = 0; i < iters; ++i) {
    uint32_t a[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { s = mix32(s + u + 1); a[u] = s; }
    unsigned long long r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) r[u] = atomicCAS(tab + (a[u] & mask), 0ull, (unsigned long long)a[u] | 1ull);
#pragma unroll
    for (int u = 0; u < U; ++u) acc += r[u];
  }
  if (acc == 0xdeadbeef) out[0] = 1;
}
template <int U>
__global__ void k_ld(const unsigned long long *tab, uint32_t mask, uint32_t iters, uint32_t *out) {
  uint32_t s = (blockIdx.x * blockDim.x + threadIdx.x) * 0x9E3779B9u;
  unsigned long long acc = 0;
  for (uint32_t i = 0; i < iters; ++i) {
    uint32_t a[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { s = mix32(s + u + 1); a[u] = s; }
    unsigned long long r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) r[u] = __ldcg(tab + (a[u] & mask));
#pragma unroll
    for (int u = 0; u < U; ++u) acc += r[u];
  }
  if (acc == 0xdeadbeef) out[0] = 1;
}
template <int U>
__global__ void k_ld16(const uint4 *tab, uint32_t mask, uint32_t iters, uint32_t *out) {
  uint32_t s = (blockIdx.x * blockDim.x + threadIdx.x) * 0x9E3779B9u;
  uint32_t acc = 0;
  for (uint32_t i = 0; i < iters; ++i) {
    uint32_t a[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { s = mix32(s + u + 1); a[u] = s; }
    uint4 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) r[u] = __ldcg(tab + (a[u] & mask));
#pragma unroll
    for (int u = 0; u < U; ++u) acc += r[u].x ^ r[u].w;
  }
  if (acc == 0xdeadbeef) out[0] = 1;
}
template <int U>
__global__ void k_or(unsigned int *tab, uint32_t mask, uint32_t iters, uint32_t *out) {
  uint32_t s = (blockIdx.x * blockDim.x + threadIdx.x) * 0x9E3779B9u;
  for (uint32_t i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < U; ++u) { s = mix32(s + u + 1); atomicOr(tab + (s & mask), 1u << (s >> 27)); }
  }
}
template <int U>
__global__ void k_st(unsigned long long *tab, uint32_t mask, uint32_t iters) {
  uint32_t s = (blockIdx.x * blockDim.x + threadIdx.x) * 0x9E3779B9u;
  for (uint32_t i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < U; ++u) { s = mix32(s + u + 1); __stcg(tab + (s & mask), (unsigned long long)s); }
  }
}
__global__ void k_clear(uint4 *p, size_t n16) {
  const uint4 z = make_uint4(0, 0, 0, 0);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) p[i] = z;
}
// coalesced streaming write then read of N keys (sequential), for the partition traffic floor
__global__ void k_seqwr(uint4 *p, size_t n16) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_uint4((uint32_t)i, 1, 2, 3);
}
__global__ void k_seqrd(const uint4 *p, size_t n16, uint32_t *out) {
  uint32_t acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
    acc ^= p[i].x;
  if (acc == 0xdeadbeef) out[0] = 1;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t *out;
  cudaMalloc(&out, 64 << 20);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](const char *name, double ops, auto launch) {
    launch();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("%-48s %9.3f ms  %9.2f G/s  (%s)\n", name, best, ops / (best * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  };
  {
    const int blocks = sms * 8, threads = 256;
    const uint32_t it = 1 << 12;
    const double folds = (double)blocks * threads * it * 8;
    timeit("fold V0 (folds/s)", folds, [&] { k_fold<0, 8><<<blocks, threads>>>(it, 1, out); });
    timeit("fold V1 (folds/s)", folds, [&] { k_fold<1, 8><<<blocks, threads>>>(it, 1, out); });
    timeit("fold V2 (folds/s)", folds, [&] { k_fold<2, 8><<<blocks, threads>>>(it, 1, out); });
    timeit("fold V3 (folds/s)", folds, [&] { k_fold<3, 8><<<blocks, threads>>>(it, 1, out); });
    timeit("fold V0 4ch (folds/s)", folds / 2, [&] { k_fold<0, 4><<<blocks, threads>>>(it, 1, out); });
    timeit("fold V1 4ch (folds/s)", folds / 2, [&] { k_fold<1, 4><<<blocks, threads>>>(it, 1, out); });
    // check equality of the variants
    uint32_t *o2; cudaMalloc(&o2, 64 << 20);
    k_fold<0, 8><<<blocks, threads>>>(64, 3, out); k_fold<1, 8><<<blocks, threads>>>(64, 3, o2);
    static uint32_t h1[1024], h2[1024];
    cudaMemcpy(h1, out, 4096, cudaMemcpyDeviceToHost); cudaMemcpy(h2, o2, 4096, cudaMemcpyDeviceToHost);
    int bad = 0; for (int i = 0; i < 1024; ++i) bad += h1[i] != h2[i];
    k_fold<2, 8><<<blocks, threads>>>(64, 3, o2); cudaMemcpy(h2, o2, 4096, cudaMemcpyDeviceToHost);
    for (int i = 0; i < 1024; ++i) bad += h1[i] != h2[i];
    k_fold<3, 8><<<blocks, threads>>>(64, 3, o2); cudaMemcpy(h2, o2, 4096, cudaMemcpyDeviceToHost);
    for (int i = 0; i < 1024; ++i) bad += h1[i] != h2[i];
    printf("fold variants mismatches: %d\n", bad);
  }
  for (int occ : {8, 16}) {
    const int blocks = sms * occ, threads = 256;
    const double nthr = (double)blocks * threads;
    for (uint32_t l2 : {21u, 22u, 23u, 24u, 25u}) {  // 16..256 MB
      unsigned long long *tab;
      const size_t bytes = 8ull << l2;
      cudaMalloc(&tab, bytes);
      const uint32_t mask = (1u << l2) - 1;
      const uint32_t it = 64;
      char nm[96];
      k_clear<<<sms * 4, 512>>>((uint4 *)tab, bytes / 16);
      cudaDeviceSynchronize();
      timeit("clear (SM stores) GB/s", bytes / 1.0, [&] { k_clear<<<sms * 4, 512>>>((uint4 *)tab, bytes / 16); });
      snprintf(nm, sizeof nm, "occ%d CAS64 U4 %zu MB (cleared)", occ, bytes >> 20);
      timeit(nm, nthr * it * 4, [&] { k_clear<<<sms * 4, 512>>>((uint4 *)tab, bytes / 16); k_cas<4><<<blocks, threads>>>(tab, mask, it, out); });
      snprintf(nm, sizeof nm, "occ%d CAS64 U8 %zu MB (cleared)", occ, bytes >> 20);
      timeit(nm, nthr * it * 8, [&] { k_clear<<<sms * 4, 512>>>((uint4 *)tab, bytes / 16); k_cas<8><<<blocks, threads>>>(tab, mask, it, out); });
      snprintf(nm, sizeof nm, "occ%d LD64 U8 %zu MB", occ, bytes >> 20);
      timeit(nm, nthr * it * 8, [&] { k_ld<8><<<blocks, threads>>>(tab, mask, it, out); });
      snprintf(nm, sizeof nm, "occ%d LD128 U8 %zu MB", occ, bytes >> 20);
      timeit(nm, nthr * it * 8, [&] { k_ld16<8><<<blocks, threads>>>((const uint4 *)tab, mask >> 1, it, out); });
      snprintf(nm, sizeof nm, "occ%d OR32 U8 %zu MB", occ, bytes >> 20);
      timeit(nm, nthr * it * 8, [&] { k_or<8><<<blocks, threads>>>((unsigned *)tab, (mask << 1) | 1, it, out); });
      snprintf(nm, sizeof nm, "occ%d ST64 U8 %zu MB", occ, bytes >> 20);
      timeit(nm, nthr * it * 8, [&] { k_st<8><<<blocks, threads>>>(tab, mask, it); });
      cudaFree(tab);
    }
  }
  {
    const size_t bytes = 1ull << 30;
    uint4 *p; cudaMalloc(&p, bytes);
    timeit("seq write 1 GB (GB/s)", bytes, [&] { k_seqwr<<<sms * 8, 256>>>(p, bytes / 16); });
    timeit("seq read 1 GB (GB/s)", bytes, [&] { k_seqrd<<<sms * 8, 256>>>(p, bytes / 16, out); });
    timeit("seq write 32 MB (GB/s)", 32 << 20, [&] { k_seqwr<<<sms * 8, 256>>>(p, (32 << 20) / 16); });
    timeit("seq read 32 MB (GB/s)", 32 << 20, [&] { k_seqrd<<<sms * 8, 256>>>(p, (32 << 20) / 16, out); });
  }
  return 0;
}
