// tools/ubench4.cu -- L2 streaming/run-write bandwidth and shared-memory random-access throughput,
// the two resources the partitioned join spends per key (not part of the product).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench4 tools/ubench4.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

__global__ void k_rd(const uint4 *p, size_t n16, int reps, uint32_t *out) {
  uint32_t acc = 0;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
      const uint4 v = __ldcg(p + i);
      acc ^= v.x ^ v.w;
    }
  if (acc == 0xdeadbeef) out[0] = acc;
}
__global__ void k_wr(uint4 *p, size_t n16, int reps) {
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
      __stcg(p + i, make_uint4((uint32_t)i, r, 2, 3));
}
// runs of K consecutive u64 at random K-aligned positions (lane i of a run group writes key i)
template <int K>
__global__ void k_runs(unsigned long long *p, uint32_t nruns, uint32_t iters) {
  const uint32_t lane = threadIdx.x & 31, grp = lane / K, sub = lane % K;
  uint32_t s = (blockIdx.x * blockDim.x + threadIdx.x) / K * 0x9E3779B9u + 17;
  for (uint32_t i = 0; i < iters; ++i) {
    s = mix32(s + grp + 1);
    const uint32_t run = s % nruns;
    __stcg(p + (size_t)run * K + sub, (unsigned long long)s);
  }
}
// runs of K keys starting at arbitrary (non-aligned) u64 positions
template <int K>
__global__ void k_runs_u(unsigned long long *p, uint32_t n, uint32_t iters) {
  const uint32_t lane = threadIdx.x & 31, grp = lane / K, sub = lane % K;
  uint32_t s = (blockIdx.x * blockDim.x + threadIdx.x) / K * 0x9E3779B9u + 17;
  for (uint32_t i = 0; i < iters; ++i) {
    s = mix32(s + grp + 1);
    const uint32_t pos = s % (n - K);
    __stcg(p + pos + sub, (unsigned long long)s);
  }
}

// shared memory: MODE 0 random atomicAdd u32 over E entries; 1 random STS.64 over 16K slots;
// 2 random LDS.64; 3 broadcast LDS.128; 4 random atomicAdd u32 + dependent STS.64 (staging)
template <int MODE>
__global__ void __launch_bounds__(512) k_smem(uint32_t iters, uint32_t E, uint32_t *out) {
  extern __shared__ unsigned long long sm[];
  uint32_t *cnt = reinterpret_cast<uint32_t *>(sm + 16384);
  for (uint32_t i = threadIdx.x; i < 16384; i += blockDim.x) sm[i] = i;
  for (uint32_t i = threadIdx.x; i < E; i += blockDim.x) cnt[i] = 0;
  __syncthreads();
  uint32_t s = (blockIdx.x * blockDim.x + threadIdx.x) * 0x9E3779B9u;
  unsigned long long acc = 0;
  for (uint32_t i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      s = s * 1664525u + 1013904223u;
      const uint32_t a = s >> 18;  // 14 bits
      if (MODE == 0) acc += atomicAdd(cnt + (a % E), 1u);
      if (MODE == 1) sm[a] = s;
      if (MODE == 2) acc += sm[a];
      if (MODE == 3) { const uint4 v = reinterpret_cast<const uint4 *>(sm)[(i * 4 + u) & 1023]; acc += v.x ^ v.w; }
      if (MODE == 4) { const uint32_t e = a & (E - 1); const uint32_t r = atomicAdd(cnt + e, 1u); sm[(e * 16 + (r & 15)) & 16383] = s; }
    }
  }
  if (acc == 0xdeadbeef) out[0] = (uint32_t)acc;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  uint32_t *out;
  cudaMalloc(&out, 1 << 20);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](const char *name, double units, const char *u, auto launch) {
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
    printf("%-52s %9.3f ms  %10.2f %s  (%s)\n", name, best, units / (best * 1e-3) / 1e9, u,
           cudaGetErrorString(cudaGetLastError()));
  };
  unsigned long long *buf;
  cudaMalloc(&buf, 1ull << 30);
  for (size_t mb : {8, 16, 32, 48, 64, 96, 128, 512}) {
    const size_t bytes = mb << 20;
    const int reps = (int)(2048 / mb) > 1 ? (int)(2048 / mb) : 1;
    char nm[96];
    snprintf(nm, sizeof nm, "L2/HBM stream read %zu MB x%d", mb, reps);
    timeit(nm, (double)bytes * reps, "GB/s", [&] { k_rd<<<sms * 4, 512>>>((const uint4 *)buf, bytes / 16, reps, out); });
    snprintf(nm, sizeof nm, "L2/HBM stream write %zu MB x%d", mb, reps);
    timeit(nm, (double)bytes * reps, "GB/s", [&] { k_wr<<<sms * 4, 512>>>((uint4 *)buf, bytes / 16, reps); });
  }
  {
    const size_t bytes = 48ull << 20;
    const uint32_t iters = 256;
    const double keys = (double)sms * 4 * 512 * iters;
#define RUNS(K)                                                                                  \
    timeit("run writes K=" #K " aligned, 48 MB (G keys/s)", keys, "Gkey/s",                      \
           [&] { k_runs<K><<<sms * 4, 512>>>(buf, (uint32_t)(bytes / 8 / K), iters); });         \
    timeit("run writes K=" #K " unaligned, 48 MB (G keys/s)", keys, "Gkey/s",                    \
           [&] { k_runs_u<K><<<sms * 4, 512>>>(buf, (uint32_t)(bytes / 8), iters); });
    RUNS(1) RUNS(2) RUNS(4) RUNS(8) RUNS(16) RUNS(32)
  }
  {
    const size_t smem = 16384 * 8 + 4096 * 4;
    cudaFuncSetAttribute(k_smem<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_smem<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_smem<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_smem<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_smem<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const uint32_t iters = 4096;
    for (int thr : {512}) {
      const double ops = (double)sms * thr * iters * 4;
      const double clkhz = clk * 1e3;
      auto per = [&](const char *nm, auto l) {
        timeit(nm, ops, "Gop/s", l);
      };
      per("smem atomicAdd.u32 random E=1024", [&] { k_smem<0><<<sms, thr, smem>>>(iters, 1024, out); });
      per("smem atomicAdd.u32 random E=2048", [&] { k_smem<0><<<sms, thr, smem>>>(iters, 2048, out); });
      per("smem atomicAdd.u32 random E=256", [&] { k_smem<0><<<sms, thr, smem>>>(iters, 256, out); });
      per("smem STS.64 random", [&] { k_smem<1><<<sms, thr, smem>>>(iters, 1024, out); });
      per("smem LDS.64 random", [&] { k_smem<2><<<sms, thr, smem>>>(iters, 1024, out); });
      per("smem LDS.128 broadcast", [&] { k_smem<3><<<sms, thr, smem>>>(iters, 1024, out); });
      per("smem atomicAdd + STS.64 (staging) E=1024", [&] { k_smem<4><<<sms, thr, smem>>>(iters, 1024, out); });
      printf("(per SM per clock: Gop/s / (%d SMs x %.3f GHz))\n", sms, clkhz / 1e9);
    }
  }
  return 0;
}
