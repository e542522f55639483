// tools/ubench3.cu -- DSMEM (cluster shared memory) random CAS / load throughput vs local smem.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench3 tools/ubench3.cu
#include <cstdio>
#include <cstdint>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
constexpr int kSlots = 16384;

template <int MODE, int U>  // MODE 0: local CAS, 1: remote CAS, 2: local load, 3: remote load
__global__ void k_dsm(uint32_t iters, uint32_t *out) {
  extern __shared__ unsigned long long tab[];
  cg::cluster_group cl = cg::this_cluster();
  for (int i = threadIdx.x; i < kSlots; i += blockDim.x) tab[i] = (MODE >= 2) ? mix32(i) : 0ull;
  cl.sync();
  const uint32_t nr = cl.num_blocks();
  uint32_t s = (blockIdx.x * blockDim.x + threadIdx.x) * 0x9E3779B9u;
  unsigned long long acc = 0;
  for (uint32_t i = 0; i < iters; ++i) {
    unsigned long long *p[U];
    uint32_t a[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      s = mix32(s + u + 1); a[u] = s;
      unsigned long long *base = (MODE == 1 || MODE == 3) ? cl.map_shared_rank(tab, (s >> 20) % nr) : tab;
      p[u] = base + (s & (kSlots - 1));
    }
    unsigned long long r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (MODE <= 1) r[u] = atomicCAS(p[u], 0ull, (unsigned long long)a[u] | 1);
      else r[u] = *(volatile unsigned long long *)p[u];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += r[u];
  }
  cl.sync();
  if (acc == 0xdeadbeef) out[0] = 1;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t *out; cudaMalloc(&out, 64);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const size_t smem = kSlots * 8;
  auto run = [&](const char *name, auto kern, int csize, int threads) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (csize > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    int maxc = 0;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = csize; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(threads); cfg.dynamicSmemBytes = smem; cfg.attrs = at; cfg.numAttrs = 1;
    cfg.gridDim = dim3(csize);
    cudaOccupancyMaxActiveClusters(&maxc, kern, &cfg);
    const int grid = maxc * csize;
    cfg.gridDim = dim3(grid);
    const uint32_t iters = 2048;
    float best = 1e30f;
    for (int r = 0; r < 4; ++r) {
      cudaEventRecord(a);
      cudaLaunchKernelEx(&cfg, kern, iters, out);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (r && ms < best) best = ms;
    }
    const double ops = (double)grid * threads * iters * 8;
    printf("%-28s cluster %2d grid %4d thr %4d: %8.3f ms %9.1f Gop/s = %.2f op/clk/SM (%s)\n", name, csize, grid, threads, best,
           ops / best / 1e6, ops / (best * 1e-3) / (grid * 1.965e9), cudaGetErrorString(cudaGetLastError()));
  };
  for (int cs : {1, 2, 4, 8, 16}) {
    run("local CAS", k_dsm<0, 8>, cs, 1024);
    run("remote CAS", k_dsm<1, 8>, cs, 1024);
    run("local load", k_dsm<2, 8>, cs, 1024);
    run("remote load", k_dsm<3, 8>, cs, 1024);
  }
  return 0;
}
