// msp_bench.cu -- INT32 roofline denominator for the join kernels.
//
// MEASURED_PEAKS.json carries HBM and bf16 peaks only; the FNV fold (LOP3 + IMAD.WIDE.U32 + IMAD +
// shift-add per coordinate) is integer-pipe bound, so the roofline needs the measured throughput of
// exactly that instruction mix.  Each thread runs 8 independent fold chains
// (enough ILP to saturate both the FMA and ALU pipes); one fold step counts as 4 INT32 ops, the
// same unit as the per-pair op counts in DESIGN.md.
#include <cstdint>
#include <cuda_runtime.h>
#include "msp_b200.h"
#include "msp_common.cuh"

namespace msp {

__global__ void __launch_bounds__(256) k_int32_peak(uint32_t iters, uint32_t seed, uint32_t *sink) {
  uint32_t lo[8], hi[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) { lo[c] = seed * (threadIdx.x + 1) + c; hi[c] = blockIdx.x ^ c; }
  uint32_t v = threadIdx.x;
  for (uint32_t i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) fnv_step(lo[c], hi[c], (v + c) & 0xFFFFu);
    v += 0x9E37u;
  }
  uint32_t acc = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) acc ^= lo[c] ^ hi[c];
  if (acc == 0x12345678u) sink[0] = acc;  // keep the chains live
}

}  // namespace msp

extern "C" double msp_int32_peak(int32_t device) {
  using namespace msp;
  if (cudaSetDevice(device) != cudaSuccess) return -1.0;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  uint32_t *sink = nullptr;
  if (cudaMalloc(&sink, 64) != cudaSuccess) return -1.0;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int blocks = sms * 8, threads = 256;
  const uint32_t iters = 1 << 14;
  k_int32_peak<<<blocks, threads>>>(iters / 16, 1u, sink);  // warm-up / clock ramp
  double best = 0.0;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(a);
    k_int32_peak<<<blocks, threads>>>(iters, 7u + rep, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    const double ops = 4.0 * 8.0 * iters * (double)blocks * threads;
    if (ms > 0) best = best > ops / (ms * 1e-3) ? best : ops / (ms * 1e-3);
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(sink);
  return cudaGetLastError() == cudaSuccess ? best : -1.0;
}
