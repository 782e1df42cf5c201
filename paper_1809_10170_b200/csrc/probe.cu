// probe.cu -- FP32 FFMA throughput probe: the measured roofline denominator
// for the FFMA direct-conv kernel (bench.py reads it live on the same GPU and
// clocks as the timed run).  32 independent FMA chains per thread, 8 CTAs of
// 256 threads per SM; ptxas pairs them into FFMA2.
#include "common.cuh"
#include "layout_kernels.h"

namespace dconv_dev {
namespace {
__global__ void __launch_bounds__(256) ffma_probe_kernel(float* out, int iters,
                                                         float a, float b) {
  float acc[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) acc[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 32; ++i) acc[i] = fmaf(acc[i], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 32; ++i) s += acc[i];
  if (s == 12345.678f) out[blockIdx.x] = s;  // keep the chains live
}
}  // namespace

double fp32_peak_probe(cudaStream_t st) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = sms * 8, iters = 20000;
  float* out = nullptr;
  if (cudaMallocAsync(&out, grid * sizeof(float), st) != cudaSuccess) return -1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double best = 0;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0, st);
    ffma_probe_kernel<<<grid, 256, 0, st>>>(out, iters, 0.999f, 1e-4f);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double tf = 2.0 * 32 * iters * (double)grid * 256 / (ms * 1e-3) / 1e12;
    if (rep > 0 && tf > best) best = tf;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFreeAsync(out, st);
  cudaStreamSynchronize(st);
  return best;
}
}  // namespace dconv_dev
