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
// The conv kernel's operand pattern without memory traffic or barriers:
// 8 px x 8 ch per thread, FFMA2 of a broadcast activation scalar and a
// weight pair, operands from LDS.128 (tools/ffma2_pattern.cu, mode 0), 8
// warps per SM.  Its rate is the practical ceiling of that instruction mix.
__global__ void __launch_bounds__(256, 1) ffma2_pattern_kernel(float* out, int iters) {
  __shared__ __align__(16) float s[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) s[i] = (i % 97) * 1e-3f;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const float* pa = s + (lane & 3) * 8 + (threadIdx.x >> 5) * 64;
  const float* pb = s + 4096 + (lane >> 2) * 68;
  uint64_t acc[8][4];
#pragma unroll
  for (int k = 0; k < 8; ++k)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[k][c] = 0;
  for (int it = 0; it < iters; ++it) {
    const int o = (it & 7) * 256;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float a[8][4];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float4 t = lds128(pa + o + k * 32 + h * 4);
        a[k][0] = t.x; a[k][1] = t.y; a[k][2] = t.z; a[k][3] = t.w;
      }
#pragma unroll
      for (int i4 = 0; i4 < 4; ++i4) {
        const float4 b0 = lds128(pb + o / 4 + (h * 4 + i4) * 8);
        const float4 b1 = lds128(pb + o / 4 + (h * 4 + i4) * 8 + 4);
        const uint64_t bp[4] = {pack2(b0.x, b0.y), pack2(b0.z, b0.w), pack2(b1.x, b1.y),
                                pack2(b1.z, b1.w)};
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int k = 0; k < 8; ++k) ffma2(acc[k][c], a[k][i4], bp[c]);
      }
    }
  }
  float sum = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const float2 f = unpack2(acc[k][c]);
      sum += f.x + f.y;
    }
  if (sum == 1234.5f) out[blockIdx.x] = sum;
}
}  // namespace

double ffma2_pattern_probe(cudaStream_t st) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int iters = 4000;
  float* out = nullptr;
  if (cudaMallocAsync(&out, sms * sizeof(float), st) != cudaSuccess) return -1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double best = 0;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0, st);
    ffma2_pattern_kernel<<<sms, 256, 0, st>>>(out, iters);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double tf = 2.0 * 8 * 8 * 8 * (double)iters * sms * 256 / (ms * 1e-3) / 1e12;
    if (rep > 0 && tf > best) best = tf;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFreeAsync(out, st);
  cudaStreamSynchronize(st);
  return best;
}

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
