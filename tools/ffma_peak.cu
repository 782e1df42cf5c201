// Microbenchmark: FP32 FFMA vs FFMA2 (fma.rn.f32x2) issue throughput on sm_100a.
// Used once to pin the FP32 roofline denominator; not part of the product path.
#include <cstdio>
#include <cuda_runtime.h>
template <int CHAINS>
__global__ void __launch_bounds__(256) ffma_kernel(float* out, int iters, float a, float b) {
  float acc[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) acc[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) acc[i] = fmaf(acc[i], a, b);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int CHAINS>
__global__ void __launch_bounds__(256) ffma2_kernel(float* out, int iters, float a, float b) {
  unsigned long long acc[CHAINS];
  float2 av = make_float2(a, a), bv = make_float2(b, b);
  unsigned long long ra = *reinterpret_cast<unsigned long long*>(&av);
  unsigned long long rb = *reinterpret_cast<unsigned long long*>(&bv);
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) { float2 t = make_float2(threadIdx.x * 1e-3f + i, i); acc[i] = *reinterpret_cast<unsigned long long*>(&t); }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i)
      asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(acc[i]) : "l"(ra), "l"(rb));
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) { float2 t = *reinterpret_cast<float2*>(&acc[i]); s += t.x + t.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("gpu %s sms %d clock_khz %d\n", p.name, p.multiProcessorCount, clk);
  float* out; cudaMalloc(&out, 148 * 8 * 256 * 4 * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000;
  for (int blocksPerSm : {4, 8}) {
    int grid = p.multiProcessorCount * blocksPerSm;
    for (int rep = 0; rep < 2; ++rep) {
      ffma_kernel<32><<<grid, 256>>>(out, iters, 0.999f, 1e-4f);
      cudaEventRecord(e0); ffma_kernel<32><<<grid, 256>>>(out, iters, 0.999f, 1e-4f); cudaEventRecord(e1);
      cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
      double fl = 2.0 * 32 * iters * (double)grid * 256;
      printf("FFMA  bps=%d  %.2f TFLOP/s\n", blocksPerSm, fl / ms / 1e9);
      ffma2_kernel<16><<<grid, 256>>>(out, iters, 0.999f, 1e-4f);
      cudaEventRecord(e0); ffma2_kernel<16><<<grid, 256>>>(out, iters, 0.999f, 1e-4f); cudaEventRecord(e1);
      cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
      fl = 2.0 * 32 * iters * (double)grid * 256;
      printf("FFMA2 bps=%d  %.2f TFLOP/s\n", blocksPerSm, fl / ms / 1e9);
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
