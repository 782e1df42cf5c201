// ffma2_pattern.cu -- how close does the conv inner loop's register pattern
// (8 px x 8 ch per thread: 32 FFMA2 accumulator pairs, 8 broadcast scalars,
// 4 weight pairs, all operands from LDS.128) get to the FFMA2 peak with 2, 3
// or 4 warps per SMSP?  No global traffic, no barriers.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ffma2_pattern tools/ffma2_pattern.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint64_t pack2(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void ffma2(uint64_t& d, float a, uint64_t b) {
  uint64_t aa;
  asm("mov.b64 %0, {%1, %1};" : "=l"(aa) : "f"(a));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(aa), "l"(b));
}

__device__ __forceinline__ void ffma2p(uint64_t& d, uint64_t a, uint64_t b) {
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(a), "l"(b));
}

// MODE 0: broadcast scalar x weight pair (the conv kernel's form)
// MODE 1: activation pair x weight pair (input channels i, i+1 in the two
//         lanes; 8 px x 8 ch x 2 partial sums = 64 accumulator pairs)
template <int TPX, int MODE>
__global__ void __launch_bounds__(256, 1) pattern(float* out, int iters) {
  __shared__ __align__(16) float s[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) s[i] = (i % 97) * 1e-3f;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const float* pa = s + (lane & 3) * 8 + (threadIdx.x >> 5) * 64;
  const float* pb = s + 4096 + (lane >> 2) * 68;
  constexpr int NC = MODE == 0 ? 4 : 8;
  uint64_t acc[TPX][NC];
#pragma unroll
  for (int k = 0; k < TPX; ++k)
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[k][c] = 0;
  for (int it = 0; it < iters; ++it) {
    const int o = (it & 7) * 256;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float a[TPX][4];
#pragma unroll
      for (int k = 0; k < TPX; ++k) {
        const float4 t = *reinterpret_cast<const float4*>(pa + o + k * 32 * 8 / 8 + h * 4);
        a[k][0] = t.x; a[k][1] = t.y; a[k][2] = t.z; a[k][3] = t.w;
      }
      if constexpr (MODE == 2) {
        // k outer, c inner: the broadcast scalar is the reused operand
#pragma unroll
        for (int i4 = 0; i4 < 4; ++i4) {
          const float4 b0 = *reinterpret_cast<const float4*>(pb + o / 4 + (h * 4 + i4) * 8);
          const float4 b1 = *reinterpret_cast<const float4*>(pb + o / 4 + (h * 4 + i4) * 8 + 4);
          uint64_t bp[4] = {pack2(b0.x, b0.y), pack2(b0.z, b0.w), pack2(b1.x, b1.y), pack2(b1.z, b1.w)};
#pragma unroll
          for (int k = 0; k < TPX; ++k)
#pragma unroll
            for (int c = 0; c < 4; ++c) ffma2(acc[k][c], a[k][i4], bp[c]);
        }
      } else if constexpr (MODE == 3) {
        // scalar FFMA, 8 px x 8 ch
#pragma unroll
        for (int i4 = 0; i4 < 4; ++i4) {
          const float4 b0 = *reinterpret_cast<const float4*>(pb + o / 4 + (h * 4 + i4) * 8);
          const float4 b1 = *reinterpret_cast<const float4*>(pb + o / 4 + (h * 4 + i4) * 8 + 4);
          const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
          for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int k = 0; k < TPX; ++k) {
              float lo, hi;
              asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(acc[k][c]));
              lo = fmaf(a[k][i4], bb[2 * c], lo);
              hi = fmaf(a[k][i4], bb[2 * c + 1], hi);
              acc[k][c] = pack2(lo, hi);
            }
        }
      } else if constexpr (MODE == 1) {
        // weights stored [c][i]: one LDS.128 = w[i..i+3][c]
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const float4 w = *reinterpret_cast<const float4*>(pb + o / 4 + c * 8 + h * 4);
          const uint64_t w01 = pack2(w.x, w.y), w23 = pack2(w.z, w.w);
#pragma unroll
          for (int k = 0; k < TPX; ++k) {
            ffma2p(acc[k][c], pack2(a[k][0], a[k][1]), w01);
            ffma2p(acc[k][c], pack2(a[k][2], a[k][3]), w23);
          }
        }
      } else
#pragma unroll
      for (int i4 = 0; i4 < 4; ++i4) {
        const float4 b0 = *reinterpret_cast<const float4*>(pb + o / 4 + (h * 4 + i4) * 8);
        const float4 b1 = *reinterpret_cast<const float4*>(pb + o / 4 + (h * 4 + i4) * 8 + 4);
        uint64_t bp[4] = {pack2(b0.x, b0.y), pack2(b0.z, b0.w), pack2(b1.x, b1.y), pack2(b1.z, b1.w)};
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int k = 0; k < TPX; ++k) ffma2(acc[k][c], a[k][i4], bp[c]);
      }
    }
  }
  float sum = 0;
#pragma unroll
  for (int k = 0; k < TPX; ++k)
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      float lo, hi;
      asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(acc[k][c]));
      sum += lo + hi;
    }
  if (sum == 1234.5f) out[blockIdx.x] = sum;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  cudaMalloc(&out, 1 << 20);
  const int iters = 4000;
  for (int mode : {0, 1, 2, 3})
  for (int threads : {128, 256}) {
    for (int ctas_per_sm : {1, 2}) {
      if (threads * ctas_per_sm > 1024) continue;
      const int grid = sms * ctas_per_sm;
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      auto k = mode == 0 ? pattern<8, 0> : mode == 1 ? pattern<8, 1> : mode == 2 ? pattern<8, 2> : pattern<8, 3>;
      k<<<grid, threads>>>(out, iters);
      cudaEventRecord(a);
      k<<<grid, threads>>>(out, iters);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double flops = 2.0 * 8 * 8 * 8 * iters * (double)grid * threads;
      printf("mode %d threads %d x %d CTA/SM (%d warps/SMSP): %.1f TFLOP/s  %s\n", mode, threads,
             ctas_per_sm, threads * ctas_per_sm / 128, flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
