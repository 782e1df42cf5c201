// tma_stride_probe.cu -- checks the TMA traversal-stride semantics the
// space-to-depth-in-place idea relies on: a 5-D tensor map over a blocked map
// {c4, half, W, H, blocks} with elementStrides {1, 1, 2, 2, 1} and box
// {4, 1, 2*PW, 2*PH, 1} should land PW x PH pixels (every other column / row)
// densely in shared memory.  Prints the first mismatches, or "ok".
// nvcc -gencode arch=compute_100a,code=sm_100a -o tools/tma_stride_probe tools/tma_stride_probe.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

__global__ void probe(const __grid_constant__ CUtensorMap map, float* out, int n_floats, int x0,
                      int y0, int blk) {
  extern __shared__ __align__(128) float sm[];
  __shared__ __align__(8) unsigned long long bar;
  const unsigned sb = (unsigned)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sb));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(sb),
                 "r"(n_floats * 4)
                 : "memory");
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"((unsigned)__cvta_generic_to_shared(sm)),
        "l"(reinterpret_cast<unsigned long long>(&map)), "r"(0), "r"(0), "r"(x0), "r"(y0),
        "r"(blk), "r"(sb)
        : "memory");
  }
  asm volatile(
      "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], 0;\n"
      "@!p bra W;\n}\n" ::"r"(sb)
      : "memory");
  for (int i = threadIdx.x; i < n_floats; i += blockDim.x) out[i] = sm[i];
}

int main() {
  const int W = 20, H = 18, B = 2, PW = 6, PH = 5, dx = 1, dy = 0, blk = 1;
  std::vector<float> h((size_t)B * H * W * 8);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (float)i;
  float *d, *o;
  cudaMalloc(&d, h.size() * 4);
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  const int nf = PH * PW * 4;
  cudaMalloc(&o, nf * 4);
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp);
  CUtensorMap map;
  const cuuint64_t dims[5] = {4, 2, W, H, B};
  const cuuint64_t strides[4] = {16, 32, (cuuint64_t)W * 32, (cuuint64_t)W * H * 32};
  const cuuint32_t box[5] = {4, 1, 2 * PW, 2 * PH, 1};
  const cuuint32_t estr[5] = {1, 1, 2, 2, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, d, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("encode failed %d\n", (int)r);
    return 1;
  }
  probe<<<1, 128, nf * 4 + 1024>>>(map, o, nf, dx, dy, blk);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("kernel: %s\n", cudaGetErrorString(e));
    return 1;
  }
  std::vector<float> got(nf);
  cudaMemcpy(got.data(), o, nf * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int y = 0; y < PH; ++y)
    for (int x = 0; x < PW; ++x)
      for (int k = 0; k < 4; ++k) {
        const int gx = dx + 2 * x, gy = dy + 2 * y;
        const float want = (gx < W && gy < H) ? h[(((size_t)blk * H + gy) * W + gx) * 8 + k] : 0.f;
        const float g = got[(y * PW + x) * 4 + k];
        if (g != want && bad++ < 8) printf("(%d,%d,%d): got %g want %g\n", y, x, k, g, want);
      }
  printf(bad ? "mismatches: %d\n" : "ok\n", bad);
  return bad != 0;
}
