// startup_probe.cu -- kernel start-up latency: entry -> 28 KB staged from L2
// (cp.async 16 B by 256 threads / cp.async.bulk issued by one warp), per-CTA clock64.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/startup_probe tools/startup_probe.cu
#include <cstdio>
#include <cstdint>
#include <vector>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void __launch_bounds__(256, 1) k_cpasync(const float* __restrict__ src, long long* dbg, int floats) {
  extern __shared__ __align__(128) float sm[];
  long long t0 = clock64();
  const float* s = src + (size_t)blockIdx.x * floats;
  for (int i = threadIdx.x * 4; i < floats; i += 256 * 4)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(sm + i)), "l"(s + i));
  asm volatile("cp.async.commit_group;");
  long long t1 = clock64();
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  long long t2 = clock64();
  float acc = 0;
  for (int i = threadIdx.x; i < floats; i += 256) acc += sm[i];
  if (threadIdx.x == 0) { dbg[blockIdx.x * 4] = t1 - t0; dbg[blockIdx.x * 4 + 1] = t2 - t0; dbg[blockIdx.x * 4 + 2] = (long long)acc; }
}
__global__ void __launch_bounds__(256, 1) k_bulk(const float* __restrict__ src, long long* dbg, int floats, int chunk) {
  extern __shared__ __align__(128) float sm[];
  __shared__ __align__(8) uint64_t bar;
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const float* s = src + (size_t)blockIdx.x * floats;
  const int n = floats / chunk;
  if (threadIdx.x < 32) {
    if (threadIdx.x == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(floats * 4));
    __syncwarp();
    for (int c = threadIdx.x; c < n; c += 32)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(su32(sm + c * chunk)), "l"(s + c * chunk), "r"(chunk * 4), "r"(su32(&bar)) : "memory");
  }
  long long t1 = clock64();
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(su32(&bar)) : "memory");
  long long t2 = clock64();
  float acc = 0;
  for (int i = threadIdx.x; i < floats; i += 256) acc += sm[i];
  if (threadIdx.x == 0) { dbg[blockIdx.x * 4] = t1 - t0; dbg[blockIdx.x * 4 + 1] = t2 - t0; dbg[blockIdx.x * 4 + 2] = (long long)acc; }
}
int main() {
  const int grid = 148, floats = 7168;  // 28 KB per CTA
  float* src; long long* dbg;
  cudaMalloc(&src, (size_t)grid * floats * 4); cudaMemset(src, 0, (size_t)grid * floats * 4);
  cudaMalloc(&dbg, grid * 32);
  cudaFuncSetAttribute(k_cpasync, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  std::vector<long long> h(grid * 4);
  auto rep = [&](const char* name) {
    cudaDeviceSynchronize();
    cudaMemcpy(h.data(), dbg, grid * 32, cudaMemcpyDeviceToHost);
    double a = 0, b = 0; for (int i = 0; i < grid; ++i) { a += h[i * 4]; b += h[i * 4 + 1]; }
    printf("%-28s issued %.0f  landed %.0f cycles (avg over CTAs)\n", name, a / grid, b / grid);
  };
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int r = 0; r < 3; ++r) { k_cpasync<<<grid, 256, 28 * 1024>>>(src, dbg, floats); rep("cp.async 16B x 256 thr"); }
  for (int chunk : {224, 512, 1792}) for (int r = 0; r < 2; ++r) {
    k_bulk<<<grid, 256, 28 * 1024>>>(src, dbg, floats, chunk);
    char nm[64]; snprintf(nm, 64, "bulk %d B x %d", chunk * 4, floats / chunk); rep(nm);
  }
  // launch-to-launch time of the lean kernel
  cudaEventRecord(e0);
  for (int r = 0; r < 20; ++r) k_cpasync<<<grid, 256, 28 * 1024>>>(src, dbg, floats);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("lean kernel back-to-back: %.2f us per launch\n", ms * 1000 / 20);
  return 0;
}
