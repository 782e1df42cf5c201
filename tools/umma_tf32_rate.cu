// umma_tf32_rate.cu -- tcgen05.mma.kind::tf32 issue-rate probe: one CTA per
// SM, one thread issues ITERS back-to-back M=128 x N x K=8 MMAs on fixed
// shared-memory operands (K-major, no swizzle, core-matrix layout as in
// conv_tf32.cu), accumulating in TMEM; reports cycles per MMA and TFLOP/s.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/umma_tf32_rate tools/umma_tf32_rate.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

// MODE 1: the conv kernel's descriptor walk -- A from a [plane][PH][PW][4]
// patch (LBO = plane bytes, SBO = PW*16), taps (n, m) shift the A start by
// (n*PW + m)*16 B, MT = 4 M-tiles at 16*PW*16 B; B walks 9 taps of 2*N*16 B.
template <int N, int NACC, int MODE = 0, int M = 128>
__global__ void __launch_bounds__(128, 1) probe(int iters, unsigned long long* out, int a_stride, int commit_every) {
  extern __shared__ __align__(1024) float smem[];
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t tslot;
  float* A = smem;                       // [2 khalf][16 mgroups][8][4]
  float* B = smem + (MODE ? 12 * 1024 : 8 * 1024);  // [2 khalf][N/8][8][4]
  for (int i = threadIdx.x; i < (MODE ? 12 * 1024 : 8 * 1024) + 4 * N * 4; i += blockDim.x)
    smem[i] = 1e-3f * (i % 7);
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar2)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) |
                         ((uint32_t)(M >> 4) << 24);
  long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    const uint32_t a0 = smem_u32(A), b0 = smem_u32(B);
    t0 = clock64();
    const int PW = a_stride ? a_stride : 8;  // MODE 1: a_stride = PW
    const uint32_t plane = (uint32_t)(66 * PW * 16);
    for (int it = 0; it < iters; ++it) {
      uint64_t ad, bd;
      uint32_t d;
      if (MODE == 0) {
        // a_stride: vary the A start like the conv's taps (16 B steps)
        ad = desc(a0 + (uint32_t)((it % 3) * a_stride), 16 * 128, 128);
        bd = desc(b0, (uint32_t)(N * 16), 128);
        d = tmem + (uint32_t)((it % NACC) * N);
      } else {
        const int mt = it & 3, tap = (it >> 2) % 9, n = tap / 3, m = tap % 3;
        ad = desc(a0 + (uint32_t)(((mt * 16 + n) * PW + m) * 16), plane, (uint32_t)(PW * 16));
        bd = desc(b0 + (uint32_t)(tap * 2 * N * 16) % (uint32_t)(2 * N * 16 * 2), (uint32_t)(N * 16), 128);
        d = tmem + (uint32_t)(mt * N);
      }
      asm volatile(
          "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
          "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
          "l"(ad), "l"(bd), "r"(idesc), "r"(it >= NACC ? 1 : 0)
          : "memory");
      if (commit_every && (it + 1) % commit_every == 0)  // like the conv's per-stage commit
        asm volatile(
            "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                smem_u32(&bar2))
            : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(&bar))
                 : "memory");
    asm volatile(
        "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(
            smem_u32(&bar))
        : "memory");
    t1 = clock64();
    out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int N, int NACC, int MODE = 0, int M = 128>
void run(int sms, int a_stride, int commit_every = 0) {
  unsigned long long* d;
  cudaMalloc(&d, sms * 8);
  const int iters = 20000;
  const size_t smem = (12 * 1024 + 4 * N * 4) * 4 + 1024;
  cudaFuncSetAttribute(probe<N, NACC, MODE, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  probe<N, NACC, MODE, M><<<sms, 128, smem>>>(iters, d, a_stride, commit_every);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe<N, NACC, MODE, M><<<sms, 128, smem>>>(iters, d, a_stride, commit_every);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double flops = 2.0 * M * N * 8 * iters * sms;
  printf("M=%d commit/%d mode %d N=%3d acc-sets=%d a_step/PW=%3d: %.1f cycles/MMA, %.0f TFLOP/s  (%s)\n", M, commit_every, MODE, N, NACC, a_stride,
         (double)h / iters, flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<64, 1>(sms, 0);
  run<128, 1>(sms, 0);
  run<256, 1>(sms, 0);
  run<128, 4>(sms, 0);
  run<128, 1>(sms, 16);
  run<256, 2>(sms, 16);
  run<128, 4, 1>(sms, 10);  // conv 3x3: PW = 10
  run<128, 4, 1>(sms, 8);   // PW = 8 (SBO 128)
  run<128, 4, 1>(sms, 16);  // PW = 16 (SBO 256)
  run<64, 4, 1>(sms, 10);
  run<64, 1, 0, 64>(sms, 0);
  run<128, 1, 0, 64>(sms, 0);
  run<256, 1, 0, 64>(sms, 0);
  return 0;
}
