// common.cuh -- sm_100a PTX helpers shared by the dconv kernels:
// mbarrier pipeline primitives and 1-D bulk async copies (cp.async.bulk,
// SASS UBLKCP) global -> shared with transaction-count completion.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "dconv_cuda.h"

namespace dconv_dev {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar,
                                                      uint32_t bytes) {
  asm volatile(
      "mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
          smem_u32(bar)),
      "r"(bytes)
      : "memory");
}

// ---- cluster (DSMEM) helpers ------------------------------------------------
__device__ __forceinline__ uint32_t mapa(uint32_t smem_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr), "r"(rank));
  return r;
}
// arrive (release at cluster scope) on the same mbarrier of CTA `rank`
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* bar, uint32_t rank) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                   mapa(smem_u32(bar), rank))
               : "memory");
}
// relaxed arrive on CTA `rank`'s barrier: pair with one fence_cluster() after
// the writes it publishes (one fence for many arrives)
__device__ __forceinline__ void mbar_arrive_remote_relaxed(uint64_t* bar, uint32_t rank) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                   mapa(smem_u32(bar), rank))
               : "memory");
}
__device__ __forceinline__ void fence_cluster() {
  asm volatile("fence.acq_rel.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITC_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAITC_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ float ld_dsmem(const float* local_equiv, uint32_t rank) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];"
               : "=f"(v)
               : "r"(mapa(smem_u32(local_equiv), rank))
               : "memory");
  return v;
}
// 16-byte store into CTA `rank`'s shared memory (same offset as local_equiv)
__device__ __forceinline__ void st_dsmem4(float* local_equiv, uint32_t rank, float4 v) {
  asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(
                   mapa(smem_u32(local_equiv), rank)),
               "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
// split cluster barrier: arrive early (non-blocking), wait just before the
// first remote access
__device__ __forceinline__ void cluster_arrive_release() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait_acquire() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Wait with back-off: for roles that idle for long stretches (epilogue
// waiting on a whole accumulator, producer far ahead), so their polling does
// not compete with the warps doing the work.
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred p;\nmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* bar, uint32_t parity, int ns) {
  while (!mbar_try(bar, parity)) __nanosleep(ns);
}

// 1-D bulk copy global -> shared::cta, completion signalled on `bar` as
// transaction bytes.  dst/src 16-byte aligned, bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src,
                                         uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// 4-byte async global->shared copy; zero-fills when !valid (src not read).
__device__ __forceinline__ void cp_async4(float* dst, const float* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(valid ? 4 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Programmatic dependent launch: a kernel launched with the
// programmatic-stream-serialization attribute may start while the previous
// kernel in the stream is still running; it must pdl_wait() before touching
// data that kernel produces.  pdl_launch_dependents() lets the next kernel
// start launching (it still waits for this grid in its own pdl_wait).
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Warm L2 with [src, src + bytes) (bytes a multiple of 16); no completion.
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// fp32 pair helpers: acc.{lo,hi} += a * b.{lo,hi} as one FFMA2 (RN per lane,
// bitwise identical to two fmaf).  ptxas folds the {a, a} pair into the
// FFMA2 scalar-broadcast operand form, so no MOV is emitted.
__device__ __forceinline__ uint64_t pack2(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float2 unpack2(uint64_t v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
__device__ __forceinline__ void ffma2(uint64_t& acc, float a, uint64_t b) {
  asm("{\n.reg .b64 aa;\nmov.b64 aa, {%1, %1};\nfma.rn.f32x2 %0, aa, %2, %0;\n}"
      : "+l"(acc)
      : "f"(a), "l"(b));
}

__device__ __forceinline__ float4 lds128(const float* p) {
  return *reinterpret_cast<const float4*>(p);
}

// One 8-channel pencil (32 bytes = one DRAM / L2 sector) from / to global
// memory in a single 256-bit access per lane (sm_100 LDG.256 / STG.256); two
// 128-bit halves would touch every sector twice, half a sector each time.
// The pencil must be 32-byte aligned (abi.cu checks the views).
__device__ __forceinline__ void ldg_pencil(const float* p, float4& a, float4& b) {
  asm("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
      : "l"(p));
}
__device__ __forceinline__ void stg_pencil(float* p, const float (&v)[8]) {
  asm volatile("st.global.v8.f32 [%8], {%0, %1, %2, %3, %4, %5, %6, %7};" ::"f"(v[0]), "f"(v[1]),
               "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "l"(p)
               : "memory");
}

// Write-ownership debug build (make own -> libdconv_b200_own.so, compiled
// with -DDCONV_DEBUG_OWNERSHIP -rdc=true): every store of a conv output
// element also counts itself in a map set by dconv_debug_set_ownership, so a
// test can assert that each element of the output view is written exactly
// once -- the GPU analogue of the reference's debug ownership map
// (SPEC.md:350).  The product build compiles the hook to nothing.
#ifdef DCONV_DEBUG_OWNERSHIP
struct OwnMap {
  unsigned* counts;
  const float* base;
  long long n;
};
extern __device__ OwnMap g_own;
__device__ __forceinline__ void own_mark(const float* p, int nf) {
  const OwnMap m = g_own;
  if (!m.counts) return;
  const long long i = p - m.base;
  for (int k = 0; k < nf; ++k)
    if (i + k >= 0 && i + k < m.n) atomicAdd(&m.counts[i + k], 1u);
}
#define DCONV_OWN(p, nf) ::dconv_dev::own_mark((p), (nf))
#else
#define DCONV_OWN(p, nf) ((void)0)
#endif

}  // namespace dconv_dev

// Host-side helpers shared by the launchers (defined in abi.cu).
namespace dconv_host {
bool pdl_enabled();  // DCONV_NO_PDL unset
int set_error(int code, const char* fmt, ...);
int check_launch(const char* kernel);
void count_launch();
// current device and its SM count (cached per device)
int current_device();
int device_sms(int dev);
// true exactly once per (kernel, device): the caller then sets that kernel's
// function attributes on the current device (attributes are per device)
bool first_use_on_device(const void* kernel, int dev);
}  // namespace dconv_host
