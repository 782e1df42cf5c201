// ref_shim.cpp -- extern "C" shim over the UNMODIFIED reference sources
// (/root/reference/proj/core/src/{shape,tensor,reference,thread_pool}.cpp),
// compiled in place by oracle/Makefile into oracle/_ref/libdconv_ref.so.
// TEST INFRASTRUCTURE ONLY: used to pin oracle/oracle.c and as the
// "reference" CPU timing of Alg. 2 (conv_reordered).  No reference source is
// copied into this repository; this file only calls the reference's API.
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "dconv/reference.hpp"
#include "dconv/shape.hpp"
#include "dconv/tensor.hpp"
#include "dconv/thread_pool.hpp"
#include "oracle.h"

using namespace dconv;

namespace {
FeatureMap make_fm(const float* p, int c, int h, int w) {
  FeatureMap f(c, h, w);
  std::memcpy(f.data.data(), p, sizeof(float) * f.data.size());
  return f;
}
KernelTensor make_k(const float* p, int ci, int co, int hf, int wf) {
  KernelTensor k(ci, co, hf, wf);
  std::memcpy(k.data.data(), p, sizeof(float) * k.data.size());
  return k;
}
}  // namespace

extern "C" {

// ConvShape ctor (shape.cpp:30-40); -1 when it throws std::invalid_argument.
int ref_conv_shape(int ci, int co, int hi, int wi, int hf, int wf, int s,
                   int* ho, int* wo) {
  try {
    ConvShape sh(ci, co, hi, wi, hf, wf, s);
    *ho = sh.h_o;
    *wo = sh.w_o;
    return 0;
  } catch (const std::invalid_argument&) {
    return -1;
  }
}

int64_t ref_conv_flops(int ci, int co, int hi, int wi, int hf, int wf, int s) {
  return conv_flops(ConvShape(ci, co, hi, wi, hf, wf, s));
}

// mode 0 = conv_oracle64, 1 = conv_naive, 2 = conv_reordered
int ref_conv(int mode, const float* in, const float* k, int ci, int co, int hi,
             int wi, int hf, int wf, int s, float* out) {
  try {
    ConvShape sh(ci, co, hi, wi, hf, wf, s);
    FeatureMap x = make_fm(in, ci, hi, wi);
    KernelTensor kt = make_k(k, ci, co, hf, wf);
    FeatureMap y = mode == 0   ? conv_oracle64(x, kt, sh)
                   : mode == 1 ? conv_naive(x, kt, sh)
                               : conv_reordered(x, kt, sh);
    std::memcpy(out, y.data.data(), sizeof(float) * y.data.size());
    return 0;
  } catch (const std::invalid_argument&) {
    return -1;
  }
}

void ref_pack_feature_map(const float* src, int c, int h, int w, int cb,
                          float* dst) {
  BlockedFeatureMap b = pack_feature_map(make_fm(src, c, h, w), cb);
  std::memcpy(dst, b.data.data(), sizeof(float) * b.data.size());
}

void ref_unpack_feature_map(const float* src, int c, int h, int w, int cb,
                            float* dst) {
  BlockedFeatureMap b(c, h, w, cb);
  std::memcpy(b.data.data(), src, sizeof(float) * b.data.size());
  FeatureMap f = unpack_feature_map(b);
  std::memcpy(dst, f.data.data(), sizeof(float) * f.data.size());
}

void ref_pack_kernel(const float* src, int ci, int co, int hf, int wf, int cob,
                     int cib, float* dst) {
  BlockedKernel b = pack_kernel(make_k(src, ci, co, hf, wf), cob, cib);
  std::memcpy(dst, b.data.data(), sizeof(float) * b.data.size());
}

void ref_unpack_kernel(const float* src, int ci, int co, int hf, int wf,
                       int cob, int cib, float* dst) {
  BlockedKernel b(ci, co, hf, wf, cob, cib);
  std::memcpy(b.data.data(), src, sizeof(float) * b.data.size());
  KernelTensor k = unpack_kernel(b);
  std::memcpy(dst, k.data.data(), sizeof(float) * k.data.size());
}

uint64_t ref_layout_transform_count() { return layout_transform_count(); }

size_t ref_blocked_kernel_offset(int ci, int co, int hf, int wf, int cob,
                                 int cib, int jb, int ib, int n, int m, int ii,
                                 int jj) {
  BlockedKernel b(ci, co, hf, wf, cob, cib);
  return b.offset(jb, ib, n, m, ii, jj);
}

// Reference Alg. 2 (conv_reordered, reference.cpp:54-68) over a batch of
// dense CHW images, one image per ThreadPool chunk (thread_pool.cpp:64-97):
// the reference's own CPU code on all host threads, used only as a timed
// CPU baseline.
struct BatchCtx {
  const float* in;
  const float* k;
  float* out;
  const ConvShape* sh;
  size_t in_img, out_img;
};
static void batch_task(void* p, int chunk) {
  BatchCtx* c = static_cast<BatchCtx*>(p);
  FeatureMap x = make_fm(c->in + chunk * c->in_img, c->sh->c_i, c->sh->h_i,
                         c->sh->w_i);
  KernelTensor kt = make_k(c->k, c->sh->c_i, c->sh->c_o, c->sh->h_f, c->sh->w_f);
  FeatureMap y = conv_reordered(x, kt, *c->sh);
  std::memcpy(c->out + chunk * c->out_img, y.data.data(),
              sizeof(float) * y.data.size());
}
int ref_conv_reordered_batch(const float* in, const float* k, int n_img,
                             int ci, int co, int hi, int wi, int hf, int wf,
                             int s, int threads, float* out) {
  try {
    ConvShape sh(ci, co, hi, wi, hf, wf, s);
    static ThreadPool* pool = nullptr;
    if (!pool) pool = new ThreadPool(threads > 1 ? threads - 1 : 0);
    pool->ensure(threads > 1 ? threads - 1 : 0);
    BatchCtx c{in, k, out, &sh, size_t(ci) * hi * wi,
               size_t(co) * sh.h_o * sh.w_o};
    pool->run(n_img, batch_task, &c);
    return 0;
  } catch (const std::invalid_argument&) {
    return -1;
  }
}

// Restated Alg. 3 (oracle.c, orc_direct_job_*) scheduled on the reference's
// own ThreadPool (thread_pool.cpp:64-97): `workers` pool threads + the
// calling thread (the caller participates, thread_pool.cpp:84-90), i.e. the
// reference's runtime with DCONV_THREADS = workers (thread_pool.cpp:23-30).
// The CPU baseline the BASELINE.md plan asks for; outputs are identical to
// orc_conv_direct (same units, same per-element order).
static void direct_task(void* p, int chunk) {
  orc_direct_job_unit(static_cast<const orc_direct_job*>(p), chunk);
}
int ref_pool_conv_direct(const float* in, const float* k, int n_img, int ci, int co,
                         int hi, int wi, int hf, int wf, int s, int cib, int cob,
                         int wob, int workers, float* out) {
  static ThreadPool* pool = nullptr;
  if (!pool) pool = new ThreadPool(workers);
  pool->ensure(workers);
  orc_direct_job job;
  const int units = orc_direct_job_init(&job, in, k, n_img, ci, co, hi, wi, hf, wf, s, cib,
                                        cob, wob, workers + 1, out);
  if (units < 0) return -1;
  pool->run(units, direct_task, &job);
  return 0;
}

}  // extern "C"
