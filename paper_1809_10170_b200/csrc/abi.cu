// abi.cu -- the extern "C" boundary (include/dconv_cuda.h): argument
// validation with the reference's error semantics, kernel selection, and
// launch accounting.  No device memory is allocated here.
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <utility>
#include <vector>

#include "common.cuh"
#include "conv_kernels.h"
#include "layout_kernels.h"

namespace {
thread_local char g_detail[512] = "";
std::atomic<int64_t> g_launches{0};

inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

bool aligned32(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 31) == 0; }
bool aligned16(const void* p) {
  return (reinterpret_cast<uintptr_t>(p) & 15) == 0;
}
}  // namespace

namespace dconv_host {
bool pdl_enabled() {
  static const bool on = getenv("DCONV_NO_PDL") == nullptr;
  return on;
}

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_detail, sizeof(g_detail), fmt, ap);
  va_end(ap);
  return code;
}
int check_launch(const char* kernel) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    return set_error(DCONV_ECUDA, "%s: %s", kernel, cudaGetErrorString(e));
  return DCONV_OK;
}
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}

namespace {
std::mutex g_dev_mu;
std::vector<std::pair<int, int>> g_sms;                 // (device, SMs)
std::vector<std::pair<int, const void*>> g_attr_done;   // (device, kernel)
}  // namespace

int device_sms(int dev) {
  std::lock_guard<std::mutex> lock(g_dev_mu);
  for (const auto& e : g_sms)
    if (e.first == dev) return e.second;
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
      sms < 1) {
    cudaGetLastError();
    return 148;  // not cached: retried on the next call
  }
  g_sms.emplace_back(dev, sms);
  return sms;
}

bool first_use_on_device(const void* kernel, int dev) {
  std::lock_guard<std::mutex> lock(g_dev_mu);
  for (const auto& e : g_attr_done)
    if (e.first == dev && e.second == kernel) return false;
  g_attr_done.emplace_back(dev, kernel);
  return true;
}
}  // namespace dconv_host

using dconv_host::set_error;

#ifdef DCONV_DEBUG_OWNERSHIP
namespace dconv_dev {
__device__ OwnMap g_own = {nullptr, nullptr, 0};
}
#endif

extern "C" {

int dconv_conv_shape(int c_i, int c_o, int h_i, int w_i, int h_f, int w_f,
                     int s, int* h_o, int* w_o) {
  // ConvShape::ConvShape, shape.cpp:32-39
  if (!(c_i >= 1 && c_o >= 1 && h_i >= 1 && w_i >= 1 && h_f >= 1 && w_f >= 1))
    return set_error(DCONV_EINVAL_SHAPE, "ConvShape: all counts must be >= 1");
  if (s < 1) return set_error(DCONV_EINVAL_SHAPE, "ConvShape: stride must be >= 1");
  if (!(h_f <= h_i && w_f <= w_i))
    return set_error(DCONV_EINVAL_SHAPE,
                     "ConvShape: filter must fit inside the input");
  if ((h_i - h_f) % s != 0)
    return set_error(DCONV_EINVAL_SHAPE,
                     "ConvShape: (h_i - h_f) must be divisible by stride");
  if ((w_i - w_f) % s != 0)
    return set_error(DCONV_EINVAL_SHAPE,
                     "ConvShape: (w_i - w_f) must be divisible by stride");
  if (h_o) *h_o = (h_i - h_f) / s + 1;
  if (w_o) *w_o = (w_i - w_f) / s + 1;
  return DCONV_OK;
}

int64_t dconv_conv_flops(int c_i, int c_o, int h_o, int w_o, int h_f, int w_f) {
  return 2LL * c_i * c_o * h_o * w_o * h_f * w_f;  // reference.cpp:106-109
}

int dconv_conv_desc_init(dconv_conv_desc* d, int n, int c_i, int c_o, int h_i,
                         int w_i, int h_f, int w_f, int stride, int c_ib,
                         int c_ob) {
  if (!d) return set_error(DCONV_EPARAM, "desc is NULL");
  std::memset(d, 0, sizeof(*d));
  if (n < 1) return set_error(DCONV_EINVAL_SHAPE, "batch must be >= 1");
  if (c_ib < 1 || c_ob < 1)
    return set_error(DCONV_EPARAM, "block sizes must be >= 1");
  int h_o = 0, w_o = 0;
  const int rc = dconv_conv_shape(c_i, c_o, h_i, w_i, h_f, w_f, stride, &h_o, &w_o);
  if (rc) return rc;
  d->n = n; d->c_i = c_i; d->c_o = c_o; d->h_i = h_i; d->w_i = w_i;
  d->h_f = h_f; d->w_f = w_f; d->stride = stride; d->h_o = h_o; d->w_o = w_o;
  d->c_ib = c_ib; d->c_ob = c_ob;
  return DCONV_OK;
}

}  // extern "C"

namespace {

struct Resolved {
  int ib_n, jb_n, jb_begin, jb_count;
  int64_t in_img, in_blk, in_row, out_img, out_blk, out_row, sk_img, sk_blk,
      sk_row;
};

int resolve(const dconv_conv_desc* d, bool dense_input, int64_t dense_img,
            const void* in, const void* w, const void* skip, const void* out,
            Resolved* r) {
  if (!d) return set_error(DCONV_EPARAM, "desc is NULL");
  if (!in || !w || !out) return set_error(DCONV_EPARAM, "NULL tensor pointer");
  int h_o = 0, w_o = 0;
  int rc = dconv_conv_shape(d->c_i, d->c_o, d->h_i, d->w_i, d->h_f, d->w_f,
                            d->stride, &h_o, &w_o);
  if (rc) return rc;
  if (d->n < 1) return set_error(DCONV_EINVAL_SHAPE, "batch must be >= 1");
  if (h_o != d->h_o || w_o != d->w_o)
    return set_error(DCONV_EINVAL_SHAPE, "desc h_o/w_o inconsistent with ConvShape");
  if (d->c_ib < 1 || d->c_ob < 1)
    return set_error(DCONV_EPARAM, "block sizes must be >= 1");
  if (d->epilogue < 0 || d->epilogue > 7)
    return set_error(DCONV_EPARAM, "unknown epilogue %d", d->epilogue);
  const bool pool = (d->epilogue & DCONV_EPI_MAXPOOL) != 0;
  if (pool && ((d->h_o | d->w_o) & 1))
    return set_error(DCONV_EINVAL_SHAPE, "fused 2x2 max-pool needs an even output (%d x %d)",
                     d->h_o, d->w_o);
  const int ph = pool ? d->h_o / 2 : d->h_o, pw = pool ? d->w_o / 2 : d->w_o;
  if ((d->epilogue & DCONV_EPI_ADD) && !skip)
    return set_error(DCONV_EPARAM, "ADD epilogue needs a skip tensor");
  const int c_ib = dense_input ? d->c_i : d->c_ib;
  r->ib_n = (d->c_i + c_ib - 1) / c_ib;
  r->jb_n = (d->c_o + d->c_ob - 1) / d->c_ob;
  r->jb_begin = d->co_block_begin;
  r->jb_count = d->co_block_count ? d->co_block_count : r->jb_n - r->jb_begin;
  if (r->jb_begin < 0 || r->jb_count < 1 || r->jb_begin + r->jb_count > r->jb_n)
    return set_error(DCONV_EPARAM, "output block range [%d, %d) outside [0, %d)",
                     r->jb_begin, r->jb_begin + r->jb_count, r->jb_n);
  if (dense_input) {
    r->in_row = d->w_i;
    r->in_blk = (int64_t)d->h_i * d->w_i;  // channel plane
    r->in_img = dense_img ? dense_img : (int64_t)d->c_i * d->h_i * d->w_i;
  } else {
    r->in_row = d->in_row_stride ? d->in_row_stride : (int64_t)d->w_i * d->c_ib;
    r->in_blk = d->in_blk_stride ? d->in_blk_stride : (int64_t)d->h_i * r->in_row;
    r->in_img = d->in_img_stride ? d->in_img_stride : (int64_t)r->ib_n * r->in_blk;
    if (r->in_row < (int64_t)d->w_i * d->c_ib ||
        r->in_blk < (int64_t)d->h_i * r->in_row)
      return set_error(DCONV_ELAYOUT, "input view strides smaller than the map");
  }
  r->out_row = d->out_row_stride ? d->out_row_stride : (int64_t)pw * d->c_ob;
  r->out_blk = d->out_blk_stride ? d->out_blk_stride : (int64_t)ph * r->out_row;
  r->out_img = d->out_img_stride ? d->out_img_stride : (int64_t)r->jb_count * r->out_blk;
  r->sk_row = d->skip_row_stride ? d->skip_row_stride : (int64_t)d->w_o * d->c_ob;
  r->sk_blk = d->skip_blk_stride ? d->skip_blk_stride : (int64_t)d->h_o * r->sk_row;
  r->sk_img = d->skip_img_stride ? d->skip_img_stride : (int64_t)r->jb_count * r->sk_blk;
  if (r->out_row < (int64_t)pw * d->c_ob || r->out_blk < (int64_t)ph * r->out_row)
    return set_error(DCONV_ELAYOUT, "output view strides smaller than the map");
  return DCONV_OK;
}

}  // namespace

extern "C" {

namespace {
int check_peers(float* const* peers, int n_peers) {
  if (n_peers < 0 || n_peers > dconv_dev::kMaxPeers)
    return set_error(DCONV_EPARAM, "n_peers %d outside [0, %d]", n_peers, dconv_dev::kMaxPeers);
  if (n_peers && !peers) return set_error(DCONV_EPARAM, "NULL peer list");
  for (int i = 0; i < n_peers; ++i)
    if (!peers[i] || !aligned16(peers[i]))
      return set_error(DCONV_EPARAM, "peer output %d is NULL or not 16-byte aligned", i);
  return DCONV_OK;
}

int conv_direct_impl(const dconv_conv_desc* d, const float* in, const float* w,
                     const float* skip, float* out, float* const* peers, int n_peers,
                     void* stream) {
  if (int rc = check_peers(peers, n_peers)) return rc;
  if (d && (d->epilogue & DCONV_EPI_MAXPOOL) &&
      (n_peers || (d->epilogue & DCONV_EPI_ADD) || d->algo == DCONV_ALGO_GENERIC))
    return set_error(DCONV_EUNSUPPORTED,
                     "fused max-pool epilogue: FFMA/TF32 paths, no skip-add, no peers");
  Resolved r;
  int rc = resolve(d, false, 0, in, w, skip, out, &r);
  if (rc) return rc;
  // input / weight rows move by 16-byte bulk copies; output and skip pencils
  // (8 channels = 32 bytes = one sector) by one 256-bit access per lane
  bool peers32 = true;
  for (int i = 0; i < n_peers; ++i) peers32 = peers32 && aligned32(peers[i]);
  const bool ffma_ok =
      d->c_ib == d->c_ob && (d->c_ib == 8 || d->c_ib == 16 || d->c_ib == 32) &&
      aligned16(in) && aligned16(w) &&
      aligned32(out) && (!skip || aligned32(skip)) && peers32 &&
      ((r.in_img | r.in_blk | r.in_row) & 3) == 0 &&
      ((r.out_img | r.out_blk | r.out_row | r.sk_img | r.sk_blk | r.sk_row) & 7) == 0;
  int algo = d->algo;
  if (algo == DCONV_ALGO_AUTO) algo = ffma_ok ? DCONV_ALGO_FFMA : DCONV_ALGO_GENERIC;
  if (algo == DCONV_ALGO_FFMA) {
    if (!ffma_ok)
      return set_error(DCONV_EUNSUPPORTED,
                       "FFMA kernel needs c_ib == c_ob in {8, 16, 32}, 16-byte aligned "
                       "input / weights and pencil-aligned (32-byte) output / skip views "
                       "(got c_ib=%d c_ob=%d)", d->c_ib, d->c_ob);
    dconv_dev::FfmaParams p{};
    p.in = in; p.w = w; p.skip = skip; p.out = out;
    p.n = d->n; p.h_i = d->h_i; p.w_i = d->w_i; p.h_o = d->h_o; p.w_o = d->w_o;
    p.h_f = d->h_f; p.w_f = d->w_f; p.s = d->stride;
    p.cbs = d->c_ib;
    p.ib_n = r.ib_n; p.jb_n = r.jb_n; p.jb_begin = r.jb_begin; p.jb_count = r.jb_count;
    p.in_img = r.in_img; p.in_blk = r.in_blk; p.in_row = r.in_row;
    p.out_img = r.out_img; p.out_blk = r.out_blk; p.out_row = r.out_row;
    p.sk_img = r.sk_img; p.sk_blk = r.sk_blk; p.sk_row = r.sk_row;
    p.epi = d->epilogue;
    p.variant = d->tile_variant > 0 ? d->tile_variant - 1 : -1;
    p.n_peers = n_peers;
    for (int i = 0; i < n_peers; ++i) p.peer_out[i] = peers[i];
    rc = dconv_dev::launch_conv_ffma(p, as_stream(stream));
    // AUTO: a configuration whose stage cannot be staged in shared memory
    // (very large filters on tiny maps) runs on the generic kernel instead.
    if (rc != DCONV_EUNSUPPORTED || d->algo != DCONV_ALGO_AUTO) return rc;
    algo = DCONV_ALGO_GENERIC;
  }
  if (algo == DCONV_ALGO_GENERIC && (n_peers || (d->epilogue & DCONV_EPI_MAXPOOL)))
    return set_error(DCONV_EUNSUPPORTED,
                     "fused peer gather / max-pool need the FFMA kernel (c_b = 8)");
  if (algo == DCONV_ALGO_GENERIC) {
    dconv_dev::GenericParams p{};
    p.in = in; p.w = w; p.skip = skip; p.out = out;
    p.n = d->n; p.c_i = d->c_i; p.h_i = d->h_i; p.w_i = d->w_i;
    p.h_o = d->h_o; p.w_o = d->w_o; p.h_f = d->h_f; p.w_f = d->w_f;
    p.s = d->stride; p.c_ib = d->c_ib; p.c_ob = d->c_ob;
    p.ib_n = r.ib_n; p.jb_n = r.jb_n; p.jb_begin = r.jb_begin; p.jb_count = r.jb_count;
    p.in_img = r.in_img; p.in_blk = r.in_blk; p.in_row = r.in_row;
    p.out_img = r.out_img; p.out_blk = r.out_blk; p.out_row = r.out_row;
    p.sk_img = r.sk_img; p.sk_blk = r.sk_blk; p.sk_row = r.sk_row;
    p.epi = d->epilogue;
    return dconv_dev::launch_conv_generic(p, as_stream(stream));
  }
  return set_error(DCONV_EUNSUPPORTED, "algo %d not available", algo);
}
}  // namespace

int dconv_cuda_conv_direct(const dconv_conv_desc* d, const float* in, const float* w,
                           const float* skip, float* out, void* stream) {
  return conv_direct_impl(d, in, w, skip, out, nullptr, 0, stream);
}

int dconv_cuda_conv_direct_peers(const dconv_conv_desc* d, const float* in, const float* w,
                                 const float* skip, float* out, float* const* peer_outs,
                                 int n_peers, void* stream) {
  return conv_direct_impl(d, in, w, skip, out, peer_outs, n_peers, stream);
}

namespace {
int tf32_prepared_size_impl(const dconv_conv_desc* d, int64_t* floats, bool x3) {
  if (!d || !floats) return set_error(DCONV_EPARAM, "NULL argument");
  Resolved r;
  static const float dummy = 0.f;
  dconv_conv_desc geom = *d;  // geometry only: the epilogue is irrelevant here
  geom.epilogue = DCONV_EPI_NONE;
  int rc = resolve(&geom, false, 0, &dummy, &dummy, nullptr, &dummy, &r);
  if (rc) return rc;
  if (d->c_ib != 8 || d->c_ob != 8)
    return set_error(DCONV_EUNSUPPORTED, "TF32 path needs c_ib == c_ob == 8");
  int ib, hf, wf;
  dconv_dev::WSrc src;
  dconv_dev::tc_geometry(r.ib_n, d->h_f, d->w_f, d->stride, ib, hf, wf, src);
  *floats = x3 ? dconv_dev::tf32x3_prepared_floats(ib, hf, wf, r.jb_count)
               : dconv_dev::tf32_prepared_floats(ib, hf, wf, r.jb_count);
  return DCONV_OK;
}

int prepare_tf32_impl(const dconv_conv_desc* d, const float* w, float* w_prepared, void* stream,
                      bool x3) {
  Resolved r;
  if (!d) return set_error(DCONV_EPARAM, "NULL argument");
  dconv_conv_desc geom = *d;
  geom.epilogue = DCONV_EPI_NONE;
  int rc = resolve(&geom, false, 0, w, w, nullptr, w_prepared, &r);
  if (rc) return rc;
  if (d->c_ib != 8 || d->c_ob != 8)
    return set_error(DCONV_EUNSUPPORTED, "TF32 path needs c_ib == c_ob == 8");
  int ib, hf, wf;
  dconv_dev::WSrc src;
  dconv_dev::tc_geometry(r.ib_n, d->h_f, d->w_f, d->stride, ib, hf, wf, src);
  return x3 ? dconv_dev::launch_prepare_tf32x3(w, ib, hf, wf, r.jb_begin, r.jb_count, src,
                                               w_prepared, as_stream(stream))
            : dconv_dev::launch_prepare_tf32(w, ib, hf, wf, r.jb_begin, r.jb_count, src,
                                             w_prepared, as_stream(stream));
}

int conv_tf32_impl(const dconv_conv_desc* d, const float* in, const float* w_prepared,
                   const float* skip, float* out, void* stream, bool x3) {
  Resolved r;
  int rc = resolve(d, false, 0, in, w_prepared, skip, out, &r);
  if (rc) return rc;
  if (d->c_ib != 8 || d->c_ob != 8 || !aligned16(in) || !aligned16(w_prepared) ||
      !aligned32(out) || (skip && !aligned32(skip)) ||
      ((r.in_img | r.in_blk | r.in_row) & 3) != 0 ||
      ((r.out_img | r.out_blk | r.out_row | r.sk_img | r.sk_blk | r.sk_row) & 7) != 0)
    return set_error(DCONV_EUNSUPPORTED,
                     "TF32 path needs c_ib == c_ob == 8, 16-byte aligned input and "
                     "pencil-aligned (32-byte) output / skip views");
  dconv_dev::FfmaParams p{};
  p.in = in; p.w = nullptr; p.skip = skip; p.out = out;
  p.n = d->n; p.h_i = d->h_i; p.w_i = d->w_i; p.h_o = d->h_o; p.w_o = d->w_o;
  p.h_f = d->h_f; p.w_f = d->w_f; p.s = d->stride;
  p.cbs = 8;
  p.ib_n = r.ib_n; p.jb_n = r.jb_n; p.jb_begin = r.jb_begin; p.jb_count = r.jb_count;
  p.in_img = r.in_img; p.in_blk = r.in_blk; p.in_row = r.in_row;
  p.out_img = r.out_img; p.out_blk = r.out_blk; p.out_row = r.out_row;
  p.sk_img = r.sk_img; p.sk_blk = r.sk_blk; p.sk_row = r.sk_row;
  p.epi = d->epilogue;
  return x3 ? dconv_dev::launch_conv_tf32x3(p, w_prepared, as_stream(stream))
            : dconv_dev::launch_conv_tf32(p, w_prepared, as_stream(stream));
}
}  // namespace

int dconv_cuda_tf32_prepared_size(const dconv_conv_desc* d, int64_t* floats) {
  return tf32_prepared_size_impl(d, floats, false);
}
int dconv_cuda_prepare_tf32_weights(const dconv_conv_desc* d, const float* w,
                                    float* w_prepared, void* stream) {
  return prepare_tf32_impl(d, w, w_prepared, stream, false);
}
int dconv_cuda_conv_direct_tf32(const dconv_conv_desc* d, const float* in,
                                const float* w_prepared, const float* skip, float* out,
                                void* stream) {
  return conv_tf32_impl(d, in, w_prepared, skip, out, stream, false);
}
int dconv_cuda_tf32x3_prepared_size(const dconv_conv_desc* d, int64_t* floats) {
  return tf32_prepared_size_impl(d, floats, true);
}
int dconv_cuda_prepare_tf32x3_weights(const dconv_conv_desc* d, const float* w,
                                      float* w_prepared, void* stream) {
  return prepare_tf32_impl(d, w, w_prepared, stream, true);
}
int dconv_cuda_conv_direct_tf32x3(const dconv_conv_desc* d, const float* in,
                                  const float* w_prepared, const float* skip, float* out,
                                  void* stream) {
  return conv_tf32_impl(d, in, w_prepared, skip, out, stream, true);
}

namespace {
int conv_first_impl(const dconv_conv_desc* d, const float* in_dense, int64_t in_img_stride,
                    const float* w, const float* skip, float* out, float* const* peers,
                    int n_peers, void* stream) {
  if (int rc = check_peers(peers, n_peers)) return rc;
  if (d && (d->epilogue & DCONV_EPI_MAXPOOL))
    return set_error(DCONV_EUNSUPPORTED, "fused max-pool epilogue: TF32 path only");
  Resolved r;
  int rc = resolve(d, true, in_img_stride, in_dense, w, skip, out, &r);
  if (rc) return rc;
  dconv_dev::GenericParams p{};
  p.in = in_dense; p.w = w; p.skip = skip; p.out = out;
  p.n = d->n; p.c_i = d->c_i; p.h_i = d->h_i; p.w_i = d->w_i;
  p.h_o = d->h_o; p.w_o = d->w_o; p.h_f = d->h_f; p.w_f = d->w_f;
  p.s = d->stride; p.c_ib = d->c_i; p.c_ob = d->c_ob;
  p.ib_n = 1; p.jb_n = r.jb_n; p.jb_begin = r.jb_begin; p.jb_count = r.jb_count;
  p.in_img = r.in_img; p.in_blk = r.in_blk; p.in_row = r.in_row;
  p.out_img = r.out_img; p.out_blk = r.out_blk; p.out_row = r.out_row;
  p.sk_img = r.sk_img; p.sk_blk = r.sk_blk; p.sk_row = r.sk_row;
  p.epi = d->epilogue;
  p.dense_input = 1;
  p.n_peers = n_peers;
  for (int i = 0; i < n_peers; ++i) p.peer_out[i] = peers[i];
  const bool fast_ok = d->c_ob == 8 && aligned16(w) && aligned16(out) &&
                       (!skip || aligned16(skip)) &&
                       ((r.out_img | r.out_blk | r.out_row | r.sk_img | r.sk_blk |
                         r.sk_row) & 3) == 0;
  static const bool no_reader = getenv("DCONV_NO_READER") != nullptr;
  if (fast_ok && d->algo != DCONV_ALGO_GENERIC && n_peers && !no_reader) {
    // the TMA-store reader writes this rank's map only: run it there, then
    // copy the rank's blocks into the peers' maps, so every copy holds the
    // same values as the all-gather of readers' slices (bitwise)
    dconv_dev::GenericParams local = p;
    local.n_peers = 0;
    rc = dconv_dev::launch_conv_reader(local, as_stream(stream));
    if (rc == DCONV_OK)
      return dconv_dev::launch_copy_pencils_peers(out, d->n, r.jb_count, d->h_o, d->w_o,
                                                  r.out_img, r.out_blk, r.out_row, peers,
                                                  n_peers, as_stream(stream));
    if (rc != DCONV_EUNSUPPORTED) return rc;
  }
  if (fast_ok && d->algo != DCONV_ALGO_GENERIC) {
    rc = dconv_dev::launch_conv_first_fast(p, as_stream(stream));
    if (rc != DCONV_EUNSUPPORTED) return rc;
  }
  if (n_peers)
    return set_error(DCONV_EUNSUPPORTED, "fused peer gather needs the register-tiled first-layer reader");
  return dconv_dev::launch_conv_first_layer(p, as_stream(stream));
}
}  // namespace

int dconv_cuda_conv_first_layer(const dconv_conv_desc* d, const float* in_dense,
                                int64_t in_img_stride, const float* w, const float* skip,
                                float* out, void* stream) {
  return conv_first_impl(d, in_dense, in_img_stride, w, skip, out, nullptr, 0, stream);
}

int dconv_cuda_conv_first_layer_peers(const dconv_conv_desc* d, const float* in_dense,
                                      int64_t in_img_stride, const float* w,
                                      const float* skip, float* out, float* const* peer_outs,
                                      int n_peers, void* stream) {
  return conv_first_impl(d, in_dense, in_img_stride, w, skip, out, peer_outs, n_peers, stream);
}

int dconv_cuda_pack_kernel(const float* src, int c_i, int c_o, int h_f, int w_f,
                           int c_ob, int c_ib, float* dst, void* stream) {
  if (!src || !dst) return set_error(DCONV_EPARAM, "NULL tensor pointer");
  if (c_i < 1 || c_o < 1 || h_f < 1 || w_f < 1)
    return set_error(DCONV_EINVAL_SHAPE, "BlockedKernel: dims must be >= 1");
  if (c_ob < 1 || c_ib < 1)
    return set_error(DCONV_EPARAM, "BlockedKernel: block sizes must be >= 1");
  return dconv_dev::launch_pack_kernel(src, c_i, c_o, h_f, w_f, c_ob, c_ib, dst,
                                       as_stream(stream));
}

int dconv_cuda_unpack_kernel(const float* src, int c_i, int c_o, int h_f,
                             int w_f, int c_ob, int c_ib, float* dst,
                             void* stream) {
  if (!src || !dst) return set_error(DCONV_EPARAM, "NULL tensor pointer");
  if (c_i < 1 || c_o < 1 || h_f < 1 || w_f < 1)
    return set_error(DCONV_EINVAL_SHAPE, "KernelTensor: dims must be >= 1");
  if (c_ob < 1 || c_ib < 1)
    return set_error(DCONV_EPARAM, "BlockedKernel: block sizes must be >= 1");
  return dconv_dev::launch_unpack_kernel(src, c_i, c_o, h_f, w_f, c_ob, c_ib,
                                         dst, as_stream(stream));
}

int dconv_cuda_pack_space_to_depth(const float* src, int n, int c, int h, int w, int f,
                                   float* dst, void* stream) {
  if (!src || !dst) return set_error(DCONV_EPARAM, "NULL tensor pointer");
  if (n < 1 || c < 1 || h < 1 || w < 1 || f < 1)
    return set_error(DCONV_EINVAL_SHAPE, "space-to-depth: dims must be >= 1");
  if (reinterpret_cast<uintptr_t>(dst) & 15)
    return set_error(DCONV_EPARAM, "space-to-depth: destination must be 16-byte aligned");
  return dconv_dev::launch_pack_s2d(src, n, c, h, w, f, dst, as_stream(stream));
}

int dconv_cuda_space_to_depth_blocked(const float* src, int64_t in_img_stride,
                                      int64_t in_blk_stride, int64_t in_row_stride, int n, int c,
                                      int h, int w, int f, float* dst, void* stream) {
  if (!src || !dst) return set_error(DCONV_EPARAM, "NULL tensor pointer");
  if (n < 1 || c < 1 || h < 1 || w < 1 || f < 1)
    return set_error(DCONV_EINVAL_SHAPE, "space-to-depth: dims must be >= 1");
  if (in_row_stride < (int64_t)w * 8 || in_blk_stride < (int64_t)h * in_row_stride ||
      in_img_stride < (int64_t)((c + 7) / 8) * in_blk_stride)
    return set_error(DCONV_ELAYOUT, "space-to-depth: input view strides smaller than the map");
  if (reinterpret_cast<uintptr_t>(dst) & 15)
    return set_error(DCONV_EPARAM, "space-to-depth: destination must be 16-byte aligned");
  return dconv_dev::launch_s2d_blocked(src, in_img_stride, in_blk_stride, in_row_stride, n, c, h,
                                       w, f, dst, as_stream(stream));
}

int dconv_cuda_pack_feature_map(const float* src, int n, int c, int h, int w,
                                int c_b, int halo, float* dst, void* stream) {
  if (!src || !dst) return set_error(DCONV_EPARAM, "NULL tensor pointer");
  if (n < 1 || c < 1 || h < 1 || w < 1)
    return set_error(DCONV_EINVAL_SHAPE, "BlockedFeatureMap: dims must be >= 1");
  if (c_b < 1) return set_error(DCONV_EPARAM, "BlockedFeatureMap: block size must be >= 1");
  if (halo < 0) return set_error(DCONV_EPARAM, "halo must be >= 0");
  return dconv_dev::launch_pack_fm(src, n, c, h, w, c_b, halo, dst,
                                   as_stream(stream));
}

int dconv_cuda_unpack_feature_map(const float* src, int n, int c, int h, int w,
                                  int c_b, int halo, float* dst, void* stream) {
  if (!src || !dst) return set_error(DCONV_EPARAM, "NULL tensor pointer");
  if (n < 1 || c < 1 || h < 1 || w < 1)
    return set_error(DCONV_EINVAL_SHAPE, "FeatureMap: dims must be >= 1");
  if (c_b < 1) return set_error(DCONV_EPARAM, "BlockedFeatureMap: block size must be >= 1");
  if (halo < 0) return set_error(DCONV_EPARAM, "halo must be >= 0");
  return dconv_dev::launch_unpack_fm(src, n, c, h, w, c_b, halo, dst,
                                     as_stream(stream));
}

int dconv_cuda_relu_blocked(float* x, int64_t count, void* stream) {
  if (!x) return set_error(DCONV_EPARAM, "NULL tensor pointer");
  if (count <= 0) return DCONV_OK;
  return dconv_dev::launch_relu(x, count, as_stream(stream));
}

int dconv_cuda_add_blocked(const float* a, const float* b, float* out,
                           int64_t count, int relu, void* stream) {
  if (!a || !b || !out) return set_error(DCONV_EPARAM, "NULL tensor pointer");
  if (count <= 0) return DCONV_OK;
  return dconv_dev::launch_add(a, b, out, count, relu, as_stream(stream));
}

int dconv_cuda_maxpool2x2_blocked(const float* in, int n, int n_blocks, int h,
                                  int w, int c_b, float* out,
                                  int64_t out_img_stride,
                                  int64_t out_blk_stride,
                                  int64_t out_row_stride, void* stream) {
  if (!in || !out) return set_error(DCONV_EPARAM, "NULL tensor pointer");
  if (n < 1 || n_blocks < 1 || h < 2 || w < 2 || c_b < 1)
    return set_error(DCONV_EINVAL_SHAPE, "maxpool2x2: bad dims");
  const int64_t row = out_row_stride ? out_row_stride : (int64_t)(w / 2) * c_b;
  const int64_t blk = out_blk_stride ? out_blk_stride : (int64_t)(h / 2) * row;
  const int64_t img = out_img_stride ? out_img_stride : (int64_t)n_blocks * blk;
  return dconv_dev::launch_maxpool2x2(in, n, n_blocks, h, w, c_b, out, img, blk,
                                      row, as_stream(stream));
}

int dconv_cuda_zero(float* x, int64_t count, void* stream) {
  if (!x) return set_error(DCONV_EPARAM, "NULL tensor pointer");
  if (count <= 0) return DCONV_OK;
  if (cudaMemsetAsync(x, 0, sizeof(float) * count, as_stream(stream)) != cudaSuccess)
    return dconv_host::check_launch("cudaMemsetAsync");
  return DCONV_OK;
}

int dconv_debug_set_ownership(unsigned* counts, const float* base, int64_t n) {
#ifdef DCONV_DEBUG_OWNERSHIP
  const dconv_dev::OwnMap m{counts, base, (long long)n};
  const cudaError_t e = cudaMemcpyToSymbol(dconv_dev::g_own, &m, sizeof(m));
  if (e != cudaSuccess) return set_error(DCONV_ECUDA, "ownership map: %s", cudaGetErrorString(e));
  return DCONV_OK;
#else
  (void)counts; (void)base; (void)n;
  return set_error(DCONV_EUNSUPPORTED, "not an ownership-debug build (make own)");
#endif
}

int dconv_cuda_ffma_cluster_slots(int tile_variant, int ks, int* cached, int* fresh) {
  if (!cached || !fresh) return set_error(DCONV_EPARAM, "null output");
  return dconv_dev::ffma_cluster_slots_probe(tile_variant, ks, cached, fresh);
}

int64_t dconv_cuda_launch_count(void) {
  return g_launches.load(std::memory_order_relaxed);
}

double dconv_cuda_fp32_peak_probe(void* stream) {
  return dconv_dev::fp32_peak_probe(as_stream(stream));
}

double dconv_cuda_ffma2_pattern_probe(void* stream) {
  return dconv_dev::ffma2_pattern_probe(as_stream(stream));
}

const char* dconv_cuda_strerror(int code) {
  switch (code) {
    case DCONV_OK: return "ok";
    case DCONV_EINVAL_SHAPE: return "invalid shape";
    case DCONV_ELAYOUT: return "layout error";
    case DCONV_EPARAM: return "parameter error";
    case DCONV_ECUDA: return "CUDA error";
    case DCONV_ENCCL: return "NCCL error";
    case DCONV_EUNSUPPORTED: return "unsupported configuration";
    case DCONV_EFORMAT: return "parse error";
    case DCONV_EBLOCKED: return "already blocked";
    case DCONV_EIO: return "I/O error";
    default: return "unknown error";
  }
}

const char* dconv_cuda_last_error_detail(void) { return g_detail; }

}  // extern "C"
