// dropin.cpp -- the reference's C++ operator API (include/dconv/*.hpp) on
// top of the C-ABI (include/dconv_cuda.h).  Every transform and convolution
// runs as a CUDA kernel; host-value overloads stage their operands through
// device memory (one upload, one download), mirroring the reference's
// by-value contract (tensor.hpp:143-159).
#include <atomic>
#include <cstring>
#include <stdexcept>
#include <string>

#include <cuda_runtime.h>

#include "dconv/direct.hpp"
#include "dconv_cuda.h"

namespace dconv {

namespace {

std::atomic<std::uint64_t> g_layout_transforms{0};  // tensor.cpp:26 semantics

void require(bool ok, const char* what) {
  if (!ok) throw std::invalid_argument(what);
}

// Map a C-ABI code back to the reference's exception types.
void check(int rc) {
  if (rc == DCONV_OK) return;
  std::string msg = std::string(dconv_cuda_strerror(rc)) + ": " + dconv_cuda_last_error_detail();
  if (rc == DCONV_EINVAL_SHAPE || rc == DCONV_ELAYOUT || rc == DCONV_EPARAM)
    throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// RAII device buffer used by the host-value overloads.
struct DevBuf {
  float* p = nullptr;
  explicit DevBuf(std::size_t n) {
    if (n) cuda_check(cudaMalloc(&p, n * sizeof(float)), "cudaMalloc");
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  void up(const std::vector<float>& h) {
    cuda_check(cudaMemcpy(p, h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice),
               "cudaMemcpy H2D");
  }
  void down(std::vector<float>& h) const {
    cuda_check(cudaMemcpy(h.data(), p, h.size() * sizeof(float), cudaMemcpyDeviceToHost),
               "cudaMemcpy D2H");
  }
};

}  // namespace

// ------------------------------------------------------------------ shape
ConvShape::ConvShape(int ci, int co, int hi, int wi, int hf, int wf, int s)
    : c_i(ci), c_o(co), h_i(hi), w_i(wi), h_f(hf), w_f(wf), stride(s), h_o(0), w_o(0) {
  // shape.cpp:30-40 rules, evaluated by the C-ABI so both layers agree
  const int rc = dconv_conv_shape(ci, co, hi, wi, hf, wf, s, &h_o, &w_o);
  if (rc != DCONV_OK) throw std::invalid_argument(dconv_cuda_last_error_detail());
}

// ------------------------------------------------------------------ tensors
FeatureMap::FeatureMap(int c, int h, int w) : channels(c), height(h), width(w) {
  require(c >= 1 && h >= 1 && w >= 1, "FeatureMap: dims must be >= 1");
  data.assign(std::size_t(c) * h * w, 0.0f);
}

BlockedFeatureMap::BlockedFeatureMap(int c, int h, int w, int cb)
    : channels(c), height(h), width(w), c_b(cb) {
  require(c >= 1 && h >= 1 && w >= 1, "BlockedFeatureMap: dims must be >= 1");
  require(cb >= 1, "BlockedFeatureMap: block size must be >= 1");
  padded_channels = detail::round_up(c, cb);
  data.assign(std::size_t(padded_channels) * h * w, 0.0f);
}

KernelTensor::KernelTensor(int ci, int co, int hf, int wf) : c_i(ci), c_o(co), h_f(hf), w_f(wf) {
  require(ci >= 1 && co >= 1 && hf >= 1 && wf >= 1, "KernelTensor: dims must be >= 1");
  data.assign(std::size_t(ci) * co * hf * wf, 0.0f);
}

BlockedKernel::BlockedKernel(int ci, int co, int hf, int wf, int cob, int cib)
    : c_i(ci), c_o(co), h_f(hf), w_f(wf), c_ob(cob), c_ib(cib) {
  require(ci >= 1 && co >= 1 && hf >= 1 && wf >= 1, "BlockedKernel: dims must be >= 1");
  require(cob >= 1 && cib >= 1, "BlockedKernel: block sizes must be >= 1");
  padded_c_i = detail::round_up(ci, cib);
  padded_c_o = detail::round_up(co, cob);
  data.assign(std::size_t(padded_c_i) * padded_c_o * hf * wf, 0.0f);
}

BlockedFeatureMap pack_feature_map(const FeatureMap& src, int c_b) {
  g_layout_transforms.fetch_add(1, std::memory_order_relaxed);
  BlockedFeatureMap dst(src.channels, src.height, src.width, c_b);
  DevBuf s(src.data.size()), d(dst.data.size());
  s.up(src.data);
  check(dconv_cuda_pack_feature_map(s.p, 1, src.channels, src.height, src.width, c_b, 0, d.p,
                                    nullptr));
  d.down(dst.data);
  return dst;
}

FeatureMap unpack_feature_map(const BlockedFeatureMap& src) {
  g_layout_transforms.fetch_add(1, std::memory_order_relaxed);
  FeatureMap dst(src.channels, src.height, src.width);
  DevBuf s(src.data.size()), d(dst.data.size());
  s.up(src.data);
  check(dconv_cuda_unpack_feature_map(s.p, 1, src.channels, src.height, src.width, src.c_b, 0,
                                      d.p, nullptr));
  d.down(dst.data);
  return dst;
}

BlockedKernel pack_kernel(const KernelTensor& src, int c_ob, int c_ib) {
  g_layout_transforms.fetch_add(1, std::memory_order_relaxed);
  BlockedKernel dst(src.c_i, src.c_o, src.h_f, src.w_f, c_ob, c_ib);
  DevBuf s(src.data.size()), d(dst.data.size());
  s.up(src.data);
  check(dconv_cuda_pack_kernel(s.p, src.c_i, src.c_o, src.h_f, src.w_f, c_ob, c_ib, d.p,
                               nullptr));
  d.down(dst.data);
  return dst;
}

KernelTensor unpack_kernel(const BlockedKernel& src) {
  g_layout_transforms.fetch_add(1, std::memory_order_relaxed);
  KernelTensor dst(src.c_i, src.c_o, src.h_f, src.w_f);
  DevBuf s(src.data.size()), d(dst.data.size());
  s.up(src.data);
  check(dconv_cuda_unpack_kernel(s.p, src.c_i, src.c_o, src.h_f, src.w_f, src.c_ob, src.c_ib,
                                 d.p, nullptr));
  d.down(dst.data);
  return dst;
}

std::uint64_t layout_transform_count() {
  return g_layout_transforms.load(std::memory_order_relaxed);
}

// ------------------------------------------------------------------ direct
namespace {

void check_operands(const BlockedFeatureMap& in, const BlockedKernel& k, const ConvShape& s,
                    const BlockingParams& p) {
  if (in.c_b != p.c_ib || k.c_ib != p.c_ib || k.c_ob != p.c_ob)
    throw std::invalid_argument("conv_direct: layout error (block sizes differ from params)");
  if (in.channels != s.c_i || in.height != s.h_i || in.width != s.w_i)
    throw std::invalid_argument("conv: input dims do not match shape");
  if (k.c_i != s.c_i || k.c_o != s.c_o || k.h_f != s.h_f || k.w_f != s.w_f)
    throw std::invalid_argument("conv: kernel dims do not match shape");
}

dconv_conv_desc make_desc(const ConvShape& s, int n, int c_ib, int c_ob, int epi) {
  dconv_conv_desc d;
  check(dconv_conv_desc_init(&d, n, s.c_i, s.c_o, s.h_i, s.w_i, s.h_f, s.w_f, s.stride, c_ib,
                             c_ob));
  d.epilogue = epi;
  return d;
}

}  // namespace

BlockedFeatureMap conv_direct(const BlockedFeatureMap& in, const BlockedKernel& kernel,
                              const ConvShape& shape, const BlockingParams& params,
                              int /*workers*/) {
  check_operands(in, kernel, shape, params);
  BlockedFeatureMap out(shape.c_o, shape.h_o, shape.w_o, params.c_ob);
  DevBuf di(in.data.size()), dw(kernel.data.size()), dout(out.data.size());
  di.up(in.data);
  dw.up(kernel.data);
  const dconv_conv_desc d = make_desc(shape, 1, params.c_ib, params.c_ob, DCONV_EPI_NONE);
  check(dconv_cuda_conv_direct(&d, di.p, dw.p, nullptr, dout.p, nullptr));
  dout.down(out.data);
  return out;
}

void relu_blocked(BlockedFeatureMap& x) {
  DevBuf d(x.data.size());
  d.up(x.data);
  check(dconv_cuda_relu_blocked(d.p, (int64_t)x.data.size(), nullptr));
  d.down(x.data);
}

BlockedFeatureMap layer_chain(const BlockedFeatureMap& in, const std::vector<Layer>& layers) {
  const std::uint64_t before = layout_transform_count();
  int c_b = in.c_b;
  for (std::size_t i = 0; i < layers.size(); ++i) {
    if (layers[i].params.c_ib != c_b)
      throw std::invalid_argument("layer_chain: layout error (c_ib != previous c_ob)");
    c_b = layers[i].params.c_ob;
  }
  if (layers.empty()) return in;
  cuda::DeviceFeatureMap cur(1, in.channels, in.height, in.width, in.c_b);
  cur.upload(in);
  for (const Layer& l : layers) {
    if (cur.channels != l.shape.c_i || cur.height != l.shape.h_i || cur.width != l.shape.w_i)
      throw std::invalid_argument("conv: input dims do not match shape");
    cuda::DeviceKernel k(l.kernel);
    cuda::DeviceFeatureMap next(1, l.shape.c_o, l.shape.h_o, l.shape.w_o, l.params.c_ob);
    cuda::conv_direct(cur, k, l.shape, next, l.relu ? DCONV_EPI_RELU : DCONV_EPI_NONE);
    cur = std::move(next);
  }
  BlockedFeatureMap out = cur.download();
  if (layout_transform_count() != before)
    throw std::runtime_error("layer_chain: layout transform inside the chain");
  return out;
}

// ------------------------------------------------------------------ device
namespace cuda {

DeviceFeatureMap::DeviceFeatureMap(int n_, int c, int h, int w, int cb)
    : n(n_), channels(c), height(h), width(w), c_b(cb) {
  require(n_ >= 1 && c >= 1 && h >= 1 && w >= 1 && cb >= 1,
          "DeviceFeatureMap: dims must be >= 1");
  cuda_check(cudaMalloc(&ptr_, elems() * sizeof(float)), "cudaMalloc");
  cuda_check(cudaMemset(ptr_, 0, elems() * sizeof(float)), "cudaMemset");
}

DeviceFeatureMap::~DeviceFeatureMap() {
  if (ptr_) cudaFree(ptr_);
}

DeviceFeatureMap::DeviceFeatureMap(DeviceFeatureMap&& o) noexcept
    : n(o.n), channels(o.channels), height(o.height), width(o.width), c_b(o.c_b), ptr_(o.ptr_) {
  o.ptr_ = nullptr;
}

DeviceFeatureMap& DeviceFeatureMap::operator=(DeviceFeatureMap&& o) noexcept {
  if (this != &o) {
    if (ptr_) cudaFree(ptr_);
    n = o.n; channels = o.channels; height = o.height; width = o.width; c_b = o.c_b;
    ptr_ = o.ptr_;
    o.ptr_ = nullptr;
  }
  return *this;
}

std::size_t DeviceFeatureMap::elems() const {
  return std::size_t(n) * detail::round_up(channels, c_b) * height * width;
}

void DeviceFeatureMap::upload(const BlockedFeatureMap& h, int image, void* stream) {
  require(h.channels == channels && h.height == height && h.width == width && h.c_b == c_b,
          "DeviceFeatureMap::upload: layout error");
  cuda_check(cudaMemcpyAsync(ptr_ + std::size_t(image) * h.data.size(), h.data.data(),
                             h.data.size() * sizeof(float), cudaMemcpyHostToDevice,
                             static_cast<cudaStream_t>(stream)),
             "cudaMemcpyAsync H2D");
  cuda_check(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)), "sync");
}

BlockedFeatureMap DeviceFeatureMap::download(int image, void* stream) const {
  BlockedFeatureMap h(channels, height, width, c_b);
  cuda_check(cudaMemcpyAsync(h.data.data(), ptr_ + std::size_t(image) * h.data.size(),
                             h.data.size() * sizeof(float), cudaMemcpyDeviceToHost,
                             static_cast<cudaStream_t>(stream)),
             "cudaMemcpyAsync D2H");
  cuda_check(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)), "sync");
  return h;
}

DeviceKernel::DeviceKernel(const BlockedKernel& h, void* stream)
    : c_i(h.c_i), c_o(h.c_o), h_f(h.h_f), w_f(h.w_f), c_ob(h.c_ob), c_ib(h.c_ib) {
  cuda_check(cudaMalloc(&ptr_, h.data.size() * sizeof(float)), "cudaMalloc");
  cuda_check(cudaMemcpyAsync(ptr_, h.data.data(), h.data.size() * sizeof(float),
                             cudaMemcpyHostToDevice, static_cast<cudaStream_t>(stream)),
             "cudaMemcpyAsync H2D");
  cuda_check(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)), "sync");
}

DeviceKernel::~DeviceKernel() {
  if (ptr_) cudaFree(ptr_);
}

void conv_direct(const DeviceFeatureMap& in, const DeviceKernel& k, const ConvShape& s,
                 DeviceFeatureMap& out, int epilogue, const DeviceFeatureMap* skip,
                 void* stream) {
  if (in.c_b != k.c_ib || out.c_b != k.c_ob)
    throw std::invalid_argument("conv_direct: layout error (block sizes)");
  if (in.channels != s.c_i || in.height != s.h_i || in.width != s.w_i || in.n != out.n)
    throw std::invalid_argument("conv: input dims do not match shape");
  if (k.c_i != s.c_i || k.c_o != s.c_o || k.h_f != s.h_f || k.w_f != s.w_f)
    throw std::invalid_argument("conv: kernel dims do not match shape");
  if (out.channels != s.c_o || out.height != s.h_o || out.width != s.w_o)
    throw std::invalid_argument("conv: output dims do not match shape");
  const dconv_conv_desc d = make_desc(s, in.n, k.c_ib, k.c_ob, epilogue);
  check(dconv_cuda_conv_direct(&d, in.data(), k.data(), skip ? skip->data() : nullptr,
                               out.data(), stream));
}

DevicePreparedKernel::DevicePreparedKernel(const DeviceKernel& k, const ConvShape& s,
                                           TensorCoreMode m, void* stream)
    : shape(s), mode(m) {
  if (k.c_ib != 8 || k.c_ob != 8)
    throw std::invalid_argument("conv_direct: layout error (tensor-core path needs c_b = 8)");
  if (k.c_i != s.c_i || k.c_o != s.c_o || k.h_f != s.h_f || k.w_f != s.w_f)
    throw std::invalid_argument("conv: kernel dims do not match shape");
  const dconv_conv_desc d = make_desc(s, 1, 8, 8, DCONV_EPI_NONE);
  const bool x3 = m == TensorCoreMode::kSplitTf32;
  int64_t floats = 0;
  check(x3 ? dconv_cuda_tf32x3_prepared_size(&d, &floats)
           : dconv_cuda_tf32_prepared_size(&d, &floats));
  cuda_check(cudaMalloc(&ptr_, std::size_t(floats) * sizeof(float)), "cudaMalloc");
  check(x3 ? dconv_cuda_prepare_tf32x3_weights(&d, k.data(), ptr_, stream)
           : dconv_cuda_prepare_tf32_weights(&d, k.data(), ptr_, stream));
  cuda_check(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)), "sync");
}

DevicePreparedKernel::~DevicePreparedKernel() {
  if (ptr_) cudaFree(ptr_);
}

void conv_direct(const DeviceFeatureMap& in, const DevicePreparedKernel& k,
                 DeviceFeatureMap& out, int epilogue, const DeviceFeatureMap* skip,
                 void* stream) {
  const ConvShape& s = k.shape;
  if (in.c_b != 8 || out.c_b != 8)
    throw std::invalid_argument("conv_direct: layout error (tensor-core path needs c_b = 8)");
  if (in.channels != s.c_i || in.height != s.h_i || in.width != s.w_i || in.n != out.n)
    throw std::invalid_argument("conv: input dims do not match shape");
  if (out.channels != s.c_o || out.height != s.h_o || out.width != s.w_o)
    throw std::invalid_argument("conv: output dims do not match shape");
  const dconv_conv_desc d = make_desc(s, in.n, 8, 8, epilogue);
  const float* sk = skip ? skip->data() : nullptr;
  check(k.mode == TensorCoreMode::kSplitTf32
            ? dconv_cuda_conv_direct_tf32x3(&d, in.data(), k.data(), sk, out.data(), stream)
            : dconv_cuda_conv_direct_tf32(&d, in.data(), k.data(), sk, out.data(), stream));
}

}  // namespace cuda
}  // namespace dconv
