// dconv/direct.hpp -- the reference's `direct` module API (
// its direct.cpp is absent from the snapshot, core/CMakeLists.txt:29),
// implemented on the B200 through include/dconv_cuda.h.
//
// Host-value overloads keep the reference signatures: inputs by const&,
// outputs returned by value in host memory (one H2D / D2H per call).
// Device overloads (dconv::cuda) keep tensors resident in HBM for chains.
#pragma once

#include <cstdint>
#include <vector>

#include "dconv/model.hpp"
#include "dconv/shape.hpp"
#include "dconv/tensor.hpp"

namespace dconv {

/// Alg. 3 direct convolution.  Preconditions: in.c_b ==
/// params.c_ib, kernel blocked with (params.c_ob, params.c_ib); dims match
/// `shape`.  Throws std::invalid_argument ("layout error" / dimension error)
/// like the reference, std::runtime_error on a CUDA failure.  `workers` is
/// the reference's CPU thread count; the result does not depend on it.
BlockedFeatureMap conv_direct(const BlockedFeatureMap& in, const BlockedKernel& kernel,
                              const ConvShape& shape, const BlockingParams& params,
                              int workers = 0);

/// In-place ReLU over every stored element, padding stays 0.
void relu_blocked(BlockedFeatureMap& x);

/// One layer of a chain.
struct Layer {
  BlockedKernel kernel;
  ConvShape shape;
  BlockingParams params;
  bool relu = false;
};

/// Runs the layers back to back on the device with zero layout transforms;
/// throws std::invalid_argument ("layer_chain: layout error") when a layer's
/// c_ib differs from the previous layer's c_ob.
BlockedFeatureMap layer_chain(const BlockedFeatureMap& in, const std::vector<Layer>& layers);

namespace cuda {

/// A blocked map resident in device memory ([n][C/c_b][H][W][c_b]).
class DeviceFeatureMap {
 public:
  DeviceFeatureMap(int n, int c, int h, int w, int cb);
  ~DeviceFeatureMap();
  DeviceFeatureMap(const DeviceFeatureMap&) = delete;
  DeviceFeatureMap& operator=(const DeviceFeatureMap&) = delete;
  DeviceFeatureMap(DeviceFeatureMap&&) noexcept;
  DeviceFeatureMap& operator=(DeviceFeatureMap&&) noexcept;
  float* data() { return ptr_; }
  const float* data() const { return ptr_; }
  std::size_t elems() const;
  int n, channels, height, width, c_b;
  void upload(const BlockedFeatureMap& host, int image = 0, void* stream = nullptr);
  BlockedFeatureMap download(int image = 0, void* stream = nullptr) const;

 private:
  float* ptr_ = nullptr;
};

/// Blocked weights resident in device memory.
class DeviceKernel {
 public:
  explicit DeviceKernel(const BlockedKernel& host, void* stream = nullptr);
  ~DeviceKernel();
  DeviceKernel(const DeviceKernel&) = delete;
  DeviceKernel& operator=(const DeviceKernel&) = delete;
  const float* data() const { return ptr_; }
  int c_i, c_o, h_f, w_f, c_ob, c_ib;

 private:
  float* ptr_ = nullptr;
};

/// Device-resident conv_direct into a preallocated output (zero workspace;
/// asynchronous on `stream`).  epilogue: DCONV_EPI_* of dconv_cuda.h.
void conv_direct(const DeviceFeatureMap& in, const DeviceKernel& kernel,
                 const ConvShape& shape, DeviceFeatureMap& out, int epilogue = 0,
                 const DeviceFeatureMap* skip = nullptr, void* stream = nullptr);

/// Tensor-core variants of conv_direct (c_ib = c_ob = 8, stride 1 or a 1x1
/// of any stride): kTf32 = one TF32 pass (looser tolerance); kSplitTf32 =
/// three TF32 passes with chunked fp32 summation, the fp32 tolerance of the
/// FFMA path.  The weights are rearranged once into the operand layout.
enum class TensorCoreMode { kTf32 = 0, kSplitTf32 = 1 };

class DevicePreparedKernel {
 public:
  DevicePreparedKernel(const DeviceKernel& k, const ConvShape& shape, TensorCoreMode mode,
                       void* stream = nullptr);
  ~DevicePreparedKernel();
  DevicePreparedKernel(const DevicePreparedKernel&) = delete;
  DevicePreparedKernel& operator=(const DevicePreparedKernel&) = delete;
  const float* data() const { return ptr_; }
  ConvShape shape;
  TensorCoreMode mode;

 private:
  float* ptr_ = nullptr;
};

/// conv_direct on the tensor cores into a preallocated output (asynchronous).
void conv_direct(const DeviceFeatureMap& in, const DevicePreparedKernel& kernel,
                 DeviceFeatureMap& out, int epilogue = 0,
                 const DeviceFeatureMap* skip = nullptr, void* stream = nullptr);

}  // namespace cuda
}  // namespace dconv
