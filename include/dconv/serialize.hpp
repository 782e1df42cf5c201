// dconv/serialize.hpp -- tensor files and the CLI `pack` step
// (SPEC.md:580-587).  The reference's serialize.cpp is absent from the
// snapshot; the format (7 int32 header words + little-endian fp32 payload) is
// documented with the C-ABI in dconv_cuda.h.  Errors: std::invalid_argument
// for parse errors ("parse error: ...") and re-packing a blocked file
// ("already blocked: ..."), std::runtime_error for I/O and CUDA failures.
#pragma once

#include <string>

#include "dconv/tensor.hpp"

namespace dconv {

void save(const std::string& path, const FeatureMap& t);
void save(const std::string& path, const BlockedFeatureMap& t);
void save(const std::string& path, const KernelTensor& t);
void save(const std::string& path, const BlockedKernel& t);

FeatureMap load_feature_map(const std::string& path);
BlockedFeatureMap load_blocked_feature_map(const std::string& path);
KernelTensor load_kernel(const std::string& path);
BlockedKernel load_blocked_kernel(const std::string& path);

/// Dense kernel file -> blocked kernel file, repacked on the GPU.
void pack_kernel_file(const std::string& in_path, int c_ob, int c_ib, const std::string& out_path);

}  // namespace dconv
