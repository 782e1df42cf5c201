// serialize.cpp -- tensor files and weight ingest.
//
// The reference describes, but does not ship (serialize.cpp is missing from
// the snapshot), a flat little-endian fp32 format with a 7-integer header
// used by the CLI's `pack` subcommand:
// "reads a dense kernel file, writes the blocked form; idempotent on
// already-packed detection via header"; packing twice -> "already blocked";
// malformed file -> parse error.  The header word order is fixed in
// include/dconv_cuda.h.  The repack itself is the GPU kernel of
// dconv_cuda_pack_kernel (the one-time cost of PAPER.md:95-101).
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <stdexcept>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "dconv/serialize.hpp"
#include "dconv_cuda.h"

namespace dconv_host {
int set_error(int code, const char* fmt, ...);
}
using dconv_host::set_error;

namespace {

int round_up(int v, int b) { return (v + b - 1) / b * b; }

bool little_endian() {
  const uint16_t one = 1;
  uint8_t b;
  std::memcpy(&b, &one, 1);
  return b == 1;
}

int read_file(const char* path, std::vector<char>& bytes) {
  if (!path) return set_error(DCONV_EPARAM, "NULL path");
  std::ifstream f(path, std::ios::binary | std::ios::ate);
  if (!f) return set_error(DCONV_EIO, "cannot open '%s'", path);
  const std::streamsize n = f.tellg();
  f.seekg(0);
  bytes.resize((size_t)n);
  if (n && !f.read(bytes.data(), n)) return set_error(DCONV_EIO, "cannot read '%s'", path);
  return DCONV_OK;
}

int parse(const std::vector<char>& bytes, const char* path, dconv_file_header* h) {
  if (bytes.size() < sizeof(dconv_file_header))
    return set_error(DCONV_EFORMAT, "'%s': %zu bytes, shorter than the 28-byte header", path,
                     bytes.size());
  std::memcpy(h, bytes.data(), sizeof(*h));
  const int64_t want = dconv_file_payload_floats(h);
  if (want < 0)
    return set_error(DCONV_EFORMAT, "'%s': invalid header {%d,%d,%d,%d,%d,%d,%d}", path, h->c,
                     h->h, h->w, h->c_b, h->c_o, h->c_ib, h->kind);
  const uint64_t have = bytes.size() - sizeof(*h);
  if (have != (uint64_t)want * 4)
    return set_error(DCONV_EFORMAT, "'%s': payload is %llu bytes, header implies %lld", path,
                     (unsigned long long)have, (long long)want * 4);
  return DCONV_OK;
}

}  // namespace

extern "C" {

int64_t dconv_file_payload_floats(const dconv_file_header* h) {
  if (!h || h->c < 1 || h->h < 1 || h->w < 1 || h->c_b < 0) return -1;
  if (h->kind == DCONV_FILE_FEATURE_MAP) {
    if (h->c_o != 0 || h->c_ib != 0) return -1;
    const int c = h->c_b ? round_up(h->c, h->c_b) : h->c;
    return (int64_t)c * h->h * h->w;
  }
  if (h->kind == DCONV_FILE_KERNEL) {
    if (h->c_o < 1) return -1;
    if ((h->c_b == 0) != (h->c_ib == 0) || h->c_ib < 0) return -1;  // both or neither
    const int ci = h->c_ib ? round_up(h->c, h->c_ib) : h->c;
    const int co = h->c_b ? round_up(h->c_o, h->c_b) : h->c_o;
    return (int64_t)ci * co * h->h * h->w;
  }
  return -1;
}

int dconv_file_read_header(const char* path, dconv_file_header* h) {
  if (!h) return set_error(DCONV_EPARAM, "NULL header");
  if (!little_endian()) return set_error(DCONV_EUNSUPPORTED, "big-endian host");
  std::vector<char> bytes;
  if (int rc = read_file(path, bytes)) return rc;
  return parse(bytes, path, h);
}

int dconv_file_read_payload(const char* path, float* host_dst, int64_t floats) {
  if (!host_dst && floats) return set_error(DCONV_EPARAM, "NULL destination");
  std::vector<char> bytes;
  if (int rc = read_file(path, bytes)) return rc;
  dconv_file_header h;
  if (int rc = parse(bytes, path, &h)) return rc;
  if (floats != dconv_file_payload_floats(&h))
    return set_error(DCONV_EPARAM, "destination holds %lld floats, file has %lld",
                     (long long)floats, (long long)dconv_file_payload_floats(&h));
  std::memcpy(host_dst, bytes.data() + sizeof(h), (size_t)floats * 4);
  return DCONV_OK;
}

int dconv_file_write(const char* path, const dconv_file_header* h, const float* host_src,
                     int64_t floats) {
  if (!path || !h || (!host_src && floats)) return set_error(DCONV_EPARAM, "NULL argument");
  if (!little_endian()) return set_error(DCONV_EUNSUPPORTED, "big-endian host");
  if (dconv_file_payload_floats(h) != floats)
    return set_error(DCONV_EPARAM, "header implies %lld floats, %lld given",
                     (long long)dconv_file_payload_floats(h), (long long)floats);
  std::ofstream f(path, std::ios::binary | std::ios::trunc);
  if (!f) return set_error(DCONV_EIO, "cannot create '%s'", path);
  f.write(reinterpret_cast<const char*>(h), sizeof(*h));
  f.write(reinterpret_cast<const char*>(host_src), (std::streamsize)floats * 4);
  if (!f) return set_error(DCONV_EIO, "cannot write '%s'", path);
  return DCONV_OK;
}

int dconv_cuda_load_kernel_file(const char* path, int c_ob, int c_ib, float* d_dst,
                                void* stream) {
  if (!d_dst) return set_error(DCONV_EPARAM, "NULL destination");
  if (c_ob < 1 || c_ib < 1) return set_error(DCONV_EPARAM, "block sizes must be >= 1");
  std::vector<char> bytes;
  if (int rc = read_file(path, bytes)) return rc;
  dconv_file_header h;
  if (int rc = parse(bytes, path, &h)) return rc;
  if (h.kind != DCONV_FILE_KERNEL) return set_error(DCONV_EFORMAT, "'%s' is not a kernel file", path);
  const float* payload = reinterpret_cast<const float*>(bytes.data() + sizeof(h));
  const int64_t n = dconv_file_payload_floats(&h);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (h.c_b != 0) {
    // already blocked: must match the requested blocking exactly
    if (h.c_b != c_ob || h.c_ib != c_ib)
      return set_error(DCONV_ELAYOUT, "file is blocked (c_ob=%d, c_ib=%d), requested (%d, %d)",
                       h.c_b, h.c_ib, c_ob, c_ib);
    cudaError_t e = cudaMemcpyAsync(d_dst, payload, (size_t)n * 4, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return set_error(DCONV_ECUDA, "upload: %s", cudaGetErrorString(e));
    return DCONV_OK;
  }
  // dense: upload, then the GPU repack (ingest only -- not the conv hot path)
  float* d_dense = nullptr;
  cudaError_t e = cudaMalloc(&d_dense, (size_t)n * 4);
  if (e != cudaSuccess) return set_error(DCONV_ECUDA, "cudaMalloc: %s", cudaGetErrorString(e));
  e = cudaMemcpyAsync(d_dense, payload, (size_t)n * 4, cudaMemcpyHostToDevice, st);
  int rc = DCONV_OK;
  if (e != cudaSuccess) rc = set_error(DCONV_ECUDA, "upload: %s", cudaGetErrorString(e));
  if (!rc) rc = dconv_cuda_pack_kernel(d_dense, h.c, h.c_o, h.h, h.w, c_ob, c_ib, d_dst, stream);
  e = cudaStreamSynchronize(st);  // the host payload must outlive the copy
  if (!rc && e != cudaSuccess) rc = set_error(DCONV_ECUDA, "sync: %s", cudaGetErrorString(e));
  cudaFree(d_dense);
  return rc;
}

int dconv_pack_kernel_file(const char* in_path, int c_ob, int c_ib, const char* out_path) {
  if (c_ob < 1 || c_ib < 1) return set_error(DCONV_EPARAM, "block sizes must be >= 1");
  dconv_file_header h;
  if (int rc = dconv_file_read_header(in_path, &h)) return rc;
  if (h.kind != DCONV_FILE_KERNEL)
    return set_error(DCONV_EFORMAT, "'%s' is not a kernel file", in_path);
  if (h.c_b != 0) return set_error(DCONV_EBLOCKED, "'%s' is already blocked", in_path);
  dconv_file_header out = h;
  out.c_b = c_ob;
  out.c_ib = c_ib;
  const int64_t n = dconv_file_payload_floats(&out);
  float* d_blk = nullptr;
  cudaError_t e = cudaMalloc(&d_blk, (size_t)n * 4);
  if (e != cudaSuccess) return set_error(DCONV_ECUDA, "cudaMalloc: %s", cudaGetErrorString(e));
  int rc = dconv_cuda_load_kernel_file(in_path, c_ob, c_ib, d_blk, nullptr);
  std::vector<float> host((size_t)n);
  if (!rc) {
    e = cudaMemcpy(host.data(), d_blk, (size_t)n * 4, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) rc = set_error(DCONV_ECUDA, "download: %s", cudaGetErrorString(e));
  }
  cudaFree(d_blk);
  if (!rc) rc = dconv_file_write(out_path, &out, host.data(), n);
  return rc;
}

}  // extern "C"

// ---------------------------------------------------------------- C++ layer
namespace dconv {

namespace {
void check_io(int rc) {
  if (rc == DCONV_OK) return;
  const std::string msg = std::string(dconv_cuda_strerror(rc)) + ": " + dconv_cuda_last_error_detail();
  if (rc == DCONV_EIO || rc == DCONV_ECUDA) throw std::runtime_error(msg);
  throw std::invalid_argument(msg);
}
dconv_file_header read_header(const std::string& path) {
  dconv_file_header h;
  check_io(dconv_file_read_header(path.c_str(), &h));
  return h;
}
}  // namespace

void save(const std::string& path, const FeatureMap& t) {
  const dconv_file_header h{t.channels, t.height, t.width, 0, 0, 0, DCONV_FILE_FEATURE_MAP};
  check_io(dconv_file_write(path.c_str(), &h, t.data.data(), (int64_t)t.data.size()));
}

void save(const std::string& path, const BlockedFeatureMap& t) {
  const dconv_file_header h{t.channels, t.height, t.width, t.c_b, 0, 0, DCONV_FILE_FEATURE_MAP};
  check_io(dconv_file_write(path.c_str(), &h, t.data.data(), (int64_t)t.data.size()));
}

void save(const std::string& path, const KernelTensor& t) {
  const dconv_file_header h{t.c_i, t.h_f, t.w_f, 0, t.c_o, 0, DCONV_FILE_KERNEL};
  check_io(dconv_file_write(path.c_str(), &h, t.data.data(), (int64_t)t.data.size()));
}

void save(const std::string& path, const BlockedKernel& t) {
  const dconv_file_header h{t.c_i, t.h_f, t.w_f, t.c_ob, t.c_o, t.c_ib, DCONV_FILE_KERNEL};
  check_io(dconv_file_write(path.c_str(), &h, t.data.data(), (int64_t)t.data.size()));
}

KernelTensor load_kernel(const std::string& path) {
  const dconv_file_header h = read_header(path);
  if (h.kind != DCONV_FILE_KERNEL || h.c_b != 0)
    throw std::invalid_argument("parse error: '" + path + "' is not a dense kernel file");
  KernelTensor t(h.c, h.c_o, h.h, h.w);
  check_io(dconv_file_read_payload(path.c_str(), t.data.data(), (int64_t)t.data.size()));
  return t;
}

BlockedKernel load_blocked_kernel(const std::string& path) {
  const dconv_file_header h = read_header(path);
  if (h.kind != DCONV_FILE_KERNEL || h.c_b == 0)
    throw std::invalid_argument("parse error: '" + path + "' is not a blocked kernel file");
  BlockedKernel t(h.c, h.c_o, h.h, h.w, h.c_b, h.c_ib);
  check_io(dconv_file_read_payload(path.c_str(), t.data.data(), (int64_t)t.data.size()));
  return t;
}

FeatureMap load_feature_map(const std::string& path) {
  const dconv_file_header h = read_header(path);
  if (h.kind != DCONV_FILE_FEATURE_MAP || h.c_b != 0)
    throw std::invalid_argument("parse error: '" + path + "' is not a dense feature-map file");
  FeatureMap t(h.c, h.h, h.w);
  check_io(dconv_file_read_payload(path.c_str(), t.data.data(), (int64_t)t.data.size()));
  return t;
}

BlockedFeatureMap load_blocked_feature_map(const std::string& path) {
  const dconv_file_header h = read_header(path);
  if (h.kind != DCONV_FILE_FEATURE_MAP || h.c_b == 0)
    throw std::invalid_argument("parse error: '" + path + "' is not a blocked feature-map file");
  BlockedFeatureMap t(h.c, h.h, h.w, h.c_b);
  check_io(dconv_file_read_payload(path.c_str(), t.data.data(), (int64_t)t.data.size()));
  return t;
}

void pack_kernel_file(const std::string& in_path, int c_ob, int c_ib, const std::string& out_path) {
  check_io(dconv_pack_kernel_file(in_path.c_str(), c_ob, c_ib, out_path.c_str()));
}

}  // namespace dconv
