// test_dropin.cpp -- the reference's operator API used exactly as the
// reference's own (missing) tests would use it (SPEC.md examples), linked
// against libdconv_b200.so instead of the CPU library.  Run by
// tests/test_dropin.py on a GPU box; exits non-zero on the first failure.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "dconv/direct.hpp"
#include "dconv/serialize.hpp"

using namespace dconv;

static int failures = 0;
#define EXPECT(cond)                                                   \
  do {                                                                 \
    if (!(cond)) {                                                     \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      ++failures;                                                      \
    }                                                                  \
  } while (0)

template <class F>
static bool throws_invalid(F f) {
  try {
    f();
  } catch (const std::invalid_argument&) {
    return true;
  }
  return false;
}

// fp64 reference of Alg. 1 (the semantic definition, reference.cpp:70-87)
static FeatureMap oracle(const FeatureMap& x, const KernelTensor& k, const ConvShape& s) {
  std::vector<double> acc(std::size_t(s.c_o) * s.h_o * s.w_o, 0.0);
  for (int i = 0; i < s.c_i; ++i)
    for (int j = 0; j < s.c_o; ++j)
      for (int xx = 0; xx < s.w_o; ++xx)
        for (int y = 0; y < s.h_o; ++y)
          for (int m = 0; m < s.w_f; ++m)
            for (int n = 0; n < s.h_f; ++n)
              acc[(std::size_t(j) * s.h_o + y) * s.w_o + xx] +=
                  double(x.at(i, y * s.stride + n, xx * s.stride + m)) * double(k.at(i, j, n, m));
  FeatureMap out(s.c_o, s.h_o, s.w_o);
  for (std::size_t q = 0; q < acc.size(); ++q) out.data[q] = float(acc[q]);
  return out;
}

static float frand(unsigned& st) {
  st = st * 1664525u + 1013904223u;
  return float(st >> 8) / float(1u << 24) * 2.0f - 1.0f;
}

static bool close_all(const FeatureMap& a, const FeatureMap& b) {
  for (std::size_t q = 0; q < a.data.size(); ++q)
    if (std::fabs(a.data[q] - b.data[q]) > 1e-4f + 1e-5f * std::fabs(b.data[q])) return false;
  return a.data.size() == b.data.size();
}

int main() {
  // ConvShape (shape.cpp:30-40)
  EXPECT(ConvShape(64, 64, 58, 58, 3, 3, 1).h_o == 56);
  EXPECT(throws_invalid([] { ConvShape(3, 64, 230, 230, 7, 7, 2); }));
  EXPECT(throws_invalid([] { ConvShape(1, 1, 2, 2, 3, 3, 1); }));

  // layouts
  {
    FeatureMap f(2, 1, 1);
    f.data = {1.0f, 2.0f};
    BlockedFeatureMap b = pack_feature_map(f, 2);
    EXPECT(b.data == std::vector<float>({1.0f, 2.0f}));
    KernelTensor k(4, 8, 1, 1);
    k.at(0, 5, 0, 0) = 7.0f;
    BlockedKernel kb = pack_kernel(k, 4, 4);
    EXPECT(kb.data[17] == 7.0f);
    EXPECT(unpack_kernel(kb).data == k.data);
    FeatureMap g(3, 5, 7);
    unsigned st = 3;
    for (float& v : g.data) v = frand(st);
    for (int cb : {1, 2, 4, 8}) EXPECT(unpack_feature_map(pack_feature_map(g, cb)).data == g.data);
  }

  // conv_direct trivial: [2] * [3] -> 6
  {
    FeatureMap x(1, 1, 1);
    x.data = {2.0f};
    KernelTensor k(1, 1, 1, 1);
    k.data = {3.0f};
    BlockedFeatureMap y = conv_direct(pack_feature_map(x, 1), pack_kernel(k, 1, 1),
                                      ConvShape(1, 1, 1, 1, 1, 1), BlockingParams{1, 1, 1});
    EXPECT(y.data.size() == 1 && y.data[0] == 6.0f);
  }

  // conv_direct vs oracle for the SPEC cases and cfg1
  struct Case { int ci, co, hi, wi, hf, wf, s, cob, cib; };
  for (const Case c : {Case{8, 16, 12, 12, 3, 3, 1, 8, 8}, Case{4, 8, 11, 11, 3, 3, 2, 8, 4},
                       Case{3, 6, 9, 9, 3, 3, 1, 8, 4}, Case{64, 64, 58, 58, 3, 3, 1, 8, 8},
                       Case{5, 7, 9, 11, 3, 3, 2, 4, 2}}) {
    ConvShape s(c.ci, c.co, c.hi, c.wi, c.hf, c.wf, c.s);
    FeatureMap x(c.ci, c.hi, c.wi);
    KernelTensor k(c.ci, c.co, c.hf, c.wf);
    unsigned st = 1809u + c.ci * 31u + c.co;
    for (float& v : x.data) v = frand(st);
    for (float& v : k.data) v = frand(st);
    BlockingParams p{c.cob, 4, c.cib};
    BlockedFeatureMap y = conv_direct(pack_feature_map(x, c.cib), pack_kernel(k, c.cob, c.cib), s, p, 4);
    BlockedFeatureMap y1 = conv_direct(pack_feature_map(x, c.cib), pack_kernel(k, c.cob, c.cib), s, p, 1);
    EXPECT(y.data == y1.data);  // bitwise independent of `workers`
    EXPECT(close_all(unpack_feature_map(y), oracle(x, k, s)));
    for (int ch = c.co; ch < y.padded_channels; ++ch)  // padded channels exact 0
      for (int yy = 0; yy < s.h_o; ++yy)
        for (int xx = 0; xx < s.w_o; ++xx) EXPECT(y.at(ch, yy, xx) == 0.0f);
  }
  // tensor-core variants through the device API: split-TF32 meets the same
  // fp32 tolerance as conv_direct (K = 4608 here); one TF32 pass does not
  {
    ConvShape s(512, 40, 9, 9, 3, 3, 1);
    FeatureMap x(s.c_i, s.h_i, s.w_i);
    KernelTensor k(s.c_i, s.c_o, 3, 3);
    unsigned st = 4608u;
    for (float& v : x.data) v = frand(st);
    for (float& v : k.data) v = frand(st);
    cuda::DeviceFeatureMap dx(1, s.c_i, s.h_i, s.w_i, 8), dy(1, s.c_o, s.h_o, s.w_o, 8);
    dx.upload(pack_feature_map(x, 8));
    cuda::DeviceKernel dk(pack_kernel(k, 8, 8));
    const FeatureMap want = oracle(x, k, s);
    cuda::DevicePreparedKernel x3(dk, s, cuda::TensorCoreMode::kSplitTf32);
    cuda::conv_direct(dx, x3, dy);
    EXPECT(close_all(unpack_feature_map(dy.download()), want));
    cuda::DevicePreparedKernel t1(dk, s, cuda::TensorCoreMode::kTf32);
    cuda::conv_direct(dx, t1, dy);
    EXPECT(!close_all(unpack_feature_map(dy.download()), want));
  }
  // layout error
  EXPECT(throws_invalid([] {
    BlockedFeatureMap x(4, 3, 3, 2);
    BlockedKernel k(4, 4, 1, 1, 4, 4);
    conv_direct(x, k, ConvShape(4, 4, 3, 3, 1, 1), BlockingParams{4, 1, 4});
  }));

  // relu_blocked
  {
    BlockedFeatureMap r(3, 1, 1, 3);
    r.data = {-1.0f, 0.0f, 2.0f};
    relu_blocked(r);
    EXPECT(r.data == std::vector<float>({0.0f, 0.0f, 2.0f}));
  }

  // layer_chain
  {
    FeatureMap x(1, 1, 1);
    x.data = {1.0f};
    KernelTensor k1(1, 1, 1, 1), k2(1, 1, 1, 1);
    k1.data = {2.0f};
    k2.data = {3.0f};
    ConvShape s(1, 1, 1, 1, 1, 1);
    BlockingParams p{8, 1, 8};
    std::vector<Layer> layers = {{pack_kernel(k1, 8, 8), s, p, false},
                                 {pack_kernel(k2, 8, 8), s, p, true}};
    BlockedFeatureMap in = pack_feature_map(x, 8);
    const auto before = layout_transform_count();
    BlockedFeatureMap y = layer_chain(in, layers);
    EXPECT(layout_transform_count() == before);
    EXPECT(y.data[0] == 6.0f);
    layers[1].params = BlockingParams{4, 1, 4};
    EXPECT(throws_invalid([&] { layer_chain(in, layers); }));
  }

  // tensor files + the CLI pack step
  {
    unsigned st = 7u;
    KernelTensor k(5, 11, 3, 3);
    for (auto& v : k.data) v = frand(st);
    const std::string dense = "/tmp/dconv_dropin_k.bin", blk = "/tmp/dconv_dropin_kb.bin",
                      back = "/tmp/dconv_dropin_kd.bin";
    save(dense, k);
    pack_kernel_file(dense, 8, 8, blk);
    const BlockedKernel kb = load_blocked_kernel(blk);
    EXPECT(kb.data == pack_kernel(k, 8, 8).data);          // GPU repack == pack_kernel
    save(back, unpack_kernel(kb));
    EXPECT(load_kernel(back).data == k.data);               // roundtrip: identical payload
    EXPECT(throws_invalid([&] { pack_kernel_file(blk, 8, 8, "/tmp/dconv_dropin_x.bin"); }));
    KernelTensor one(1, 1, 1, 1);                           // 1-weight kernel file
    one.data = {0.5f};
    save(dense, one);
    pack_kernel_file(dense, 8, 8, blk);
    const BlockedKernel ob = load_blocked_kernel(blk);
    EXPECT(ob.data.size() == 64 && ob.data[0] == 0.5f);
  }

  if (failures) {
    std::fprintf(stderr, "%d failure(s)\n", failures);
    return 1;
  }
  std::printf("test_dropin: all checks passed\n");
  return 0;
}
