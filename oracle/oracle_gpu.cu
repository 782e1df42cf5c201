// oracle_gpu.cu -- conv_oracle64 (reference.cpp:70-87) on the GPU, in fp64.
//
// TEST INFRASTRUCTURE ONLY (see oracle.h): the checker for whole-output
// parity at the bench sizes (VGG-16 b32, ResNet-50 b256, GoogLeNet b64), where
// the CPU oracle would take hours.  Nothing in paper_1809_10170_b200/ links or
// loads this library; only tests/ do.
//
// Same arithmetic as the reference's fp64 referee, element by element: the
// products double(x) * double(w) are exact (24 + 24 bits < 53), and every
// output element sums them in the reference's order -- input channel i
// ascending, then filter column m, then filter row n (the i, j, x, y, m, n
// loop nest of reference.cpp:76-83 restricted to one (j, y, x)) -- starting
// from +0.0.  So `double -> float` of the result is bit-identical to
// conv_oracle64 (tests/test_oracle_gpu.py checks it against the golden
// fixtures the reference produced).
//
// Input: any blocked view [n][C/cb][H][W][cb] with strides (cb = 1 is the
// dense CHW first-layer input).  Kernel: the dense KernelTensor
// [C_i][C_o][H_f][W_f] (tensor.hpp:83-103), independent of the packing under
// test.  Output: fp64 [n][ceil(C_o/8)][H_o][W_o][8] (padded channels 0).
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

struct OgParams {
  const float* in;
  long long in_img, in_blk, in_row;
  int in_cb;
  const float* k;
  double* out;
  int n, c_i, c_o, h_i, w_i, h_o, w_o, h_f, w_f, s;
  int TW, PPT, TH, PH, PW, tiles_x, tiles_y;
};

constexpr int kThreads = 128;
constexpr int kMaxPpt = 4;

__global__ void __launch_bounds__(kThreads) og_conv64(const OgParams p) {
  extern __shared__ float sm[];
  float* patch = sm;                          // [8][PH][PW]
  float* wsm = sm + 8 * p.PH * p.PW;          // [8 ii][h_f][w_f][8 jj]
  const int t = threadIdx.x;
  const int tile = blockIdx.x, jb = blockIdx.y;
  const int img = tile / (p.tiles_x * p.tiles_y);
  const int rem = tile - img * p.tiles_x * p.tiles_y;
  const int ty0 = (rem / p.tiles_x) * p.TH, tx0 = (rem % p.tiles_x) * p.TW;
  const int rows_per_pass = kThreads / p.TW;
  const int tx = t % p.TW, try0 = t / p.TW;

  double acc[kMaxPpt][8];
#pragma unroll
  for (int k = 0; k < kMaxPpt; ++k)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[k][j] = 0.0;

  const int taps = p.h_f * p.w_f;
  for (int c0 = 0; c0 < p.c_i; c0 += 8) {
    const int cnt = min(8, p.c_i - c0);
    __syncthreads();
    const int plane = p.PH * p.PW;
    for (int idx = t; idx < cnt * plane; idx += kThreads) {
      const int ii = idx / plane, r = idx - ii * plane;
      const int pr = r / p.PW, pc = r - pr * p.PW;
      const int y = ty0 * p.s + pr, x = tx0 * p.s + pc;
      const int c = c0 + ii;
      float v = 0.f;
      if (y < p.h_i && x < p.w_i)
        v = p.in[(long long)img * p.in_img + (long long)(c / p.in_cb) * p.in_blk +
                 (long long)y * p.in_row + (long long)x * p.in_cb + c % p.in_cb];
      patch[idx] = v;
    }
    for (int idx = t; idx < cnt * taps * 8; idx += kThreads) {
      const int ii = idx / (taps * 8), r = idx - ii * taps * 8;
      const int tap = r >> 3, jj = r & 7;
      const int j = jb * 8 + jj;
      wsm[idx] = j < p.c_o ? p.k[((long long)(c0 + ii) * p.c_o + j) * taps + tap] : 0.f;
    }
    __syncthreads();
    for (int ii = 0; ii < cnt; ++ii)
      for (int m = 0; m < p.w_f; ++m)       // reference order: i, then m, then n
        for (int n = 0; n < p.h_f; ++n) {
          const float* wp = wsm + ((ii * p.h_f + n) * p.w_f + m) * 8;
          double w[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) w[j] = (double)wp[j];
          const float* pp = patch + ii * plane + n * p.PW + tx * p.s + m;
#pragma unroll
          for (int k = 0; k < kMaxPpt; ++k) {
            if (k >= p.PPT) break;
            const double x = (double)pp[(try0 + k * rows_per_pass) * p.s * p.PW];
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[k][j] = fma(x, w[j], acc[k][j]);
          }
        }
  }
  const int jb_n = (p.c_o + 7) / 8;
#pragma unroll
  for (int k = 0; k < kMaxPpt; ++k) {
    if (k >= p.PPT) break;
    const int y = ty0 + try0 + k * rows_per_pass, x = tx0 + tx;
    if (y >= p.h_o || x >= p.w_o) continue;
    double* o = p.out + ((((long long)img * jb_n + jb) * p.h_o + y) * p.w_o + x) * 8;
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = acc[k][j];
  }
}

}  // namespace

extern "C" {

// Returns 0, -1 on a shape error, or the CUDA error code.
int orcg_conv_oracle64(const float* in, int n, int c_i, int h_i, int w_i, int in_cb,
                       long long in_img, long long in_blk, long long in_row,
                       const float* k_dense, int c_o, int h_f, int w_f, int s, double* out,
                       void* stream) {
  if (n < 1 || c_i < 1 || c_o < 1 || h_f < 1 || w_f < 1 || s < 1 || in_cb < 1) return -1;
  if (h_f > h_i || w_f > w_i || (h_i - h_f) % s || (w_i - w_f) % s) return -1;
  OgParams p{};
  p.in = in; p.in_img = in_img; p.in_blk = in_blk; p.in_row = in_row; p.in_cb = in_cb;
  p.k = k_dense; p.out = out;
  p.n = n; p.c_i = c_i; p.c_o = c_o; p.h_i = h_i; p.w_i = w_i;
  p.h_f = h_f; p.w_f = w_f; p.s = s;
  p.h_o = (h_i - h_f) / s + 1;
  p.w_o = (w_i - w_f) / s + 1;
  // largest pixel tile whose 8-channel patch + weights fit 190 KB
  const size_t w_bytes = (size_t)8 * h_f * w_f * 8 * 4;
  bool found = false;
  for (int tw : {32, 16, 8, 4}) {
    for (int ppt = kMaxPpt; ppt >= 1 && !found; --ppt) {
      const int th = (kThreads / tw) * ppt;
      const int ph = (th - 1) * s + h_f, pw = (tw - 1) * s + w_f;
      if ((size_t)8 * ph * pw * 4 + w_bytes <= 190 * 1024) {
        p.TW = tw; p.PPT = ppt; p.TH = th; p.PH = ph; p.PW = pw;
        found = true;
      }
    }
    if (found) break;
  }
  if (!found) return -1;
  p.tiles_x = (p.w_o + p.TW - 1) / p.TW;
  p.tiles_y = (p.h_o + p.TH - 1) / p.TH;
  const size_t smem = (size_t)8 * p.PH * p.PW * 4 + w_bytes;
  cudaFuncSetAttribute(og_conv64, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  dim3 grid((unsigned)(n * p.tiles_x * p.tiles_y), (unsigned)((c_o + 7) / 8));
  og_conv64<<<grid, kThreads, smem, static_cast<cudaStream_t>(stream)>>>(p);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : (int)e;
}

}  // extern "C"
