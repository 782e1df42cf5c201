// conv_generic.cu -- any-(c_ib, c_ob) direct convolution and the first-layer
// (dense-input) reader.
//
// The generic kernel keeps the reference's per-element accumulation order of
// Alg. 3: i' -> n -> m -> ii, fp32 FMA, one thread per
// output element of the (padded) blocked output.  It exists so that every
// (c_ob, c_ib) the reference API accepts (BlockingParams, model.hpp:54-61)
// has a CUDA path; the FFMA kernel (conv_ffma.cu) is the fast path.
//
// The first-layer kernel reads the unblocked network input [N][C_i][H][W]
// directly (the blocked layout is not imposed on the first
// layer's input) with weights packed at c_ib = C_i, so no channel padding and
// no wasted FLOPs for C_i = 3.
#include "common.cuh"
#include "conv_kernels.h"

namespace dconv_dev {

namespace {

__device__ __forceinline__ float epilogue(float v, const GenericParams& p,
                                          int img, int jl, int y, int x,
                                          int jj) {
  if (p.epi & DCONV_EPI_ADD)
    v += p.skip[(int64_t)img * p.sk_img + (int64_t)jl * p.sk_blk +
                (int64_t)y * p.sk_row + (int64_t)x * p.c_ob + jj];
  if (p.epi & DCONV_EPI_RELU) v = fmaxf(v, 0.f);
  return v;
}

__global__ void conv_generic_kernel(const GenericParams p) {
  // element index over [img][jl][y][x][jj] of the computed output blocks
  const int64_t total =
      (int64_t)p.n * p.jb_count * p.h_o * p.w_o * p.c_ob;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t t = e;
    const int jj = (int)(t % p.c_ob); t /= p.c_ob;
    const int x = (int)(t % p.w_o); t /= p.w_o;
    const int y = (int)(t % p.h_o); t /= p.h_o;
    const int jl = (int)(t % p.jb_count); t /= p.jb_count;
    const int img = (int)t;
    const int jb = p.jb_begin + jl;
    const float* in = p.in + (int64_t)img * p.in_img;
    float acc = 0.f;
    for (int ib = 0; ib < p.ib_n; ++ib) {
      const float* wb =
          p.w + ((int64_t)jb * p.ib_n + ib) * p.h_f * p.w_f * p.c_ib * p.c_ob;
      const float* ib_base = in + (int64_t)ib * p.in_blk;
      for (int n = 0; n < p.h_f; ++n)
        for (int m = 0; m < p.w_f; ++m) {
          const float* ip = ib_base + (int64_t)(y * p.s + n) * p.in_row +
                            (int64_t)(x * p.s + m) * p.c_ib;
          const float* wp = wb + ((int64_t)(n * p.w_f + m) * p.c_ib) * p.c_ob + jj;
          for (int ii = 0; ii < p.c_ib; ++ii)
            acc = fmaf(ip[ii], wp[(int64_t)ii * p.c_ob], acc);
        }
    }
    float* o = p.out + (int64_t)img * p.out_img + (int64_t)jl * p.out_blk +
               (int64_t)y * p.out_row + (int64_t)x * p.c_ob + jj;
    DCONV_OWN(o, 1);
    *o = epilogue(acc, p, img, jl, y, x, jj);
  }
}

// First layer: dense input, one input block holding all C_i channels.
__global__ void conv_first_layer_kernel(const GenericParams p) {
  const int64_t total =
      (int64_t)p.n * p.jb_count * p.h_o * p.w_o * p.c_ob;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t t = e;
    const int jj = (int)(t % p.c_ob); t /= p.c_ob;
    const int x = (int)(t % p.w_o); t /= p.w_o;
    const int y = (int)(t % p.h_o); t /= p.h_o;
    const int jl = (int)(t % p.jb_count); t /= p.jb_count;
    const int img = (int)t;
    const int jb = p.jb_begin + jl;
    const float* in = p.in + (int64_t)img * p.in_img;
    const float* wb = p.w + (int64_t)jb * p.h_f * p.w_f * p.c_i * p.c_ob;
    float acc = 0.f;
    for (int n = 0; n < p.h_f; ++n)
      for (int m = 0; m < p.w_f; ++m) {
        const float* wp = wb + ((int64_t)(n * p.w_f + m) * p.c_i) * p.c_ob + jj;
        for (int ii = 0; ii < p.c_i; ++ii)
          acc = fmaf(in[(int64_t)ii * p.in_blk + (int64_t)(y * p.s + n) * p.in_row +
                        x * p.s + m],
                     wp[(int64_t)ii * p.c_ob], acc);
      }
    float* o = p.out + (int64_t)img * p.out_img + (int64_t)jl * p.out_blk +
               (int64_t)y * p.out_row + (int64_t)x * p.c_ob + jj;
    DCONV_OWN(o, 1);
    *o = epilogue(acc, p, img, jl, y, x, jj);
  }
}

int grid_for(int64_t total) {
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 64) blocks = 148 * 64;
  if (blocks < 1) blocks = 1;
  return (int)blocks;
}

}  // namespace

int launch_conv_generic(const GenericParams& p, cudaStream_t stream) {
  const int64_t total = (int64_t)p.n * p.jb_count * p.h_o * p.w_o * p.c_ob;
  conv_generic_kernel<<<grid_for(total), 256, 0, stream>>>(p);
  dconv_host::count_launch();
  return dconv_host::check_launch("conv_generic_kernel");
}

int launch_conv_first_layer(const GenericParams& p, cudaStream_t stream) {
  const int64_t total = (int64_t)p.n * p.jb_count * p.h_o * p.w_o * p.c_ob;
  conv_first_layer_kernel<<<grid_for(total), 256, 0, stream>>>(p);
  dconv_host::count_launch();
  return dconv_host::check_launch("conv_first_layer_kernel");
}

}  // namespace dconv_dev
