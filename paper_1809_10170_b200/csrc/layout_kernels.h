// layout_kernels.h -- internal launchers for layout.cu (not public).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace dconv_dev {
int launch_pack_kernel(const float* src, int c_i, int c_o, int h_f, int w_f,
                       int c_ob, int c_ib, float* dst, cudaStream_t st);
int launch_unpack_kernel(const float* src, int c_i, int c_o, int h_f, int w_f,
                         int c_ob, int c_ib, float* dst, cudaStream_t st);
int launch_pack_s2d(const float* src, int n, int c, int h, int w, int f, float* dst,
                    cudaStream_t st);
int launch_s2d_blocked(const float* src, int64_t in_img, int64_t in_blk, int64_t in_row, int n,
                       int c, int h, int w, int f, float* dst, cudaStream_t st);
int launch_pack_fm(const float* src, int n, int c, int h, int w, int c_b,
                   int halo, float* dst, cudaStream_t st);
int launch_unpack_fm(const float* src, int n, int c, int h, int w, int c_b,
                     int halo, float* dst, cudaStream_t st);
int launch_relu(float* x, int64_t count, cudaStream_t st);
int launch_add(const float* a, const float* b, float* o, int64_t count,
               int relu, cudaStream_t st);
int launch_maxpool2x2(const float* in, int n, int n_blocks, int h, int w,
                      int c_b, float* out, int64_t o_img, int64_t o_blk,
                      int64_t o_row, cudaStream_t st);
// copy [n][n_blocks][h][w][8] pencils of a strided map into each peer's copy
// at the same offsets (the reader's fused C_o-shard gather)
int launch_copy_pencils_peers(const float* src, int n, int n_blocks, int h, int w,
                              int64_t img_s, int64_t blk_s, int64_t row_s,
                              float* const* peers, int n_peers, cudaStream_t st);
double fp32_peak_probe(cudaStream_t st);
double ffma2_pattern_probe(cudaStream_t st);
}  // namespace dconv_dev
