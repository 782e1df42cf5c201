/*
 * dconv_cuda.h -- C-ABI of the B200-native direct-convolution hot path.
 *
 * This is the drop-in boundary: plain pointers, sizes and integer error codes,
 * no C++ or torch types.  Every device pointer is a CUDA global-memory
 * address; every call is asynchronous on `stream` (a cudaStream_t passed as
 * void*, NULL = legacy default stream).  The library owns no device memory:
 * the callers pass every buffer, so the "zero memory overhead" contract of the
 * reference holds -- no im2col buffer, no
 * split-K scratch, no staging copy in global memory.
 *
 * Layouts are the reference's (tensor.hpp:50-141), with an outermost image
 * dimension added (each image slice is byte-identical to the reference's
 * batch-1 BlockedFeatureMap):
 *   blocked map     [N][ceil(C/c_b)][H][W][c_b]    fp32, padded channels == 0
 *   blocked kernel  [C_o/c_ob][C_i/c_ib][H_f][W_f][c_ib][c_ob]
 *   dense map       [N][C][H][W]                   (first-layer reader input)
 *   dense kernel    [C_i][C_o][H_f][W_f]           (KernelTensor, tensor.hpp:83-103)
 *
 * Reference interfaces replaced (file:line in /root/reference/proj/core/):
 *   dconv_cuda_conv_direct      <- conv_direct (direct.cpp is
 *                                  absent from the snapshot, CMakeLists.txt:29)
 *                                  + the tile registry micro_kernel.hpp:37-51
 *   dconv_cuda_conv_first_layer <- the unblocked first layer (PAPER.md:18-21,
 *                                  SPEC.md:121 zero-pad alternative)
 *   dconv_cuda_pack_kernel      <- pack_kernel        tensor.cpp:85-95
 *   dconv_cuda_unpack_kernel    <- unpack_kernel      tensor.cpp:97-108
 *   dconv_cuda_pack_feature_map <- pack_feature_map   tensor.cpp:65-73
 *   dconv_cuda_unpack_feature_map <- unpack_feature_map tensor.cpp:75-83
 *   dconv_cuda_relu_blocked     <- relu_blocked
 *   dconv_cuda_add_blocked      <- skip layer, PAPER.md:4-7 (no reference code)
 *   dconv_cuda_maxpool2x2_blocked <- subsampling, PAPER.md:9-10 (no reference code)
 *   dconv_conv_shape            <- ConvShape::ConvShape shape.cpp:30-40
 *   dconv_conv_flops            <- conv_flops         reference.cpp:106-109
 *   dconv_file_*                <- tensor file format (serialize.cpp
 *                                  is absent from the snapshot) and the CLI's
 *                                  `pack` subcommand
 */
#ifndef DCONV_CUDA_H
#define DCONV_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Error codes (the C++ layer maps them back to the reference's exceptions:
 * EINVAL_SHAPE/EPARAM -> std::invalid_argument, ELAYOUT -> std::invalid_argument
 * "layout error", ECUDA/ENCCL -> std::runtime_error). */
enum {
  DCONV_OK = 0,
  DCONV_EINVAL_SHAPE = 1,  /* ConvShape rules violated (shape.cpp:32-37) */
  DCONV_ELAYOUT = 2,       /* block sizes / strides inconsistent */
  DCONV_EPARAM = 3,        /* bad parameter (null pointer, bad epilogue...) */
  DCONV_ECUDA = 4,         /* a CUDA runtime call failed */
  DCONV_ENCCL = 5,         /* reserved for the multi-GPU layer */
  DCONV_EUNSUPPORTED = 6,  /* no kernel for this configuration */
  DCONV_EFORMAT = 7,       /* malformed tensor file (parse error) */
  DCONV_EBLOCKED = 8,      /* "already blocked": packing a packed file */
  DCONV_EIO = 9            /* file open / read / write failed */
};

/* Fused epilogue applied to the fp32 accumulator before the single store. */
enum {
  DCONV_EPI_NONE = 0,
  DCONV_EPI_RELU = 1,      /* relu_blocked fused */
  DCONV_EPI_ADD = 2,       /* + skip (same blocked geometry as the output) */
  DCONV_EPI_ADD_RELU = 3,  /* relu(conv + skip): ResNet block tail */
  DCONV_EPI_MAXPOOL = 4    /* flag: 2x2/s2 max-pool fused after the above; the
                              output view is the pooled map (h_o/2 x w_o/2,
                              h_o and w_o even).  FFMA (no skip-add, no
                              peers) and TF32 paths. */
};

/* Kernel selection. */
enum {
  DCONV_ALGO_AUTO = 0,     /* fast FFMA path when c_ib == c_ob == 8, else generic */
  DCONV_ALGO_FFMA = 1,     /* register-blocked FFMA kernel (c_ib == c_ob == 8) */
  DCONV_ALGO_GENERIC = 2,  /* any (c_ib, c_ob); slow reference-order kernel */
  DCONV_ALGO_TF32 = 3,     /* tcgen05/TMEM TF32 variant (looser tolerance) */
  DCONV_ALGO_TF32X3 = 4    /* split-TF32 tensor-core variant, fp32 tolerance */
};

/* One convolution layer over a batch of blocked feature maps.
 * Geometry follows ConvShape (shape.hpp:29-45): valid convolution, exact
 * stride division; h_o/w_o are filled in by dconv_conv_desc_init.
 * Strides are in floats; 0 selects the dense value:
 *   *_blk_stride = H*W*c_b, *_img_stride = n_blocks*blk_stride,
 *   *_row_stride = W*c_b.
 * Non-dense strides express views: a halo'd (pre-padded) buffer, a crop
 * (ResNet stride-2 projections) or a C_o-shard of a larger map.  The pointers
 * passed to the calls point at element (0, 0, 0) of the view. */
typedef struct dconv_conv_desc {
  int n, c_i, c_o, h_i, w_i, h_f, w_f, stride;
  int h_o, w_o;
  int c_ib, c_ob;
  int64_t in_img_stride, in_blk_stride, in_row_stride;
  int64_t out_img_stride, out_blk_stride, out_row_stride;
  int64_t skip_img_stride, skip_blk_stride, skip_row_stride;
  int epilogue;            /* DCONV_EPI_* */
  int algo;                /* DCONV_ALGO_* */
  int co_block_begin;      /* first output block j' computed (C_o sharding) */
  int co_block_count;      /* number of output blocks computed; 0 = all */
  int tile_variant;        /* FFMA CTA tile: 0 = selector, 1 = 128 px x 128 ch,
                              2 = 256 px x 64 ch, 3 = 128 px x 64 ch,
                              4 = 256 px x 32 ch (c_b = 8);
                              see Plan.autotune in nets.py */
} dconv_conv_desc;

/* Fills `d` for a dense layer and validates it like ConvShape's constructor.
 * Returns DCONV_EINVAL_SHAPE when the reference would throw. */
int dconv_conv_desc_init(dconv_conv_desc* d, int n, int c_i, int c_o, int h_i,
                         int w_i, int h_f, int w_f, int stride, int c_ib,
                         int c_ob);

/* ConvShape validation alone (shape.cpp:30-40). */
int dconv_conv_shape(int c_i, int c_o, int h_i, int w_i, int h_f, int w_f,
                     int stride, int* h_o, int* w_o);

/* conv_flops (reference.cpp:106-109) for one image. */
int64_t dconv_conv_flops(int c_i, int c_o, int h_o, int w_o, int h_f, int w_f);

/* Direct convolution (Alg. 3) on blocked tensors.
 * in:   blocked input view, c_b == d->c_ib
 * w:    blocked kernel (c_ob, c_ib), full C_o (sharding selects blocks)
 * skip: blocked map like the output, read when epilogue has ADD (else NULL)
 * out:  blocked output view, c_b == d->c_ob.  Every valid element of the
 *       selected output blocks is written with its final value exactly once
 *       (no zero-init pass; a stream-K launch stores a partial tile into the
 *       <= #SMs tiles it cuts first); padded channel slots are written as
 *       exact 0.
 * Alignment (FFMA and tensor-core kernels): `in` and `w` 16 bytes with view
 * strides that are multiples of 4 floats (bulk copies); `out` and `skip`
 * pencil-aligned -- 32 bytes, view strides multiples of 8 floats -- because a
 * pencil moves as one 256-bit access.  cudaMalloc / torch allocations and any
 * pencil offset into them qualify.  Other views run on the generic kernel
 * (DCONV_ALGO_AUTO) or return DCONV_EUNSUPPORTED (DCONV_ALGO_FFMA).
 * Stream-K (layers whose tile count does not fill whole waves of SMs, or is
 * between a quarter of the SMs and all of them): while
 * the launch runs, `out` also carries partial tiles, so `out` must not alias
 * `skip` for such a launch to use it (aliasing launches keep the split-K
 * tail); its per-stream flags live in the module, nothing is allocated.
 * Launches of ONE stream never overlap, which the flags rely on: a CUDA
 * graph captured from stream A must not be replayed concurrently with itself
 * or with other work captured from / launched on stream A. */
int dconv_cuda_conv_direct(const dconv_conv_desc* d, const float* in,
                           const float* w, const float* skip, float* out,
                           void* stream);

/* tcgen05/TMEM TF32 variant (north_star "tensor-core variant"; looser
 * tolerance).  c_ib == c_ob == 8; stride 1, a 1x1 of any
 * stride (subsampled view), or a k x k stride-s layer (computed as a
 * stride-1 layer over the space-to-depth view of the input, which the TMA
 * reads in place with element strides s: no copy).  The weights are
 * rearranged once (like pack_kernel, tensor.cpp:85-95) into the tensor-core
 * operand layout; the caller owns that buffer (no hidden allocation).
 *   dconv_cuda_tf32_prepared_size   -> floats of the prepared weight buffer
 *   dconv_cuda_prepare_tf32_weights -> blocked kernel -> prepared weights
 *   dconv_cuda_conv_direct_tf32     -> same contract as dconv_cuda_conv_direct */
int dconv_cuda_tf32_prepared_size(const dconv_conv_desc* d, int64_t* floats);
int dconv_cuda_prepare_tf32_weights(const dconv_conv_desc* d, const float* w_blocked,
                                    float* w_prepared, void* stream);
int dconv_cuda_conv_direct_tf32(const dconv_conv_desc* d, const float* in,
                                const float* w_prepared, const float* skip, float* out,
                                void* stream);

/* Split-TF32 tensor-core variant with the fp32 tolerance of the FFMA path
 * (|a-b| <= 1e-4 + 1e-5|b| against conv_oracle64, reference.cpp:70-87):
 * x = x_hi + x_lo, w = w_hi + w_lo, three TF32 MMAs per tap
 * (x_hi*w_lo + x_lo*w_hi + x_hi*w_hi) with the reduction summed in chunks
 * of ~144 products (TMEM chunk accumulators, fp32 register totals).  Same
 * geometry limits and contract as the TF32 calls; the activation split
 * happens in shared memory (no workspace); the prepared weights hold hi and
 * lo halves (2x the TF32 buffer). */
int dconv_cuda_tf32x3_prepared_size(const dconv_conv_desc* d, int64_t* floats);
int dconv_cuda_prepare_tf32x3_weights(const dconv_conv_desc* d, const float* w_blocked,
                                      float* w_prepared, void* stream);
int dconv_cuda_conv_direct_tf32x3(const dconv_conv_desc* d, const float* in,
                                  const float* w_prepared, const float* skip, float* out,
                                  void* stream);

/* First layer: dense [N][C_i][H_i][W_i] input (the paper does not impose the
 * blocked layout on network inputs) -> blocked output.
 * d->c_ib is ignored for the input; the weights must be packed with
 * c_ib = C_i (one input block holding every channel, no zero padding). */
int dconv_cuda_conv_first_layer(const dconv_conv_desc* d, const float* in_dense,
                                int64_t in_img_stride, const float* w,
                                const float* skip, float* out, void* stream);

/* Fused gather for C_o sharding: identical to
 * dconv_cuda_conv_direct / _conv_first_layer, and every output pencil this
 * rank computes is also stored, at the same offset, into each of
 * `n_peers` (<= 7) peer copies of the output map -- device pointers that are
 * P2P-mapped over NVLink (e.g. torch symmetric memory), addressed exactly
 * like `out`.  After a barrier every rank holds the full map, with no
 * separate all-gather.  FFMA / register-tiled first-layer kernels only. */
int dconv_cuda_conv_direct_peers(const dconv_conv_desc* d, const float* in,
                                 const float* w, const float* skip, float* out,
                                 float* const* peer_outs, int n_peers, void* stream);
int dconv_cuda_conv_first_layer_peers(const dconv_conv_desc* d, const float* in_dense,
                                      int64_t in_img_stride, const float* w,
                                      const float* skip, float* out,
                                      float* const* peer_outs, int n_peers,
                                      void* stream);

/* pack_kernel: dense [C_i][C_o][H_f][W_f] -> blocked.  Bit-exact permutation,
 * padded slots written 0.  `dst` holds round_up(C_o,c_ob)*round_up(C_i,c_ib)*H_f*W_f. */
int dconv_cuda_pack_kernel(const float* src, int c_i, int c_o, int h_f, int w_f,
                           int c_ob, int c_ib, float* dst, void* stream);
int dconv_cuda_unpack_kernel(const float* src, int c_i, int c_o, int h_f,
                             int w_f, int c_ob, int c_ib, float* dst,
                             void* stream);

/* pack_feature_map over n images: dense [n][c][h][w] -> blocked
 * [n][ceil(c/c_b)][h + 2*halo][w + 2*halo][c_b]; the data lands in the
 * interior, the halo ring and padded channels are written 0 (halo = 0 gives
 * the reference layout exactly). */
int dconv_cuda_pack_feature_map(const float* src, int n, int c, int h, int w,
                                int c_b, int halo, float* dst, void* stream);
int dconv_cuda_unpack_feature_map(const float* src, int n, int c, int h, int w,
                                  int c_b, int halo, float* dst, void* stream);

/* Space-to-depth repack of a dense image batch [n][c][h][w] into the blocked
 * layout [n][ceil(c*f*f/8)][ceil(h/f)][ceil(w/f)][8]: channel (dy*f + dx)*c + ch
 * of the result is pixel (f*y + dy, f*x + dx) of channel ch (zero outside).
 * A stride-f first layer becomes a stride-1 blocked layer over it (the TF32
 * path's stems); not part of the reference API. */
int dconv_cuda_pack_space_to_depth(const float* src, int n, int c, int h, int w, int f,
                                   float* dst, void* stream);

/* The same for a blocked (c_b = 8) map view with strides in floats: a stride-f
 * blocked layer becomes a stride-1 layer over the result.  (The tensor-core
 * conv calls read this view in place with strided TMA and need no copy; this
 * materialises it, e.g. for other consumers.) */
int dconv_cuda_space_to_depth_blocked(const float* src, int64_t in_img_stride,
                                      int64_t in_blk_stride, int64_t in_row_stride, int n, int c,
                                      int h, int w, int f, float* dst, void* stream);

/* Element-wise / pooling kernels in the blocked layout (count in floats). */
int dconv_cuda_relu_blocked(float* x, int64_t count, void* stream);
int dconv_cuda_add_blocked(const float* a, const float* b, float* out,
                           int64_t count, int relu, void* stream);
/* 2x2 stride-2 max-pool per image block; writes into an output view with
 * row stride / block stride / image stride (0 = dense) so it can land in the
 * interior of the next layer's halo buffer. */
int dconv_cuda_maxpool2x2_blocked(const float* in, int n, int n_blocks, int h,
                                  int w, int c_b, float* out,
                                  int64_t out_img_stride,
                                  int64_t out_blk_stride,
                                  int64_t out_row_stride, void* stream);

/* Zeroes a float buffer (halo buffers are zeroed once, outside timing). */
int dconv_cuda_zero(float* x, int64_t count, void* stream);

/* Write-ownership check (the GPU analogue of the reference's debug ownership
 * map), in the debug build libdconv_b200_own.so only (csrc
 * `make own`; the product build returns DCONV_EUNSUPPORTED): while set,
 * every conv kernel store of an output element at address a with
 * base <= a < base + n also does atomicAdd(&counts[a - base], 1), so each
 * element of an output view must end at exactly 1.  counts = NULL clears. */
int dconv_debug_set_ownership(unsigned* counts, const float* base, int64_t n);

/* Test hook for the FFMA launcher's per-(device, kernel, ks) cache of
 * co-resident clusters: the cached answer for CTA tile `tile_variant`
 * (1..4, as dconv_conv_desc.tile_variant) and cluster size ks next to a fresh
 * cudaOccupancyMaxActiveClusters query of the same instantiation. */
int dconv_cuda_ffma_cluster_slots(int tile_variant, int ks, int* cached, int* fresh);

/* Launch accounting: number of device kernels this library launched since
 * load (for bench.py's gpu_launches claim) and the name of the last kernel. */
int64_t dconv_cuda_launch_count(void);

/* Peak FP32 FFMA throughput probe (TFLOP/s) measured with CUDA events on the
 * current device: the roofline denominator for the FFMA kernel. */
double dconv_cuda_fp32_peak_probe(void* stream);
/* The conv kernel's FFMA2 operand pattern (broadcast scalar x pair, LDS.128
 * operands, 8 px x 8 ch per thread) with no memory traffic: its practical
 * ceiling, reported beside the peak (tools/ffma2_pattern.cu). */
double dconv_cuda_ffma2_pattern_probe(void* stream);

/* ---- Tensor files --------------------------------
 * Flat little-endian file: 7 int32 header words, then the fp32 payload.
 *   feature map: {C,   H,   W,   c_b  (0 = dense CHW),  0,   0,    0}
 *   kernel:      {C_i, H_f, W_f, c_ob (0 = dense),      C_o, c_ib, 1}
 * Payload: dense CHW / [C_i][C_o][H_f][W_f], or the blocked layout with its
 * zero-padded channel slots.  (serialize.cpp is absent from the reference
 * snapshot; this is the header the SPEC describes, word order fixed here.) */
typedef struct dconv_file_header {
  int32_t c, h, w, c_b, c_o, c_ib, kind;
} dconv_file_header;
enum { DCONV_FILE_FEATURE_MAP = 0, DCONV_FILE_KERNEL = 1 };

/* Payload length in floats implied by a header (-1 if the header is invalid). */
int64_t dconv_file_payload_floats(const dconv_file_header* h);
/* Host-side I/O.  read_header validates the header and the file length. */
int dconv_file_read_header(const char* path, dconv_file_header* h);
int dconv_file_read_payload(const char* path, float* host_dst, int64_t floats);
int dconv_file_write(const char* path, const dconv_file_header* h,
                     const float* host_src, int64_t floats);
/* The CLI `pack` step: dense kernel file -> blocked kernel file, repacked on
 * the GPU (dconv_cuda_pack_kernel).  DCONV_EBLOCKED if the input is already
 * blocked. */
int dconv_pack_kernel_file(const char* in_path, int c_ob, int c_ib,
                           const char* out_path);
/* Weight ingest: a kernel file (dense or already blocked with the same
 * c_ob/c_ib) into device memory in the blocked layout `d_dst`
 * (dconv_cuda_pack_kernel's size).  Dense files are repacked on the GPU. */
int dconv_cuda_load_kernel_file(const char* path, int c_ob, int c_ib,
                                float* d_dst, void* stream);

const char* dconv_cuda_strerror(int code);
const char* dconv_cuda_last_error_detail(void);

#ifdef __cplusplus
}
#endif
#endif
