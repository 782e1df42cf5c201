// conv_kernels.h -- internal launcher interfaces between the C-ABI layer
// (abi.cu) and the kernels.  Not part of the public boundary.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace dconv_dev {

// Parameters of the FFMA direct-conv kernel (c_ib = c_ob = 8).  All strides
// in floats.  Tiling / staging fields are filled in by the launcher.
constexpr int kMaxPeers = 7;  // fused C_o-shard gather: up to 8 GPUs

struct FfmaParams {
  const float* in;
  const float* w;
  const float* skip;
  float* out;
  int n, h_i, w_i, h_o, w_o, h_f, w_f, s;
  int cbs;                  // channel block of maps and kernel (c_ib = c_ob): 8, 16, 32
  int ib_n;                 // input channel blocks (padded C_i / cbs)
  int jb_n;                 // output channel blocks in the weights (of cbs)
  int jb_begin, jb_count;   // output 8-channel sub-blocks computed (launcher: * cbs/8)
  int64_t in_img, in_blk, in_row;
  int64_t out_img, out_blk, out_row;
  int64_t sk_img, sk_blk, sk_row;
  int epi;
  // launcher-filled
  int TH, TW, TWe, tiles_x, tiles_y;  // tiles over the batch-stacked output
  int G, R, n_g, n_r, PH, PW;
  int slab_floats, patch_floats, wstride_floats, stage_floats, NS;
  int flush_every;          // stages per partial sum before the TMEM fold
  int ksplit;               // CTAs per cluster sharing one unit's K range (1,2,4,8)
  int red_floats;           // smem floats of the split-K partial buffer
  int unit_begin, unit_count;  // work units of this launch
  int variant;                 // requested CTA tile (-1 = selector)
  int skip_prefetch;           // ADD epilogue: L2-prefetch the skip tile a unit ahead
  int sy;                      // row stride of the staged patch (s, or 1 for 1x1 re-viewed)
  unsigned tw_magic;           // ceil(2^32 / TW)
  unsigned h_o_magic;          // ceil(2^32 / h_o) when n * h_o^2 < 2^32, else 0
  // fused gather: every output store is repeated at the same offset from
  // each peer's copy of the output map (P2P-mapped over NVLink)
  int n_peers;
  float* peer_out[kMaxPeers];
  int epi_wg;                  // 1: compute warps hand tiles to the epilogue warpgroup
  // stream-K (whole-K launches whose units do not fill whole waves): CTA b
  // runs stages [b*W/P, (b+1)*W/P) of the launch's units x S stages; a unit
  // cut by a range boundary is finished by the CTA holding its first stages,
  // which adds the partial tile the next CTA left in the output map itself
  // (flag sk_flags[b + 1]); no workspace
  int streamk;
  int sk_base;                 // units [0, sk_base) run whole, round-robin, before the stream-K range
  unsigned* sk_flags;          // one flag per CTA (device-resident, self-resetting)
  int dense1x1;                // 1: 1x1/s1 stage whose patch is the tile itself (pixel q at q * c_b)
  long long* dbg;              // DCONV_FFMA_PROFILE: per-CTA phase clocks (else null)
};

int launch_conv_ffma(const FfmaParams& p, cudaStream_t stream);
int ffma_cluster_slots_probe(int tile_variant, int ks, int* cached, int* fresh);

// tcgen05/TMEM TF32 variant (conv_tf32.cu): weights prepared once into the
// UMMA K-major layout by launch_prepare_tf32.  A k x k stride-s layer is
// computed as a stride-1 layer over the space-to-depth view of its input
// (s*s*C_i channels, ceil(k/s) filter, read in place by strided TMA); its
// prepared weights are rearranged accordingly from the original ones (WSrc).
struct WSrc {
  int s, ib_o, hf_o, wf_o;  // space-to-depth factor, original input blocks and filter
};
// computed-layer geometry (ib_n, h_f, w_f) and weight source for a layer
inline void tc_geometry(int ib_o, int h_f, int w_f, int stride, int& ib_n, int& hf, int& wf,
                        WSrc& src) {
  const int s = (stride > 1 && (h_f > 1 || w_f > 1)) ? stride : 1;
  ib_n = ib_o * s * s;
  hf = (h_f + s - 1) / s;
  wf = (w_f + s - 1) / s;
  src = WSrc{s, ib_o, h_f, w_f};
}
int64_t tf32_prepared_floats(int ib_n, int h_f, int w_f, int jb_count);
int launch_prepare_tf32(const float* w, int ib_n, int h_f, int w_f, int jb_begin, int jb_count,
                        const WSrc& src, float* out, cudaStream_t stream);
int launch_conv_tf32(const FfmaParams& p, const float* w_prepared, cudaStream_t stream);

// split-TF32 variant (conv_tf32x3.cu): fp32 tolerance on the tensor cores;
// weights prepared once into hi/lo operand pairs.
int64_t tf32x3_prepared_floats(int ib_n, int h_f, int w_f, int jb_count);
int launch_prepare_tf32x3(const float* w, int ib_n, int h_f, int w_f, int jb_begin, int jb_count,
                          const WSrc& src, float* out, cudaStream_t stream);
int launch_conv_tf32x3(const FfmaParams& p, const float* w_prepared, cudaStream_t stream);

// Generic (any c_ib / c_ob) reference-order kernel and the first-layer reader.
struct GenericParams {
  const float* in;
  const float* w;
  const float* skip;
  float* out;
  int n, c_i, h_i, w_i, h_o, w_o, h_f, w_f, s, c_ib, c_ob;
  int ib_n, jb_n, jb_begin, jb_count;
  int64_t in_img, in_blk, in_row;    // for dense input: in_blk = H*W, in_row = W
  int64_t out_img, out_blk, out_row;
  int64_t sk_img, sk_blk, sk_row;
  int epi;
  int dense_input;                   // 1: first layer, input [N][C_i][H][W]
  int n_peers;                       // fused gather (first-layer reader only)
  float* peer_out[kMaxPeers];
};

int launch_conv_generic(const GenericParams& p, cudaStream_t stream);
int launch_conv_first_layer(const GenericParams& p, cudaStream_t stream);
// register-tiled first-layer reader (c_ob = 8); DCONV_EUNSUPPORTED if no
// specialisation matches (the caller then uses launch_conv_first_layer).
int launch_conv_first_fast(const GenericParams& p, cudaStream_t stream);
// first-layer reader with TMA-stored output tiles (conv_reader.cu): 3x3/s1 and
// 7x7/s2 on many tiles, ReLU / plain epilogue; DCONV_EUNSUPPORTED otherwise.
int launch_conv_reader(const GenericParams& p, cudaStream_t stream);

}  // namespace dconv_dev
