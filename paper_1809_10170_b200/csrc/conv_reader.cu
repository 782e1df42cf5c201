// conv_reader.cu -- first-layer reader with TMA-stored output tiles.
//
// The network input is the dense image [N][C_i][H][W] (C_i = 3, PAPER.md:18-21:
// the first layer keeps its input layout); the output is the blocked map
// [N][C_o/8][H_o][W_o][8].  A 3-channel input with 64 output channels is an
// output-heavy layer: VGG conv1_1 at batch 32 moves 20 MB in and 411 MB out
// for 5.5 GFLOP, so the FP32 pipe and the output stream have to run
// concurrently.  Design (persistent CTAs, 256 threads, 1-2 per SM):
//
//  * warp w owns output block j' = w of the CTA's 8 blocks (64 channels), lane
//    x one output column of the tile; each thread keeps an 8-row x 8-channel
//    accumulator tile (32 FFMA2 pairs), so the weights of a tap are one
//    broadcast LDS.128 pair per warp and the input column segment of
//    7*S + W_F values is reused across the W_F filter rows;
//  * the input patch (all C_i planes, zero outside the image) is staged with
//    4-byte cp.async by all threads for the NEXT tile while this one computes,
//    in a 3-deep ring that needs one __syncthreads per tile.  The dense rows
//    start at arbitrary 4-byte offsets (W = 226, 229, 227 floats per row) and
//    a tensor map needs 16-byte row strides, so the input cannot be a TMA
//    tensor.  Strided layers store the patch de-interleaved by column phase
//    so lanes read consecutive words;
//  * each warp writes its finished block (ReLU applied) to its own staging
//    tile in exactly the blocked layout [TH rows][TW px][8 ch] and stores it
//    with its own TMA tensor store (cp.async.bulk.tensor, SASS UTMASTG):
//    whole 32-byte pencils, ragged tiles clipped at the map edge, no CTA
//    barrier, overlapping the next tile's FFMA2s (the warp awaits only the
//    store's shared-memory read before reusing its staging tile).  The
//    register-tiled reader stored each pencil as two half-sector STG.128s
//    from 32 different rows per warp instruction -- 32 sectors per request,
//    twice the L2 write traffic.
//  * all tile geometry is compile-time (C_i = 3): every shared-memory offset
//    of the inner loop is an immediate.
// Measured (B200, tools/one_layer.py): VGG conv1_1 b32 271 -> 138 us,
// GoogLeNet 7x7/s2 stem b64 381 -> 305 us (ResNet b256: 1.15 ms, 52.7 TFLOP/s).
//
// Zero workspace: the staging tile, patch and weights live in shared memory.
// Fallbacks (the register-tiled reader in conv_first.cu): fused skip-add,
// fused peer stores, filters/strides without a specialisation, few tiles.
#include <algorithm>
#include <cstdlib>
#include <cuda.h>

#include "common.cuh"
#include "conv_kernels.h"
#include "tf32_common.cuh"  // encode_fn (cuTensorMapEncodeTiled)

namespace dconv_dev {

namespace {

constexpr int kRThreads = 256;
constexpr int kBlocks = 8;     // output blocks per CTA (one per warp)

struct ReaderParams {
  const float* in;
  const float* w;
  float* out;                  // (ownership debug build: the TMA store's elements)
  int64_t in_img, in_blk, in_row;
  int64_t out_img, out_blk, out_row;
  int n, c_i, h_i, w_i, h_o, w_o;
  int jb_begin, jb_count, co_groups;
  int tiles_x, tiles_y;
  int relu;
};

__device__ __forceinline__ void tma_store_5d(const CUtensorMap* map, const void* src, int c0,
                                             int c1, int c2, int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4, %5, %6}], "
      "[%1];" ::"l"(reinterpret_cast<uint64_t>(map)),
      "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Compile-time tile geometry (C_i = CI channels, stride S, W_F x W_F filter,
// TW-wide tiles, R accumulator rows per thread): every shared-memory offset
// of the inner loops is an immediate.
template <int CI, int S, int WF, int TW, int R>
struct RGeom {
  static constexpr int NB = 3;                   // patch ring depth
  static constexpr int TH = R * (32 / TW);       // tile rows: R (TW 32) or 2R (TW 16)
  static constexpr int L = (R - 1) * S + WF;     // input rows feeding R output rows
  static constexpr int PH = (TH - 1) * S + WF;   // patch rows
  static constexpr int PWC = (TW - 1) * S + WF;  // patch columns
  static constexpr int PQ = (PWC + S - 1) / S;   // words per column phase
  // floats per patch row (S phases); TW = 16: the second row band starts
  // R*S rows later -- pad so that offset is 16 banks mod 32
  static constexpr int rowlen_for(int v) {
    return (TW != 16 || (R * S * v) % 32 == 16) ? v : rowlen_for(v + 1);
  }
  static constexpr int ROWLEN = rowlen_for(S * PQ);
  static constexpr int PATCH = (CI * PH * ROWLEN + 31) & ~31;  // one buffer, floats
  static constexpr int WFLOATS = (WF * WF * CI * 8 * 8 + 31) & ~31;
  static constexpr int OUTW = TH * TW * 8;                     // one warp's staging tile
  static constexpr size_t SMEM = (size_t)(8 * OUTW + WFLOATS + NB * PATCH) * 4;
};

// Warps 0-7: warp w computes output block w of the CTA's 8 and stores it with
// its own TMA store (no CTA barrier in the epilogue).  All 256 threads stage
// the patch of tile t+1 with cp.async while computing tile t; a 3-deep patch
// ring makes ONE __syncthreads per tile enough: at tile t the warps write
// slot (t+1) % 3, last read at tile t-2, which every warp finished before
// passing tile t-1's barrier.
// TW: tile width in output columns (32: one lane per column; 16: lanes
// 16-31 take the tile's second band of R rows).
template <int CI, int S, int WF, int TW, int R, int MINB>
__global__ void __launch_bounds__(kRThreads, MINB)
    conv_reader_kernel(const __grid_constant__ CUtensorMap omap, const ReaderParams p) {
  using G = RGeom<CI, S, WF, TW, R>;
  constexpr int NB = G::NB, TH = G::TH, L = G::L, PH = G::PH, PWC = G::PWC, PQ = G::PQ;
  constexpr int ROWLEN = G::ROWLEN;
  constexpr int TAPS_C = WF * WF * CI;
  extern __shared__ __align__(1024) float smem[];
  float* stage_out = smem;                     // [8 warps][TH][TW][8]
  float* wsm = stage_out + 8 * G::OUTW;        // [(n*WF + m)*CI + c][8 blk][8]
  float* patch0 = wsm + G::WFLOATS;            // NB x [c][PH][S][PQ (+pad)]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int tiles_img = p.tiles_x * p.tiles_y;
  const int n_tiles = tiles_img * p.n;
  const int cgi = blockIdx.y;
  const int jb0 = p.jb_begin + cgi * kBlocks;
  const int cg_valid = min(kBlocks, p.jb_begin + p.jb_count - jb0);

  pdl_wait();
  pdl_launch_dependents();
  // weights of the CTA's 8 blocks, once
  for (int e = tid; e < TAPS_C * kBlocks * 2; e += kRThreads) {
    const int half = e & 1, b = (e >> 1) % kBlocks, row = (e >> 1) / kBlocks;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (b < cg_valid)
      v = *reinterpret_cast<const float4*>(p.w + ((int64_t)(jb0 + b) * TAPS_C + row) * 8 +
                                           half * 4);
    *reinterpret_cast<float4*>(wsm + (row * kBlocks + b) * 8 + half * 4) = v;
  }
  // patch of a tile = CI x PH rows x PWC columns from input column x0*S;
  // column q stored at phase q % S, word q / S (zero outside the image)
  auto stage = [&](int tile, float* sp) {
    const int img = tile / tiles_img, tt = tile - img * tiles_img;
    const int ty = tt / p.tiles_x;
    const int iy0 = ty * TH * S, ix0 = (tt - ty * p.tiles_x) * TW * S;
    const float* in = p.in + (int64_t)img * p.in_img + ix0;
    const int cols = min(PWC, p.w_i - ix0);  // columns inside the image
#pragma unroll 1
    for (int rr = warp; rr < CI * PH; rr += kRThreads / 32) {
      const int c = rr / PH, row = rr - c * PH;
      const int gy = iy0 + row;
      const bool row_ok = gy < p.h_i;
      const float* src = in + (int64_t)c * p.in_blk + (int64_t)gy * p.in_row;
      float* dst = sp + rr * ROWLEN;
#pragma unroll
      for (int q0 = 0; q0 < PWC; q0 += 32) {
        const int q = q0 + lane;
        if (q < PWC) {
          const bool ok = row_ok && q < cols;
          cp_async4(dst + (q % S) * PQ + q / S, ok ? src + q : p.in, ok);
        }
      }
    }
    cp_async_commit();
  };

  const int cb = warp;                        // output block within the CTA
  const int x = lane % TW, band = lane / TW;  // tile column, row band
  float* my_out = stage_out + warp * G::OUTW;
  if ((int)blockIdx.x < n_tiles) stage(blockIdx.x, patch0);
  int it = 0;
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++it) {
    const int next = tile + gridDim.x;
    if (next < n_tiles) {
      stage(next, patch0 + ((it + 1) % NB) * G::PATCH);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();  // this tile's patch (and, first time, the weights) visible
    const float* sp = patch0 + (it % NB) * G::PATCH;
    const int img = tile / tiles_img, tt = tile - img * tiles_img;
    const int ty = tt / p.tiles_x;
    const int y0 = ty * TH, x0 = (tt - ty * p.tiles_x) * TW;

    uint64_t acc[R][4];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[r][q] = 0ull;
    const float* wcb = wsm + cb * 8;
    const float* pband = sp + band * (R * S) * ROWLEN + x;
#pragma unroll
    for (int c = 0; c < CI; ++c) {
#pragma unroll
      for (int m = 0; m < WF; ++m) {
        // input column x*S + m of the band's L rows (phase m % S, word x + m / S)
        const float* col = pband + c * PH * ROWLEN + (m % S) * PQ + m / S;
        float seg[L];
#pragma unroll
        for (int i = 0; i < L; ++i) seg[i] = col[i * ROWLEN];
#pragma unroll
        for (int n = 0; n < WF; ++n) {
          const float* wp = wcb + ((n * WF + m) * CI + c) * (kBlocks * 8);
          const float4 b0 = lds128(wp), b1 = lds128(wp + 4);
          const uint64_t bp0 = pack2(b0.x, b0.y), bp1 = pack2(b0.z, b0.w);
          const uint64_t bp2 = pack2(b1.x, b1.y), bp3 = pack2(b1.z, b1.w);
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const float a = seg[r * S + n];
            ffma2(acc[r][0], a, bp0);
            ffma2(acc[r][1], a, bp1);
            ffma2(acc[r][2], a, bp2);
            ffma2(acc[r][3], a, bp3);
          }
        }
      }
    }
    // ---- epilogue: this warp's block -> staging tile -> its own TMA store
    if (lane == 0) bulk_wait_read0();  // its previous store has read the staging tile
    __syncwarp();
    float* ob = my_out + ((band * R) * TW + x) * 8;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      float v[8];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 f = unpack2(acc[r][q]);
        v[2 * q] = f.x;
        v[2 * q + 1] = f.y;
      }
      if (p.relu) {
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = fmaxf(v[i], 0.f);
      }
      float* o = ob + r * TW * 8;
#ifdef DCONV_DEBUG_OWNERSHIP
      {  // the elements the TMA store writes (clipped at the map edge)
        const int y = y0 + band * R + r, xx = x0 + x;
        if (y < p.h_o && xx < p.w_o && cb < cg_valid)
          DCONV_OWN(p.out + (int64_t)img * p.out_img + (int64_t)(cgi * kBlocks + cb) * p.out_blk +
                        (int64_t)y * p.out_row + (int64_t)xx * 8, 8);
      }
#endif
      // lanes 4-7 of each quarter-warp write the high half first: the 8
      // lanes' 16-byte stores then hit 8 distinct bank groups
      const float4 lo = make_float4(v[0], v[1], v[2], v[3]);
      const float4 hi = make_float4(v[4], v[5], v[6], v[7]);
      const bool swp = (x >> 2) & 1;
      *reinterpret_cast<float4*>(o + (swp ? 4 : 0)) = swp ? hi : lo;
      *reinterpret_cast<float4*>(o + (swp ? 0 : 4)) = swp ? lo : hi;
    }
    fence_proxy_async_smem();  // generic-proxy writes -> visible to the TMA engine
    __syncwarp();
    if (lane == 0 && cb < cg_valid) {
      tma_store_5d(&omap, my_out, 0, x0, y0, cgi * kBlocks + cb, img);
      bulk_commit();
    }
  }
  if (lane == 0) bulk_wait0();  // stores complete before the CTA's shared memory goes away
}

template <int CI, int S, int WF, int TW, int R, int MINB>
int launch_reader(const GenericParams& g, cudaStream_t stream) {
  using Gm = RGeom<CI, S, WF, TW, R>;
  ReaderParams p{};
  p.in = g.in; p.w = g.w; p.out = g.out;
  p.in_img = g.in_img; p.in_blk = g.in_blk; p.in_row = g.in_row;
  p.out_img = g.out_img; p.out_blk = g.out_blk; p.out_row = g.out_row;
  p.n = g.n; p.c_i = g.c_i; p.h_i = g.h_i; p.w_i = g.w_i; p.h_o = g.h_o; p.w_o = g.w_o;
  p.jb_begin = g.jb_begin; p.jb_count = g.jb_count;
  p.co_groups = (g.jb_count + kBlocks - 1) / kBlocks;
  p.tiles_x = (g.w_o + TW - 1) / TW;
  p.tiles_y = (g.h_o + Gm::TH - 1) / Gm::TH;
  p.relu = (g.epi & DCONV_EPI_RELU) ? 1 : 0;
  const size_t smem = Gm::SMEM;
  if (smem > 220 * 1024) return DCONV_EUNSUPPORTED;

  // output tensor map: {8 ch, W_o, H_o, blocks, images} over the (view) output
  CUtensorMap map;
  if (!tf32::encode_fn()) return DCONV_EUNSUPPORTED;
  const cuuint64_t dims[5] = {8, (cuuint64_t)g.w_o, (cuuint64_t)g.h_o, (cuuint64_t)g.jb_count,
                              (cuuint64_t)g.n};
  const cuuint64_t strides[4] = {32, (cuuint64_t)g.out_row * 4, (cuuint64_t)g.out_blk * 4,
                                 (cuuint64_t)g.out_img * 4};
  const cuuint32_t box[5] = {8, (cuuint32_t)TW, (cuuint32_t)Gm::TH, 1, 1};  // one block
  const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  if (tf32::encode_fn()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, g.out, dims, strides, box,
                        estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
      CUDA_SUCCESS)
    return DCONV_EUNSUPPORTED;

  auto kernel = conv_reader_kernel<CI, S, WF, TW, R, MINB>;
  const int dev = dconv_host::current_device();
  const int sms = dconv_host::device_sms(dev);
  if (dconv_host::first_use_on_device(reinterpret_cast<const void*>(kernel), dev))
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kRThreads, smem) !=
          cudaSuccess ||
      occ < 1) {
    cudaGetLastError();
    return DCONV_EUNSUPPORTED;
  }
  const int n_tiles = p.tiles_x * p.tiles_y * p.n;
  const int per_group = std::max(1, sms * std::min(occ, MINB) / p.co_groups);
  dim3 grid((unsigned)std::min(n_tiles, per_group), (unsigned)p.co_groups);
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.gridDim = grid;
  cfg.blockDim = dim3(kRThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cfg.attrs = attr;
  cfg.numAttrs = dconv_host::pdl_enabled() ? 1 : 0;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, map, p);
  if (e != cudaSuccess)
    return dconv_host::set_error(DCONV_ECUDA, "conv_reader: %s", cudaGetErrorString(e));
  dconv_host::count_launch();
  return dconv_host::check_launch("conv_reader_kernel");
}

template <int S, int WF>
int pick_width(const GenericParams& g, cudaStream_t stream) {
  // tile width 32 unless the map width wastes less with 16 (112 = 7 x 16)
  const int waste32 = (g.w_o + 31) / 32 * 32 - g.w_o;
  const int waste16 = (g.w_o + 15) / 16 * 16 - g.w_o;
  const bool w16 = waste16 < waste32;
  const int sms = dconv_host::device_sms(dconv_host::current_device());
  const int64_t groups = (g.jb_count + kBlocks - 1) / kBlocks;
  auto tiles = [&](int tw, int r) {
    const int th = r * (32 / tw);
    return (int64_t)g.n * ((g.h_o + th - 1) / th) * ((g.w_o + tw - 1) / tw) * groups;
  };
  // few tiles (batch-1 maps): 2 accumulator rows per thread, 4x the tiles
  if (WF > 7 || tiles(w16 ? 16 : 32, 8) < sms) {
    if (w16) return launch_reader<3, S, WF, 16, 2, 1>(g, stream);
    return launch_reader<3, S, WF, 32, 2, 1>(g, stream);
  }
  // 3x3: two CTAs per SM (one CTA's barrier / epilogue overlaps the other's
  // FFMA2s; 120 registers).  7x7/s2: one CTA per SM with the full register
  // file -- measured on B200 (GoogLeNet stem b64 / b256): 304 / 1146 us
  // against 309 / 1193 us with two CTAs of 4-row threads.
  if constexpr (WF == 7) {
    if (w16) return launch_reader<3, S, WF, 16, 8, 1>(g, stream);
    return launch_reader<3, S, WF, 32, 8, 1>(g, stream);
  } else if constexpr (WF == 3) {
    if (w16) return launch_reader<3, S, WF, 16, 8, 2>(g, stream);
    return launch_reader<3, S, WF, 32, 8, 2>(g, stream);
  }
  return DCONV_EUNSUPPORTED;
}

}  // namespace

int launch_conv_reader(const GenericParams& g, cudaStream_t stream) {
  // many-tile layers with a ReLU / plain epilogue written to this rank's map only
  if (g.c_ob != 8 || g.c_i != 3 || g.h_f != g.w_f || g.n_peers || (g.epi & ~DCONV_EPI_RELU))
    return DCONV_EUNSUPPORTED;
  if (g.s == 1 && g.w_f == 3) return pick_width<1, 3>(g, stream);
  if (g.s == 2 && g.w_f == 7) return pick_width<2, 7>(g, stream);
  if (g.s == 4 && g.w_f == 11) return pick_width<4, 11>(g, stream);
  return DCONV_EUNSUPPORTED;
}

}  // namespace dconv_dev
