// conv_first.cu -- first-layer reader: direct convolution that consumes the
// dense network input [N][C_i][H][W] (C_i = 3 for every config) and writes the
// blocked layout (c_ob = 8).  The paper keeps the first layer's input in its
// original layout; reading it directly avoids both a packing
// pass and the 8/3x wasted FLOPs of zero-padding C_i to a channel block.
//
// CTA: 256 threads = 32 pixel groups x 8 output blocks (64 channels).  A
// pixel group is 8 consecutive output pixels of one row; each thread keeps an
// 8-pixel x 8-channel accumulator tile (FFMA2 pairs).  The CTA stages the
// weights of its 8 output blocks in shared memory once and then walks its
// pixel tiles persistently: while it computes tile i from one patch buffer
// (all C_i planes, zero-filled outside the image), cp.async fills the other
// with tile i+1.  For every (c, n) a thread loads a register row segment of
// 7*S + WF input values and reuses it across the WF filter columns
// (s*(k'*w_ob + kk) + m indexing).
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "conv_kernels.h"

namespace dconv_dev {

namespace {

constexpr int kCG = 8;     // output blocks per CTA
constexpr int kPGN = 32;   // pixel groups per CTA

struct FirstTile {
  int CX, TH;              // column groups (PX px each) x rows per CTA
  int tiles_x, tiles_y;
  int PH, PW, PWs;         // patch rows, cols, padded row stride (floats)
};

// PX: output pixels per thread (8; 2 for batch-1 maps, where 256-pixel
// tiles would leave most SMs idle)
template <int S, int WF, int PX>
__global__ void __launch_bounds__(256, 2)
    conv_first_kernel(const GenericParams p, const FirstTile t) {
  extern __shared__ __align__(16) float smem[];
  const int taps_c = p.h_f * WF * p.c_i;  // (n, m, c) rows of the weight tile
  float* sw = smem;                                   // [taps_c][2][kCG][4]
  const int patch_floats = (p.c_i * t.PH * t.PWs + 3) & ~3;
  float* sp0 = smem + taps_c * kCG * 8;               // 2 x [c_i][PH][PWs]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int tiles_img = t.tiles_x * t.tiles_y;
  const int n_tiles = tiles_img * p.n;
  const int jb0 = p.jb_begin + blockIdx.y * kCG;
  const int cg_valid = min(kCG, p.jb_begin + p.jb_count - jb0);

  pdl_wait();  // programmatic dependent launch: input readable from here on
  pdl_launch_dependents();
  // ---- stage weights once: global [jb][n][m][c][8] -> smem [(n,m,c)][half][cb][4]
  for (int e = tid; e < taps_c * kCG * 2; e += 256) {
    const int half = e & 1;
    const int cb = (e >> 1) % kCG;
    const int row = (e >> 1) / kCG;  // (n*WF + m)*c_i + c
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (cb < cg_valid)
      v = *reinterpret_cast<const float4*>(p.w + ((int64_t)(jb0 + cb) * taps_c + row) * 8 +
                                           half * 4);
    *reinterpret_cast<float4*>(sw + ((row * 2 + half) * kCG + cb) * 4) = v;
  }
  // ---- async patch staging (zero outside the image)
  auto stage = [&](int tile, float* sp) {
    const int img = tile / tiles_img, tt = tile - img * tiles_img;
    const int iy0 = (tt / t.tiles_x) * t.TH * S, ix0 = (tt % t.tiles_x) * t.CX * PX * S;
    const float* in = p.in + (int64_t)img * p.in_img;
    const int patch = p.c_i * t.PH * t.PW;
    for (int e = tid; e < patch; e += 256) {
      const int col = e % t.PW;
      const int rc = e / t.PW;
      const int row = rc % t.PH, c = rc / t.PH;
      const int gy = iy0 + row, gx = ix0 + col;
      const bool ok = gy < p.h_i && gx < p.w_i;
      cp_async4(sp + (c * t.PH + row) * t.PWs + col,
                ok ? in + (int64_t)c * p.in_blk + (int64_t)gy * p.in_row + gx : p.in, ok);
    }
    cp_async_commit();
  };

  const int pg = (lane & 3) + 4 * warp;
  const int cb = lane >> 2;
  const int r = pg % t.TH, cx = pg / t.TH;
  const bool active = cx < t.CX;

  int buf = 0;
  if ((int)blockIdx.x < n_tiles) stage(blockIdx.x, sp0);
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, buf ^= 1) {
    const int next = tile + gridDim.x;
    if (next < n_tiles) {
      stage(next, sp0 + (buf ^ 1) * patch_floats);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();  // this tile's patch (and, first time, the weights) visible
    const float* sp = sp0 + buf * patch_floats;
    const int img = tile / tiles_img, tt = tile - img * tiles_img;
    const int y0 = (tt / t.tiles_x) * t.TH, x0 = (tt % t.tiles_x) * t.CX * PX;

    // ---- compute: pixel group pg = (row r, column group cx); block cb
    uint64_t acc[PX][4];
#pragma unroll
    for (int j = 0; j < PX; ++j)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[j][q] = 0ull;
    if (active) {
      constexpr int L = (PX - 1) * S + WF;  // input columns feeding PX pixels x WF taps
      for (int c = 0; c < p.c_i; ++c) {
        // h_f == WF (square filters, checked at launch): unrolled, so the
        // accumulators stay in place across filter rows
#pragma unroll
        for (int n = 0; n < WF; ++n) {
          const float* row = sp + (c * t.PH + r * S + n) * t.PWs + cx * PX * S;
          float seg[L];
#pragma unroll
          for (int i = 0; i < L; ++i) seg[i] = row[i];
          const float* wrow = sw + ((n * WF) * p.c_i + c) * (2 * kCG * 4) + cb * 4;
#pragma unroll
          for (int m = 0; m < WF; ++m) {
            const float* wp = wrow + m * p.c_i * (2 * kCG * 4);
            const float4 b0 = lds128(wp);
            const float4 b1 = lds128(wp + kCG * 4);
            const uint64_t bp0 = pack2(b0.x, b0.y), bp1 = pack2(b0.z, b0.w);
            const uint64_t bp2 = pack2(b1.x, b1.y), bp3 = pack2(b1.z, b1.w);
#pragma unroll
            for (int j = 0; j < PX; ++j) {
              const float a = seg[j * S + m];
              ffma2(acc[j][0], a, bp0);
              ffma2(acc[j][1], a, bp1);
              ffma2(acc[j][2], a, bp2);
              ffma2(acc[j][3], a, bp3);
            }
          }
        }
      }
    }
    __syncthreads();  // everyone is done with this buffer before it is refilled

    const int y = y0 + r;
    if (!active || cb >= cg_valid || y >= p.h_o) continue;
    const int jl = jb0 + cb - p.jb_begin;
    float* obase = p.out + (int64_t)img * p.out_img + (int64_t)jl * p.out_blk +
                   (int64_t)y * p.out_row;
    const float* sbase = p.skip ? p.skip + (int64_t)img * p.sk_img + (int64_t)jl * p.sk_blk +
                                      (int64_t)y * p.sk_row
                                : nullptr;
#pragma unroll
    for (int j = 0; j < PX; ++j) {
      const int x = x0 + cx * PX + j;
      if (x >= p.w_o) break;
      const float2 c0 = unpack2(acc[j][0]), c1 = unpack2(acc[j][1]);
      const float2 c2 = unpack2(acc[j][2]), c3 = unpack2(acc[j][3]);
      float4 v0 = make_float4(c0.x, c0.y, c1.x, c1.y);
      float4 v1 = make_float4(c2.x, c2.y, c3.x, c3.y);
      if (p.epi & DCONV_EPI_ADD) {
        const float4 s0 = *reinterpret_cast<const float4*>(sbase + x * 8);
        const float4 s1 = *reinterpret_cast<const float4*>(sbase + x * 8 + 4);
        v0.x += s0.x; v0.y += s0.y; v0.z += s0.z; v0.w += s0.w;
        v1.x += s1.x; v1.y += s1.y; v1.z += s1.z; v1.w += s1.w;
      }
      if (p.epi & DCONV_EPI_RELU) {
        v0.x = fmaxf(v0.x, 0.f); v0.y = fmaxf(v0.y, 0.f);
        v0.z = fmaxf(v0.z, 0.f); v0.w = fmaxf(v0.w, 0.f);
        v1.x = fmaxf(v1.x, 0.f); v1.y = fmaxf(v1.y, 0.f);
        v1.z = fmaxf(v1.z, 0.f); v1.w = fmaxf(v1.w, 0.f);
      }
      DCONV_OWN(obase + x * 8, 8);
      *reinterpret_cast<float4*>(obase + x * 8) = v0;
      *reinterpret_cast<float4*>(obase + x * 8 + 4) = v1;
      for (int q = 0; q < p.n_peers; ++q) {  // fused C_o-shard gather
        float* po = p.peer_out[q] + (obase - p.out) + x * 8;
        *reinterpret_cast<float4*>(po) = v0;
        *reinterpret_cast<float4*>(po + 4) = v1;
      }
    }
  }
}

FirstTile pick_first_tile(const GenericParams& p, size_t w_bytes, size_t budget, int PX) {
  FirstTile best{};
  double best_eff = -1;
  size_t best_patch = 0;
  const int max_cx = std::min(kPGN, (p.w_o + PX - 1) / PX);
  for (int cx = 1; cx <= max_cx; ++cx) {
    const int th = std::min(kPGN / cx, p.h_o);
    if (th < 1) continue;
    const int tx = (p.w_o + cx * PX - 1) / (cx * PX);
    const int ty = (p.h_o + th - 1) / th;
    const int ph = (th - 1) * p.s + p.h_f;
    const int pw = (cx * PX - 1) * p.s + p.w_f;
    const int pws = pw | 1;  // odd row stride: rows of a warp hit distinct banks
    const size_t patch = (size_t)p.c_i * ph * pws * 4;
    if (w_bytes + 2 * patch > budget) continue;  // double-buffered
    const double eff = (double)p.h_o * p.w_o / ((double)tx * ty * kPGN * PX);
    if (eff > best_eff + 1e-9 || (eff > best_eff - 1e-9 && patch < best_patch)) {
      best = FirstTile{cx, th, tx, ty, ph, pw, pws};
      best_eff = eff;
      best_patch = patch;
    }
  }
  return best;
}

template <int S, int WF, int PX>
int launch_first_px(const GenericParams& p, const FirstTile& t, cudaStream_t stream) {
  const size_t w_bytes = (size_t)p.h_f * WF * p.c_i * kCG * 8 * 4;
  if (t.CX == 0) return DCONV_EUNSUPPORTED;
  const size_t patch = (((size_t)p.c_i * t.PH * t.PWs + 3) & ~size_t(3)) * 4;
  const size_t smem = w_bytes + 2 * patch;  // weights + double-buffered patch
  auto kernel = conv_first_kernel<S, WF, PX>;
  const int dev = dconv_host::current_device();
  const int sms = dconv_host::device_sms(dev);
  if (dconv_host::first_use_on_device(reinterpret_cast<const void*>(kernel), dev))
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, 256, smem) != cudaSuccess ||
      occ < 1) {
    cudaGetLastError();
    return dconv_host::set_error(DCONV_EUNSUPPORTED, "conv_first: %zu B smem per CTA", smem);
  }
  const int co_groups = (p.jb_count + kCG - 1) / kCG;
  const int n_tiles = t.tiles_x * t.tiles_y * p.n;
  // persistent: enough CTAs to fill every SM's resident slots, split over
  // the output-block groups
  const int slots = std::max(1, sms * occ / co_groups);
  dim3 grid((unsigned)std::min(n_tiles, slots), (unsigned)co_groups);
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.gridDim = grid;
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cfg.attrs = attr;
  cfg.numAttrs = dconv_host::pdl_enabled() ? 1 : 0;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, p, t);
  if (e != cudaSuccess)
    return dconv_host::set_error(DCONV_ECUDA, "conv_first: %s", cudaGetErrorString(e));
  dconv_host::count_launch();
  return dconv_host::check_launch("conv_first_kernel");
}

template <int S, int WF>
int launch_first(const GenericParams& p, cudaStream_t stream) {
  const int sms = dconv_host::device_sms(dconv_host::current_device());
  const size_t w_bytes = (size_t)p.h_f * WF * p.c_i * kCG * 8 * 4;
  const size_t budget = 220 * 1024;
  const int co_groups = (p.jb_count + kCG - 1) / kCG;
  // 8 pixels per thread unless that leaves SMs idle (batch-1 maps): then 2
  const FirstTile t8 = pick_first_tile(p, w_bytes, budget, 8);
  if (t8.CX == 0) return DCONV_EUNSUPPORTED;
  if ((int64_t)t8.tiles_x * t8.tiles_y * p.n * co_groups >= sms)
    return launch_first_px<S, WF, 8>(p, t8, stream);
  const FirstTile t2 = pick_first_tile(p, w_bytes, budget, 2);
  if (t2.CX == 0) return launch_first_px<S, WF, 8>(p, t8, stream);
  return launch_first_px<S, WF, 2>(p, t2, stream);
}

}  // namespace

int launch_conv_first_fast(const GenericParams& p, cudaStream_t stream) {
  if (p.c_ob != 8 || p.h_f != p.w_f) return DCONV_EUNSUPPORTED;
  // many-tile layers: the TMA-store reader (conv_reader.cu)
  static const bool no_reader = getenv("DCONV_NO_READER") != nullptr;
  if (!no_reader) {
    const int rc = launch_conv_reader(p, stream);
    if (rc != DCONV_EUNSUPPORTED) return rc;
  }
  if (p.s == 1 && p.w_f == 3) return launch_first<1, 3>(p, stream);
  if (p.s == 2 && p.w_f == 7) return launch_first<2, 7>(p, stream);
  if (p.s == 4 && p.w_f == 11) return launch_first<4, 11>(p, stream);
  if (p.s == 1 && p.w_f == 5) return launch_first<1, 5>(p, stream);
  if (p.s == 1 && p.w_f == 1) return launch_first<1, 1>(p, stream);
  if (p.s == 2 && p.w_f == 3) return launch_first<2, 3>(p, stream);
  return DCONV_EUNSUPPORTED;
}

}  // namespace dconv_dev
