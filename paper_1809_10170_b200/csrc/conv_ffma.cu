// conv_ffma.cu -- register-blocked FP32 FFMA direct convolution for sm_100a.
//
// GPU restatement of Alg. 3 in the blocked layout with
// c_ib = c_ob = 8 (one 32-byte pencil = one DRAM sector per pixel):
//   * j' (output blocks, "in Parallel")      -> blockIdx.y, CG blocks per CTA
//   * l, k' (output rows / row tiles)        -> blockIdx.x, a TH x TW pixel tile
//   * i' (input blocks, cache blocking)      -> the smem pipeline stage
//   * (n, m, ii) reduction                   -> per-stage loop from smem
//   * (kk, jj) register tile                 -> 8 pixels x 8 channels / thread
// The input index is s*(k'*w_ob + kk) + m (SPEC.md:354 stride fix).
//
// Data movement: a dedicated producer warp streams each stage -- the input
// patch rows of G i'-blocks (each patch row is contiguous in the blocked
// layout) and the matching (j', i') weight slab rows (contiguous,
// tensor.hpp:138-140) -- with 1-D bulk async copies (cp.async.bulk -> UBLKCP)
// into an NS-deep ring of shared-memory stages guarded by full/empty
// mbarriers.  Eight compute warps consume.  Nothing is written to global
// memory except the output, once, from registers (zero workspace).
#include <algorithm>
#include <cstdio>

#include "common.cuh"
#include "conv_kernels.h"

namespace dconv_dev {

namespace {

constexpr int kCB = 8;             // channel block of this kernel (c_ib = c_ob)
constexpr int kComputeWarps = 8;   // 256 compute threads, 8x8 outputs each
constexpr int kThreads = (kComputeWarps + 1) * 32;  // + producer warp
constexpr int kMaxStages = 8;

template <int BM, int BN>
__global__ void __launch_bounds__(kThreads, 1)
    conv_ffma_kernel(const FfmaParams p) {
  constexpr int PG = BM / 8;  // pixel groups
  constexpr int CG = BN / 8;  // channel groups == output blocks per CTA
  constexpr int WR = PG / 4;  // warps along pixels
  static_assert(PG * CG == kComputeWarps * 32, "thread tile mismatch");

  extern __shared__ __align__(128) float smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.NS * p.stage_floats);
  uint64_t* empty = full + kMaxStages;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int img = blockIdx.x / p.tiles_per_img;
  const int tile = blockIdx.x - img * p.tiles_per_img;
  const int ty0 = (tile / p.tiles_x) * p.TH;
  const int tx0 = (tile % p.tiles_x) * p.TW;
  const int jb0 = p.jb_begin + blockIdx.y * CG;  // first output block (global)
  const int cg_valid = min(CG, p.jb_begin + p.jb_count - jb0);
  const int S = p.n_g * p.n_r;

  if (tid == 0) {
    for (int i = 0; i < p.NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kComputeWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == kComputeWarps) {
    // ------------------------------------------------------------ producer
    const float* in_img = p.in + (int64_t)img * p.in_img;
    const int col0 = tx0 * p.s;
    const int cols = min(p.PW, p.w_i - col0);
    for (int st = 0; st < S; ++st) {
      const int buf = st % p.NS;
      if (st >= p.NS) mbar_wait(&empty[buf], ((st / p.NS) - 1) & 1);
      const int g = st / p.n_r, r = st - g * p.n_r;
      const int ib0 = g * p.G, Ge = min(p.G, p.ib_n - ib0);
      const int n0 = r * p.R, Re = min(p.R, p.h_f - n0);
      const int row0 = ty0 * p.s + n0;
      const int rows = min((p.THe - 1) * p.s + Re, p.h_i - row0);
      const uint32_t patch_bytes = (uint32_t)(Ge * rows * cols * kCB * 4);
      const uint32_t wbytes = (uint32_t)(Re * p.w_f * kCB * kCB * 4) * Ge;
      float* sp = smem + buf * p.stage_floats;
      float* sw = sp + p.patch_floats;
      if (lane == 0)
        mbar_arrive_expect_tx(&full[buf], patch_bytes + wbytes * cg_valid);
      __syncwarp();
      const int n_patch = Ge * rows;
      const int tasks = n_patch + cg_valid;
      for (int t = lane; t < tasks; t += 32) {
        if (t < n_patch) {
          const int gi = t / rows, pr = t - gi * rows;
          const float* src = in_img + (int64_t)(ib0 + gi) * p.in_blk +
                             (int64_t)(row0 + pr) * p.in_row +
                             (int64_t)col0 * kCB;
          float* dst = sp + ((gi * p.PH + pr) * p.PW) * kCB;
          bulk_g2s(dst, src, (uint32_t)(cols * kCB * 4), &full[buf]);
        } else {
          const int c = t - n_patch;
          const float* src =
              p.w + ((int64_t)(jb0 + c) * p.ib_n + ib0) * p.slab_floats +
              (int64_t)n0 * p.w_f * kCB * kCB;
          bulk_g2s(sw + c * p.wstride_floats, src, wbytes, &full[buf]);
        }
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const int wr = warp % WR, wc = warp / WR;
  const int pg = wr * 4 + (lane & 3);
  const int cg = wc * 8 + (lane >> 2);

  int poff[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int q = pg + PG * k;
    const int ty = q / p.TW, tx = q - (q / p.TW) * p.TW;
    // pixels beyond the clamped patch never store; point them at offset 0
    poff[k] = (ty < p.THe && tx < p.TWe) ? (ty * p.s * p.PW + tx * p.s) * kCB : 0;
  }

  // acc[k][c2] holds channels (2*c2, 2*c2+1) of pixel k as an fp32 pair so
  // every update is one FFMA2 (fma.rn.f32x2, scalar-broadcast input).
  uint64_t acc[8][4];
#pragma unroll
  for (int k = 0; k < 8; ++k)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[k][c] = 0ull;

  const int wf = p.w_f;
  for (int st = 0; st < S; ++st) {
    const int buf = st % p.NS;
    mbar_wait(&full[buf], (st / p.NS) & 1);
    const int g = st / p.n_r, r = st - g * p.n_r;
    const int Ge = min(p.G, p.ib_n - g * p.G);
    const int Re = min(p.R, p.h_f - r * p.R);
    const float* sp = smem + buf * p.stage_floats;
    const float* sw = sp + p.patch_floats + cg * p.wstride_floats;
    for (int gi = 0; gi < Ge; ++gi) {
      for (int n = 0; n < Re; ++n) {
        const float* pa_row = sp + ((gi * p.PH + n) * p.PW) * kCB;
        const float* pw_row = sw + ((gi * p.R + n) * wf) * (kCB * kCB);
        for (int m = 0; m < wf; ++m) {
          const float* pa = pa_row + m * kCB;
          const float* pw = pw_row + m * (kCB * kCB);
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            float4 a[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) a[k] = lds128(pa + poff[k] + half * 4);
#pragma unroll
            for (int i4 = 0; i4 < 4; ++i4) {
              const float4 b0 = lds128(pw + (half * 4 + i4) * kCB);
              const float4 b1 = lds128(pw + (half * 4 + i4) * kCB + 4);
              const uint64_t bp0 = pack2(b0.x, b0.y), bp1 = pack2(b0.z, b0.w);
              const uint64_t bp2 = pack2(b1.x, b1.y), bp3 = pack2(b1.z, b1.w);
#pragma unroll
              for (int k = 0; k < 8; ++k) {
                const float av = i4 == 0 ? a[k].x
                                 : i4 == 1 ? a[k].y
                                 : i4 == 2 ? a[k].z
                                           : a[k].w;
                ffma2(acc[k][0], av, bp0);
                ffma2(acc[k][1], av, bp1);
                ffma2(acc[k][2], av, bp2);
                ffma2(acc[k][3], av, bp3);
              }
            }
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[buf]);
  }

  // -------------------------------------------------------------- epilogue
  if (cg >= cg_valid) return;
  const int jl = jb0 + cg - p.jb_begin;  // block index within the output view
  float* obase = p.out + (int64_t)img * p.out_img + (int64_t)jl * p.out_blk;
  const float* sbase =
      p.skip ? p.skip + (int64_t)img * p.sk_img + (int64_t)jl * p.sk_blk
             : nullptr;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int q = pg + PG * k;
    const int ty = q / p.TW, tx = q - (q / p.TW) * p.TW;
    const int y = ty0 + ty, x = tx0 + tx;
    if (y >= p.h_o || x >= p.w_o) continue;
    const float2 c0 = unpack2(acc[k][0]), c1 = unpack2(acc[k][1]);
    const float2 c2 = unpack2(acc[k][2]), c3 = unpack2(acc[k][3]);
    float4 v0 = make_float4(c0.x, c0.y, c1.x, c1.y);
    float4 v1 = make_float4(c2.x, c2.y, c3.x, c3.y);
    if (p.epi & DCONV_EPI_ADD) {
      const float* sk = sbase + (int64_t)y * p.sk_row + (int64_t)x * kCB;
      const float4 s0 = *reinterpret_cast<const float4*>(sk);
      const float4 s1 = *reinterpret_cast<const float4*>(sk + 4);
      v0.x += s0.x; v0.y += s0.y; v0.z += s0.z; v0.w += s0.w;
      v1.x += s1.x; v1.y += s1.y; v1.z += s1.z; v1.w += s1.w;
    }
    if (p.epi & DCONV_EPI_RELU) {
      v0.x = fmaxf(v0.x, 0.f); v0.y = fmaxf(v0.y, 0.f);
      v0.z = fmaxf(v0.z, 0.f); v0.w = fmaxf(v0.w, 0.f);
      v1.x = fmaxf(v1.x, 0.f); v1.y = fmaxf(v1.y, 0.f);
      v1.z = fmaxf(v1.z, 0.f); v1.w = fmaxf(v1.w, 0.f);
    }
    float* o = obase + (int64_t)y * p.out_row + (int64_t)x * kCB;
    *reinterpret_cast<float4*>(o) = v0;
    *reinterpret_cast<float4*>(o + 4) = v1;
  }
}

struct TilePick {
  int TH, TW;
  int64_t tiles;
};

TilePick pick_tile(int BM, int h_o, int w_o, int s, int h_f, int w_f) {
  TilePick best{0, 0, -1};
  int64_t best_patch = 0;
  for (int TW = 4; TW <= BM && TW <= 128; TW *= 2) {
    const int TH = BM / TW;
    const int64_t tiles =
        (int64_t)((h_o + TH - 1) / TH) * ((w_o + TW - 1) / TW);
    const int64_t patch =
        (int64_t)((TH - 1) * s + h_f) * ((TW - 1) * s + w_f);
    if (best.tiles < 0 || tiles < best.tiles ||
        (tiles == best.tiles && patch < best_patch)) {
      best = TilePick{TH, TW, tiles};
      best_patch = patch;
    }
  }
  return best;
}

template <int BM, int BN>
int launch(FfmaParams p, cudaStream_t stream) {
  constexpr int CG = BN / 8;
  const TilePick t = pick_tile(BM, p.h_o, p.w_o, p.s, p.h_f, p.w_f);
  p.TH = t.TH;
  p.TW = t.TW;
  p.tiles_x = (p.w_o + p.TW - 1) / p.TW;
  p.tiles_per_img = (int)t.tiles;
  // The patch only has to cover output pixels that exist: clamp the tile
  // extents to the output before sizing it (pixels outside map to offset 0).
  p.TWe = std::min(p.TW, p.w_o);
  p.THe = std::min(p.TH, p.h_o);
  p.PW = (p.TWe - 1) * p.s + p.w_f;
  p.slab_floats = p.h_f * p.w_f * kCB * kCB;

  // Stage decomposition (i'-groups x filter-row groups), sized for smem.
  const int kWeightBudget = 40 * 1024, kPatchBudget = 32 * 1024;
  const int full_taps_bytes = CG * p.h_f * p.w_f * kCB * kCB * 4;
  if (full_taps_bytes <= kWeightBudget) {
    p.R = p.h_f;
    p.PH = (p.THe - 1) * p.s + p.R;
    const int patch1 = p.PH * p.PW * kCB * 4;
    p.G = std::max(1, std::min(kWeightBudget / full_taps_bytes,
                               kPatchBudget / std::max(1, patch1)));
    p.G = std::min(p.G, p.ib_n);
  } else {
    p.G = 1;
    p.R = std::max(1, kWeightBudget / (CG * p.w_f * kCB * kCB * 4));
    p.R = std::min(p.R, p.h_f);
    p.PH = (p.THe - 1) * p.s + p.R;
  }
  p.n_g = (p.ib_n + p.G - 1) / p.G;
  p.n_r = (p.h_f + p.R - 1) / p.R;
  p.patch_floats = p.G * p.PH * p.PW * kCB;
  p.wstride_floats = p.G * p.R * p.w_f * kCB * kCB + 4;  // +16 B: bank spread
  p.stage_floats = p.patch_floats + CG * p.wstride_floats;
  p.stage_floats = (p.stage_floats + 31) & ~31;  // 128-byte aligned stages
  const int stage_bytes = p.stage_floats * 4;
  const int kSmemBudget = 220 * 1024;
  p.NS = std::min(kMaxStages, (kSmemBudget - 2 * kMaxStages * 8) / stage_bytes);
  const int S = p.n_g * p.n_r;
  p.NS = std::min(p.NS, std::max(2, S));
  if (p.NS < 2 || p.PH > 256 || p.PW > 256)
    return dconv_host::set_error(DCONV_EUNSUPPORTED,
                                 "conv_ffma: stage of %d bytes does not fit "
                                 "shared memory twice",
                                 stage_bytes);
  const size_t smem = (size_t)p.NS * stage_bytes + 2 * kMaxStages * 8;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(conv_ffma_kernel<BM, BN>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                         227 * 1024);
    attr_set = true;
  }
  dim3 grid((unsigned)(p.tiles_per_img * p.n), (unsigned)((p.jb_count + CG - 1) / CG));
  conv_ffma_kernel<BM, BN><<<grid, kThreads, smem, stream>>>(p);
  dconv_host::count_launch();
  return dconv_host::check_launch("conv_ffma_kernel");
}

}  // namespace

int launch_conv_ffma(const FfmaParams& p, cudaStream_t stream) {
  if (p.jb_count >= 12) return launch<128, 128>(p, stream);
  return launch<256, 64>(p, stream);
}

}  // namespace dconv_dev
