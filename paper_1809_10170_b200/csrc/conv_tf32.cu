// conv_tf32.cu -- tcgen05/TMEM TF32 variant of the direct convolution
// (north_star: "optional tcgen05/TMEM TF32 implicit-tile variant").
//
// Same algorithm and layout as conv_ffma.cu (Alg. 3, blocked
// c_b = 8), executed on the 5th-generation tensor cores:
//   D[128 px x N ch] (TMEM, fp32) += A[128 px x 8 ch] * B[8 ch x N ch]
// per filter tap (n, m) and input block i' -- one tcgen05.mma.kind::tf32
// with K = 8 = c_ib.
//
// A operand straight from the blocked map: a tensor-map TMA splits each
// 32-byte pencil of the input patch into two 16-byte channel planes
// (channels 0-3 and 4-7).  With 8-pixel-wide tiles, 8 consecutive pixels of
// one plane are one 128-byte UMMA core matrix (K-major, no swizzle), the next
// tile row is SBO = PW*16 bytes away and the second K chunk LBO = one plane
// away -- so every tap (n, m) is just a different descriptor start address
// into the same staged patch (no im2col, no copies).
// B operand: the weights, rearranged once (prepare kernel below) into
// [co-group][i'][n][m][k-half][N][4] so each stage is one contiguous bulk
// copy already in the K-major core-matrix layout.
//
// Roles: warp 0 = TMA producer, warp 1 = MMA issuer (one thread), warps 2-5
// = epilogue (tcgen05.ld of their TMEM lane quarter -> fused skip/ReLU ->
// blocked pencil stores).  A unit = MT <= 4 M-tiles (16*MT rows x 8 cols)
// x N channels, accumulated in up to 512 TMEM columns.
//
// Precision: TF32 inputs (10-bit mantissa), fp32 accumulation; tolerance is
// stated separately (tests/test_gpu_parity.py::test_tf32_*).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include <vector>
#include "tf32_common.cuh"

namespace dconv_dev {

namespace {

using namespace tf32;
constexpr int kEpiWarps = 8;   // 2 per TMEM lane quarter, each half of the columns
constexpr int kThreadsT = (2 + kEpiWarps) * 32;
// Per-role wait clocks (DCONV_TF32_PROFILE=1): compiled in only with
// -DDCONV_TF32_PROF (tools/build_prof.sh), no cost in the product build.
#ifdef DCONV_TF32_PROF
constexpr bool kTf32Prof = true;
#else
constexpr bool kTf32Prof = false;
#endif

// WF_T / MT_T: filter width and M-tiles per unit as compile-time constants
// (0 = runtime), so the per-stage MMA walk unrolls into straight-line issue.
// VAR: the tap walk (kWalkPlain / kWalkS2D / kWalkWide), one per instantiation
// -- the MMA issuer is latency-bound on N = 64 and small-map layers, and a
// runtime choice between walks measured 3-19% slower than a single walk.
template <int WF_T, int MT_T, int VAR>
__global__ void __launch_bounds__(kThreadsT, 1)
    conv_tf32_kernel(const __grid_constant__ CUtensorMap tmap, const Tf32Params p) {
  extern __shared__ __align__(1024) float smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.NS * p.stage_floats);
  uint64_t* empty = full + kMaxStagesT;
  // accumulators: nacc = 2 TMEM sets (MT*N <= 256) so the MMAs of unit u+1
  // overlap the epilogue of unit u, else 1
  uint64_t* acc_full = empty + kMaxStagesT;   // [2]
  uint64_t* acc_empty = acc_full + 2;         // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = p.n_g * p.n_r;
  long long prof[6] = {0, 0, 0, 0, 0, 0};  // DCONV_TF32_PROFILE only
  const long long prof_t0 = kTf32Prof && p.dbg ? clock64() : 0;
  const uint32_t tmem_cols = 512;
  const int nacc = p.MT * p.N <= 256 ? 2 : 1;
  const uint32_t acc_cols = (uint32_t)(p.MT * p.N);

  if (threadIdx.x == 0) {
    for (int i = 0; i < p.NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], kEpiWarps);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();  // programmatic dependent launch: input readable from here on
  pdl_launch_dependents();

  auto decode = [&](int u, int& img, int& y0, int& x0, int& cg) {
    decode_unit(p, u, img, y0, x0, cg);
  };

  if (warp == 0) {
    // ----------------------------------------------------------- producer
    if (lane == 0) {
      // ring slot and phase advance incrementally (no per-stage division)
      int gs = 0, buf = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
        int img, y0, x0, cg;
        decode(u, img, y0, x0, cg);
        int g = 0, r = 0;
        for (int st = 0; st < S; ++st, ++gs) {
          if (st > 0 && ++r == p.n_r) { r = 0; ++g; }
          if (gs > 0 && ++buf == p.NS) { buf = 0; phase ^= 1u; }
          if (gs >= p.NS) {
            const long long t0 = kTf32Prof && p.dbg ? clock64() : 0;
            mbar_wait_backoff(&empty[buf], phase ^ 1u, 64);
            if (kTf32Prof && p.dbg) prof[0] += clock64() - t0;
          }
          const int ib0 = g * p.G, n0 = r * p.R;
          const int Ge = min(p.G, p.ib_n - ib0), Re = min(p.R, p.h_f - n0);
          float* sp = smem + buf * p.stage_floats;
          // the TMA box always lands whole (OOB elements zero-filled)
          const uint32_t patch_bytes = 2u * (uint32_t)(p.G * p.PH * p.PW * 4) * 4u;
          const uint32_t wbytes = (uint32_t)(Ge * Re * p.w_f * 2 * p.N * 4) * 4u;
          if (p.stack > 1) {
            // image-stacked tile: one box per (image slot, input block) at
            // patch row k * SP of that block (see conv_tf32x3.cu)
            const int slots = min(p.stack, p.n - img);
            const uint32_t box = (uint32_t)(p.SP * p.PW * 4) * 4u;
            mbar_arrive_expect_tx(&full[buf], 2u * box * (uint32_t)(slots * Ge) + wbytes);
            // the stage's blocks lie in one space-to-depth phase: coordinates
            // once per stage (a division per copy made the producer the limit)
            int cx, cy, c40;
            tma_block_coords(p, img, ib0, x0, n0, cx, cy, c40);
            for (int k = 0; k < slots; ++k)
              for (int gi = 0; gi < Ge; ++gi) {
                const int c4 = c40 + k * p.ib_o + gi;
                if (p.wide) {  // whole pencils: 8 floats per pixel, one box
                  tma_load_4d(sp + (gi * p.PH + k * p.SP) * p.PW * 8, &tmap, 0, cx, cy, c4,
                              &full[buf]);
                  continue;
                }
                float* dst = sp + (gi * p.PH + k * p.SP) * p.PW * 4;
                tma_load_5d(dst, &tmap, 0, 0, cx, cy, c4, &full[buf]);
                tma_load_5d(dst + p.plane_floats, &tmap, 0, 1, cx, cy, c4, &full[buf]);
              }
          } else {
            mbar_arrive_expect_tx(&full[buf], patch_bytes + wbytes);
            int cx, cy, c4;  // a stage's G blocks lie in one space-to-depth phase
            tma_block_coords(p, img, ib0, x0, y0 + n0, cx, cy, c4);
            if (p.wide) {  // whole pencils, one box (32-byte swizzle)
              tma_load_4d(sp, &tmap, 0, cx, cy, c4, &full[buf]);
            } else {
              tma_load_5d(sp, &tmap, 0, 0, cx, cy, c4, &full[buf]);
              tma_load_5d(sp + p.plane_floats, &tmap, 0, 1, cx, cy, c4, &full[buf]);
            }
          }
          const float* wsrc =
              p.w + (((int64_t)cg * p.ib_n + ib0) * p.h_f + n0) * (int64_t)p.w_f * 2 * p.N * 4;
          bulk_g2s(sp + 2 * p.plane_floats, wsrc, wbytes, &full[buf]);
        }
      }
    }
  } else if (warp == 1) {
    // ----------------------------------------------------------- MMA issuer
    int gs = 0, ui = 0, buf = 0;
    uint32_t phase = 0;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x, ++ui) {
      int img, y0, x0, cg;
      decode(u, img, y0, x0, cg);
      const int valid_rows = p.stack > 1 ? p.MT * kTileRows : min(p.MT * kTileRows, p.h_o - y0);
      const int mts = (valid_rows + kTileRows - 1) / kTileRows;
      const int ab = nacc == 2 ? (ui & 1) : 0, au = nacc == 2 ? (ui >> 1) : ui;
      const uint32_t acc_base = tmem_base + (uint32_t)ab * acc_cols;
      if (au > 0) {
        const long long t0 = kTf32Prof && p.dbg ? clock64() : 0;
        mbar_wait(&acc_empty[ab], (au - 1) & 1);  // epilogue drained this TMEM set
        if (kTf32Prof && p.dbg) prof[2] += clock64() - t0;
      }
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      int g = 0, r = 0;
      for (int st = 0; st < S; ++st, ++gs) {
        if (st > 0 && ++r == p.n_r) { r = 0; ++g; }
        if (gs > 0 && ++buf == p.NS) { buf = 0; phase ^= 1u; }
        {
          const long long t0 = kTf32Prof && p.dbg ? clock64() : 0;
          mbar_wait(&full[buf], phase);
          if (kTf32Prof && p.dbg) prof[1] += clock64() - t0;
        }
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const long long t_issue = kTf32Prof && p.dbg ? clock64() : 0;
        const int Ge = min(p.G, p.ib_n - g * p.G);
        const int Re = min(p.R, p.h_f - r * p.R);
        const float* sp = smem + buf * p.stage_floats;
        const uint32_t a_base = smem_u32(sp);
        const uint32_t b_base = smem_u32(sp + 2 * p.plane_floats);
        // The whole warp walks the taps (every value is warp-uniform, so it
        // stays in the uniform datapath); one elected lane issues each MMA.
        // A descriptor's low word (start >> 4 | LBO >> 4 << 16) advances by
        // the byte offset >> 4 (smem < 256 KB: no carry), the high word
        // (SBO, version) is fixed -- a 32-bit add per MMA.
        const ADesc ad = a_desc(p, a_base);
        const uint32_t a_lo0 = ad.lo0, a_hi = ad.hi, au = ad.unit;
        const uint32_t b_lo0 = ((b_base >> 4) & 0x3FFFu) | (((uint32_t)(p.N * 16) >> 4) << 16);
        const uint32_t b_hi = (128u >> 4) | (1u << 14);
        const uint32_t a_mt = (uint32_t)(kTileRows * p.PW) * au;  // next M-tile (16 B units)
        const uint32_t b_tap = (uint32_t)(2 * p.N);          // next (n, m) tap
        uint32_t accum = st == 0 ? 0u : 1u;
        const int wf = WF_T > 0 ? WF_T : p.w_f;
        // space-to-depth: skip the taps of this stage's phase that multiply
        // structurally zero weights (the first MMA of a unit is always issued
        // so the accumulator is initialised)
        int nmax, mmax;
        s2d_valid_taps(p, g * p.G, nmax, mmax);
        // the tap walk, specialised: without space-to-depth no tap is
        // skipped and the issuer loop carries no per-tap test (the test
        // cost 15-19% on N = 64 / 14x14 layers: the issuer is latency-bound)
        auto walk = [&](auto s2d_tag, auto wide_tag) {
          constexpr bool S2D = decltype(s2d_tag)::value;
          constexpr uint32_t AU = decltype(wide_tag)::value ? 2u : 1u;  // A start unit
          for (int gi = 0; gi < Ge; ++gi)
            for (int n = 0; n < Re; ++n) {
              const bool row_ok = !S2D || r * p.R + n < nmax;
              const uint32_t arow = a_lo0 + (uint32_t)((gi * p.PH + n) * p.PW) * AU;
              const uint32_t brow = b_lo0 + (uint32_t)((gi * p.R + n) * wf) * b_tap;
              if (MT_T > 0 && mts == MT_T) {
#pragma unroll
                for (int m = 0; m < (WF_T > 0 ? WF_T : 1); ++m) {
                  if (S2D && accum && !(row_ok && m < mmax)) continue;
#pragma unroll
                  for (int mt = 0; mt < MT_T; ++mt)
                    umma_tf32_elect(acc_base + (uint32_t)(mt * p.N),
                                    arow + (uint32_t)m * AU + (uint32_t)mt * a_mt, a_hi,
                                    brow + (uint32_t)m * b_tap, b_hi, p.idesc, accum);
                  accum = 1u;
                }
                if (WF_T > 0) continue;
                for (int m = 1; m < wf; ++m) {
                  if (S2D && accum && !(row_ok && m < mmax)) continue;
#pragma unroll
                  for (int mt = 0; mt < MT_T; ++mt)
                    umma_tf32_elect(acc_base + (uint32_t)(mt * p.N),
                                    arow + (uint32_t)m * AU + (uint32_t)mt * a_mt, a_hi,
                                    brow + (uint32_t)m * b_tap, b_hi, p.idesc, S2D ? accum : 1u);
                  accum = 1u;
                }
                continue;
              }
              for (int m = 0; m < wf; ++m) {
                if (S2D && accum && !(row_ok && m < mmax)) continue;
                const uint32_t blo = brow + (uint32_t)m * b_tap;
                uint32_t alo = arow + (uint32_t)m * AU;
                for (int mt = 0; mt < mts; ++mt, alo += a_mt)
                  umma_tf32_elect(acc_base + (uint32_t)(mt * p.N), alo, a_hi, blo, b_hi, p.idesc,
                                  accum);
                accum = 1u;
              }
            }
        };
        if constexpr (VAR == kWalkS2D) {
          walk(std::true_type{}, std::false_type{});
        } else if constexpr (VAR == kWalkWide) {
          walk(std::false_type{}, std::true_type{});
        } else {
          walk(std::false_type{}, std::false_type{});
        }
        if (kTf32Prof && p.dbg) prof[4] += clock64() - t_issue;
        umma_commit_elect(&empty[buf]);  // stage smem free once these MMAs retire
        if (st == S - 1) umma_commit_elect(&acc_full[ab]);
        __syncwarp();
        if (kTf32Prof && p.dbg) prof[5] += clock64() - t_issue;
      }
    }
  } else {
    // ----------------------------------------------------------- epilogue
    const int q = warp & 3;  // TMEM lane quarter of this warp
    const int ch = (warp - 2) / 4;  // which half of the N columns
    const int r = q * 32 + lane;  // pixel row of the M-tile
    const int ty = r / kTW, tx = r % kTW;
    int ui = 0;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x, ++ui) {
      int img, y0, x0, cg;
      decode(u, img, y0, x0, cg);
      const int ab = nacc == 2 ? (ui & 1) : 0, au = nacc == 2 ? (ui >> 1) : ui;
      const uint32_t acc_base = tmem_base + (uint32_t)ab * acc_cols;
      mbar_wait_backoff(&acc_full[ab], au & 1, 256);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int x = x0 + tx;
      for (int mt = 0; mt < p.MT; ++mt) {
        if (p.stack == 1 && y0 + mt * kTileRows >= p.h_o) break;  // warp-uniform
        int im, y;
        bool ok;
        tile_row_pixel(p, img, y0, mt * kTileRows + ty, im, y, ok);
        const bool valid = ok && x < p.w_o;
        const int half_n = p.N / 2;  // >= 32
        for (int c0 = ch * half_n; c0 < (ch + 1) * half_n; c0 += 32) {
          float v[32];
          tmem_ld32x32(acc_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(mt * p.N + c0), v);
          emit32(p, v, im, y, x, valid, tx, ty, cg, c0);
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[ab]);
    }
  }

  if (kTf32Prof && p.dbg) {  // per-role cycle sums, kept in registers during the loop
    if (threadIdx.x == 0) p.dbg[blockIdx.x * 8 + 0] = prof[0];
    if (threadIdx.x == 32)
      for (int i = 1; i < 6; ++i) p.dbg[blockIdx.x * 8 + i] = prof[i];
    if (threadIdx.x == 32) p.dbg[blockIdx.x * 8 + 6] = clock64() - prof_t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(tmem_cols));
  }
}

// Prepared weights: [cg][i'][n][m][k-half][N][4] from the blocked kernel
// [jb][i'][n][m][ii][jj] (tensor.hpp:131-137); channel slots beyond jb_count
// blocks are zero.  Bit-exact permutation.
__global__ void prepare_tf32_weights_kernel(const float* __restrict__ w, int ib_n, int h_f,
                                            int w_f, int jb_begin, int jb_count, int N,
                                            const WSrc src, int64_t total, float* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t t = e;
    const int k4 = (int)(t % 4); t /= 4;
    const int co = (int)(t % N); t /= N;
    const int kh = (int)(t % 2); t /= 2;
    const int m = (int)(t % w_f); t /= w_f;
    const int n = (int)(t % h_f); t /= h_f;
    const int ib = (int)(t % ib_n); t /= ib_n;
    const int cg = (int)t;
    const int jl = cg * (N / 8) + co / 8;  // block within the computed range
    float v = 0.f;
    if (jl < jb_count) {
      const int jb = jb_begin + jl, jj = co % 8, ii = kh * 4 + k4;
      v = weight_src(w, jb, ib, n, m, ii, jj, src);
    }
    out[e] = v;
  }
}

}  // namespace

using Tf32Kernel = void (*)(const CUtensorMap, const Tf32Params);
// instantiated walks: 3x3 plain / space-to-depth (11x11/s4 -> 3x3), 1x1 plain /
// wide (a strided 1x1 is a subsampled view, never space-to-depth), generic
// plain / space-to-depth (3x3/s2 -> 2x2, 7x7/s2 -> 4x4)
template <int V>
Tf32Kernel tf32_kernel_for(int wf, int mt) {
  static const Tf32Kernel k3[4] = {conv_tf32_kernel<3, 1, V>, conv_tf32_kernel<3, 2, V>,
                                   conv_tf32_kernel<3, 3, V>, conv_tf32_kernel<3, 4, V>};
  if (wf == 3) return k3[mt - 1];
  return conv_tf32_kernel<0, 0, V>;
}
Tf32Kernel pick_tf32_kernel(const Tf32Params& p) {
  static const Tf32Kernel k1[2][4] = {
      {conv_tf32_kernel<1, 1, kWalkPlain>, conv_tf32_kernel<1, 2, kWalkPlain>,
       conv_tf32_kernel<1, 3, kWalkPlain>, conv_tf32_kernel<1, 4, kWalkPlain>},
      {conv_tf32_kernel<1, 1, kWalkWide>, conv_tf32_kernel<1, 2, kWalkWide>,
       conv_tf32_kernel<1, 3, kWalkWide>, conv_tf32_kernel<1, 4, kWalkWide>}};
  if (p.w_f == 1) return k1[p.wide ? 1 : 0][p.MT - 1];
  return p.s2d > 1 ? tf32_kernel_for<kWalkS2D>(p.w_f, p.MT)
                   : tf32_kernel_for<kWalkPlain>(p.w_f, p.MT);
}

// Channels per unit: an M=128 MMA costs ~71 cycles for any N <= 128 and ~128
// cycles at N = 256 (tools/umma_tf32_rate.cu), so wide layers use N = 256.
int tf32_channels(int jb_count) {
  static const int force = getenv("DCONV_TF32_N") ? atoi(getenv("DCONV_TF32_N")) : 0;
  if (force == 64 || force == 128 || force == 256) return force;
  return jb_count * 8 >= 256 ? 256 : (jb_count * 8 > 64 ? 128 : 64);
}

int64_t tf32_prepared_floats(int ib_n, int h_f, int w_f, int jb_count) {
  const int N = tf32_channels(jb_count);
  const int n_cg = (jb_count * 8 + N - 1) / N;
  return (int64_t)n_cg * ib_n * h_f * w_f * 2 * N * 4;
}

int launch_prepare_tf32(const float* w, int ib_n, int h_f, int w_f, int jb_begin, int jb_count,
                        const WSrc& src, float* out, cudaStream_t stream) {
  const int N = tf32_channels(jb_count);
  const int64_t total = tf32_prepared_floats(ib_n, h_f, w_f, jb_count);
  int64_t blocks = std::min<int64_t>((total + 255) / 256, 148 * 32);
  prepare_tf32_weights_kernel<<<(unsigned)blocks, 256, 0, stream>>>(w, ib_n, h_f, w_f, jb_begin,
                                                                    jb_count, N, src, total, out);
  dconv_host::count_launch();
  return dconv_host::check_launch("prepare_tf32_weights_kernel");
}

int launch_conv_tf32(const FfmaParams& f0, const float* w_prepared, cudaStream_t stream) {
  FfmaParams f = f0;  // (f0: the original filter, before the space-to-depth view)
  InView view;
  if (int rc = prepare_view(f, view, "conv_tf32")) return rc;
  Tf32Params p{};
  p.w = w_prepared;
  copy_geometry(p, f);
  p.s2d = view.s2d;
  p.ib_o = view.ib;
  p.hf_o = f0.h_f;
  p.wf_o = f0.w_f;
  p.N = tf32_channels(f.jb_count);
  p.n_cg = (f.jb_count * 8 + p.N - 1) / p.N;
  // stage = G input blocks x R filter rows, <= 48 KB of weights
  const int wtap = 2 * p.N * 4 * 4;  // bytes per (i', n, m)
  // M-tiles per unit: more tiles share each weight stage (less L2/smem
  // traffic per MAC); fewer give more units.  Score = useful rows x SM-wave
  // balance (a ragged last wave costs a full round) / load-bound cost; ties
  // go to the larger MT.
  {
    const int sms = tf32::sm_count();
    const int strips = (p.w_o + kTW - 1) / kTW;
    // time = rounds x per-unit cycles; a unit streams ib_n input blocks, each
    // max(MMA time, load time): 9*MT MMAs of ~78 cycles (N <= 128) against its
    // patch + weight bytes at ~40 B/cycle/SM when every SM loads (L2 bound),
    // plus ~3000 cycles of fill and epilogue per unit.
    double best = -1;
    for (int mt = kMaxMT; mt >= 1; --mt) {
      if (mt * p.N > 512) continue;  // accumulators: MT x N TMEM columns
      // TMA box rows of a strided (space-to-depth) read: (PH) x s <= 256
      if (mt > 1 && (mt * kTileRows - 1 + p.h_f) * p.s2d > 256) continue;
      // small maps stack images along the tile rows (below)
      const int sp = p.h_o + p.h_f - 1;
      const int st = !(p.epi & DCONV_EPI_MAXPOOL) && p.h_o + sp <= mt * kTileRows
                         ? std::min(p.n, (mt * kTileRows - p.h_o) / sp + 1)
                         : 1;
      const int rg = st > 1 ? 1 : (p.h_o + mt * kTileRows - 1) / (mt * kTileRows);
      const int64_t units = (int64_t)((p.n + st - 1) / st) * rg * strips * p.n_cg;
      const double taps = (double)p.h_f * p.w_f;
      const double mma = taps * mt * (p.N > 128 ? 128.0 : 78.0);
      const double bytes = (double)(mt * kTileRows - 1 + p.h_f) * (kTW - 1 + p.w_f) * 32.0 +
                           taps * p.N * 32.0;
      // double-buffered accumulators (MT*N <= 256) hide most of the epilogue
      const double unit = p.ib_n * std::max(mma, bytes / 40.0) + (mt * p.N <= 256 ? 800.0 : 3000.0);
      const double rounds = (double)((units + sms - 1) / sms);
      const double score = 1.0 / (rounds * unit);
      if (score > best * (1 + 1e-9)) {
        best = score;
        p.MT = mt;
      }
    }
    static const char* force_mt = getenv("DCONV_TF32_MT");
    if (const char* e = force_mt)
      p.MT = std::max(1, std::min(std::min(kMaxMT, 512 / p.N), atoi(e)));
  }
  // filter rows per stage, then image stacking for small maps (h_o = 7:
  // slot k of a unit holds image img + k at tile row k * SP; not with the
  // fused pool), then the input blocks per stage
  p.R = p.h_f * p.w_f * wtap <= 48 * 1024
            ? p.h_f
            : std::max(1, std::min(p.h_f, (48 * 1024) / (p.w_f * wtap)));
  p.SP = p.h_o + p.R - 1;
  p.stack = 1;
  static const bool no_stack = getenv("DCONV_NO_STACK") != nullptr;
  if (!no_stack && !(p.epi & DCONV_EPI_MAXPOOL) && p.h_o + p.SP <= p.MT * kTileRows) {
    int pw = p.PW;
    while ((p.SP * pw) % 8) ++pw;  // 128-B aligned slot boxes
    if (pw <= 16) {
      p.PW = pw;
      p.stack = std::min(p.n, (p.MT * kTileRows - p.h_o) / p.SP + 1);
    }
  }
  p.PH = std::max(p.MT * kTileRows - 1 + p.R, p.stack > 1 ? p.stack * p.SP : 0);
  if (p.stack > 1)
    while ((p.PH * p.PW) % 8) ++p.PH;
  const int patch_blk_bytes = 2 * p.PH * p.PW * 16;  // both planes
  // space-to-depth layers: a 72 KB weight budget (two input blocks of a 2x2
  // phase filter at N = 256): their stages carry few valid taps, and the
  // per-stage hand-offs, not the loads, bound them
  static const int s2d_wkb = getenv("DCONV_S2D_WKB") ? atoi(getenv("DCONV_S2D_WKB")) : 72;
  const int wbudget = (p.s2d > 1 ? s2d_wkb : 48) * 1024;
  p.G = p.R == p.h_f ? std::max(1, std::min({p.ib_n, wbudget / (p.h_f * p.w_f * wtap),
                                             (40 * 1024) / patch_blk_bytes}))
                     : 1;
  // 1x1 layers with >= 256 input channels: at least 4 ring stages (as the
  // split-TF32 kernel: with 2 the TMA -> MMA hand-off is exposed)
  {
    static const bool shallow = getenv("DCONV_X3_SHALLOW") != nullptr;  // A/B only
    const int bar = (2 * kMaxStagesT + 4) * 8 + 16;
    auto stage_of = [&](int g) {
      const int plane = (g * p.PH * p.PW * 4 + 31) & ~31;
      return ((2 * plane + g * p.R * p.w_f * 2 * p.N * 4) + 255) & ~255;
    };
    if (p.h_f * p.w_f == 1 && p.ib_n >= 32 && !shallow)
      while (p.G > 1 && 4 * stage_of(p.G) * 4 > 220 * 1024 - bar) --p.G;
  }
  // space-to-depth: a stage's blocks must lie in one phase
  if (p.s2d > 1)
    while (p.ib_o % p.G) --p.G;
  p.n_g = (p.ib_n + p.G - 1) / p.G;
  p.n_r = (p.h_f + p.R - 1) / p.R;
  if (p.PH > 256 || p.PW > 256 || p.G > 256)
    return dconv_host::set_error(DCONV_EUNSUPPORTED, "conv_tf32: TMA box too large");
  p.plane_floats = (p.G * p.PH * p.PW * 4 + 31) & ~31;  // TMA destinations 128 B aligned
  p.wstage_floats = p.G * p.R * p.w_f * 2 * p.N * 4;
  p.stage_floats = ((2 * p.plane_floats + p.wstage_floats) + 255) & ~255;  // 1 KB aligned
  const int stage_bytes = p.stage_floats * 4;
  const int bar_bytes = (2 * kMaxStagesT + 4) * 8 + 16;
  p.NS = std::min(kMaxStagesT, (220 * 1024 - bar_bytes) / stage_bytes);
  if (p.NS < 2)
    return dconv_host::set_error(DCONV_EUNSUPPORTED, "conv_tf32: stage of %d bytes", stage_bytes);
  p.row_groups = p.stack > 1 ? 1 : (p.h_o + p.MT * kTileRows - 1) / (p.MT * kTileRows);
  p.strips = (p.w_o + kTW - 1) / kTW;
  p.units = (p.n + p.stack - 1) / p.stack * p.row_groups * p.strips * p.n_cg;
  // instruction descriptor: D f32, A/B tf32, K-major both, N, M = 128
  p.idesc = tf32_idesc(p.N);

  // tensor map over the input view: {c4, half, W, H, image*block}
  CUtensorMap map;
  // 1x1 layers: whole pencils per TMA box (DCONV_TF32_NO_WIDE=1: half planes)
  static const bool no_wide = getenv("DCONV_TF32_NO_WIDE") != nullptr;
  // (stacked tiles: one box of SP rows per image slot; slot rows start on
  // 8-pixel = 256-byte swizzle atoms since PW = 8)
  p.wide = (!no_wide && p.h_f == 1 && p.w_f == 1 && p.PW == kTW && p.s2d == 1 &&
            (p.PH % 4) == 0) ? 1 : 0;
  if (int rc = p.wide ? encode_input_map_wide(&map, view, p.PW, p.stack > 1 ? p.SP : p.PH,
                                              p.stack > 1 ? 1 : p.G)
               : p.stack > 1 ? encode_input_map(&map, view, p.PW, p.SP, 1)
                             : encode_input_map(&map, view, p.PW, p.PH, p.G))
    return rc;

  const int dev = dconv_host::current_device();
  const int sms = dconv_host::device_sms(dev);
  {
    const Tf32Kernel k = pick_tf32_kernel(p);
    if (dconv_host::first_use_on_device(reinterpret_cast<const void*>(k), dev))
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  }
  const size_t smem = (size_t)p.NS * stage_bytes + bar_bytes;
  const int grid = std::min(p.units, sms);
  static const bool dbg = getenv("DCONV_DEBUG") != nullptr;
  if (dbg)
    fprintf(stderr, "conv_tf32 N=%d MT=%d G=%d R=%d NS=%d stage=%d B stack=%d s2d=%d units=%d\n",
            p.N, p.MT, p.G, p.R, p.NS, stage_bytes, p.stack, p.s2d, p.units);
  static const bool prof = kTf32Prof && getenv("DCONV_TF32_PROFILE") != nullptr;  // profiling builds only
  if (prof) {  // debugging aid: where do the roles wait?  (not for timed runs)
    cudaMalloc(&p.dbg, (size_t)grid * 8 * 8);
    cudaMemsetAsync(p.dbg, 0, (size_t)grid * 8 * 8, stream);
    long long start = 0;
    pick_tf32_kernel(p)<<<grid, kThreadsT, smem, stream>>>(map, p);
    std::vector<unsigned long long> h((size_t)grid * 8);
    cudaMemcpy(h.data(), p.dbg, h.size() * 8, cudaMemcpyDeviceToHost);
    double w_empty = 0, w_full = 0, w_acc = 0, issue = 0, issue_commit = 0, total = 0;
    for (int b = 0; b < grid; ++b) {
      w_empty += h[b * 8]; w_full += h[b * 8 + 1]; w_acc += h[b * 8 + 2];
      issue += h[b * 8 + 4]; issue_commit += h[b * 8 + 5]; total += h[b * 8 + 6];
    }
    (void)start;
    fprintf(stderr,
            "conv_tf32 N=%d MT=%d G=%d R=%d NS=%d stage=%d B units=%d S=%d: per CTA avg wait "
            "cycles producer(empty)=%.0f mma(full)=%.0f mma(acc_empty)=%.0f issue=%.0f "
            "issue+commit=%.0f total=%.0f\n",
            p.N, p.MT, p.G, p.R, p.NS, stage_bytes, p.units, p.n_g * p.n_r, w_empty / grid,
            w_full / grid, w_acc / grid, issue / grid, issue_commit / grid, total / grid);
    cudaFree(p.dbg);
    p.dbg = nullptr;
  }
  {
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreadsT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cfg.attrs = attr;
    cfg.numAttrs = dconv_host::pdl_enabled() ? 1 : 0;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, pick_tf32_kernel(p), map, p);
    if (e != cudaSuccess)
      return dconv_host::set_error(DCONV_ECUDA, "conv_tf32: %s", cudaGetErrorString(e));
  }
  dconv_host::count_launch();
  return dconv_host::check_launch("conv_tf32_kernel");
}

}  // namespace dconv_dev
