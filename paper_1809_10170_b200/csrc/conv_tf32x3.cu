// conv_tf32x3.cu -- split-TF32 ("3xTF32") tcgen05 direct convolution that
// meets the fp32 tolerance of the FFMA path (|a-b| <= 1e-4 + 1e-5|b| against
// conv_oracle64, reference.cpp:70-87).
//
// Same algorithm, layout and tiling as conv_tf32.cu (Alg. 3, PAPER.md:326-363,
// blocked c_b = 8; one tcgen05.mma.kind::tf32 per filter tap and input block),
// with every operand split into a TF32 head and an fp32 remainder:
//   x = x_hi + x_lo, x_hi = x with the low 13 mantissa bits cleared,
//   conv(x, w) ~= T(x_hi, w_hi) + T(x_hi, w_lo) + T(x_lo, w_hi)
// (the dropped x_lo*w_lo term is ~2^-22 of a product).
//   * Weights: hi and lo are prepared once (bit-exact split of the blocked
//     kernel, like pack_kernel tensor.cpp:85-95) and streamed by bulk copy.
//   * Activations: TMA stages the raw fp32 patch (x_hi: the tensor core
//     reads only an operand's TF32 bits); two "split" warps write the
//     remainders x - trunc(x) into a second pair of planes of the same
//     stage -- on chip, so no workspace is added.
//   * Accumulation: the tensor core adds into its fp32 accumulator with an
//     error that grows with the accumulator's magnitude (K = 4608 in one
//     accumulator fails the fp32 bar: profiles/r1_tf32x3_accuracy.txt).  The
//     reduction is therefore cut into chunks of ~144 products (288 with the
//     separate correction accumulator of 64-channel layers): the MMAs of a
//     chunk go to one of two TMEM accumulator sets while the epilogue warps
//     add the previous chunk into fp32 register totals (IEEE adds), the same
//     two-level summation the FFMA kernel does with its TMEM fold
//     (profiles/r1_tf32x3_kernel_accuracy.txt: chunk K vs accuracy).
//
// Roles (12 warps): warp 0 TMA producer, warp 1 MMA issuer (elect.sync),
// warps 2-3 operand split, warps 4-11 epilogue (chunk drain into registers,
// then fused skip/ReLU/pool and blocked pencil stores).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "tf32_common.cuh"

namespace dconv_dev {

int tf32_channels(int jb_count);  // conv_tf32.cu

namespace {

using namespace tf32;
constexpr int kSplitWarps = 2;
constexpr int kEpiWarpsX = 8;
constexpr int kThreadsX = (4 + kEpiWarpsX) * 32;
constexpr uint32_t kHiMask = 0xFFFFE000u;  // TF32: sign, exponent, 10 mantissa bits
// Role wait-cycle instrumentation (DCONV_TF32_PROFILE), compiled in only when
// built with -DDCONV_X3_PROF (tools/build_prof.sh): it costs registers in
// the 56-register producer/MMA/split group.
#ifdef DCONV_X3_PROF
constexpr bool kProf = true;
#else
constexpr bool kProf = false;
#endif

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, "
      "%8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
        "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]),
        "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ float4 hi4(float4 v) {
  return make_float4(__uint_as_float(__float_as_uint(v.x) & kHiMask),
                     __uint_as_float(__float_as_uint(v.y) & kHiMask),
                     __uint_as_float(__float_as_uint(v.z) & kHiMask),
                     __uint_as_float(__float_as_uint(v.w) & kHiMask));
}

// COLS = MT * N / 2: accumulator columns each epilogue thread totals in
// registers (two epilogue warps per TMEM lane quarter, each half of N).
// DA ("dual accumulator", used for N = 64): per tap and M-tile one N' = 2N MMA
// A_hi x [B_hi | B_lo] writes the head product and the first correction into
// adjacent column blocks [main | corr], and A_lo x B_hi accumulates into corr:
// two MMAs instead of three, A_hi read once, and the small terms are summed
// apart from the head (no bits lost in its accumulator).  Weights per k-half
// are [hi N rows | lo N rows]; TMEM per M-tile 2N columns.
template <int WF_T, int MT_T, int COLS, bool DA, int VAR>  // VAR: tap walk (conv_tf32.cu)
__global__ void __launch_bounds__(kThreadsX, 1)
    conv_tf32x3_kernel(const __grid_constant__ CUtensorMap tmap, const Tf32Params p) {
  extern __shared__ __align__(1024) float smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.NS * p.stage_floats);
  uint64_t* split = full + kMaxStagesT;       // stage split into hi / lo planes
  uint64_t* empty = split + kMaxStagesT;
  uint64_t* chunk_full = empty + kMaxStagesT;  // [2] chunk accumulator sets
  uint64_t* chunk_empty = chunk_full + 2;      // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(chunk_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = p.n_g * p.n_r;
  const int n_chunks = (S + p.chunk_st - 1) / p.chunk_st;
  constexpr uint32_t kSetCols = 256;  // chunk set c & 1 at column (c & 1) * 256
  const uint32_t tmem_cols = 512;

  if (threadIdx.x == 0) {
    for (int i = 0; i < p.NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&split[i], kSplitWarps);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&chunk_full[i], 1);
      mbar_init(&chunk_empty[i], kEpiWarpsX);
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
  // DCONV_TF32_PROFILE: per-role wait cycles (lane 0 of warps 0, 1, 2)
  long long prof = 0, prof2 = 0;
  const long long prof_t0 = kProf && p.dbg ? clock64() : 0;
  pdl_wait();  // programmatic dependent launch: input readable from here on
  pdl_launch_dependents();

  // register split per warpgroup (one setmaxnreg per warpgroup, dominating
  // its roles' code): WG0 = producer, MMA issuer, split warps; WG1-2 = epilogue
  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
  if (warp == 0) {
    // ----------------------------------------------------------- producer
    if (lane == 0) {
      int gs = 0, buf = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
        int img, y0, x0, cg;
        decode_unit(p, u, img, y0, x0, cg);
        int g = 0, r = 0;
        for (int st = 0; st < S; ++st, ++gs) {
          if (st > 0 && ++r == p.n_r) { r = 0; ++g; }
          if (gs > 0 && ++buf == p.NS) { buf = 0; phase ^= 1u; }
          if (gs >= p.NS) {
            const long long t0 = kProf && p.dbg ? clock64() : 0;
            mbar_wait_backoff(&empty[buf], phase ^ 1u, 64);
            if (kProf && p.dbg) prof += clock64() - t0;
          }
          const int ib0 = g * p.G, n0 = r * p.R;
          const int Ge = min(p.G, p.ib_n - ib0), Re = min(p.R, p.h_f - n0);
          float* sp = smem + buf * p.stage_floats;
          // the TMA box always lands whole (OOB elements zero-filled)
          const uint32_t patch_bytes = 2u * (uint32_t)(p.G * p.PH * p.PW * 4) * 4u;
          const uint32_t wbytes = (uint32_t)(Ge * Re * p.w_f * 4 * p.N * 4) * 4u;
          if (p.stack > 1) {
            // one box per (image slot, input block): slot k of block g lands
            // at patch row k * SP of that block's rows
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
              p.w + (((int64_t)cg * p.ib_n + ib0) * p.h_f + n0) * (int64_t)p.w_f * 4 * p.N * 4;
          bulk_g2s(sp + 4 * p.plane_floats, wsrc, wbytes, &full[buf]);
        }
      }
    }
  } else if (warp == 1) {
    // ----------------------------------------------------------- MMA issuer
    int gs = 0, buf = 0, cs = 0;
    uint32_t phase = 0;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
      int img, y0, x0, cg;
      decode_unit(p, u, img, y0, x0, cg);
      const int valid_rows = p.stack > 1 ? p.MT * kTileRows : min(p.MT * kTileRows, p.h_o - y0);
      const int mts = (valid_rows + kTileRows - 1) / kTileRows;
      int g = 0, r = 0, ci = 0;
      uint32_t acc_base = 0, accum = 0;
      for (int st = 0; st < S; ++st, ++gs) {
        if (st > 0 && ++r == p.n_r) { r = 0; ++g; }
        if (gs > 0 && ++buf == p.NS) { buf = 0; phase ^= 1u; }
        if (ci == 0) {
          // new chunk: its accumulator set must have been drained
          const int set = cs & 1;
          if (cs >= 2) {
            const long long t0 = kProf && p.dbg ? clock64() : 0;
            mbar_wait(&chunk_empty[set], ((cs >> 1) - 1) & 1);
            if (kProf && p.dbg) prof2 += clock64() - t0;
          }
          acc_base = tmem_base + (uint32_t)set * kSetCols;
          accum = 0u;
        }
        {
          const long long t0 = kProf && p.dbg ? clock64() : 0;
          mbar_wait(&split[buf], phase);
          if (kProf && p.dbg) prof += clock64() - t0;
        }
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const int Ge = min(p.G, p.ib_n - g * p.G);
        const int Re = min(p.R, p.h_f - r * p.R);
        const float* sp = smem + buf * p.stage_floats;
        const uint32_t a_base = smem_u32(sp);
        const uint32_t b_base = smem_u32(sp + 4 * p.plane_floats);
        // descriptor low words (start >> 4 | LBO >> 4 << 16) advance by 32-bit
        // adds (see conv_tf32.cu); lo planes / lo weights at fixed offsets
        const ADesc ad = a_desc(p, a_base);
        const uint32_t a_lo0 = ad.lo0, a_hi = ad.hi, au = ad.unit;
        const uint32_t b_lo0 =
            ((b_base >> 4) & 0x3FFFu) | (((uint32_t)((DA ? 2 : 1) * p.N * 16) >> 4) << 16);
        const uint32_t b_hi = (128u >> 4) | (1u << 14);
        const uint32_t a_mt = (uint32_t)(kTileRows * p.PW) * au;  // next M-tile (16 B units)
        const uint32_t b_tap = (uint32_t)(4 * p.N);          // next (n, m) tap: hi + lo
        const uint32_t a_rem = (uint32_t)(p.plane_floats / 2);  // lo planes (16 B units)
        const uint32_t b_rem = (uint32_t)(2 * p.N);             // lo weights of a tap
        const int wf = WF_T > 0 ? WF_T : p.w_f;
        constexpr int kMtLoop = MT_T > 0 ? MT_T : kMaxMT;
        // space-to-depth: skip the taps of this stage's phase that multiply
        // structurally zero weights (the first MMA of a chunk is always
        // issued, initialising its accumulator set)
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
#pragma unroll
              for (int m = 0; m < (WF_T > 0 ? WF_T : 1); ++m) {
                if (S2D && accum && !(row_ok && m < mmax)) continue;
#pragma unroll
                for (int mt = 0; mt < kMtLoop; ++mt) {
                  if (mt >= mts) break;
                  const uint32_t a = arow + (uint32_t)m + (uint32_t)mt * a_mt;
                  const uint32_t b = brow + (uint32_t)m * b_tap;
                  if constexpr (DA) {
                    const uint32_t d = acc_base + (uint32_t)(mt * 2 * p.N);
                    umma_tf32_elect(d, a, a_hi, b, b_hi, p.idesc2, accum);  // [main | corr]
                    umma_tf32_elect(d + (uint32_t)p.N, a + a_rem, a_hi, b, b_hi, p.idesc, 1u);
                  } else {
                    const uint32_t d = acc_base + (uint32_t)(mt * p.N);
                    // small terms first, the head product last
                    umma_tf32_elect(d, a, a_hi, b + b_rem, b_hi, p.idesc, accum);
                    umma_tf32_elect(d, a + a_rem, a_hi, b, b_hi, p.idesc, 1u);
                    umma_tf32_elect(d, a, a_hi, b, b_hi, p.idesc, 1u);
                  }
                }
                accum = 1u;
              }
              if (WF_T > 0) continue;
              for (int m = 1; m < wf; ++m) {
                if (S2D && accum && !(row_ok && m < mmax)) continue;
                for (int mt = 0; mt < mts; ++mt) {
                  const uint32_t a = arow + (uint32_t)m + (uint32_t)mt * a_mt;
                  const uint32_t b = brow + (uint32_t)m * b_tap;
                  if constexpr (DA) {
                    const uint32_t d = acc_base + (uint32_t)(mt * 2 * p.N);
                    umma_tf32_elect(d, a, a_hi, b, b_hi, p.idesc2, S2D ? accum : 1u);
                    umma_tf32_elect(d + (uint32_t)p.N, a + a_rem, a_hi, b, b_hi, p.idesc, 1u);
                  } else {
                    const uint32_t d = acc_base + (uint32_t)(mt * p.N);
                    umma_tf32_elect(d, a, a_hi, b + b_rem, b_hi, p.idesc, S2D ? accum : 1u);
                    umma_tf32_elect(d, a + a_rem, a_hi, b, b_hi, p.idesc, 1u);
                    umma_tf32_elect(d, a, a_hi, b, b_hi, p.idesc, 1u);
                  }
                }
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
        umma_commit_elect(&empty[buf]);  // stage smem free once these MMAs retire
        if (++ci == p.chunk_st || st == S - 1) {
          umma_commit_elect(&chunk_full[cs & 1]);
          ci = 0;
          ++cs;
        }
        __syncwarp();
      }
    }
  } else {
    // ----------------------------------------------------------- operand split
    // x_lo = x - x_hi into the second plane pair.  x_hi is the raw patch:
    // kind::tf32 reads only the top 19 bits of an fp32 operand (truncation;
    // a rounding tensor core would make x_hi + x_lo != x and fail the fp32
    // tolerance tests by orders of magnitude, tests/test_gpu_parity.py).
    const int t = threadIdx.x - 64;
    int gs = 0, buf = 0;
    uint32_t phase = 0;
    const int n4 = p.plane_floats / 2;  // float4s in the two hi planes
    for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
      for (int st = 0; st < S; ++st, ++gs) {
        if (gs > 0 && ++buf == p.NS) { buf = 0; phase ^= 1u; }
        const long long t0 = kProf && p.dbg ? clock64() : 0;
        mbar_wait(&full[buf], phase);
        if (kProf && p.dbg) prof += clock64() - t0;
        const float4* hi = reinterpret_cast<const float4*>(smem + buf * p.stage_floats);
        float4* lo = reinterpret_cast<float4*>(smem + buf * p.stage_floats) + n4;
        // batches of 8 loads in flight before any store (the stores could
        // alias later loads for the compiler, which would serialise them)
        constexpr int kStep = kSplitWarps * 32;
        for (int i0 = t; i0 < n4; i0 += 8 * kStep) {
          float4 v[8];
#pragma unroll
          for (int k = 0; k < 8; ++k)
            if (i0 + k * kStep < n4) v[k] = hi[i0 + k * kStep];
#pragma unroll
          for (int k = 0; k < 8; ++k)
            if (i0 + k * kStep < n4) {
              const float4 h = hi4(v[k]);
              lo[i0 + k * kStep] = make_float4(v[k].x - h.x, v[k].y - h.y, v[k].z - h.z,
                                               v[k].w - h.w);
            }
        }
        fence_proxy_async_smem();  // generic-proxy writes -> tcgen05.mma operands
        __syncwarp();
        if (lane == 0) mbar_arrive(&split[buf]);
      }
    }
  }
  } else {
    // ----------------------------------------------------------- epilogue
    asm volatile("setmaxnreg.inc.sync.aligned.u32 224;");
    const int q = warp & 3;         // TMEM lane quarter of this warp
    const int ch = (warp - 4) / 4;  // which half of the N columns
    const int r = q * 32 + lane;    // pixel row of the M-tile
    const int ty = r / kTW, tx = r % kTW;
    const int cpm = p.N / 64;       // 32-column chunks per M-tile per thread
    const uint32_t lane_base = tmem_base + ((uint32_t)(q * 32) << 16);
    int cs = 0;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
      int img, y0, x0, cg;
      decode_unit(p, u, img, y0, x0, cg);
      const int valid_rows = p.stack > 1 ? p.MT * kTileRows : min(p.MT * kTileRows, p.h_o - y0);
      const int mts = (valid_rows + kTileRows - 1) / kTileRows;
      float tot[COLS];
      for (int c = 0; c < n_chunks; ++c, ++cs) {
        const int set = cs & 1;
        mbar_wait_backoff(&chunk_full[set], (cs >> 1) & 1, 32);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
        for (int j = 0; j < COLS / 32; ++j) {
          const int mt = j / cpm;
          const int c0 = ch * (p.N / 2) + (j - mt * cpm) * 32;
          if (mt < mts) {  // warp-uniform
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              float v[16];
              const uint32_t col = (uint32_t)((DA ? 2 : 1) * mt * p.N + c0 + h * 16);
              tmem_ld16(lane_base + (uint32_t)set * kSetCols + col, v);
              if constexpr (DA) {  // + the chunk's correction terms
                float w[16];
                tmem_ld16(lane_base + (uint32_t)set * kSetCols + col + (uint32_t)p.N, w);
#pragma unroll
                for (int i = 0; i < 16; ++i) v[i] += w[i];
              }
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                float& t = tot[j * 32 + h * 16 + i];
                t = c == 0 ? v[i] : t + v[i];
              }
            }
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&chunk_empty[set]);
      }
      const int x = x0 + tx;
#pragma unroll
      for (int j = 0; j < COLS / 32; ++j) {
        const int mt = j / cpm;
        const int c0 = ch * (p.N / 2) + (j - mt * cpm) * 32;
        if (mt < mts) {
          int im, y;
          bool ok;
          tile_row_pixel(p, img, y0, mt * kTileRows + ty, im, y, ok);
          emit32(p, *reinterpret_cast<float(*)[32]>(&tot[j * 32]), im, y, x, ok && x < p.w_o, tx,
                 ty, cg, c0);
        }
      }
    }
  }

  if (kProf && p.dbg && lane == 0 && warp <= 2) {
    p.dbg[blockIdx.x * 8 + warp] = prof;
    if (warp == 1) p.dbg[blockIdx.x * 8 + 4] = prof2;
    if (warp == 1) p.dbg[blockIdx.x * 8 + 5] = clock64() - prof_t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(tmem_cols));
  }
}

// Prepared weights: [cg][i'][n][m][hi/lo][k-half][N][4], or
// [cg][i'][n][m][k-half][hi/lo][N][4] for DA (N = 64), from the blocked
// kernel [jb][i'][n][m][ii][jj] (tensor.hpp:131-137): w_hi = w with the low
// 13 mantissa bits cleared, w_lo = w - w_hi (exact).  Channel slots beyond
// jb_count blocks are zero.
__global__ void prepare_tf32x3_weights_kernel(const float* __restrict__ w, int ib_n, int h_f,
                                              int w_f, int jb_begin, int jb_count, int N,
                                              int da, const WSrc src, int64_t total, float* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t t = e;
    const int k4 = (int)(t % 4); t /= 4;
    const int co = (int)(t % N); t /= N;
    int kh, hl;
    if (da) {  // [k-half][hi/lo][N][4]: per k-half 2N rows, hi then lo
      hl = (int)(t % 2); t /= 2;
      kh = (int)(t % 2); t /= 2;
    } else {   // [hi/lo][k-half][N][4]
      kh = (int)(t % 2); t /= 2;
      hl = (int)(t % 2); t /= 2;
    }
    const int m = (int)(t % w_f); t /= w_f;
    const int n = (int)(t % h_f); t /= h_f;
    const int ib = (int)(t % ib_n); t /= ib_n;
    const int cg = (int)t;
    const int jl = cg * (N / 8) + co / 8;
    float v = 0.f;
    if (jl < jb_count) {
      const int jb = jb_begin + jl, jj = co % 8, ii = kh * 4 + k4;
      v = weight_src(w, jb, ib, n, m, ii, jj, src);
    }
    const float h = __uint_as_float(__float_as_uint(v) & kHiMask);
    out[e] = hl ? v - h : h;
  }
}

using X3Kernel = void (*)(const CUtensorMap, const Tf32Params);

// (WF, MT, COLS) instantiations: WF in {3, 1, generic}, MT * N in {128, 256};
// DA (N <= 128): MT * N = 128
template <int WF, int V>
X3Kernel pick_wf(int MT, int cols, bool da) {
  if (da)
    return MT == 1 ? conv_tf32x3_kernel<WF, 1, 64, true, V> : conv_tf32x3_kernel<WF, 2, 64, true, V>;
  if (MT == 1)
    return cols == 64 ? conv_tf32x3_kernel<WF, 1, 64, false, V>
                      : conv_tf32x3_kernel<WF, 1, 128, false, V>;
  if (MT == 2)
    return cols == 64 ? conv_tf32x3_kernel<WF, 2, 64, false, V>
                      : conv_tf32x3_kernel<WF, 2, 128, false, V>;
  return conv_tf32x3_kernel<WF, 4, 128, false, V>;
}
// walks as in conv_tf32.cu: 3x3 / generic plain or space-to-depth, 1x1 plain or wide
X3Kernel pick_x3_kernel(const Tf32Params& p) {
  const int cols = p.MT * p.N / 2;
  if (p.w_f == 1)
    return p.wide ? pick_wf<1, kWalkWide>(p.MT, cols, p.da) : pick_wf<1, kWalkPlain>(p.MT, cols, p.da);
  if (p.s2d > 1)
    return p.w_f == 3 ? pick_wf<3, kWalkS2D>(p.MT, cols, p.da) : pick_wf<0, kWalkS2D>(p.MT, cols, p.da);
  return p.w_f == 3 ? pick_wf<3, kWalkPlain>(p.MT, cols, p.da) : pick_wf<0, kWalkPlain>(p.MT, cols, p.da);
}

void set_x3_attrs(X3Kernel k) {
  // attributes are per device: once for each (kernel, device)
  if (dconv_host::first_use_on_device(reinterpret_cast<const void*>(k),
                                      dconv_host::current_device()))
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
}

// separate correction accumulator for N = 64 (DCONV_X3_NO_DA: off); the
// prepared weight layout follows it.  Measured: N = 64 layers +9..18% (two
// MMAs per tap instead of three, an N = 64 MMA costing as much as N = 128);
// N = 128 loses (MT halves to 1: twice the weight traffic per pixel; 512->128
// 1x1 -30%), so it keeps three MMAs into one accumulator.
bool use_da(int N) {
  static const bool off = getenv("DCONV_X3_NO_DA") != nullptr;
  return !off && N == 64;
}

}  // namespace

int64_t tf32x3_prepared_floats(int ib_n, int h_f, int w_f, int jb_count) {
  const int N = tf32_channels(jb_count);
  const int n_cg = (jb_count * 8 + N - 1) / N;
  return (int64_t)n_cg * ib_n * h_f * w_f * 4 * N * 4;
}

int launch_prepare_tf32x3(const float* w, int ib_n, int h_f, int w_f, int jb_begin, int jb_count,
                          const WSrc& src, float* out, cudaStream_t stream) {
  const int N = tf32_channels(jb_count);
  const int64_t total = tf32x3_prepared_floats(ib_n, h_f, w_f, jb_count);
  const int64_t blocks = std::min<int64_t>((total + 255) / 256, 148 * 32);
  prepare_tf32x3_weights_kernel<<<(unsigned)blocks, 256, 0, stream>>>(
      w, ib_n, h_f, w_f, jb_begin, jb_count, N, use_da(N) ? 1 : 0, src, total, out);
  dconv_host::count_launch();
  return dconv_host::check_launch("prepare_tf32x3_weights_kernel");
}

int launch_conv_tf32x3(const FfmaParams& f0, const float* w_prepared, cudaStream_t stream) {
  FfmaParams f = f0;  // (f0: the original filter, before the space-to-depth view)
  InView view;
  if (int rc = prepare_view(f, view, "conv_tf32x3")) return rc;
  Tf32Params p{};
  p.w = w_prepared;
  copy_geometry(p, f);
  p.s2d = view.s2d;
  p.ib_o = view.ib;
  p.hf_o = f0.h_f;
  p.wf_o = f0.w_f;
  p.N = tf32_channels(f.jb_count);
  p.n_cg = (f.jb_count * 8 + p.N - 1) / p.N;
  const int sms = sm_count();
  const int wtap = 4 * p.N * 4 * 4;  // bytes per (i', n, m): hi + lo
  // Filter rows per stage when the whole filter's hi/lo weights of one
  // input block fit the 72 KB weight budget: all of them, else as many as fit.
  auto rows_for = [&](int r_cap) {
    return p.h_f * p.w_f * wtap <= 72 * 1024 && r_cap == p.h_f
               ? p.h_f
               : std::max(1, std::min(r_cap, (72 * 1024) / (p.w_f * wtap)));
  };
  // Image slots per unit: small maps (h_o = 7) stack images along the tile
  // rows, slot k at patch row k * SP (SP = h_o + R - 1), instead of leaving
  // most of a 16-row M-tile empty.  Not with the fused pool (its windows
  // pair tile rows).
  auto stack_for = [&](int mt, int R) {
    const int sp = p.h_o + R - 1;
    if ((p.epi & DCONV_EPI_MAXPOOL) || p.h_o + sp > mt * kTileRows) return 1;
    static const bool no_stack = getenv("DCONV_NO_STACK") != nullptr;
    return no_stack ? 1 : std::min(p.n, (mt * kTileRows - p.h_o) / sp + 1);
  };
  // M-tiles per unit (MT * N in {128, 256}: two chunk sets fit TMEM, the
  // totals fit the epilogue registers).  Cost per input block = max(3 MMAs
  // per tap and M-tile; shared-memory traffic at ~120 B/cycle (MMA operand
  // reads, TMA writes, the split's read + write); L2 -> SM loads at ~40
  // B/cycle (patch + hi/lo weights)) + per-unit fill / epilogue; rounds of
  // units over the SMs.
  {
    double best = -1;
    const bool da = use_da(p.N);
    for (int mt = kMaxMT; mt >= 1; --mt) {
      const int cols = mt * p.N / 2;
      if (da ? cols != 64 : (cols != 64 && cols != 128)) continue;
      // TMA box rows of a strided (space-to-depth) read: (PH) x s <= 256
      if ((mt * kTileRows - 1 + p.h_f) * p.s2d > 256) continue;
      const int st = stack_for(mt, rows_for(p.h_f));
      const int rg = st > 1 ? 1 : (p.h_o + mt * kTileRows - 1) / (mt * kTileRows);
      const int64_t units =
          (int64_t)((p.n + st - 1) / st) * rg * ((p.w_o + kTW - 1) / kTW) * p.n_cg;
      const double taps = (double)p.h_f * p.w_f;
      const double mma_cyc = p.N > 128 ? 128.0 : 71.0;
      // DA: one N' = 2N MMA + one N MMA per tap and M-tile
      const double mma = da ? taps * mt * ((p.N > 64 ? 128.0 : 71.0) + 71.0)
                            : taps * mt * 3 * mma_cyc;
      const double patch = (double)(mt * kTileRows - 1 + p.h_f) * (kTW - 1 + p.w_f) * 32.0;
      const double operands = da ? 2 * 4096.0 + 3 * p.N * 32.0 : 3 * (4096.0 + p.N * 32.0);
      const double smem_bytes = taps * mt * operands + taps * wtap + patch * 3;
      const double l2_bytes = taps * wtap + patch;
      const double unit =
          p.ib_n * std::max({mma, smem_bytes / 120.0, l2_bytes / 40.0}) + 1500.0;
      const double rounds = (double)((units + sms - 1) / sms);
      const double score = 1.0 / (rounds * unit);
      if (score > best * (1 + 1e-9)) {
        best = score;
        p.MT = mt;
      }
    }
    if (best < 0)
      return dconv_host::set_error(DCONV_EUNSUPPORTED,
                                   "conv_tf32x3: no M-tile count for N = %d, stride %d", p.N, p.s2d);
    static const char* force_mt = getenv("DCONV_TF32_MT");
    if (force_mt) {
      const int mt = atoi(force_mt);
      if (mt >= 1 && mt <= kMaxMT && (mt * p.N == 128 || (!da && mt * p.N == 256))) p.MT = mt;
    }
  }
  // stage = G input blocks x R filter rows: <= 72 KB of hi/lo weights,
  // <= 40 KB of patch (hi + lo planes); at least two stages in 220 KB --
  // else fewer filter rows per stage, then fewer M-tiles
  const int bar_bytes = (3 * kMaxStagesT + 4) * 8 + 16;
  static const bool no_deep = getenv("DCONV_X3_SHALLOW") != nullptr;  // A/B only
  int stage_bytes = 0;
  for (int r_cap = p.h_f;; ) {
    p.R = rows_for(r_cap);
    p.stack = stack_for(p.MT, p.R);
    p.SP = p.h_o + p.R - 1;
    p.PW = kTW - 1 + p.w_f;
    if (p.stack > 1) {
      // every slot's TMA destination (row k*SP of a block) 128-byte aligned:
      // widen the smem row pitch (= box width; the extra columns are
      // out-of-bounds zero fill or unused pixels) so SP*PW % 8 == 0
      int pw = p.PW;
      while ((p.SP * pw) % 8) ++pw;
      if (pw <= 16) p.PW = pw; else p.stack = 1;
    }
    // patch rows per input block (stacked: every slot's rows; rows read by
    // never-stored tile rows stay inside the block; blocks 128-B aligned)
    p.PH = std::max(p.MT * kTileRows - 1 + p.R, p.stack > 1 ? p.stack * p.SP : 0);
    if (p.stack > 1)
      while ((p.PH * p.PW) % 8) ++p.PH;
    const int patch_blk_bytes = 4 * p.PH * p.PW * 16;
    p.G = p.R == p.h_f ? std::max(1, std::min({p.ib_n, (72 * 1024) / (p.h_f * p.w_f * wtap),
                                               (40 * 1024) / patch_blk_bytes}))
                       : 1;
    // 1x1 layers: at least 4 ring stages (smaller G) -- their stages are
    // short, and with 2 the TMA -> split -> MMA hand-off is exposed
    // (ResNet-50 1024->256 1x1 b256: the split warps waited on TMA half the time)
    // (>= 32 input blocks: the short-K layers are epilogue-bound, measured
    // 2% slower with the deeper ring: ResNet-50 64->256 1x1 + skip-add)
    if (p.h_f * p.w_f == 1 && p.ib_n >= 32 && !no_deep)
      while (p.G > 1 &&
             4 * (((4 * ((p.G * p.PH * p.PW * 4 + 31) & ~31) + p.G * p.R * p.w_f * 4 * p.N * 4) +
                   255) & ~255) * 4 > 220 * 1024 - bar_bytes)
        --p.G;
    // space-to-depth: a stage's blocks must lie in one phase
    if (p.s2d > 1)
      while (p.ib_o % p.G) --p.G;
    p.plane_floats = (p.G * p.PH * p.PW * 4 + 31) & ~31;  // 128 B aligned planes
    p.wstage_floats = p.G * p.R * p.w_f * 4 * p.N * 4;
    p.stage_floats = ((4 * p.plane_floats + p.wstage_floats) + 255) & ~255;  // 1 KB aligned
    stage_bytes = p.stage_floats * 4;
    p.NS = std::min(kMaxStagesT, (220 * 1024 - bar_bytes) / stage_bytes);
    if (p.NS >= 2) break;
    if (p.R > 1) {
      r_cap = p.R - 1;
    } else if (p.MT > 1 && (p.MT / 2) * p.N >= 128 && !use_da(p.N)) {
      p.MT /= 2;
      r_cap = p.h_f;
    } else {
      return dconv_host::set_error(DCONV_EUNSUPPORTED, "conv_tf32x3: stage of %d bytes",
                                   stage_bytes);
    }
  }
  p.n_g = (p.ib_n + p.G - 1) / p.G;
  p.n_r = (p.h_f + p.R - 1) / p.R;
  if (p.PH > 256 || p.PW > 256 || p.G > 256)
    return dconv_host::set_error(DCONV_EUNSUPPORTED, "conv_tf32x3: TMA box too large");
  // accumulator chunk: ~144 products (DCONV_X3_CHUNK_K), whole stages
  // (profiles/r1_tf32x3_kernel_accuracy.txt: worst element at 0.52 of the
  // fp32 tolerance at K = 4608; 288 reaches 0.90, 576 fails)
  // (DA: the correction terms have their own accumulator; chunk 288)
  p.da = use_da(p.N) ? 1 : 0;
  static const int chunk_env = getenv("DCONV_X3_CHUNK_K") ? atoi(getenv("DCONV_X3_CHUNK_K")) : 0;
  const int chunk_k = chunk_env ? chunk_env : (p.da ? 288 : 144);
  const int k_stage = p.G * p.R * p.w_f * 8;
  p.chunk_st = std::max(1, chunk_k / k_stage);
  p.row_groups = p.stack > 1 ? 1 : (p.h_o + p.MT * kTileRows - 1) / (p.MT * kTileRows);
  p.strips = (p.w_o + kTW - 1) / kTW;
  p.units = (p.n + p.stack - 1) / p.stack * p.row_groups * p.strips * p.n_cg;
  p.idesc = tf32_idesc(p.N);
  p.idesc2 = tf32_idesc(2 * p.N);

  CUtensorMap map;
  // stacked: one box per (image slot, block), SP rows; else PH rows x G blocks;
  // 1x1 layers: whole pencils per box (DCONV_TF32_NO_WIDE=1: half planes)
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
  set_x3_attrs(pick_x3_kernel(p));
  const size_t smem = (size_t)p.NS * stage_bytes + bar_bytes;
  const int grid = std::min(p.units, sms);
  static const bool dbg = getenv("DCONV_DEBUG") != nullptr;
  if (dbg)
    fprintf(stderr,
            "conv_tf32x3 N=%d MT=%d G=%d R=%d NS=%d stage=%d B chunk_st=%d stack=%d da=%d "
            "units=%d\n",
            p.N, p.MT, p.G, p.R, p.NS, stage_bytes, p.chunk_st, p.stack, p.da, p.units);
  static const bool prof = kProf && getenv("DCONV_TF32_PROFILE") != nullptr;
  if (prof) {  // debugging aid: where do the roles wait?  (not for timed runs)
    cudaMalloc(&p.dbg, (size_t)grid * 8 * 8);
    cudaMemsetAsync(p.dbg, 0, (size_t)grid * 8 * 8, stream);
    pick_x3_kernel(p)<<<grid, kThreadsX, smem, stream>>>(map, p);
    std::vector<unsigned long long> h((size_t)grid * 8);
    cudaMemcpy(h.data(), p.dbg, h.size() * 8, cudaMemcpyDeviceToHost);
    double a[6] = {0, 0, 0, 0, 0, 0};
    for (int b = 0; b < grid; ++b)
      for (int i = 0; i < 6; ++i) a[i] += (double)h[b * 8 + i] / grid;
    fprintf(stderr,
            "conv_tf32x3 profile: avg cycles producer(empty)=%.0f mma(split)=%.0f "
            "mma(chunk_empty)=%.0f split(full)=%.0f total=%.0f\n",
            a[0], a[1], a[4], a[2], a[5]);
    cudaFree(p.dbg);
    p.dbg = nullptr;
  }
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreadsX);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cfg.attrs = attr;
  cfg.numAttrs = dconv_host::pdl_enabled() ? 1 : 0;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, pick_x3_kernel(p), map, p);
  if (e != cudaSuccess)
    return dconv_host::set_error(DCONV_ECUDA, "conv_tf32x3: %s", cudaGetErrorString(e));
  dconv_host::count_launch();
  return dconv_host::check_launch("conv_tf32x3_kernel");
}

}  // namespace dconv_dev
