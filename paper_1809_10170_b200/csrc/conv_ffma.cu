// conv_ffma.cu -- register-blocked FP32 direct convolution for sm_100a.
//
// GPU restatement of Alg. 3 in the blocked layout with
// c_ib = c_ob = 8 (one 32-byte pencil = one DRAM sector per pixel):
//   * j' (output blocks, "in Parallel")      -> blockIdx.y, BN/8 blocks per CTA
//   * l, k' (output rows / row tiles)        -> work unit: TH x TW pixel tile of
//                                               the batch-stacked output
//   * i' (input blocks, cache blocking)      -> the shared-memory pipeline stage
//   * (n, m, ii) reduction                   -> per-stage loop from smem
//   * (kk, jj) register tile                 -> 8 pixels x TCO channels / thread
// Input index s*(k'*w_ob + kk) + m (SPEC.md:354 stride fix).
//
// Data movement: warp 0 streams each stage NS-1 stages ahead -- the input
// patch rows of G i'-blocks (each row of a blocked map is contiguous) and the
// matching (j', i') weight slab rows (contiguous, tensor.hpp:138-140) -- with
// 1-D bulk async copies (cp.async.bulk, SASS UBLKCP) into an NS-deep ring of
// smem stages guarded by full/empty mbarriers; all NW warps compute.
//
// Arithmetic: FFMA2 (fma.rn.f32x2, each lane an IEEE fp32 fma).  Accuracy:
// two-level summation -- each thread accumulates ~256 products in registers,
// then folds that partial sum into a running total kept in TMEM
// (tcgen05.st / tcgen05.ld, no register cost).  For K = 4608 the worst-case
// per-element error drops well below a single fp32 accumulator's (the
// reference's own conv_naive reaches 3e-4 there), keeping every element
// inside |a-b| <= 1e-4 + 1e-5|b| of conv_oracle64.
//
// Zero workspace: nothing is written to global memory except the output,
// once, from registers (smem ring and TMEM are on-chip).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "conv_kernels.h"

namespace dconv_dev {

namespace {

constexpr int kCB = 8;          // channels per math sub-block (a thread's 8 output channels,
                                // one input slice of a tap); storage blocks are CBS = 8/16/32
constexpr int kMaxStages = 8;
constexpr int kMaxKs = 16;      // split-K cluster size (> 8 is the non-portable opt-in)

// Per-CTA phase clocks (DCONV_FFMA_PROFILE=1): compiled in only with
// -DDCONV_FFMA_PROF (tools/build_prof.sh) -- the stamps' tests cost the
// product build 1.7% on VGG-16 b32 and 7% on 1x1 layers.
#ifdef DCONV_FFMA_PROF
constexpr bool kFfmaProf = true;
#else
constexpr bool kFfmaProf = false;
#endif

// Tuning / debugging overrides, read once per process --
// except DCONV_KSPLIT, read at every launch so a test can force several
// split factors in one process.
struct Knobs {
  int force_g = 0, flush_every = 0;
  bool no_splitk = false, no_tailsplit = false, debug = false;
  Knobs() {
    if (const char* e = getenv("DCONV_FORCE_G")) force_g = atoi(e);
    if (const char* e = getenv("DCONV_FLUSH_EVERY")) flush_every = atoi(e);
    no_splitk = getenv("DCONV_NO_SPLITK") != nullptr;
    no_tailsplit = getenv("DCONV_NO_TAILSPLIT") != nullptr;
    debug = getenv("DCONV_DEBUG") != nullptr;
  }
};
const Knobs& knobs() {
  static const Knobs k;
  return k;
}
int ksplit_knob() {
  const char* e = getenv("DCONV_KSPLIT");
  return e ? atoi(e) : 0;
}
constexpr int kComputeWarps = 8;  // default: 2 compute warpgroups, 8x8 outputs / thread
constexpr int kThreads = (kComputeWarps + 4) * 32;  // + producer warpgroup

// ---- TMEM helpers (32 lanes x 32 columns of 32-bit per warp) ----------------
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, "
      "%8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, "
      "%23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]),
      "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]),
      "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
      "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
      "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]),
      "r"(v[31])
      : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, "
      "%8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, "
      "%23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
        "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]),
        "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
        "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]),
        "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, "
      "%8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
        "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]),
        "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

// acc (NP pairs) -> TMEM at taddr (+ optional fold of the previous total)
template <int NP>
__device__ __forceinline__ void tmem_fold(uint32_t taddr, uint64_t* acc,
                                          bool have_total, bool store) {
  static_assert(NP % 16 == 0, "32-column chunks");
#pragma unroll
  for (int c = 0; c < NP / 16; ++c) {
    uint32_t v[32];
    const uint32_t ta = taddr + c * 32;
    if (have_total) {
      tmem_ld32(ta, v);
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        uint64_t t;
        asm("mov.b64 %0, {%1, %2};" : "=l"(t) : "r"(v[2 * i]), "r"(v[2 * i + 1]));
        acc[c * 16 + i] = fadd2(acc[c * 16 + i], t);
      }
    }
    if (store) {
#pragma unroll
      for (int i = 0; i < 16; ++i)
        asm("mov.b64 {%0, %1}, %2;" : "=r"(v[2 * i]), "=r"(v[2 * i + 1]) : "l"(acc[c * 16 + i]));
      tmem_st32(ta, v);
    }
  }
}

// final = (running total) + acc -> TMEM result columns t_res, handed to the
// epilogue warpgroup
template <int NP>
__device__ __forceinline__ void tmem_finalize(uint32_t t_tot, uint32_t t_res, const uint64_t* acc,
                                              bool have_total) {
#pragma unroll
  for (int c = 0; c < NP / 16; ++c) {
    uint32_t v[32];
    if (have_total) {
      tmem_ld32(t_tot + c * 32, v);
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        uint64_t t;
        asm("mov.b64 %0, {%1, %2};" : "=l"(t) : "r"(v[2 * i]), "r"(v[2 * i + 1]));
        t = fadd2(acc[c * 16 + i], t);
        asm("mov.b64 {%0, %1}, %2;" : "=r"(v[2 * i]), "=r"(v[2 * i + 1]) : "l"(t));
      }
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i)
        asm("mov.b64 {%0, %1}, %2;" : "=r"(v[2 * i]), "=r"(v[2 * i + 1]) : "l"(acc[c * 16 + i]));
    }
    tmem_st32(t_res + c * 32, v);
  }
}

// Pixel tiles live on the batch-stacked "virtual image": image i occupies
// virtual output rows [i*h_o, (i+1)*h_o).  A TH x TW tile starting at virtual
// row vy0 therefore covers a run of row segments -- the tail of image img0,
// then whole images, then the head of another -- so maps of any height
// (56, 28, 14, 7, 13 ...) fill whole tiles.  In shared memory the patch rows
// of the segments are stacked: segment 0 holds (cnt0-1)*s + R rows, every
// later segment (h_o-1)*s + R rows.
struct TileRows {
  int vy0, img0, y0, cnt0, th;  // th: valid virtual rows of this tile
};

// v / h_o for 0 <= v < n * h_o (multiply-high by a host-computed reciprocal)
__device__ __forceinline__ int div_ho(const FfmaParams& p, int v) {
  return p.h_o_magic ? (int)__umulhi((unsigned)v, p.h_o_magic) : v / p.h_o;
}

__device__ __forceinline__ TileRows tile_rows(const FfmaParams& p, int tile_y) {
  TileRows t;
  t.vy0 = tile_y * p.TH;
  t.img0 = div_ho(p, t.vy0);
  t.y0 = t.vy0 - t.img0 * p.h_o;
  t.th = min(p.TH, p.n * p.h_o - t.vy0);
  t.cnt0 = min(p.h_o - t.y0, t.th);
  return t;
}

// tile row ty -> (image, output row, first patch row)
__device__ __forceinline__ void tile_row(const FfmaParams& p, const TileRows& t, int ty,
                                         int& img, int& y, int& prow) {
  if (ty < t.cnt0) {
    img = t.img0;
    y = t.y0 + ty;
    prow = ty * p.sy;
  } else {
    const int d = ty - t.cnt0;
    const int j = div_ho(p, d);  // full segments before this one (segment j+1)
    y = d - j * p.h_o;
    img = t.img0 + 1 + j;
    prow = (t.cnt0 - 1) * p.sy + p.R + j * ((p.h_o - 1) * p.sy + p.R) + y * p.sy;
  }
}

// NW compute warps (8: 232 registers each; 12: 152 registers, 3 warps per
// SMSP for latency hiding, activations loaded 2 channels at a time).
// Weight chunk of output block c inside a stage: TCO = 8 pads each chunk by
// 16 B, TCO = 16 (a thread reads blocks 2t and 2t+1) skews every block pair by
// 16 B -- either way the 8 lanes of a warp that read different blocks hit
// distinct 16-byte bank groups.
template <int TCO>
__host__ __device__ __forceinline__ int wchunk(int c, int wstride) {
  return TCO == 16 ? c * wstride + (c >> 1) * 4 : c * wstride;
}

// Roles: NW compute warps (two warpgroups), a producer warpgroup (one active
// warp) and an epilogue warpgroup: when p.epi_wg, the compute warps hand each
// finished tile to the epilogue warps through TMEM and go straight on to the
// next unit, so skip-add / ReLU / stores overlap the next tile's FFMA2s.
// CBS: channel block of the stored maps and kernels (c_ib = c_ob = CBS, 8 /
// 16 / 32).  A pixel of a staged row is CBS floats; the math walks it as
// CBS / 8 sub-blocks of 8 channels, and an 8-channel output sub-block jl8 is
// storage block jl8 / SUB at channel offset (jl8 % SUB) * 8 of the pencil.
// jb_begin / jb_count count 8-channel sub-blocks, ib_n storage blocks.
template <int CBS>
__device__ __forceinline__ int64_t sub_off(int jl8, int64_t blk) {
  return (int64_t)(jl8 / (CBS / 8)) * blk + (jl8 % (CBS / 8)) * 8;
}

template <int BM, int BN, int WF, int NW, int TPX, int TCO, int CBS>
__global__ void __launch_bounds__((NW + 8) * 32, 1)
    conv_ffma_kernel(const FfmaParams p) {
  constexpr int SUB = CBS / kCB;  // 8-channel sub-blocks per storage block
  // TCO: channels per thread (1 or 2 output blocks)
  constexpr int NBLK = TCO / 8;
  constexpr int AV = NW == 8 ? 4 : 2;  // activation channels per LDS
  // TMEM running totals: NW/4 warp slots x TPX*TCO columns
  constexpr int kTmemCols = (NW / 4) * TPX * TCO <= 128 ? 128 : ((NW / 4) * TPX * TCO <= 256 ? 256 : 512);
  constexpr int PG = BM / TPX;   // pixel groups (TPX pixels each)
  constexpr int CGT = BN / TCO;  // channel thread groups == output blocks
  // warp shape: PPW pixel groups x CPW channel groups per warp (4 x 8; the
  // 32-channel tile, CGT = 4: 8 x 4)
  constexpr int PPW = CGT >= 8 ? 4 : 8, CPW = 32 / PPW;
  static_assert(CGT % CPW == 0 || CGT == CPW, "warp shape");
  constexpr int WPG = PG / PPW;  // warps along pixels
  constexpr int NP = TPX * TCO / 2;  // accumulator pairs per thread
  static_assert(PG * CGT == NW * 32, "thread tile mismatch");
  constexpr int CG = BN / 8;     // output blocks per CTA tile

  extern __shared__ __align__(128) float smem[];
  float* red = smem + p.NS * p.stage_floats;   // split-K partials [64][256]
  uint64_t* full = reinterpret_cast<uint64_t*>(red + p.red_floats);
  uint64_t* empty = full + kMaxStages;
  uint64_t* ready = empty + kMaxStages;        // all ranks' partials written
  uint64_t* done = ready + 1;                  // all ranks finished reading mine
  uint64_t* res_full = done + 1;               // [2] tile results in TMEM
  uint64_t* res_empty = res_full + 2;          // [2] epilogue drained them
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(res_empty + 2);

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const long long t_start = kFfmaProf && p.dbg ? clock64() : 0;
  if (kFfmaProf && p.dbg && threadIdx.x == 0) p.dbg[blockIdx.x * 16 + 0] = (long long)globaltimer_ns();
  const int S = p.n_g * p.n_r;                 // stages per work unit
  const int co_groups = (p.jb_count + CG - 1) / CG;
  const int n_units = p.unit_count;             // this launch's units: [unit_begin, +count)
  // Split-K over a thread-block cluster of ks CTAs: rank r runs stages
  // [st0, st1) of every unit, the partial tiles are reduced through DSMEM.
  const int ks = p.ksplit;
  const int rank = blockIdx.x % ks;            // == %cluster_ctarank (1-D cluster)
  const int cluster_id = blockIdx.x / ks, n_clusters = gridDim.x / ks;
  const int st0 = rank * S / ks, st1 = (rank + 1) * S / ks;
  const bool use_tmem = (p.streamk ? S : st1 - st0) > p.flush_every;
  // Work pieces of this CTA: (unit, [s0, s1) of its S stages).  Default: the
  // units cluster_id, cluster_id + n_clusters, ... with the rank's stage
  // range.  Stream-K: a contiguous range of the launch's units x S stages.
  struct Pieces {
    int sk, S, n_units, step, u, st0, st1, g, g_end, sk_base;
    __device__ bool next(int& uu, int& s0, int& s1) {
      if (sk) {
        // whole waves first, round-robin like the default (neighbouring CTAs
        // on neighbouring tiles: contiguous ranges alone cost the memory-heavy
        // 1x1 + skip layers 4-5%), then the last 1.x waves as stage ranges
        if (u + step < sk_base) {
          u += step;
          uu = u; s0 = 0; s1 = S;
          return true;
        }
        if (g >= g_end) return false;
        uu = g / S;
        s0 = g - uu * S;
        uu += sk_base;
        s1 = min(S, s0 + (g_end - g));
        g += s1 - s0;
        return true;
      }
      u += step;
      if (u >= n_units) return false;
      uu = u; s0 = st0; s1 = st1;
      return true;
    }
  };
  auto make_pieces = [&]() {
    Pieces it;
    it.sk = p.streamk; it.S = S; it.n_units = n_units; it.step = n_clusters;
    it.u = cluster_id - n_clusters; it.st0 = st0; it.st1 = st1;
    it.sk_base = p.sk_base;
    const long long W = (long long)(n_units - p.sk_base) * S;
    it.g = (int)(W * blockIdx.x / gridDim.x);
    it.g_end = (int)(W * (blockIdx.x + 1) / gridDim.x);
    return it;
  };

  if (tid == 0) {
    for (int i = 0; i < p.NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], NW);
    }
    mbar_init(ready, ks);  // one arrive per rank (thread 0, after a named barrier)
    mbar_init(done, ks);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&res_full[i], NW);
      mbar_init(&res_empty[i], 4);
    }
    fence_mbar_init();
    if (p.dbg) p.dbg[blockIdx.x * 16 + 14] = clock64() - t_start;  // barriers initialised
  }
  // TMEM: running totals [0, 128) + (epilogue hand-off) 2 result buffers
  constexpr int kResCols = (NW / 4) * TPX * TCO;
  const bool tmem_on = use_tmem || p.epi_wg;
  const uint32_t tmem_cols = p.epi_wg ? 512u : (uint32_t)kTmemCols;
  if (tmem_on && warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // setup above overlaps the previous kernel's tail (programmatic dependent
  // launch); its output is read only from here on
  pdl_wait();
  pdl_launch_dependents();
  // every rank's barriers and smem must exist before the first remote access:
  // arrive now, wait only right before the first publish (the ranks' setup
  // and main loops overlap the barrier instead of waiting on it)
  if (ks > 1) cluster_arrive_release();
  if (kFfmaProf && p.dbg && tid == 0) p.dbg[blockIdx.x * 16 + 15] = clock64() - t_start;  // setup done

  // unit u -> (co group fastest: concurrently running CTAs share the pixel
  // tile's patch rows in L2, consecutive waves reuse the weight slabs)
  auto decode = [&](int u, TileRows& tr, int& tx0, int& jb0, int& cg_valid) {
    u += p.unit_begin;
    const int cgi = u % co_groups;
    const int t = u / co_groups;
    const int tile_y = t / p.tiles_x;
    tr = tile_rows(p, tile_y);
    tx0 = (t - tile_y * p.tiles_x) * p.TW;
    jb0 = p.jb_begin + cgi * CG;
    cg_valid = min(CG, p.jb_begin + p.jb_count - jb0);
  };

  if (warp >= NW + 4) {
    // ------------------------------------------------------------ epilogue WG
    asm volatile("setmaxnreg.dec.sync.aligned.u32 96;");
    if constexpr (NW == 8 && TCO == 8) {
      if (p.epi_wg) {
        const uint32_t tmem_base = *tmem_slot;
        const int qd = warp & 3;  // TMEM lane quarter = compute warps qd, qd + 4
        // a lane's consecutive pixels are PG apart in the tile: PG / TW rows, PG % TW columns
        const int e_dty = (int)__umulhi((unsigned)PG, p.tw_magic), e_dtx = PG - e_dty * p.TW;
        int unit_iter = 0;  // whole units (the ones handed over through TMEM)
        Pieces pieces = make_pieces();
        for (int u, ps0, ps1; pieces.next(u, ps0, ps1);) {
          if (ps0 != 0) continue;  // a stream-K contributor piece is stored raw by the compute warps
          TileRows tr;
          int tx0, jb0, cg_valid;
          decode(u, tr, tx0, jb0, cg_valid);
          const int rb = unit_iter & 1;
          mbar_wait(&res_full[rb], (unit_iter >> 1) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll 1
          for (int half = 0; half < 2; ++half) {
            const int cw = qd + 4 * half;  // the compute warp whose tile this lane holds
            const int pg = (cw % WPG) * PPW + (lane % PPW);
            const int cb = (cw / WPG) * CPW + lane / PPW;
            const int jl = jb0 + cb - p.jb_begin;
            const uint32_t tr_addr = tmem_base + ((uint32_t)(qd * 32) << 16) +
                                     (uint32_t)(kResCols * (1 + rb) + half * TPX * TCO);
            // Every lane runs the tcgen05.ld (warp-collective); blocks past
            // cg_valid only skip their stores.
            const bool blk_ok = cb < cg_valid;
            // This lane's pixels are q = pg + PG * k: tile coordinates and
            // the output / skip offsets advance by a fixed step (dty rows,
            // dtx columns, a carry when the column wraps), so only pixel 0
            // pays the divisions and 64-bit multiplies (the epilogue warps
            // were instruction-bound on short-K 1x1 layers: ~100
            // instructions per pixel, ncu source page).  Tile row ty is
            // row vy0 + ty of the batch-stacked output.
            int ty = (int)__umulhi((unsigned)pg, p.tw_magic), tx = pg - ty * p.TW;
            int img = div_ho(p, tr.vy0 + ty), y = tr.vy0 + ty - img * p.h_o;
            int64_t o_off = sub_off<CBS>(jl, p.out_blk) + (int64_t)img * p.out_img +
                            (int64_t)y * p.out_row + (int64_t)(tx0 + tx) * CBS;
            int64_t s_off = 0;
            if (p.epi & DCONV_EPI_ADD)
              s_off = sub_off<CBS>(jl, p.sk_blk) + (int64_t)img * p.sk_img +
                      (int64_t)y * p.sk_row + (int64_t)(tx0 + tx) * CBS;
            // 4 pixels at a time: their skip pencils first (4 256-bit loads
            // in flight per thread), then the TMEM chunks are read and stored.
#pragma unroll 1
            for (int k4 = 0; k4 < TPX; k4 += 4) {
              int64_t ooff[4];
              float4 sk4[8];
#pragma unroll
              for (int kk = 0; kk < 4; ++kk) {
                const bool ok = blk_ok && ty < tr.th && tx0 + tx < p.w_o;
                ooff[kk] = ok ? o_off : -1;
                if ((p.epi & DCONV_EPI_ADD) && ok)
                  ldg_pencil(p.skip + s_off, sk4[2 * kk], sk4[2 * kk + 1]);
                // next pixel of this lane
                int dy = e_dty;
                tx += e_dtx;
                int dx = e_dtx;
                if (tx >= p.TW) { tx -= p.TW; dx -= p.TW; ++dy; }
                ty += dy;
                y += dy;
                o_off += (int64_t)dy * p.out_row + dx * CBS;
                s_off += (int64_t)dy * p.sk_row + dx * CBS;
                while (y >= p.h_o) {  // into the next image of the stack
                  y -= p.h_o;
                  o_off += p.out_img - (int64_t)p.h_o * p.out_row;
                  s_off += p.sk_img - (int64_t)p.h_o * p.sk_row;
                }
              }
#pragma unroll
              for (int kc = 0; kc < 2; ++kc) {
                uint32_t v[16];
                tmem_ld16(tr_addr + (k4 * 8 + kc * 16), v);
#pragma unroll
                for (int kj = 0; kj < 2; ++kj) {
                  const int kk = kc * 2 + kj;
                  if (ooff[kk] < 0) continue;
                  float o[8];
#pragma unroll
                  for (int c = 0; c < 8; ++c) o[c] = __uint_as_float(v[kj * 8 + c]);
                  if (p.epi & DCONV_EPI_ADD) {
                    o[0] += sk4[2 * kk].x; o[1] += sk4[2 * kk].y;
                    o[2] += sk4[2 * kk].z; o[3] += sk4[2 * kk].w;
                    o[4] += sk4[2 * kk + 1].x; o[5] += sk4[2 * kk + 1].y;
                    o[6] += sk4[2 * kk + 1].z; o[7] += sk4[2 * kk + 1].w;
                  }
                  if (p.epi & DCONV_EPI_RELU) {
#pragma unroll
                    for (int c = 0; c < 8; ++c) o[c] = fmaxf(o[c], 0.f);
                  }
                  float* dst = p.out + ooff[kk];
                  DCONV_OWN(dst, 8);
                  stg_pencil(dst, o);
                  for (int pi = 0; pi < p.n_peers; ++pi) stg_pencil(p.peer_out[pi] + ooff[kk], o);
                }
              }
            }
          }
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(&res_empty[rb]);
          ++unit_iter;
        }
      }
    }
    // TMEM is freed only after every compute and epilogue warp is done
    if (tmem_on) asm volatile("bar.sync 2, %0;" ::"n"((NW + 4) * 32) : "memory");
    return;
  }
  if (warp >= NW) {
    // ------------------------------------------------------------ producer
    // One warpgroup, register budget handed to the compute warpgroups; its
    // warps stream every stage of every unit of this CTA through the NS-deep
    // ring (prefetch runs across unit boundaries, so the epilogue of one tile
    // overlaps the loads of the next).  A bulk copy takes uniform operands,
    // so a warp issues its lanes' copies one after another: the stage's
    // copies are spread over kProdWarps warps to issue them in parallel
    // (1x1 layers need ~130 row copies per unit).
    asm volatile("setmaxnreg.dec.sync.aligned.u32 32;");
    constexpr int kProdWarps = 4;
    const int pw = warp - NW;
    const int pt = pw * 32 + lane;  // producer thread index
    if (kFfmaProf && p.dbg && pt == 0) p.dbg[blockIdx.x * 16 + 8] = clock64() - t_start;
    int gs = 0;
    int pbuf = 0;            // ring slot of stage gs (gs % NS)
    uint32_t pphase = 0u;    // (gs / NS) & 1
    const int seg_rows_full = (p.h_o - 1) * p.sy;  // + Re per full segment
    Pieces pieces = make_pieces();
    for (int u, st0, st1; pieces.next(u, st0, st1);) {  // (shadow the rank's range)
      TileRows tr;
      int tx0, jb0, cg_valid;
      decode(u, tr, tx0, jb0, cg_valid);
      if (kFfmaProf && p.dbg && pt == 0 && gs == 0) p.dbg[blockIdx.x * 16 + 12] = clock64() - t_start;
      const int col0 = tx0 * p.s;
      const int cols = min(p.PW, p.w_i - col0);
      const int n_seg = 1 + (tr.th - tr.cnt0 + p.h_o - 1) / p.h_o;
      if ((p.epi & DCONV_EPI_ADD) && rank == 0 && p.skip_prefetch) {
        // the epilogue reads this unit's skip tile once: pull it into L2 now,
        // a unit ahead of the read, so the ADD epilogue does not wait on HBM
        const uint32_t row_bytes = (uint32_t)(min(p.TW, p.w_o - tx0) * CBS * 4);
        for (int t = pt; t < cg_valid * tr.th; t += 32 * kProdWarps) {
          const int c = t / tr.th, ty = t - c * tr.th;
          int img, y, prow;
          tile_row(p, tr, ty, img, y, prow);
          if ((c % SUB) == 0)  // one prefetch per storage block row
            bulk_prefetch_l2(p.skip + sub_off<CBS>(jb0 + c - p.jb_begin, p.sk_blk) +
                                 (int64_t)img * p.sk_img + (int64_t)y * p.sk_row +
                                 (int64_t)tx0 * CBS,
                             row_bytes);
        }
      }
      int g = st0 / p.n_r, r = st0 - g * p.n_r;
      for (int st = st0; st < st1; ++st, ++gs) {
        const int buf = pbuf;
        if (gs >= p.NS) mbar_wait(&empty[buf], pphase ^ 1u);
        if (++pbuf == p.NS) { pbuf = 0; pphase ^= 1u; }
        if (st > st0 && ++r == p.n_r) { r = 0; ++g; }
        const int ib0 = g * p.G, Ge = min(p.G, p.ib_n - ib0);
        const int n0 = r * p.R, Re = min(p.R, p.h_f - n0);
        // rows of each segment this stage: (cnt-1)*s + Re
        const int rows_first = (tr.cnt0 - 1) * p.sy + Re;
        const int rest = tr.th - tr.cnt0;  // rows in later segments
        const int n_full = rest / p.h_o, last_cnt = rest - n_full * p.h_o;
        const int total_rows = rows_first + n_full * (seg_rows_full + Re) +
                               (last_cnt ? (last_cnt - 1) * p.sy + Re : 0);
        const uint32_t patch_bytes = (uint32_t)(Ge * total_rows * cols * CBS * 4);
        const uint32_t wbytes = (uint32_t)(Re * p.w_f * CBS * CBS * 4) * Ge;
        const int n_wblk = (cg_valid + SUB - 1) / SUB;  // storage blocks of weights
        float* sp = smem + buf * p.stage_floats;
        float* sw = sp + p.patch_floats;
        // one expect_tx per stage; copies of other warps may complete before
        // it (the transaction count is allowed to run ahead within a phase)
        if (pt == 0) mbar_arrive_expect_tx(&full[buf], patch_bytes + wbytes * n_wblk);
        __syncwarp();
        if (kFfmaProf && p.dbg && pt == 0 && gs == 0) p.dbg[blockIdx.x * 16 + 13] = clock64() - t_start;
        // the stage's copies are numbered in one sequence (segments' rows,
        // then weight chunks) and dealt round-robin over the producer warps
        // (copy c -> warp c % 4, lane c / 4 % 32): a bulk copy takes uniform
        // operands, so a warp issues its lanes' copies one after another, and
        // few-row stages (batch 1) would otherwise all land on warp 0
        const int me = pw + kProdWarps * lane;
        int cbase = 0;
        auto first_mine = [&](int base) {
          return base + ((me - base) % (32 * kProdWarps) + 32 * kProdWarps) % (32 * kProdWarps);
        };
        for (int j = 0; j < n_seg; ++j) {
          int img, y_start, rows, prow0;
          if (j == 0) {
            img = tr.img0; y_start = tr.y0; rows = rows_first; prow0 = 0;
          } else {
            const int cnt = min(p.h_o, rest - (j - 1) * p.h_o);
            img = tr.img0 + j; y_start = 0; rows = (cnt - 1) * p.sy + Re;
            prow0 = (tr.cnt0 - 1) * p.sy + p.R + (j - 1) * (seg_rows_full + p.R);
          }
          const float* src0 = p.in + (int64_t)img * p.in_img +
                              (int64_t)(y_start * p.sy + n0) * p.in_row + (int64_t)col0 * CBS;
          const int n_cp = Ge * rows;
          for (int c = first_mine(cbase); c < cbase + n_cp; c += 32 * kProdWarps) {
            const int t = c - cbase;
            const int gi = t / rows, pr = t - gi * rows;
            const float* src = src0 + (int64_t)(ib0 + gi) * p.in_blk + (int64_t)pr * p.in_row;
            float* dst = sp + ((gi * p.PH + prow0 + pr) * p.PW) * CBS;
            bulk_g2s(dst, src, (uint32_t)(cols * CBS * 4), &full[buf]);
          }
          cbase += n_cp;
        }
        for (int cc = first_mine(cbase); cc < cbase + n_wblk; cc += 32 * kProdWarps) {
          const int c = cc - cbase;
          // storage block J = jb0 / SUB + c of the blocked kernel
          const float* src = p.w + ((int64_t)(jb0 / SUB + c) * p.ib_n + ib0) * p.slab_floats +
                             (int64_t)n0 * p.w_f * CBS * CBS;
          bulk_g2s(sw + wchunk<TCO>(c, p.wstride_floats), src, wbytes, &full[buf]);
        }
        if (kFfmaProf && p.dbg && pt == 0 && gs == 0) p.dbg[blockIdx.x * 16 + 9] = clock64() - t_start;
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  if constexpr (NW == 8) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 192;");
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 152;");
  }
  const int wr = warp % WPG, wc = warp / WPG;
  const int pg = wr * PPW + (lane % PPW);
  const int cb = (wc * CPW + lane / PPW) * NBLK;  // first output block within the CTA tile

  const uint32_t tmem_base = tmem_on ? *tmem_slot : 0u;
  if (kFfmaProf && p.dbg && tid == 0) p.dbg[blockIdx.x * 16 + 1] = clock64() - t_start;  // setup done
  const uint32_t taddr = tmem_base + ((uint32_t)((warp & 3) * 32) << 16) +
                         (uint32_t)((warp >> 2) * TPX * TCO);
  const int wf = WF > 0 ? WF : p.w_f;

  int gs = 0, unit_iter = 0;
  int rbuf = 0;            // ring slot of stage gs (gs % NS)
  uint32_t rphase = 0u;    // its full-barrier phase ((gs / NS) & 1)
  int wu_iter = 0;  // units handed to the epilogue warpgroup (all but stream-K contributor pieces)
  Pieces pieces = make_pieces();
  for (int u, st0, st1; pieces.next(u, st0, st1); ++unit_iter) {  // (shadow the rank's range)
    const bool whole = !p.streamk || (st0 == 0 && st1 == S);
    // stream-K boundary pieces: 1 = last stages of a unit begun by the
    // previous CTA (store the raw partial tile into the output map, raise
    // this CTA's flag), 2 = first stages of a unit continued by the next CTA
    // (wait for its flag, add its partial, run the epilogue), 3 = middle
    // stages (fewer units than SMs: a unit spans three or more CTAs): wait,
    // add, store the raw sum back, raise the flag
    const int sk_mode = whole ? 0 : (st0 > 0 ? (st1 < S ? 3 : 1) : 2);
    TileRows tr{};
    int tx0 = 0, jb0 = 0, cg_valid = 0;
    // dense 1x1 tiles handed to the epilogue warpgroup need no tile geometry
    // in the compute warps: pixels are addressed from one pointer and the
    // epilogue warps decode the unit themselves (short-K units: the decode's
    // divisions were ~10% of a 64-channel unit)
    const bool geom = !(WF == 1 && p.dense1x1 && p.epi_wg && whole);
    if (geom) decode(u, tr, tx0, jb0, cg_valid);
    // per-pixel patch offsets of this tile (pixels that do not exist read
    // offset 0 and are never stored)
    int poff[TPX];
#pragma unroll
    for (int k = 0; k < TPX; ++k) poff[k] = 0;
    if (geom && !(WF == 1 && p.dense1x1))  // dense 1x1 tiles address pixels from one pointer
#pragma unroll
    for (int k = 0; k < TPX; ++k) {
      const int q = pg + PG * k;
      const int ty = (int)__umulhi((unsigned)q, p.tw_magic), tx = q - ty * p.TW;
      int img, y, prow;
      tile_row(p, tr, ty, img, y, prow);
      poff[k] = (ty < tr.th && tx0 + tx < p.w_o) ? (prow * p.PW + tx * p.s) * CBS : 0;
    }
    uint64_t acc[TPX][TCO / 2];
#pragma unroll
    for (int k = 0; k < TPX; ++k)
#pragma unroll
      for (int c = 0; c < TCO / 2; ++c) acc[k][c] = 0ull;
    bool have_total = false;
    // per-stage bookkeeping by counters, not divisions (scalar work in this
    // loop showed up in the headline: a modulo per stage cost 1%)
    int fold_in = p.flush_every;  // stages until the next TMEM fold
    int g = st0 / p.n_r, r = st0 - g * p.n_r;

    for (int st = st0; st < st1; ++st, ++gs) {
      const int buf = rbuf;
      if (kFfmaProf && p.dbg && tid == 0 && gs == 0) p.dbg[blockIdx.x * 16 + 10] = clock64() - t_start;
      mbar_wait(&full[buf], rphase);
      if (++rbuf == p.NS) { rbuf = 0; rphase ^= 1u; }
      if (kFfmaProf && p.dbg && tid == 0 && gs == 0) p.dbg[blockIdx.x * 16 + 2] = clock64() - t_start;
      if (st > st0 && ++r == p.n_r) { r = 0; ++g; }
      const int Ge = min(p.G, p.ib_n - g * p.G);
      const int Re = min(p.R, p.h_f - r * p.R);
      const float* sp = smem + buf * p.stage_floats;
      // this thread's output sub-block cb: weight chunk of storage block
      // cb / SUB, column offset (cb % SUB) * 8 in its CBS-wide rows
      const float* sw = sp + p.patch_floats + wchunk<TCO>(cb / SUB, p.wstride_floats) +
                        (cb % SUB) * kCB;
      const int sw2 = NBLK > 1 ? wchunk<TCO>(cb + 1, p.wstride_floats) - wchunk<TCO>(cb, p.wstride_floats) : 0;
      // per-pixel patch pointers once per stage; rows and taps then add a
      // warp-uniform offset (measured +1%; swapping the channel-half order
      // between warpgroups to de-phase their LDS bubbles measured -2.5%).
      const float* pk[TPX];
#pragma unroll
      for (int k = 0; k < TPX; ++k) pk[k] = sp + poff[k];
      // one filter tap of one input block: 8 channels x (8 px x TCO ch)
      // c_b = 32: a pixel is one 128-byte pencil, so the 4 lanes of a
      // quarter-warp that read 4 pixels' same channel quarter hit one bank
      // group; odd lanes take the two channel halves in the other order
      // (activations 2-way instead of 4-way, weights 2-way instead of none)
      // 8 x 4 warp shape: a quarter-warp reads 8 pixels 32 B apart (two
      // bank rows); lanes 4-7 of it take the channel halves in the other order
      // so its 16-byte reads land on 8 distinct bank groups
      const int hswap = CBS == 32 ? (lane & 1) : (PPW == 8 ? ((lane >> 2) & 1) : 0);
      // dense (1x1/s1 tiles no wider than the map): the staged patch is the
      // tile itself, pixel q at q * CBS floats, so a thread's TPX pixels sit
      // at compile-time offsets from ONE pointer (pd): no per-pixel address
      // arithmetic per input block (it cost the 1x1 loop ~8%: ncu source
      // page, profiles/r2_ncu_src_1x1.txt)
      const float* pd = sp + pg * CBS;
      auto tap = [&](const float* pw, int aoff, auto dense) {
#pragma unroll
        for (int half_i = 0; half_i < 8 / AV; ++half_i) {
          const int half = half_i ^ hswap;
          float a[TPX][AV];
#pragma unroll
          for (int k = 0; k < TPX; ++k) {
            const float* pa = decltype(dense)::value ? pd + k * (PG * CBS) : pk[k];
            if constexpr (AV == 4) {
              const float4 t = lds128(pa + aoff + half * 4);
              a[k][0] = t.x; a[k][1] = t.y; a[k][2] = t.z; a[k][3] = t.w;
            } else {
              const float2 t = *reinterpret_cast<const float2*>(pa + aoff + half * 2);
              a[k][0] = t.x; a[k][1] = t.y;
            }
          }
#pragma unroll
          for (int i4 = 0; i4 < AV; ++i4) {
#pragma unroll
            for (int bb = 0; bb < NBLK; ++bb) {
              const float* pb = pw + bb * sw2 + (half * AV + i4) * CBS;
              const float4 b0 = lds128(pb);
              const float4 b1 = lds128(pb + 4);
              uint64_t bp[4];
              bp[0] = pack2(b0.x, b0.y);
              bp[1] = pack2(b0.z, b0.w);
              bp[2] = pack2(b1.x, b1.y);
              bp[3] = pack2(b1.z, b1.w);
#pragma unroll
              for (int c = 0; c < 4; ++c)
#pragma unroll
                for (int k = 0; k < TPX; ++k) ffma2(acc[k][bb * 4 + c], a[k][i4], bp[c]);
            }
          }
        }
      };
      if (WF == 1 && Re == 1) {
        // 1x1 filters: a stage is Ge input blocks of one tap each; unrolled
        // so the accumulators stay put across blocks (no register rotation)
        const int gstride = p.PH * p.PW * CBS, wgstride = p.R * CBS * CBS;
        if (p.dense1x1) {
#pragma unroll 4
          for (int gi = 0; gi < Ge * SUB; ++gi)  // 8-channel input sub-blocks
            tap(sw + (gi / SUB) * wgstride + (gi % SUB) * kCB * CBS,
                (gi / SUB) * gstride + (gi % SUB) * kCB, std::true_type{});
        } else {
#pragma unroll 4
          for (int gi = 0; gi < Ge * SUB; ++gi)
            tap(sw + (gi / SUB) * wgstride + (gi % SUB) * kCB * CBS,
                (gi / SUB) * gstride + (gi % SUB) * kCB, std::false_type{});
        }
      } else {
        for (int gi = 0; gi < Ge; ++gi) {
#pragma unroll 1
          for (int sb = 0; sb < SUB; ++sb) {  // 8-channel input sub-blocks
            for (int n = 0; n < Re; ++n) {
              const int row_off = ((gi * p.PH + n) * p.PW) * CBS + sb * kCB;
              const float* pw_row = sw + ((gi * p.R + n) * wf) * (CBS * CBS) + sb * kCB * CBS;
#pragma unroll(WF > 0 ? WF : 1)
              for (int m = 0; m < wf; ++m) tap(pw_row + m * (CBS * CBS), row_off + m * CBS, std::false_type{});
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[buf]);
      // fold the partial sum into the TMEM running total every flush_every
      // stages (never after the last stage: the epilogue folds it)
      if (use_tmem && --fold_in == 0 && st + 1 < st1) {
        fold_in = p.flush_every;
        tmem_fold<NP>(taddr, &acc[0][0], have_total, true);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        have_total = true;
#pragma unroll
        for (int k = 0; k < TPX; ++k)
#pragma unroll
          for (int c = 0; c < TCO / 2; ++c) acc[k][c] = 0ull;
      }
    }
    if (kFfmaProf && p.dbg && tid == 0) p.dbg[blockIdx.x * 16 + 3] = clock64() - t_start;  // loop end
    if (sk_mode >= 2) {
      // stream-K finisher (or middle piece): the next CTA stored this unit's later-stage
      // partial tile into the output map first thing; add it to the
      // registers (first stages + later stages, in that order) and go on as
      // for a whole unit.  The flag is cleared for the next launch.
      if (tid == 0) {
        unsigned f;
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(p.sk_flags + blockIdx.x + 1) : "memory");
        } while (f == 0u);
        asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p.sk_flags + blockIdx.x + 1), "r"(0u) : "memory");
      }
      asm volatile("bar.sync 1, %0;" ::"n"(NW * 32) : "memory");
#pragma unroll
      for (int bb = 0; bb < NBLK; ++bb) {
        if (cb + bb >= cg_valid) continue;
        const int jl = jb0 + cb + bb - p.jb_begin;
#pragma unroll
        for (int k4 = 0; k4 < TPX; k4 += 4) {
          float4 t[8];
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const int q = pg + PG * (k4 + kk);
            const int ty = (int)__umulhi((unsigned)q, p.tw_magic), tx = q - ty * p.TW;
            const int x = tx0 + tx;
            t[2 * kk] = t[2 * kk + 1] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (ty < tr.th && x < p.w_o) {
              int img, y, prow;
              tile_row(p, tr, ty, img, y, prow);
              const float4* o = reinterpret_cast<const float4*>(
                  p.out + sub_off<CBS>(jl, p.out_blk) + (int64_t)img * p.out_img +
                  (int64_t)y * p.out_row + (int64_t)x * CBS);
              t[2 * kk] = __ldcg(o);
              t[2 * kk + 1] = __ldcg(o + 1);
            }
          }
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            uint64_t* a = acc[k4 + kk] + bb * 4;
            a[0] = fadd2(a[0], pack2(t[2 * kk].x, t[2 * kk].y));
            a[1] = fadd2(a[1], pack2(t[2 * kk].z, t[2 * kk].w));
            a[2] = fadd2(a[2], pack2(t[2 * kk + 1].x, t[2 * kk + 1].y));
            a[3] = fadd2(a[3], pack2(t[2 * kk + 1].z, t[2 * kk + 1].w));
          }
        }
      }
    }
    if (p.epi_wg && (sk_mode == 0 || sk_mode == 2)) {
      // hand the finished tile to the epilogue warpgroup (TMEM result buffer
      // wu_iter & 1) and go on with the next unit
      const int rb = wu_iter & 1;
      if (wu_iter >= 2) mbar_wait(&res_empty[rb], ((wu_iter >> 1) - 1) & 1);
      ++wu_iter;
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      tmem_finalize<NP>(taddr, taddr + (uint32_t)(kResCols * (1 + rb)), &acc[0][0], have_total);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&res_full[rb]);
      continue;
    }
    if (have_total) tmem_fold<NP>(taddr, &acc[0][0], true, false);

    // ------------------------------------------------------------ epilogue
    // Split-K: every rank publishes its partial tile in its own smem, then
    // rank r sums pixels [r*8/ks, (r+1)*8/ks) of every thread's 8x8 tile over
    // ranks 0..ks-1 in that fixed order (deterministic, no global workspace).
    // pixel k of this thread, output block jl of the view: skip-add, ReLU,
    // one pencil store (+ the same pencil into every peer's map)
    auto emit = [&](int k, int jl, float (&v)[8]) {
      const int q = pg + PG * k;
      const int ty = (int)__umulhi((unsigned)q, p.tw_magic), tx = q - ty * p.TW;
      const int x = tx0 + tx;
      if (ty >= tr.th || x >= p.w_o) return;
      int img, y, prow;
      tile_row(p, tr, ty, img, y, prow);
      float* o = p.out + sub_off<CBS>(jl, p.out_blk) + (int64_t)img * p.out_img +
                 (int64_t)y * p.out_row + (int64_t)x * CBS;
      if (sk_mode & 1) {  // raw partial tile, finished by the previous CTA
#pragma unroll
        for (int c = 0; c < 8; c += 4)
          __stcg(reinterpret_cast<float4*>(o + c), make_float4(v[c], v[c + 1], v[c + 2], v[c + 3]));
        return;
      }
      if (p.epi & DCONV_EPI_ADD) {
        const float* sk = p.skip + sub_off<CBS>(jl, p.sk_blk) + (int64_t)img * p.sk_img +
                          (int64_t)y * p.sk_row + (int64_t)x * CBS;
        float4 s0, s1;
        ldg_pencil(sk, s0, s1);
        v[0] += s0.x; v[1] += s0.y; v[2] += s0.z; v[3] += s0.w;
        v[4] += s1.x; v[5] += s1.y; v[6] += s1.z; v[7] += s1.w;
      }
      if (p.epi & DCONV_EPI_RELU) {
#pragma unroll
        for (int c = 0; c < 8; ++c) v[c] = fmaxf(v[c], 0.f);
      }
      DCONV_OWN(o, 8);
      stg_pencil(o, v);
      // fused C_o-shard gather: the same pencil into every peer's map
      for (int pi = 0; pi < p.n_peers; ++pi) stg_pencil(p.peer_out[pi] + (o - p.out), v);
    };

    if (TCO == 8 && ks > 1) {
      // Split-K, push model: a thread's tile is 16 items (pixel k, channel
      // half); item i belongs to rank owner(i) (ranks own contiguous item
      // ranges [i*ks/16 ...]).  Every rank stores its partial of item i
      // straight into the owner's smem slot [source rank][slot] (remote
      // st.shared::cluster, fire-and-forget), then each owner sums its slots
      // locally in rank order 0..ks-1: deterministic, no global workspace,
      // and no remote-load latency on the critical path.
      constexpr int kItems = 2 * TPX;
      const int ipo = (kItems + ks - 1) / ks;  // items per owner, at most
      const bool last_unit = u + n_clusters >= n_units;  // cluster-uniform
      // owners must have read the previous unit before we overwrite
      if (unit_iter == 0) cluster_wait_acquire();
      if (unit_iter > 0) mbar_wait_cluster(done, (unit_iter - 1) & 1);
#pragma unroll
      for (int i = 0; i < kItems; ++i) {
        const int k = i >> 1, hf = i & 1;
        const int owner = ((i + 1) * ks + kItems - 1) / kItems - 1;
        const int slot = i - owner * kItems / ks;
        const float2 a = unpack2(acc[k][2 * hf]), b = unpack2(acc[k][2 * hf + 1]);
        st_dsmem4(red + ((rank * ipo + slot) * (NW * 32) + tid) * 4, owner,
                  make_float4(a.x, a.y, b.x, b.y));
      }
      // every compute warp's stores issued: one fence, ks relaxed arrives
      asm volatile("bar.sync 1, %0;" ::"n"(NW * 32) : "memory");
      if (kFfmaProf && p.dbg && tid == 0) p.dbg[blockIdx.x * 16 + 4] = clock64() - t_start;  // published
      if (tid == 0) {
        fence_cluster();
        for (int q = 0; q < ks; ++q) mbar_arrive_remote_relaxed(ready, q);
      }
      mbar_wait_cluster(ready, unit_iter & 1);
      if (kFfmaProf && p.dbg && tid == 0) p.dbg[blockIdx.x * 16 + 5] = clock64() - t_start;  // all ready
      if (cb < cg_valid) {
        const int jl = jb0 + cb - p.jb_begin;
        const int i_lo = rank * kItems / ks, i_hi = (rank + 1) * kItems / ks;
#pragma unroll 1
        for (int i = i_lo; i < i_hi; ++i) {
          float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
          const float* rp = red + ((i - i_lo) * (NW * 32) + tid) * 4;
#pragma unroll 4
          for (int src = 0; src < ks; ++src) {
            const float4 t = lds128(rp + src * ipo * (NW * 32) * 4);
            v.x += t.x; v.y += t.y; v.z += t.z; v.w += t.w;
          }
          // pixel i/2, channels (i&1)*4 .. +3
          const int k = i >> 1, hf = i & 1;
          const int q = pg + PG * k;
          const int ty = (int)__umulhi((unsigned)q, p.tw_magic), tx = q - ty * p.TW;
          const int x = tx0 + tx;
          if (ty >= tr.th || x >= p.w_o) continue;
          int img, y, prow;
          tile_row(p, tr, ty, img, y, prow);
          if (p.epi & DCONV_EPI_ADD) {
            const float4 s4 = __ldg(reinterpret_cast<const float4*>(
                p.skip + sub_off<CBS>(jl, p.sk_blk) + (int64_t)img * p.sk_img +
                (int64_t)y * p.sk_row + (int64_t)x * CBS + hf * 4));
            v.x += s4.x; v.y += s4.y; v.z += s4.z; v.w += s4.w;
          }
          if (p.epi & DCONV_EPI_RELU) {
            v.x = fmaxf(v.x, 0.f); v.y = fmaxf(v.y, 0.f);
            v.z = fmaxf(v.z, 0.f); v.w = fmaxf(v.w, 0.f);
          }
          const int64_t off = sub_off<CBS>(jl, p.out_blk) + (int64_t)img * p.out_img +
                              (int64_t)y * p.out_row + (int64_t)x * CBS + hf * 4;
          DCONV_OWN(p.out + off, 4);
          *reinterpret_cast<float4*>(p.out + off) = v;
          for (int pi = 0; pi < p.n_peers; ++pi)
            *reinterpret_cast<float4*>(p.peer_out[pi] + off) = v;
        }
      }
      if (kFfmaProf && p.dbg && tid == 0) p.dbg[blockIdx.x * 16 + 6] = clock64() - t_start;  // reduced
      if (!last_unit) {
        // every compute warp has read its slots: the ranks may publish again
        asm volatile("bar.sync 1, %0;" ::"n"(NW * 32) : "memory");
        if (tid == 0) {
          fence_cluster();
          for (int q = 0; q < ks; ++q) mbar_arrive_remote_relaxed(done, q);
        }
      }
    } else if (p.epi & DCONV_EPI_MAXPOOL) {
      // fused ReLU + 2x2/s2 max-pool: vertical partner in-thread (pixel
      // k + TW/PG), horizontal partner in lane ^ 1; the even-column lane
      // stores the pooled pencil (windows are all valid or all invalid:
      // even h_o, w_o and tile origins)
      const int kv = p.TW / PG;
      const int jl = jb0 + cb - p.jb_begin;
      auto pool_pair = [&](int k, int k2) {
        float v[8];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float2 a = unpack2(acc[k][c]), b = unpack2(acc[k2][c]);
          v[2 * c] = fmaxf(a.x, b.x);
          v[2 * c + 1] = fmaxf(a.y, b.y);
        }
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          v[c] = fmaxf(v[c], __shfl_xor_sync(0xffffffffu, v[c], 1));
          if (p.epi & DCONV_EPI_RELU) v[c] = fmaxf(v[c], 0.f);
        }
        const int q = pg + PG * k;
        const int ty = (int)__umulhi((unsigned)q, p.tw_magic), tx = q - ty * p.TW;
        const int x = tx0 + tx;
        if (cb >= cg_valid || (tx & 1) || ty >= tr.th || x >= p.w_o) return;
        int img, y, prow;
        tile_row(p, tr, ty, img, y, prow);
        float* o = p.out + sub_off<CBS>(jl, p.out_blk) + (int64_t)img * p.out_img +
                   (int64_t)(y >> 1) * p.out_row + (int64_t)(x >> 1) * CBS;
        DCONV_OWN(o, 8);
        *reinterpret_cast<float4*>(o) = make_float4(v[0], v[1], v[2], v[3]);
        *reinterpret_cast<float4*>(o + 4) = make_float4(v[4], v[5], v[6], v[7]);
      };
      if (kv == 1) {
#pragma unroll
        for (int k = 0; k < TPX; k += 2) pool_pair(k, k + 1);
      } else if (kv == 2) {
#pragma unroll
        for (int k = 0; k < TPX; ++k)
          if ((k & 2) == 0) pool_pair(k, k + 2);
      } else {
#pragma unroll
        for (int k = 0; k < TPX; ++k)
          if ((k & 4) == 0 && k + 4 < TPX) pool_pair(k, k + 4);
      }
    } else {
#pragma unroll
      for (int bb = 0; bb < NBLK; ++bb) {
        if (cb + bb >= cg_valid) continue;
        const int jl = jb0 + cb + bb - p.jb_begin;  // block index within the output view
#pragma unroll
        for (int k = 0; k < TPX; ++k) {
          float v[8];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const float2 f = unpack2(acc[k][bb * 4 + c]);
            v[2 * c] = f.x;
            v[2 * c + 1] = f.y;
          }
          emit(k, jl, v);
        }
      }
      if (sk_mode & 1) {
        // partial tile stored: publish it to the finishing CTA
        __threadfence();
        asm volatile("bar.sync 1, %0;" ::"n"(NW * 32) : "memory");
        if (tid == 0)
          asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p.sk_flags + blockIdx.x), "r"(1u) : "memory");
      }
    }
  }
  // (push model: every remote access to this CTA's smem -- the peers'
  // partial stores and arrives -- completes before its last `ready` wait, so
  // no exit barrier is needed)
  if (kFfmaProf && p.dbg && tid == 0) {
    p.dbg[blockIdx.x * 16 + 7] = clock64() - t_start;  // exit
    p.dbg[blockIdx.x * 16 + 11] = (long long)globaltimer_ns();
  }

  if (tmem_on) {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    // every compute and epilogue warp is done with TMEM before warp 0 frees it
    asm volatile("bar.sync 2, %0;" ::"n"((NW + 4) * 32) : "memory");
    if (warp == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "r"(tmem_cols));
    }
  }
}

// Rows of the stacked patch for a tile starting at output row y0 of an image
// (segment layout of tile_row), with R filter rows per stage.
int patch_rows(int y0, int th, int h_o, int s, int R) {
  const int cnt0 = std::min(h_o - y0, th);
  int rows = (cnt0 - 1) * s + R, rest = th - cnt0;
  while (rest > 0) {
    const int c = std::min(h_o, rest);
    rows += (c - 1) * s + R;
    rest -= c;
  }
  return rows;
}

int max_patch_rows(const FfmaParams& p, int R) {
  // every tile start residue that occurs (vy0 = tile_y * TH)
  int best = 0;
  const int vh = p.n * p.h_o;
  for (int vy0 = 0, seen = 0; vy0 < vh && seen <= p.h_o; vy0 += p.TH, ++seen)
    best = std::max(best, patch_rows(vy0 % p.h_o, std::min(p.TH, vh - vy0), p.h_o, p.sy, R));
  return best;
}

// Tile selector: pixel-tile width TW (powers of two, or the map width and its
// halves/thirds), TH = BM / TW rows of the stacked batch.  Score = useful
// pixels / launched pixel-slots, where the launch takes floor(units/sms)
// full waves plus a ragged tail that the tail-split launch finishes in about
// 1/2, 1/4 or 1/8 of a wave when it fits on sms/2, /4, /8 clusters -- divided
// by how far the producer's bulk copies (one per patch row and input block,
// ~kCopyCycles each, measured) outrun the unit's FFMA2 time: narrow tiles of
// 1x1 layers are copy-bound (TW = 4 on a 56-wide map ran at 16 TFLOP/s).
// Ties go to the smaller patch.
double tail_rounds(int64_t units, int sms) {
  const int64_t full = units / sms, tail = units - full * sms;
  double t = 0.0;
  if (tail > 0) {
    if (full == 0) {
      // fewer units than SMs: one split-K launch over clusters of ks CTAs
      // (co-resident clusters ~ sms/2, sms/4 - 1, sms/8 - 2)
      t = 1.0;
      if (tail * 8 <= sms - 16) t = 0.125 + 0.4;
      else if (tail * 4 <= sms - 4) t = 0.25 + 0.2;
      else if (tail * 2 <= sms) t = 0.5 + 0.1;
    } else if (tail * 8 <= sms / 2) t = 0.125 + 0.05;
    else if (tail * 4 <= sms) t = 0.25 + 0.05;
    else if (tail * 2 <= sms) t = 0.5 + 0.05;
    else t = 1.0;
    // stream-K balances a ragged tail over all SMs (stage granularity and
    // the boundary pieces cost ~0.1 of a unit)
    if (full > 0) t = std::min(t, (double)tail / sms + 0.1);
  }
  return (double)full + t;
}

constexpr double kCopyCycles = 50.0;     // per bulk copy (row of one input block)
constexpr double kFfmaPerCycle = 102.0;  // FMA / cycle / SM sustained (80% of 128)
constexpr double kUnitOverhead = 1500.0; // per-unit prologue + epilogue, cycles
constexpr double kLaunchFill = 2500.0;   // first stage in flight, cycles

// One unit's FFMA2 cycles (BM x BN outputs x the whole reduction) + overhead.
double unit_cycles(const FfmaParams& p, int BM, int BN) {
  return (double)BM * BN * p.ib_n * p.cbs * p.h_f * p.w_f / kFfmaPerCycle + kUnitOverhead;
}

// Few units (< SMs): every unit's K range split over a cluster of ks CTAs,
// ceil(units / slots[ks]) rounds of (unit / ks + DSMEM reduction).
double split_cycles(int64_t units, int ks, int slots, double unit) {
  const double rounds = (double)((units + slots - 1) / slots);
  const double red = ks > 1 ? 1500.0 + 300.0 * ks : 0.0;
  return rounds * (unit / ks + red) + kLaunchFill;
}

// Cheapest split factor for `units` (< SMs) given the co-resident cluster
// counts slots[ks] (slots[1] = SMs); ks <= max_ks (stages to split).
int best_split(int64_t units, const int* slots, int max_ks, double unit, double* cycles) {
  int best = 1;
  double best_c = split_cycles(units, 1, slots[1], unit);
  for (int ks = 2; ks <= kMaxKs && ks <= max_ks; ++ks) {
    if (slots[ks] < 1) continue;
    const double c = split_cycles(units, ks, slots[ks], unit);
    if (c < best_c - 1e-9) {
      best_c = c;
      best = ks;
    }
  }
  if (cycles) *cycles = best_c;
  return best;
}

void pick_tile(FfmaParams& p, int BM, int BN, int co_groups, int sms, const int* slots,
               bool allow_split) {
  int cand[16], nc = 0;
  const int PG = BM / 8;  // pixel groups (8 px per thread)
  if (p.epi & DCONV_EPI_MAXPOOL) {
    // fused 2x2 pool: a thread's vertical window partner is pixel k + TW/PG
    // (TW a multiple of PG, TH even), the horizontal one is lane ^ 1
    for (int tw = PG; tw <= 128 && tw <= BM / 2; tw *= 2)
      if ((BM / tw) % 2 == 0) cand[nc++] = tw;
  } else {
    for (int tw = 4; tw <= 128 && tw <= BM; tw *= 2) cand[nc++] = tw;
    for (int d = 1; d <= 4; ++d) {
      const int tw = (p.w_o + d - 1) / d;
      if (tw >= 2 && tw <= BM && tw <= 128) cand[nc++] = tw;
    }
  }
  double best_score = -1;
  int64_t best_patch = 0;
  const int64_t vh = (int64_t)p.n * p.h_o;
  const double unit = unit_cycles(p, BM, BN);
  FfmaParams q = p;
  for (int i = 0; i < nc; ++i) {
    const int tw = cand[i], th = BM / tw;
    const int64_t ty = (vh + th - 1) / th, tx = (p.w_o + tw - 1) / tw;
    const int64_t units = ty * tx * co_groups;
    double cycles;
    if (units < sms && allow_split)
      best_split(units, slots, p.ib_n, unit, &cycles);
    else
      cycles = tail_rounds(units, sms) * unit + kLaunchFill;
    q.TH = th;
    q.TW = tw;
    const double rows = max_patch_rows(q, p.h_f);
    // producer copies per input block vs FFMA2 cycles per input block
    const double copy_ratio = kCopyCycles * rows /
                              ((double)BM * BN * p.cbs * p.h_f * p.w_f / kFfmaPerCycle);
    const double score = 1.0 / (cycles * std::max(1.0, copy_ratio));
    const int64_t patch = (int64_t)((std::min<int64_t>(th, vh) - 1) * p.sy + p.h_f) *
                          ((std::min(tw, p.w_o) - 1) * p.s + p.w_f);
    static const int force_tw = getenv("DCONV_FORCE_TW") ? atoi(getenv("DCONV_FORCE_TW")) : 0;
    if (force_tw && tw != force_tw) continue;  // tuning experiments only
    if (score > best_score * (1 + 1e-9) ||
        (score > best_score * (1 - 1e-9) && patch < best_patch)) {
      best_score = score;
      best_patch = patch;
      p.TH = th;
      p.TW = tw;
      p.tiles_y = (int)ty;
      p.tiles_x = (int)tx;
    }
  }
}

// Stage geometry for split factor ks: G input blocks x R filter rows per
// stage under a 40 KB weight / 32 KB patch budget (G = 1 when `fine`: few
// units, or split-K whose 64 KB partial buffer shares smem with the ring),
// NS ring depth, TMEM fold interval.  Returns the dynamic smem bytes, or 0 if
// two stages do not fit.
template <int BN, int NW, int TPX, int TCO, int CBS>
size_t configure(FfmaParams& p, int ks, bool fine) {
  constexpr int CG = BN / CBS;  // weight chunks (output storage blocks) per stage
  // patch budget: 1x1 layers stage twice the input blocks per stage (their
  // stages are short: one tap per block; ResNet-50 256->64 at 56x56 +17%)
  static const int patch_kb = getenv("DCONV_PATCH_BUDGET") ? atoi(getenv("DCONV_PATCH_BUDGET")) : 0;
  const int kWeightBudget = 40 * 1024;
  const int kPatchBudget = (patch_kb ? patch_kb : (p.h_f * p.w_f == 1 ? 64 : 32)) * 1024;
  const int full_taps_bytes = CG * p.h_f * p.w_f * CBS * CBS * 4;
  if (full_taps_bytes <= kWeightBudget) {
    p.R = p.h_f;
    p.PH = max_patch_rows(p, p.R);
    const int patch1 = p.PH * p.PW * CBS * 4;
    p.G = std::max(1, std::min(kWeightBudget / full_taps_bytes,
                               kPatchBudget / std::max(1, patch1)));
    p.G = std::min(p.G, p.ib_n);
    if (fine || ks > 1) {
      // finer stages (split-K shares smem with its 64 KB partial buffer):
      // keep each stage <= 36 KB so the ring stays >= 4 deep; 1x1 layers
      // still group several input blocks per stage
      const int per_block = patch1 + CG * p.R * p.w_f * CBS * CBS * 4;
      p.G = std::max(1, std::min(p.G, (36 * 1024) / per_block));
    }
    // 1x1 layers: the consumers' block loop is unrolled by 4 (its remainder
    // loop rotates the accumulators through 28 MOVs per block)
    if (p.h_f * p.w_f == 1 && CBS == 8 && p.G > 4) p.G &= ~3;
    if (knobs().force_g) p.G = std::max(1, std::min(p.ib_n, knobs().force_g));
  } else {
    p.G = 1;
    p.R = std::max(1, kWeightBudget / (CG * p.w_f * CBS * CBS * 4));
    p.R = std::min(p.R, p.h_f);
    p.PH = max_patch_rows(p, p.R);
  }
  p.n_g = (p.ib_n + p.G - 1) / p.G;
  p.n_r = (p.h_f + p.R - 1) / p.R;
  p.patch_floats = p.G * p.PH * p.PW * CBS;
  // +16 B per block chunk: the 8 lanes of a warp that read different output
  // blocks hit distinct 16-byte bank groups of the weight stage.
  p.wstride_floats = p.G * p.R * p.w_f * CBS * CBS + (TCO == 8 ? 4 : 0);
  p.stage_floats = (p.patch_floats + wchunk<TCO>(CG, p.wstride_floats) + 31) & ~31;  // 128 B aligned
  const int S = p.n_g * p.n_r;
  const int kSmemBudget = 220 * 1024;
  const int bar_bytes = (2 * kMaxStages + 6) * 8 + 16;
  // split-K slots: ks sources x ceil(16 / ks) items x 4 floats per thread
  const int red_bytes = ks * ((2 * TPX + ks - 1) / ks) * NW * 32 * 16;
  p.ksplit = ks;
  p.red_floats = ks > 1 ? red_bytes / 4 : 0;
  const int ring_budget = kSmemBudget - bar_bytes - (ks > 1 ? red_bytes : 0);
  p.NS = std::min(kMaxStages, ring_budget / (p.stage_floats * 4));
  // the ring spans unit boundaries (the producer prefetches the next unit), so
  // its depth is set by shared memory alone, not by the stages per unit
  // partial sums cover >= 256 products before folding into the TMEM total
  const int k_stage = p.G * p.R * p.w_f * CBS;
  p.flush_every = std::max(1, (256 + k_stage - 1) / k_stage);
  if (knobs().flush_every) p.flush_every = std::max(1, knobs().flush_every);
  if (p.NS < 2) return 0;
  // 1x1/s1 tiles no wider than the map: the patch is the tile itself (tile
  // row r = patch row r, PW = TW), so the consumers address a thread's pixels
  // from one pointer.  Pixels past the tile's last row read on into the
  // stage (never stored): the stage must hold BM pixels from the last block.
  constexpr int BM = NW * 32 * TPX * TCO / BN;
  static const bool no_dense = getenv("DCONV_NO_DENSE1X1") != nullptr;
  p.dense1x1 = (!no_dense && p.h_f == 1 && p.w_f == 1 && p.s == 1 && p.sy == 1 && p.TWe == p.TW &&
                p.PW == p.TW &&
                (p.G - 1) * p.PH * p.PW * CBS + BM * CBS <= p.stage_floats) ? 1 : 0;
  return (size_t)p.NS * p.stage_floats * 4 + (ks > 1 ? red_bytes : 0) + bar_bytes;
}

// co-resident clusters of ks CTAs at ~200 KB smem (GPC-limited).  Cached per
// (device, kernel instantiation, ks): every conv_ffma_kernel<...> has its own
// register / smem footprint, so the occupancy answer of one must not be
// reused for another.
int device_index() { return dconv_host::current_device(); }

template <class K>
int cluster_slots(K kernel, int ks, int sms, int threads) {
  if (ks == 1) return sms;
  struct Entry {
    int dev;
    const void* fn;
    int ks, n;
  };
  static std::mutex mu;
  static std::vector<Entry> cache;
  const int dev = device_index();
  const void* fn = reinterpret_cast<const void*>(kernel);
  {
    std::lock_guard<std::mutex> lock(mu);
    for (const Entry& e : cache)
      if (e.dev == dev && e.fn == fn && e.ks == ks) return e.n;
  }
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = ks;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(ks * 64);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = 200 * 1024;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kernel, &cfg) != cudaSuccess || n < 1) {
    cudaGetLastError();
    n = -1;
  }
  std::lock_guard<std::mutex> lock(mu);
  cache.push_back({dev, fn, ks, n});
  return n;
}

template <class K>
int launch_units(K kernel, int threads, FfmaParams p, size_t smem, int unit_begin,
                 int unit_count, int clusters, cudaStream_t stream) {
  p.unit_begin = unit_begin;
  p.unit_count = unit_count;
  // epilogue warpgroup hand-off for whole-K units (split-K reduces in the
  // compute warps; the fused pool pairs pixels across lanes there)
  static const bool no_epi_wg = getenv("DCONV_NO_EPI_WG") != nullptr;
  p.epi_wg = (p.ksplit == 1 && !(p.epi & DCONV_EPI_MAXPOOL) && !no_epi_wg) ? 1 : 0;
  // the epilogue warpgroup hides the skip reads behind the next tile; a
  // producer L2 prefetch would cost a bulk op per 256-B skip row and make
  // the single producer warp the bottleneck (measured on 1x1 layers)
  if (p.epi_wg) p.skip_prefetch = 0;
  static const bool prof = kFfmaProf && getenv("DCONV_FFMA_PROFILE") != nullptr;  // profiling builds only
  if (prof) {  // debugging aid: per-CTA phase clocks of one extra launch
    const int grid = p.ksplit == 1 ? clusters : clusters * p.ksplit;
    cudaMalloc(&p.dbg, (size_t)grid * 16 * 8);
    cudaMemset(p.dbg, 0, (size_t)grid * 16 * 8);
    if (p.ksplit == 1) {
      kernel<<<clusters, threads, smem, stream>>>(p);
    } else {
      cudaLaunchConfig_t cfg{};
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = p.ksplit;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(threads);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = stream;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, kernel, p);
    }
    std::vector<long long> h((size_t)grid * 16);
    cudaMemcpy(h.data(), p.dbg, h.size() * 8, cudaMemcpyDeviceToHost);
    double a[16] = {};
    long long g0 = h[0], g1 = h[11], gmax0 = h[0];
    for (int b = 0; b < grid; ++b) {
      for (int i = 1; i < 16; ++i) a[i] += h[b * 16 + i];
      g0 = std::min(g0, h[b * 16]);
      gmax0 = std::max(gmax0, h[b * 16]);
      g1 = std::max(g1, h[b * 16 + 11]);
    }
    for (double& v : a) v /= grid;
    fprintf(stderr, "conv_ffma profile: grid=%d ks=%d avg cycles: setup=%.0f first_data=%.0f "
            "loop_end=%.0f published=%.0f all_ready=%.0f reduced=%.0f exit=%.0f | bars_init=%.0f "
            "common_setup=%.0f | producer "
            "start=%.0f decoded=%.0f expect_tx=%.0f stage0_issued=%.0f | compute first_wait=%.0f | CTA start spread %lld ns, "
            "first start -> last exit %lld ns\n", grid, p.ksplit, a[1], a[2], a[3], a[4], a[5],
            a[6], a[7], a[14], a[15], a[8], a[12], a[13], a[9], a[10], gmax0 - g0, g1 - g0);
    cudaFree(p.dbg);
    p.dbg = nullptr;
  }
  {
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (p.ksplit > 1) {
      attr[na].id = cudaLaunchAttributeClusterDimension;
      attr[na].val.clusterDim.x = p.ksplit;
      attr[na].val.clusterDim.y = 1;
      attr[na].val.clusterDim.z = 1;
      ++na;
    }
    if (dconv_host::pdl_enabled()) {
      attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[na].val.programmaticStreamSerializationAllowed = 1;
      ++na;
    }
    cfg.gridDim = dim3(clusters * p.ksplit);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cfg.attrs = attr;
    cfg.numAttrs = na;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, p);
    if (e != cudaSuccess)
      return dconv_host::set_error(DCONV_ECUDA, "conv_ffma (cluster %d): %s", p.ksplit,
                                   cudaGetErrorString(e));
  }
  dconv_host::count_launch();
  return dconv_host::check_launch("conv_ffma_kernel");
}

// Stream-K flags: one self-resetting flag per CTA, in a slot owned by the
// launching stream (launches of one stream never overlap; up to kSkSlots
// streams per device, later ones run without stream-K).  Module-resident:
// nothing is allocated.
constexpr int kSkSlots = 32, kSkFlagsPerSlot = 160;
__device__ unsigned g_sk_flags[kSkSlots * kSkFlagsPerSlot];

unsigned* sk_flags_for(cudaStream_t stream, int dev) {
  struct Dev {
    unsigned* base = nullptr;
    bool tried = false;
    std::vector<cudaStream_t> streams;
  };
  static std::mutex mu;
  static std::vector<Dev> devs;
  std::lock_guard<std::mutex> lock(mu);
  if ((int)devs.size() <= dev) devs.resize(dev + 1);
  Dev& d = devs[dev];
  if (!d.tried) {
    d.tried = true;
    // (the first launch of a process may already be under stream capture:
    // the symbol lookup is no stream operation, keep it legal there)
    cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
    cudaThreadExchangeStreamCaptureMode(&mode);
    void* sym = nullptr;
    if (cudaGetSymbolAddress(&sym, g_sk_flags) == cudaSuccess) d.base = static_cast<unsigned*>(sym);
    else cudaGetLastError();
    cudaThreadExchangeStreamCaptureMode(&mode);
  }
  if (!d.base) return nullptr;
  for (size_t i = 0; i < d.streams.size(); ++i)
    if (d.streams[i] == stream) return d.base + i * kSkFlagsPerSlot;
  if ((int)d.streams.size() >= kSkSlots) return nullptr;
  d.streams.push_back(stream);
  return d.base + (d.streams.size() - 1) * kSkFlagsPerSlot;
}

template <int BM, int BN, int WF, int NW, int TPX, int TCO, int CBS>
int launch_variant(FfmaParams p, cudaStream_t stream) {
  constexpr int threads = (NW + 8) * 32;
  constexpr int CG = BN / 8;
  const int dev = device_index();
  const int sms = dconv_host::device_sms(dev);
  const int co_groups = (p.jb_count + CG - 1) / CG;
  auto kernel = conv_ffma_kernel<BM, BN, WF, NW, TPX, TCO, CBS>;
  // kernel attributes are per device: set once for each device this
  // instantiation is launched on
  if (dconv_host::first_use_on_device(reinterpret_cast<const void*>(kernel), dev)) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  }
  // the DSMEM split-K reduction: 8 warps, 8 channels x 4 or 8 pixels/thread
  const bool no_split = knobs().no_splitk || NW != 8 || (TPX != 8 && TPX != 4) ||
                        TCO != 8 || (p.epi & DCONV_EPI_MAXPOOL);
  int slots[kMaxKs + 1] = {0};
  slots[1] = sms;
  if (!no_split)
    for (int ks = 2; ks <= kMaxKs; ++ks) slots[ks] = cluster_slots(kernel, ks, sms, threads);
  pick_tile(p, BM, BN, co_groups, sms, slots, !no_split);
  if ((p.epi & DCONV_EPI_MAXPOOL) && p.TW == 0)
    return dconv_host::set_error(DCONV_EUNSUPPORTED, "conv_ffma: no pool-compatible tile");
  p.TWe = std::min(p.TW, p.w_o);
  // q / TW for q < BM by multiply-high (exact: BM * TW < 2^32)
  p.tw_magic = (unsigned)(((uint64_t(1) << 32) + p.TW - 1) / p.TW);
  p.PW = (p.TWe - 1) * p.s + p.w_f;
  p.slab_floats = p.h_f * p.w_f * CBS * CBS;
  const int units = p.tiles_y * p.tiles_x * co_groups;
  const bool fine = (int64_t)units * 2 < sms;  // batch-1 layers: split-K over fine stages

  FfmaParams q = p;
  if (!configure<BN, NW, TPX, TCO, CBS>(q, 1, fine))
    return dconv_host::set_error(DCONV_EUNSUPPORTED, "conv_ffma: stage does not fit smem twice");
  const int S = q.n_g * q.n_r;

  // (1) fewer units than SMs (batch 1): one split-K launch with the cheapest
  // cluster size (the same cycle model as the tile selector).
  int best_ks = 1;
  double split_cycles_est = unit_cycles(p, BM, BN) + kLaunchFill;
  if (units < sms && !no_split) {
    FfmaParams t = p;
    if (configure<BN, NW, TPX, TCO, CBS>(t, 2, true))
      best_ks = best_split(units, slots, t.n_g * t.n_r, unit_cycles(p, BM, BN), &split_cycles_est);
  }
  if (const int kf = ksplit_knob(); kf && !no_split)
    best_ks = std::max(1, std::min(kf, std::min(kMaxKs, S)));
  // (1b) between a quarter of the SMs and all of them (small per-rank
  // batches, VGG b1's 112x112 / 56x56 layers): stream-K over every SM, a unit
  // cut into up to 5 pieces chained through the output map, when its estimate
  // (stage-granular share per CTA + ~4K cycles per piece of the chain) beats
  // the cluster split
  static const int sk_few_div = getenv("DCONV_STREAMK_FEW_DIV") ? atoi(getenv("DCONV_STREAMK_FEW_DIV")) : 4;
  static const bool no_streamk_few = getenv("DCONV_NO_STREAMK") != nullptr ||
                                     getenv("DCONV_NO_STREAMK_FEW") != nullptr;
  if (!no_streamk_few && !ksplit_knob() && units < sms && units * sk_few_div >= sms && S >= 2 &&
      (int64_t)units * S >= sms &&  // every CTA holds a stage: piece b continues in CTA b + 1
      sms + 1 < kSkFlagsPerSlot && !(p.epi & DCONV_EPI_MAXPOOL) && p.skip != p.out &&
      NW == 8 && TCO == 8) {
    const int64_t per_cta = ((int64_t)units * S + sms - 1) / sms;  // stages
    const int pieces = (int)((S + per_cta - 1) / per_cta) + 1;
    const double c_sk = (double)per_cta / S * unit_cycles(p, BM, BN) + pieces * 4000.0 + kLaunchFill;
    if (c_sk < split_cycles_est) {
      if (unsigned* flags = sk_flags_for(stream, dev)) {
        const size_t smem_sk = configure<BN, NW, TPX, TCO, CBS>(q, 1, fine);
        q.streamk = 1;
        q.sk_flags = flags;
        q.sk_base = 0;
        if (knobs().debug)
          fprintf(stderr, "conv_ffma<%d,%d,%d>: stream-K (few units) TH=%d TW=%d units=%d S=%d "
                  "stages/CTA=%lld pieces<=%d\n", BM, BN, WF, q.TH, q.TW, units, S,
                  (long long)per_cta, pieces);
        return launch_units(kernel, threads, q, smem_sk, 0, units, sms, stream);
      }
    }
  }
  if (best_ks > 1) {
    FfmaParams r = p;
    const size_t smem = configure<BN, NW, TPX, TCO, CBS>(r, best_ks, true);
    if (!smem) return dconv_host::set_error(DCONV_EUNSUPPORTED, "conv_ffma: split stage");
    const int clusters = std::min(units, std::max(1, cluster_slots(kernel, best_ks, sms, threads)));
    if (knobs().debug)
      fprintf(stderr, "conv_ffma<%d,%d,%d>: split TH=%d TW=%d units=%d ks=%d clusters=%d S=%d\n",
              BM, BN, WF, r.TH, r.TW, units, best_ks, clusters, r.n_g * r.n_r);
    return launch_units(kernel, threads, r, smem, 0, units, clusters, stream);
  }

  // (2) many units: full waves without splitting; a ragged last wave (< 75%
  // of the SMs) runs as a second launch whose units are split over clusters,
  // so the SMs that would idle help finish the tail.
  const int main_units = units / sms * sms, tail = units - main_units;
  // Stream-K: ragged unit counts (1.3 or 2.65 waves) run as ONE launch whose
  // CTAs each take units * S / sms stages; the <= 2 cut units per CTA are
  // finished through the output map (see FfmaParams::streamk).  Needs whole-K
  // units with a stage count to cut, the plain epilogue, and an output that
  // is not also the skip input (the partial tile passes through it).
  static const bool no_streamk = getenv("DCONV_NO_STREAMK") != nullptr;
  // worth it when the waves + split tail estimate is > 1% over units / sms
  double est_tail = 1.0;
  if (!no_split && tail * 4 < sms * 3)
    for (int ks = kMaxKs; ks >= 2; --ks)
      if (ks <= S && slots[ks] >= tail) {
        est_tail = 1.0 / ks + 0.12;  // cluster launches of 3 / 5 / 6 CTAs run erratically (+-3%)
        break;
      }
  static const bool sk_always = getenv("DCONV_STREAMK_ALWAYS") != nullptr;
  static const int sk_min_s = getenv("DCONV_STREAMK_MIN_S") ? atoi(getenv("DCONV_STREAMK_MIN_S")) : 2;
  // stream-K estimate: the whole waves but one, then (sms + tail) units cut
  // at stage granularity, + the boundary pieces' partial store / load
  const int sk_rr = (units / sms - 1) * sms;
  const double t_sk = (units / sms - 1) +
                      (double)(((int64_t)(units - sk_rr) * S + sms - 1) / sms) / S + 0.03;
  // (short-K skip-add layers lose more at the cut units than the model says:
  // 256->1024 + skip at 14x14 b256, S = 4: -1.5%)
  const bool sk_pays = sk_always || (t_sk < units / sms + est_tail &&
                                     !((p.epi & DCONV_EPI_ADD) && S < 8));
  if (!no_streamk && sk_pays && main_units > 0 && tail > 0 && S >= sk_min_s && sms + 1 < kSkFlagsPerSlot &&
      !(p.epi & DCONV_EPI_MAXPOOL) && p.skip != p.out && (int64_t)units * S < (1 << 30)) {
    if (unsigned* flags = sk_flags_for(stream, dev)) {
      const size_t smem_sk = configure<BN, NW, TPX, TCO, CBS>(q, 1, fine);
      q.streamk = 1;
      q.sk_flags = flags;
      static const bool sk_contig = getenv("DCONV_STREAMK_CONTIGUOUS") != nullptr;
      q.sk_base = sk_contig ? 0 : (units / sms - 1) * sms;
      if (knobs().debug)
        fprintf(stderr, "conv_ffma<%d,%d,%d>: stream-K TH=%d TW=%d units=%d S=%d G=%d R=%d NS=%d "
                "(%.2f waves)\n", BM, BN, WF, q.TH, q.TW, units, S, q.G, q.R, q.NS,
                (double)units / sms);
      return launch_units(kernel, threads, q, smem_sk, 0, units, sms, stream);
    }
  }
  int tail_ks = 1;
  if (main_units > 0 && tail > 0 && tail * 4 < sms * 3 && !no_split &&
      !knobs().no_tailsplit) {
    static const bool pow2_only = getenv("DCONV_TAIL_POW2") != nullptr;
    for (int ks = kMaxKs; ks >= 2; ks = pow2_only ? ks / 2 : ks - 1) {
      FfmaParams t = p;
      if (!configure<BN, NW, TPX, TCO, CBS>(t, ks, true)) continue;
      if (ks > t.n_g * t.n_r) continue;
      const int slots = cluster_slots(kernel, ks, sms, threads);
      if (slots >= tail) {
        tail_ks = ks;
        break;
      }
    }
  }
  const size_t smem_main = configure<BN, NW, TPX, TCO, CBS>(q, 1, fine);
  if (knobs().debug && tail_ks > 1)
    for (int ks = 2; ks <= kMaxKs; ++ks)
      fprintf(stderr, "  cluster_slots(%d) = %d\n", ks, cluster_slots(kernel, ks, sms, threads));
  if (knobs().debug)
    fprintf(stderr,
            "conv_ffma<%d,%d,%d>: %dx%d tiles TH=%d TW=%d units=%d S=%d G=%d R=%d NS=%d "
            "main=%d tail=%d tail_ks=%d\n",
            BM, BN, WF, q.tiles_y, q.tiles_x, q.TH, q.TW, units, S, q.G, q.R, q.NS, main_units,
            tail, tail_ks);
  if (tail_ks == 1)
    return launch_units(kernel, threads, q, smem_main, 0, units, std::min(units, sms), stream);
  int rc = launch_units(kernel, threads, q, smem_main, 0, main_units, sms, stream);
  if (rc) return rc;
  FfmaParams t = p;
  const size_t smem_tail = configure<BN, NW, TPX, TCO, CBS>(t, tail_ks, true);
  return launch_units(kernel, threads, t, smem_tail, main_units, tail, tail, stream);
}

template <int BM, int BN, int NW = 8, int TPX = 8, int TCO = 8, int CBS = 8>
int launch_wf(const FfmaParams& p, cudaStream_t stream) {
  if constexpr (CBS != 8) {
    // c_b = 16 / 32: filter widths 1 and 3 specialised, any other at run time
    switch (p.w_f) {
      case 1: return launch_variant<BM, BN, 1, NW, TPX, TCO, CBS>(p, stream);
      case 3: return launch_variant<BM, BN, 3, NW, TPX, TCO, CBS>(p, stream);
      default: return launch_variant<BM, BN, 0, NW, TPX, TCO, CBS>(p, stream);
    }
  }
  switch (p.w_f) {
    case 1: return launch_variant<BM, BN, 1, NW, TPX, TCO, 8>(p, stream);
    case 3: return launch_variant<BM, BN, 3, NW, TPX, TCO, 8>(p, stream);
    case 5: return launch_variant<BM, BN, 5, NW, TPX, TCO, 8>(p, stream);
    default: return launch_variant<BM, BN, 0, NW, TPX, TCO, 8>(p, stream);
  }
}

// fresh (uncached) occupancy query, for the cache check below
template <class K>
int cluster_slots_fresh(K kernel, int ks, int threads) {
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = ks;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(ks * 64);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = 200 * 1024;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kernel, &cfg) != cudaSuccess || n < 1) {
    cudaGetLastError();
    n = -1;
  }
  return n;
}

template <int BM, int BN, int NW, int TPX, int TCO>
int probe_slots(int ks, int* cached, int* fresh) {
  auto kernel = conv_ffma_kernel<BM, BN, 3, NW, TPX, TCO, 8>;
  const int dev = device_index();
  if (dconv_host::first_use_on_device(reinterpret_cast<const void*>(kernel), dev)) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  }
  constexpr int threads = (NW + 8) * 32;
  *cached = cluster_slots(kernel, ks, dconv_host::device_sms(dev), threads);
  *fresh = cluster_slots_fresh(kernel, ks, threads);
  return DCONV_OK;
}

}  // namespace

// Test hook: the cached co-resident cluster count of one CTA-tile
// instantiation (3x3 filters) next to a fresh occupancy query.
int ffma_cluster_slots_probe(int tile_variant, int ks, int* cached, int* fresh) {
  if (ks < 2 || ks > kMaxKs) return dconv_host::set_error(DCONV_EPARAM, "ks %d", ks);
  switch (tile_variant) {
    case 1: return probe_slots<128, 128, 8, 8, 8>(ks, cached, fresh);
    case 2: return probe_slots<256, 64, 8, 8, 8>(ks, cached, fresh);
    case 3: return probe_slots<128, 64, 8, 4, 8>(ks, cached, fresh);
    case 4: return probe_slots<256, 32, 8, 4, 8>(ks, cached, fresh);
    default: return dconv_host::set_error(DCONV_EPARAM, "tile_variant %d", tile_variant);
  }
}

int launch_conv_ffma(const FfmaParams& p0, cudaStream_t stream) {
  FfmaParams p = p0;
  // 1x1 stride-s layers read only every s-th input row: view the input with
  // an s-times row pitch so the patch stages just those rows (column
  // stride stays s)
  p.sy = p.s;
  if (p.h_f == 1 && p.s > 1) {
    p.in_row *= p.s;
    p.h_i = p.h_o;
    p.sy = 1;
  }
  p.h_o_magic = (int64_t)p.n * p.h_o * p.h_o < (int64_t(1) << 32)
                    ? (unsigned)(((uint64_t(1) << 32) + p.h_o - 1) / p.h_o)
                    : 0u;
  static const bool no_skip_prefetch = getenv("DCONV_NO_SKIP_PREFETCH") != nullptr;
  p.skip_prefetch = (p.epi & DCONV_EPI_ADD) && !no_skip_prefetch;
  // c_b = 16 / 32 storage blocks: the kernel counts output blocks in
  // 8-channel sub-blocks (a thread's channel tile)
  const int sub = p.cbs / kCB;
  if (p.cbs != 8 && p.cbs != 16 && p.cbs != 32)
    return dconv_host::set_error(DCONV_EUNSUPPORTED, "conv_ffma: c_b %d", p.cbs);
  p.jb_begin *= sub;
  p.jb_count *= sub;
  int v = p.variant;  // desc.tile_variant - 1; -1 = selector
  // measured (tools/sweep_variants.py): 256 px x 64 ch wins on every 3x3 /
  // 5x5 layer of the configs; 1x1 layers with >= 128 output channels
  // (little reuse per staged pixel) prefer 128 px x 128 ch
  // (the 32-channel tile by default only for layers of <= 32 channels, not
  // for <= 32-channel C_o slices of wider layers: a slice then runs the
  // unsharded layer's tiling, so C_o-sharded ranks reproduce it bitwise)
  if (v < 0)
    v = (p.h_f * p.w_f == 1 && p.jb_count >= 16) ? 0
        : (p.jb_n * sub <= 4 && !(p.epi & DCONV_EPI_MAXPOOL)) ? 3 : 1;
  if (p.cbs != 8) {
    // c_b = 16 / 32: the two main CTA tiles (the 128 x 64 batch-1 tile
    // runs as 256 x 64)
    if (p.epi & DCONV_EPI_MAXPOOL)
      return dconv_host::set_error(DCONV_EUNSUPPORTED, "conv_ffma: fused pool needs c_b = 8");
    if (p.cbs == 16)
      return v == 0 ? launch_wf<128, 128, 8, 8, 8, 16>(p, stream)
                    : launch_wf<256, 64, 8, 8, 8, 16>(p, stream);
    return v == 0 ? launch_wf<128, 128, 8, 8, 8, 32>(p, stream)
                  : launch_wf<256, 64, 8, 8, 8, 32>(p, stream);
  }
  switch (v) {
    // Measured on B200 and not instantiated (tools/variant_run.sh): 12
    // compute warps with 2-channel activation loads (<192,128,12>,
    // <384,64,12>) -6..-12%; 16 px x 8 ch per thread (<512,64,8,16>,
    // <256,128,8,16>, spills at 229 registers) -13%; 8 px x 16 ch per thread
    // (<256,128,8,8,16>, 25% fewer LDS per FFMA2) +-0% at 128 ch, -6% at
    // 256/512 ch.  tools/ffma2_pattern.cu: this operand pattern tops out at
    // ~59 TFLOP/s with any warp count (83% of the FFMA2 probe).
    case 0: return launch_wf<128, 128>(p, stream);  // 128 px x 128 channels
    case 2:  // 128 px x 64 channels, 4 px x 8 ch per thread: twice the units
             // of the 256 x 64 tile for batch-1 layers (less split-K)
      if (p.epi & DCONV_EPI_MAXPOOL)
        return dconv_host::set_error(DCONV_EUNSUPPORTED, "conv_ffma: 128x64 tile has no fused pool");
      return launch_wf<128, 64, 8, 4, 8>(p, stream);
    case 3:  // 256 px x 32 channels, 4 px x 8 ch per thread: layers with C_o = 32
             // (or C_o / 32 odd: no half-empty 64-channel group)
      if (p.epi & DCONV_EPI_MAXPOOL)
        return dconv_host::set_error(DCONV_EUNSUPPORTED, "conv_ffma: 256x32 tile has no fused pool");
      return launch_wf<256, 32, 8, 4, 8>(p, stream);
    default: return launch_wf<256, 64>(p, stream);  // 256 px x 64 channels
  }
}

}  // namespace dconv_dev
