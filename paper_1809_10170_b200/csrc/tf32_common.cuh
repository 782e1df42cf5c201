// tf32_common.cuh -- tcgen05 / TMA helpers and the blocked-pencil epilogue
// shared by the TF32 tensor-core kernels (conv_tf32.cu: one TF32 pass;
// conv_tf32x3.cu: split-TF32, fp32 tolerance).
#pragma once
#include <algorithm>
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "conv_kernels.h"

namespace dconv_dev {
namespace tf32 {

constexpr int kMaxMT = 4;       // M-tiles (128 pixels each) per work unit, at most
constexpr int kTileRows = 16;   // an M-tile is 16 output rows x 8 columns
constexpr int kTW = 8;
constexpr int kMaxStagesT = 8;

struct Tf32Params {
  const float* w;     // prepared weights
  const float* skip;
  float* out;
  int n, h_i, w_i, h_o, w_o, h_f, w_f;
  int ib_n, jb_begin, jb_count;
  int N;              // channels per work unit (64, 128 or 256), 8 | N
  int n_cg;           // channel groups
  int64_t out_img, out_blk, out_row, sk_img, sk_blk, sk_row;
  int epi;
  int G, R, n_g, n_r, PH, PW;
  int plane_floats;   // one channel half-plane of a stage: G*PH*PW*4
  int wstage_floats;  // G*R*w_f*2*N*4 (x2 for split-TF32: hi and lo)
  int stage_floats;
  int NS;
  int row_groups, strips, units;
  int MT;             // M-tiles per unit (1..4)
  int chunk_st;       // split-TF32: stages per TMEM accumulator chunk
  int s2d, ib_o;      // in-place space-to-depth factor (1 = off); original input blocks
  int hf_o, wf_o;     // original filter (s2d: taps s*n'+dy >= hf_o are structurally zero)
  int wide;           // 1x1 layers: whole 32-byte pencils by one TMA box, 32-byte-swizzled
                      // K-major A (see encode_input_map_wide); 0: two 16-byte half planes
  int stack;          // images stacked along the tile rows (small maps), 1 = off
  int SP;             // stacked mode: patch rows per image slot (h_o + R - 1)
  uint32_t idesc;
  uint32_t idesc2;    // split-TF32 DA: the N' = 2N instruction descriptor
  int da;             // split-TF32: separate correction accumulator (N <= 128)
  unsigned long long* dbg;  // DCONV_TF32_PROFILE: per-CTA wait cycles (else null)
};

__device__ __forceinline__ void tma_load_5d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, int c3, int c4, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4),
      "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, int c3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
      "r"(smem_u32(bar))
      : "memory");
}

// Issued by one elected lane of a converged warp (elect.sync); the
// descriptors come in as 32-bit halves so the loop arithmetic stays 32-bit.
__device__ __forceinline__ void umma_tf32_elect(uint32_t d_tmem, uint32_t a_lo, uint32_t a_hi,
                                                uint32_t b_lo, uint32_t b_hi, uint32_t idesc,
                                                uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred e, p;\n.reg .b64 ad, bd;\n"
      "mov.b64 ad, {%1, %2};\nmov.b64 bd, {%3, %4};\n"
      "setp.ne.b32 p, %6, 0;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], ad, bd, %5, p;\n}\n" ::"r"(d_tmem),
      "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(
          smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tmem_ld32x32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, "
      "%8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, "
      "%23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
        "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]),
        "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
        "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]),
        "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// unit u -> (channel group fastest, then strip, row group, image (group));
// with p.stack > 1 a unit holds images img .. img + stack - 1 (one row group)
__device__ __forceinline__ void decode_unit(const Tf32Params& p, int u, int& img, int& y0, int& x0,
                                            int& cg) {
  cg = u % p.n_cg;
  int t = u / p.n_cg;
  const int strip = t % p.strips;
  t /= p.strips;
  const int rg = t % p.row_groups;
  img = (t / p.row_groups) * p.stack;
  y0 = rg * p.MT * kTileRows;
  x0 = strip * kTW;
}

// Tile row j (0 .. MT*16-1) of a unit -> (image, output row).  Stacked
// images: slot k = j / SP holds image img + k, output row j - k*SP (rows
// h_o .. SP-1 of a slot mix two images' patch rows and are never stored).
__device__ __forceinline__ void tile_row_pixel(const Tf32Params& p, int img, int y0, int j,
                                               int& im, int& y, bool& ok) {
  if (p.stack > 1) {
    const int k = j / p.SP;
    im = img + k;
    y = j - k * p.SP;
    ok = k < p.stack && y < p.h_o && im < p.n;
  } else {
    im = img;
    y = y0 + j;
    ok = y < p.h_o;
  }
}

// Epilogue for 32 accumulator columns (4 output blocks starting at channel c0
// of channel group cg) of pixel (img, y, x): fused skip-add / ReLU / 2x2
// max-pool, then blocked pencil stores.  Every lane of the warp must call it
// (the pool exchanges values across lanes); `valid` masks the stores.
__device__ __forceinline__ void emit32(const Tf32Params& p, float (&v)[32], int img, int y, int x,
                                       bool valid, int tx, int ty, int cg, int c0) {
  if (p.epi & DCONV_EPI_MAXPOOL) {
    // 2x2 window = lanes {l, l^1, l^8, l^9} (8-px tile rows, even
    // origins, even h_o/w_o: a window is all valid or all invalid)
    if (valid && (p.epi & DCONV_EPI_ADD)) {
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int jb = cg * (p.N / 8) + (c0 / 8) + b;
        if (jb >= p.jb_count) break;
        const float* sk = p.skip + (int64_t)img * p.sk_img + (int64_t)jb * p.sk_blk +
                          (int64_t)y * p.sk_row + (int64_t)x * 8;
#pragma unroll
        for (int i = 0; i < 8; ++i) v[b * 8 + i] += sk[i];
      }
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      v[i] = fmaxf(v[i], __shfl_xor_sync(0xffffffffu, v[i], 1));
      v[i] = fmaxf(v[i], __shfl_xor_sync(0xffffffffu, v[i], 8));
      if (p.epi & DCONV_EPI_RELU) v[i] = fmaxf(v[i], 0.f);
    }
    if (!valid || (tx & 1) || (ty & 1)) return;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int jb = cg * (p.N / 8) + (c0 / 8) + b;
      if (jb >= p.jb_count) break;
      float* o = p.out + (int64_t)img * p.out_img + (int64_t)jb * p.out_blk +
                 (int64_t)(y >> 1) * p.out_row + (int64_t)(x >> 1) * 8;
      DCONV_OWN(o, 8);
      stg_pencil(o, *reinterpret_cast<const float(*)[8]>(v + b * 8));
    }
    return;
  }
  if (!valid) return;
  if (p.epi & DCONV_EPI_ADD) {
    // all of the chunk's skip pencils in flight before any store
    // (read-only path: the loads do not wait behind the stores)
    float4 s4[8];
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int jb = min(cg * (p.N / 8) + (c0 / 8) + b, p.jb_count - 1);
      // one 256-bit load per pencil (a warp's lanes are 32 adjacent pixels:
      // 1 KB contiguous per instruction)
      ldg_pencil(p.skip + (int64_t)img * p.sk_img + (int64_t)jb * p.sk_blk + (int64_t)y * p.sk_row +
                     (int64_t)x * 8,
                 s4[2 * b], s4[2 * b + 1]);
    }
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      float* vv = v + b * 8;
      vv[0] += s4[2 * b].x; vv[1] += s4[2 * b].y; vv[2] += s4[2 * b].z; vv[3] += s4[2 * b].w;
      vv[4] += s4[2 * b + 1].x; vv[5] += s4[2 * b + 1].y;
      vv[6] += s4[2 * b + 1].z; vv[7] += s4[2 * b + 1].w;
    }
  }
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const int jb = cg * (p.N / 8) + (c0 / 8) + b;  // block within the computed range
    if (jb >= p.jb_count) break;
    float* o = p.out + (int64_t)img * p.out_img + (int64_t)jb * p.out_blk +
               (int64_t)y * p.out_row + (int64_t)x * 8;
    float* vv = v + b * 8;
    if (p.epi & DCONV_EPI_RELU) {
#pragma unroll
      for (int i = 0; i < 8; ++i) vv[i] = fmaxf(vv[i], 0.f);
    }
    DCONV_OWN(o, 8);
    stg_pencil(o, *reinterpret_cast<const float(*)[8]>(vv));
  }
}

inline PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  // driver entry point, resolved once (thread-safe static initialisation)
  static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    return PFN_cuTensorMapEncodeTiled_v12000(nullptr);
  }();
  return fn;
}

// The input as the TMA sees it: the original view, even when the kernel
// computes a re-shaped layer (below).
struct InView {
  const float* base;
  int n, w_i, h_i, ib;     // original dims and input blocks per image
  int64_t px_floats, row, blk;
  int s2d;                 // space-to-depth factor (1 = off)
};

// Host side shared by both launchers.
//   * A 1x1 stride-s layer becomes a stride-1 1x1 layer over the subsampled
//     view (pixel stride 8s floats, row stride s rows).
//   * A k x k stride-s layer becomes a stride-1 layer with s*s*C_i channels
//     and a ceil(k/s) filter (space-to-depth: channel block phase*ib + b,
//     phase = dy*s + dx, is pixel (s*y + dy, s*x + dx) of block b), read in
//     place: the TMA traverses the original map with element strides s
//     (tools/tma_stride_probe.cu), so no repacked copy exists.  The prepared
//     weights follow the same channel order (prepare kernels).
// Then the checks.
inline int prepare_view(FfmaParams& f, InView& v, const char* who) {
  v = InView{f.in, f.n, f.w_i, f.h_i, f.ib_n, 8, f.in_row, f.in_blk, 1};
  if (f.in_img != (int64_t)f.ib_n * f.in_blk)
    return dconv_host::set_error(DCONV_EUNSUPPORTED,
                                 "%s: input view must stack blocks densely per image", who);
  if (f.s > 1 && f.h_f == 1 && f.w_f == 1) {
    v.px_floats = 8 * (int64_t)f.s;
    v.row = f.in_row * f.s;
    v.h_i = f.h_o;
    v.w_i = f.w_o;
    f.h_i = f.h_o;
    f.w_i = f.w_o;
    f.s = 1;
  } else if (f.s > 1) {
    const int s = f.s;
    // the TMA traverses the original map with element strides s: the tensor
    // map encoder allows strides of at most 8
    if (s > 8)
      return dconv_host::set_error(DCONV_EUNSUPPORTED,
                                   "%s: k x k stride %d > 8 (TMA element stride limit)", who, s);
    v.s2d = s;
    f.ib_n *= s * s;
    f.h_f = (f.h_f + s - 1) / s;
    f.w_f = (f.w_f + s - 1) / s;
    f.h_i = f.h_o + f.h_f - 1;
    f.w_i = f.w_o + f.w_f - 1;
    f.s = 1;
  }
  if (!encode_fn()) return dconv_host::set_error(DCONV_ECUDA, "cuTensorMapEncodeTiled unavailable");
  return DCONV_OK;
}

// 5-D tensor map {c4, half, W, H, image*block} over the original view; the
// box lands PW x PH pixels x G blocks (with element strides s2d: every s-th
// column and row).
inline int encode_input_map(CUtensorMap* map, const InView& v, int PW, int PH, int G) {
  const cuuint64_t dims[5] = {4, 2, (cuuint64_t)v.w_i, (cuuint64_t)v.h_i, (cuuint64_t)v.n * v.ib};
  const cuuint64_t strides[4] = {16, (cuuint64_t)v.px_floats * 4, (cuuint64_t)v.row * 4,
                                 (cuuint64_t)v.blk * 4};
  const cuuint32_t box[5] = {4, 1, (cuuint32_t)(PW * v.s2d), (cuuint32_t)(PH * v.s2d),
                             (cuuint32_t)G};
  const cuuint32_t estr[5] = {1, 1, (cuuint32_t)v.s2d, (cuuint32_t)v.s2d, 1};
  if (box[2] > 256 || box[3] > 256)
    return dconv_host::set_error(DCONV_EUNSUPPORTED, "TMA box %u x %u too large", box[2], box[3]);
  const CUresult cr = encode_fn()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float*>(v.base),
                                  dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS)
    return dconv_host::set_error(DCONV_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)cr);
  return DCONV_OK;
}

// 1x1 layers ("wide" A): 4-D map {8 ch, W, H, image*block} whose innermost box
// row is a whole 32-byte pencil, stored with the 32-byte swizzle: the canonical
// K-major SWIZZLE_32B UMMA layout (8 pixels x 32 B atoms, SBO 256 B), so one
// box replaces the two 16-byte half-plane boxes -- each 32-byte sector crosses
// the L2->SM crossbar once instead of twice (ncu: 2.0 GB of TMA reads for an
// 822 MB input on ResNet-50's 256->64 1x1 at 56x56 b256 with half planes).
inline int encode_input_map_wide(CUtensorMap* map, const InView& v, int PW, int PH, int G) {
  const cuuint64_t dims[4] = {8, (cuuint64_t)v.w_i, (cuuint64_t)v.h_i, (cuuint64_t)v.n * v.ib};
  const cuuint64_t strides[3] = {(cuuint64_t)v.px_floats * 4, (cuuint64_t)v.row * 4,
                                 (cuuint64_t)v.blk * 4};
  const cuuint32_t box[4] = {8, (cuuint32_t)PW, (cuuint32_t)PH, (cuuint32_t)G};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  if (box[1] > 256 || box[2] > 256 || box[3] > 256)
    return dconv_host::set_error(DCONV_EUNSUPPORTED, "TMA box %u x %u x %u too large", box[1],
                                 box[2], box[3]);
  const CUresult cr = encode_fn()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(v.base),
                                  dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                  CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS)
    return dconv_host::set_error(DCONV_ECUDA, "cuTensorMapEncodeTiled (wide) failed (%d)", (int)cr);
  return DCONV_OK;
}

// A-operand descriptor words of a stage: low word (start >> 4 | LBO >> 4 << 16)
// and high word (SBO >> 4, version 1, layout).  Half planes: no swizzle,
// core matrices 8 px x 16 B, LBO = one plane (the second K half), SBO = one
// tile row.  Wide: SWIZZLE_32B K-major (layout type 6), 8 px x 32 B atoms,
// SBO 256 B.  `unit` = 16-byte units per pixel step (2 when wide).
// tap-walk variants of the tensor-core kernels (template parameter VAR)
constexpr int kWalkPlain = 0;  // stride-1 layers, half-plane A
constexpr int kWalkS2D = 1;    // space-to-depth view: skip structurally zero taps
constexpr int kWalkWide = 2;   // 1x1 whole-pencil (32-byte swizzled) A
struct ADesc {
  uint32_t lo0, hi, unit;
};
__device__ __forceinline__ ADesc a_desc(const Tf32Params& p, uint32_t a_base) {
  ADesc d;
  if (p.wide) {
    d.lo0 = ((a_base >> 4) & 0x3FFFu) | (1u << 16);
    d.hi = (256u >> 4) | (1u << 14) | (6u << 29);
    d.unit = 2u;
  } else {
    d.lo0 = ((a_base >> 4) & 0x3FFFu) | (((uint32_t)(p.plane_floats * 4) >> 4) << 16);
    d.hi = ((uint32_t)(p.PW * 16) >> 4) | (1u << 14);
    d.unit = 1u;
  }
  return d;
}

// Original blocked weight [jb][b][n][m][ii][jj] behind element (jb, ib, n, m,
// ii, jj) of the computed (possibly space-to-depth) layer; 0 for the taps
// the re-shaped filter adds past the original edge.
__device__ __forceinline__ float weight_src(const float* __restrict__ w, int jb, int ib, int n,
                                            int m, int ii, int jj, const WSrc& q) {
  const int ph = ib / q.ib_o, b = ib - ph * q.ib_o;
  const int dy = ph / q.s, dx = ph - dy * q.s;
  const int no = q.s * n + dy, mo = q.s * m + dx;
  if (no >= q.hf_o || mo >= q.wf_o) return 0.f;
  return w[(((((int64_t)jb * q.ib_o + b) * q.hf_o + no) * q.wf_o + mo) * 8 + ii) * 8 + jj];
}

// TMA coordinates of input block ib (of the computed layer) for a tile at
// (x0, row y) of image img: with space-to-depth, block ib = phase*ib_o + b
// is pixel (s*y + dy, s*x + dx) of original block b.
__device__ __forceinline__ void tma_block_coords(const Tf32Params& p, int img, int ib, int x0,
                                                 int y, int& cx, int& cy, int& c4) {
  const int s = p.s2d;
  if (s == 1) {  // no space-to-depth (the common case: no divisions)
    cx = x0;
    cy = y;
    c4 = img * p.ib_o + ib;
    return;
  }
  const int ph = ib / p.ib_o, b = ib - ph * p.ib_o;
  const int dy = ph / s, dx = ph - dy * s;
  cx = s * x0 + dx;
  cy = s * y + dy;
  c4 = img * p.ib_o + b;
}

// Space-to-depth layers: a stage holds input blocks of one phase (dy, dx);
// its taps (n', m') with s*n'+dy >= hf_o or s*m'+dx >= wf_o multiply zero
// weights.  Returns the valid tap rows / columns of the stage's phase (the
// MMA issuers skip the rest: 3x3/s2 computes 9 of 16 taps, 7x7/s2 49 of 64).
__device__ __forceinline__ void s2d_valid_taps(const Tf32Params& p, int ib0, int& nmax,
                                               int& mmax) {
  if (p.s2d <= 1) {
    nmax = p.h_f;
    mmax = p.w_f;
    return;
  }
  const int phase = ib0 / p.ib_o, dy = phase / p.s2d, dx = phase - dy * p.s2d;
  nmax = (p.hf_o - dy + p.s2d - 1) / p.s2d;
  mmax = (p.wf_o - dx + p.s2d - 1) / p.s2d;
}

inline void copy_geometry(Tf32Params& p, const FfmaParams& f) {
  p.skip = f.skip;
  p.out = f.out;
  p.n = f.n; p.h_i = f.h_i; p.w_i = f.w_i; p.h_o = f.h_o; p.w_o = f.w_o;
  p.h_f = f.h_f; p.w_f = f.w_f;
  p.ib_n = f.ib_n; p.jb_begin = f.jb_begin; p.jb_count = f.jb_count;
  p.out_img = f.out_img; p.out_blk = f.out_blk; p.out_row = f.out_row;
  p.sk_img = f.sk_img; p.sk_blk = f.sk_blk; p.sk_row = f.sk_row;
  p.epi = f.epi;
  p.PW = kTW - 1 + p.w_f;
}

// instruction descriptor: D f32, A/B tf32, K-major both, N, M = 128
inline uint32_t tf32_idesc(int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(128 >> 4) << 24);
}

inline int sm_count() { return dconv_host::device_sms(dconv_host::current_device()); }

}  // namespace tf32
}  // namespace dconv_dev
