/*
 * oracle.c -- CPU restatement of the reference dconv hot path.
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Citations are into
 * /root/reference/proj/core/ unless they name SPEC.md / PAPER.md.
 */
#include "oracle.h"

#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

int orc_round_up(int value, int block) {  /* tensor.hpp:28-30 */
  return (value + block - 1) / block * block;
}

int orc_conv_shape(int c_i, int c_o, int h_i, int w_i, int h_f, int w_f,
                   int s, int* h_o, int* w_o) {
  /* shape.cpp:32-39: counts >= 1, stride >= 1, filter fits, exact division */
  if (!(c_i >= 1 && c_o >= 1 && h_i >= 1 && w_i >= 1 && h_f >= 1 && w_f >= 1))
    return -1;
  if (s < 1) return -1;
  if (!(h_f <= h_i && w_f <= w_i)) return -1;
  if ((h_i - h_f) % s != 0) return -1;
  if ((w_i - w_f) % s != 0) return -1;
  if (h_o) *h_o = (h_i - h_f) / s + 1;
  if (w_o) *w_o = (w_i - w_f) / s + 1;
  return 0;
}

int64_t orc_conv_flops(int c_i, int c_o, int h_o, int w_o, int h_f, int w_f) {
  /* reference.cpp:106-109 */
  return 2LL * c_i * c_o * h_o * w_o * h_f * w_f;
}

/* BlockedFeatureMap::offset (tensor.hpp:71-74) */
static inline size_t bfm_off(int c, int y, int x, int h, int w, int c_b) {
  return (size_t)(c / c_b) * ((size_t)h * w * c_b) +
         ((size_t)y * w + x) * c_b + (size_t)(c % c_b);
}

/* BlockedKernel::offset (tensor.hpp:131-137) */
static inline size_t bk_off(int jb, int ib, int n, int m, int ii, int jj,
                            int in_blocks, int h_f, int w_f, int c_ib,
                            int c_ob) {
  return (((((size_t)jb * in_blocks + ib) * h_f + n) * w_f + m) * c_ib + ii) *
             c_ob + jj;
}

void orc_pack_feature_map(const float* src, int c, int h, int w, int c_b,
                          float* dst) {
  /* tensor.cpp:65-73: zero-initialised destination, element-wise copy */
  const int pc = orc_round_up(c, c_b);
  memset(dst, 0, sizeof(float) * (size_t)pc * h * w);
  for (int ch = 0; ch < c; ++ch)
    for (int y = 0; y < h; ++y)
      for (int x = 0; x < w; ++x)
        dst[bfm_off(ch, y, x, h, w, c_b)] = src[((size_t)ch * h + y) * w + x];
}

void orc_unpack_feature_map(const float* src, int c, int h, int w, int c_b,
                            float* dst) {
  /* tensor.cpp:75-83: padded channels dropped */
  for (int ch = 0; ch < c; ++ch)
    for (int y = 0; y < h; ++y)
      for (int x = 0; x < w; ++x)
        dst[((size_t)ch * h + y) * w + x] = src[bfm_off(ch, y, x, h, w, c_b)];
}

void orc_pack_kernel(const float* src, int c_i, int c_o, int h_f, int w_f,
                     int c_ob, int c_ib, float* dst) {
  /* tensor.cpp:85-95 (BlockedKernel ctor zero-fills, tensor.cpp:60-62) */
  const int pci = orc_round_up(c_i, c_ib), pco = orc_round_up(c_o, c_ob);
  const int ib_n = pci / c_ib;
  memset(dst, 0, sizeof(float) * (size_t)pci * pco * h_f * w_f);
  for (int i = 0; i < c_i; ++i)
    for (int j = 0; j < c_o; ++j)
      for (int n = 0; n < h_f; ++n)
        for (int m = 0; m < w_f; ++m)
          dst[bk_off(j / c_ob, i / c_ib, n, m, i % c_ib, j % c_ob, ib_n, h_f,
                     w_f, c_ib, c_ob)] =
              src[(((size_t)i * c_o + j) * h_f + n) * w_f + m];
}

void orc_unpack_kernel(const float* src, int c_i, int c_o, int h_f, int w_f,
                       int c_ob, int c_ib, float* dst) {
  /* tensor.cpp:97-108 */
  const int ib_n = orc_round_up(c_i, c_ib) / c_ib;
  for (int i = 0; i < c_i; ++i)
    for (int j = 0; j < c_o; ++j)
      for (int n = 0; n < h_f; ++n)
        for (int m = 0; m < w_f; ++m)
          dst[(((size_t)i * c_o + j) * h_f + n) * w_f + m] =
              src[bk_off(j / c_ob, i / c_ib, n, m, i % c_ib, j % c_ob, ib_n,
                         h_f, w_f, c_ib, c_ob)];
}

void orc_conv_oracle64(const float* in, const float* k, int c_i, int c_o,
                       int h_i, int w_i, int h_f, int w_f, int s, float* out) {
  /* reference.cpp:70-87: loops i, j, x, y, m, n; fp64 accumulate */
  int h_o = (h_i - h_f) / s + 1, w_o = (w_i - w_f) / s + 1;
  size_t n_out = (size_t)c_o * h_o * w_o;
  double* acc = (double*)calloc(n_out, sizeof(double));
  for (int i = 0; i < c_i; ++i)
    for (int j = 0; j < c_o; ++j)
      for (int x = 0; x < w_o; ++x)
        for (int y = 0; y < h_o; ++y)
          for (int m = 0; m < w_f; ++m)
            for (int n = 0; n < h_f; ++n)
              acc[((size_t)j * h_o + y) * w_o + x] +=
                  (double)in[((size_t)i * h_i + y * s + n) * w_i + x * s + m] *
                  (double)k[(((size_t)i * c_o + j) * h_f + n) * w_f + m];
  for (size_t q = 0; q < n_out; ++q) out[q] = (float)acc[q];
  free(acc);
}

void orc_conv_naive(const float* in, const float* k, int c_i, int c_o, int h_i,
                    int w_i, int h_f, int w_f, int s, float* out) {
  /* reference.cpp:34-52: fp32, FeatureMap output zero-initialised */
  int h_o = (h_i - h_f) / s + 1, w_o = (w_i - w_f) / s + 1;
  memset(out, 0, sizeof(float) * (size_t)c_o * h_o * w_o);
  for (int i = 0; i < c_i; ++i)
    for (int j = 0; j < c_o; ++j)
      for (int x = 0; x < w_o; ++x)
        for (int y = 0; y < h_o; ++y)
          for (int m = 0; m < w_f; ++m)
            for (int n = 0; n < h_f; ++n)
              out[((size_t)j * h_o + y) * w_o + x] +=
                  in[((size_t)i * h_i + y * s + n) * w_i + x * s + m] *
                  k[(((size_t)i * c_o + j) * h_f + n) * w_f + m];
}

void orc_conv_oracle64_blocked(const float* in, const float* k, int c_i,
                               int c_o, int h_i, int w_i, int h_f, int w_f,
                               int s, int c_ib, int c_ob, int y0, int y1,
                               float* out) {
  /* Same per-output fp64 summation order as reference.cpp:75-83 (i outer,
   * then m, then n), read through the blocked offsets of tensor.hpp:71-74 and
   * :131-137.  Parallel over output channels: order per element unchanged. */
  const int h_o = (h_i - h_f) / s + 1, w_o = (w_i - w_f) / s + 1;
  const int ib_n = orc_round_up(c_i, c_ib) / c_ib;
  const int pco = orc_round_up(c_o, c_ob);
  if (y0 < 0) y0 = 0;
  if (y1 > h_o) y1 = h_o;
#pragma omp parallel for schedule(dynamic)
  for (int j = 0; j < pco; ++j) {
    for (int y = y0; y < y1; ++y)
      for (int x = 0; x < w_o; ++x) {
        double acc = 0.0;
        if (j < c_o)
          for (int i = 0; i < c_i; ++i)
            for (int m = 0; m < w_f; ++m)
              for (int n = 0; n < h_f; ++n)
                acc += (double)in[bfm_off(i, y * s + n, x * s + m, h_i, w_i,
                                          c_ib)] *
                       (double)k[bk_off(j / c_ob, i / c_ib, n, m, i % c_ib,
                                        j % c_ob, ib_n, h_f, w_f, c_ib, c_ob)];
        out[bfm_off(j, y, x, h_o, w_o, c_ob)] = (float)acc;
      }
  }
}

/* ---- conv_direct restatement (Alg. 3) ---------------------------------- */

/* Micro-kernel contract, micro_kernel.hpp:21-38: `in` points at input element
 * (l*s, k'*w_ob*s) of block i', `w` at slab(j', i'), `out` at a contiguous
 * w_ob*c_ob tile.  Load tile, accumulate the full (n, m, ii) slab with kk, jj
 * innermost (jj unit stride), store. */
#define DEF_TILE(COB, WOB)                                                    \
  static void tile_##COB##_##WOB(const float* in, const float* w, float* out, \
                                 int h_f, int w_f, int c_ib, int row_pitch,   \
                                 int col_stride) {                            \
    float acc[WOB][COB];                                                      \
    for (int kk = 0; kk < WOB; ++kk)                                          \
      for (int jj = 0; jj < COB; ++jj) acc[kk][jj] = out[kk * COB + jj];      \
    for (int n = 0; n < h_f; ++n)                                             \
      for (int m = 0; m < w_f; ++m)                                           \
        for (int ii = 0; ii < c_ib; ++ii) {                                   \
          const float* ip = in + (size_t)n * row_pitch + m * c_ib + ii;       \
          const float* wp = w + ((size_t)(n * w_f + m) * c_ib + ii) * COB;    \
          for (int kk = 0; kk < WOB; ++kk) {                                  \
            const float a = ip[(size_t)kk * col_stride];                      \
            for (int jj = 0; jj < COB; ++jj) acc[kk][jj] += a * wp[jj];       \
          }                                                                   \
        }                                                                     \
    for (int kk = 0; kk < WOB; ++kk)                                          \
      for (int jj = 0; jj < COB; ++jj) out[kk * COB + jj] = acc[kk][jj];      \
  }

/* AVX2 register model (model.hpp:63-73 with n_vec=8, n_reg=16, 2 operand
 * registers reserved): (c_ob/8)*w_ob + 2 <= 16. */
DEF_TILE(8, 14)
DEF_TILE(16, 7)
DEF_TILE(32, 3)

/* tile_kernel_generic (micro_kernel.hpp:48-51): runtime sizes, same order */
static void tile_generic(const float* in, const float* w, float* out, int h_f,
                         int w_f, int c_ib, int row_pitch, int col_stride,
                         int c_ob, int w_ob) {
  for (int n = 0; n < h_f; ++n)
    for (int m = 0; m < w_f; ++m)
      for (int ii = 0; ii < c_ib; ++ii) {
        const float* ip = in + (size_t)n * row_pitch + m * c_ib + ii;
        const float* wp = w + ((size_t)(n * w_f + m) * c_ib + ii) * c_ob;
        for (int kk = 0; kk < w_ob; ++kk) {
          const float a = ip[(size_t)kk * col_stride];
          for (int jj = 0; jj < c_ob; ++jj) out[kk * c_ob + jj] += a * wp[jj];
        }
      }
}

typedef void (*tile_fn)(const float*, const float*, float*, int, int, int, int,
                        int);

static tile_fn find_tile(int c_ob, int w_ob) {  /* micro_kernel.hpp:43-46 */
  if (c_ob == 8 && w_ob == 14) return tile_8_14;
  if (c_ob == 16 && w_ob == 7) return tile_16_7;
  if (c_ob == 32 && w_ob == 3) return tile_32_3;
  return NULL;
}

static int conv_direct_impl(const float* in, const float* k, int n_img,
                            int c_i, int c_o, int h_i, int w_i, int h_f,
                            int w_f, int s, int c_ib, int c_ob, int w_ob,
                            int threads, float* out, int literal) {
  int h_o, w_o;
  if (orc_conv_shape(c_i, c_o, h_i, w_i, h_f, w_f, s, &h_o, &w_o)) return -1;
  if (c_ib < 1 || c_ob < 1 || w_ob < 1) return -1;
  const int ib_n = orc_round_up(c_i, c_ib) / c_ib;
  const int jb_n = orc_round_up(c_o, c_ob) / c_ob;
  const size_t in_img = (size_t)ib_n * h_i * w_i * c_ib;
  const size_t out_img = (size_t)jb_n * h_o * w_o * c_ob;
  const size_t out_blk = (size_t)h_o * w_o * c_ob;
  const size_t slab = (size_t)h_f * w_f * c_ib * c_ob;
  const int row_pitch = w_i * c_ib;
  const int col_stride = s * c_ib;
  tile_fn full = literal ? NULL : find_tile(c_ob, w_ob);
  const int units = n_img * jb_n;
#ifdef _OPENMP
  if (threads <= 0) threads = omp_get_max_threads();
#else
  threads = 1;
#endif
  /* j' in parallel; whole-block ownership so the
   * result is bitwise independent of the thread count. */
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads)
  for (int u = 0; u < units; ++u) {
    const int img = u / jb_n, jb = u % jb_n;
    const float* inp = in + (size_t)img * in_img;
    float* ob = out + (size_t)img * out_img + (size_t)jb * out_blk;
    memset(ob, 0, sizeof(float) * out_blk);
    for (int ib = 0; ib < ib_n; ++ib) {               /* i' */
      const float* w = k + ((size_t)jb * ib_n + ib) * slab;  /* tensor.hpp:138-140 */
      const float* inb = inp + (size_t)ib * h_i * w_i * c_ib;
      for (int l = 0; l < h_o; ++l)                   /* l */
        for (int kb = 0; kb * w_ob < w_o; ++kb) {     /* k' */
          const int wob = (w_o - kb * w_ob) < w_ob ? (w_o - kb * w_ob) : w_ob;
          float* ot = ob + ((size_t)l * w_o + (size_t)kb * w_ob) * c_ob;
          if (literal) {
            /* PAPER.md:349 literal: column s*k'*w_ob + kk + m (wrong for s>1) */
            for (int n = 0; n < h_f; ++n)
              for (int m = 0; m < w_f; ++m)
                for (int ii = 0; ii < c_ib; ++ii)
                  for (int kk = 0; kk < wob; ++kk) {
                    const int col = s * kb * w_ob + kk + m;
                    const float a =
                        inb[((size_t)(l * s + n) * w_i + col) * c_ib + ii];
                    const float* wp = w + ((size_t)(n * w_f + m) * c_ib + ii) * c_ob;
                    for (int jj = 0; jj < c_ob; ++jj) ot[kk * c_ob + jj] += a * wp[jj];
                  }
            continue;
          }
          /* stride fix SPEC.md:354: column s*(k'*w_ob + kk) + m */
          const float* it =
              inb + ((size_t)(l * s) * w_i + (size_t)kb * w_ob * s) * c_ib;
          if (full && wob == w_ob)
            full(it, w, ot, h_f, w_f, c_ib, row_pitch, col_stride);
          else  /* edge tile, identical order */
            tile_generic(it, w, ot, h_f, w_f, c_ib, row_pitch, col_stride,
                         c_ob, wob);
        }
    }
  }
  return 0;
}

int orc_conv_direct(const float* in, const float* k, int n_img, int c_i,
                    int c_o, int h_i, int w_i, int h_f, int w_f, int s,
                    int c_ib, int c_ob, int w_ob, int threads, float* out) {
  return conv_direct_impl(in, k, n_img, c_i, c_o, h_i, w_i, h_f, w_f, s, c_ib,
                          c_ob, w_ob, threads, out, 0);
}

int orc_conv_direct_literal_alg3(const float* in, const float* k, int c_i,
                                 int c_o, int h_i, int w_i, int h_f, int w_f,
                                 int s, int c_ib, int c_ob, int w_ob,
                                 float* out) {
  /* the literal index can run past the row for s > 1; callers pass inputs
   * large enough or accept garbage -- we clamp by construction in the test */
  return conv_direct_impl(in, k, 1, c_i, c_o, h_i, w_i, h_f, w_f, s, c_ib,
                          c_ob, w_ob, 1, out, 1);
}

void orc_relu(float* x, int64_t n) {
  for (int64_t i = 0; i < n; ++i) x[i] = x[i] > 0.0f ? x[i] : 0.0f;
}

void orc_add(const float* a, const float* b, float* out, int64_t n) {
  for (int64_t i = 0; i < n; ++i) out[i] = a[i] + b[i];
}

void orc_maxpool2x2(const float* in, int n_cblk, int h, int w, int c_b,
                    float* out) {
  const int ho = h / 2, wo = w / 2;
  for (int b = 0; b < n_cblk; ++b)
    for (int y = 0; y < ho; ++y)
      for (int x = 0; x < wo; ++x)
        for (int c = 0; c < c_b; ++c) {
          const float* p = in + (((size_t)b * h + 2 * y) * w + 2 * x) * c_b + c;
          float v = p[0];
          float t = p[c_b];
          v = t > v ? t : v;
          t = p[(size_t)w * c_b];
          v = t > v ? t : v;
          t = p[(size_t)w * c_b + c_b];
          v = t > v ? t : v;
          out[(((size_t)b * ho + y) * wo + x) * c_b + c] = v;
        }
}

static inline uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

void orc_fill_uniform(float* dst, int64_t n, uint64_t seed, uint64_t stream) {
  const uint64_t base = seed * 0xD1B54A32D192ED03ULL ^ (stream * 0x8CB92BA72F3D8DD7ULL);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    const uint64_t r = splitmix64(base + (uint64_t)i);
    /* 24-bit integer in [0, 2^24) -> exactly representable value in [-1, 1) */
    dst[i] = (float)(int32_t)(r >> 40) * (1.0f / 8388608.0f) - 1.0f;
  }
}
