/*
 * oracle.h -- CPU restatement of the reference `dconv` hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (paper_1809_10170_b200/,
 * include/) may link or call this library.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs load it, as the checker or
 * the timed CPU baseline.
 *
 * Every function cites the reference file:line it restates (paths relative to
 * /root/reference/proj/core/).  Parity of this restatement with the reference
 * itself is pinned by tests/test_oracle.py against oracle/_ref (the reference
 * sources compiled unmodified, see oracle/Makefile) and against the SPEC.md
 * known-answer examples committed in tests/golden/.
 *
 * Layouts (all fp32):
 *   dense map     [C][H][W]                                tensor.hpp:33-48
 *   blocked map   [ceil(C/c_b)][H][W][c_b] (zero padded)   tensor.hpp:50-81
 *   dense kernel  [C_i][C_o][H_f][W_f]                     tensor.hpp:83-103
 *   blocked kern  [C_o/c_ob][C_i/c_ib][H_f][W_f][c_ib][c_ob]  tensor.hpp:105-141
 * The batched variants add an outermost image dimension; each image slice is
 * byte-identical to the reference's batch-1 type.
 */
#ifndef DCONV_ORACLE_H
#define DCONV_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ConvShape (shape.hpp:29-45, ctor shape.cpp:30-40).  Returns 0 and fills
 * h_o/w_o on success, -1 (the reference throws std::invalid_argument) on an
 * invalid geometry. */
int orc_conv_shape(int c_i, int c_o, int h_i, int w_i, int h_f, int w_f,
                   int stride, int* h_o, int* w_o);

/* detail::round_up (tensor.hpp:28-30). */
int orc_round_up(int value, int block);

/* conv_flops (reference.cpp:106-109): 2*c_i*c_o*h_o*w_o*h_f*w_f. */
int64_t orc_conv_flops(int c_i, int c_o, int h_o, int w_o, int h_f, int w_f);

/* pack_feature_map / unpack_feature_map (tensor.cpp:65-83).  `dst` of the
 * pack must hold round_up(c, c_b)*h*w floats; it is fully written (padding
 * channels set to exact 0). */
void orc_pack_feature_map(const float* src, int c, int h, int w, int c_b,
                          float* dst);
void orc_unpack_feature_map(const float* src, int c, int h, int w, int c_b,
                            float* dst);

/* pack_kernel / unpack_kernel (tensor.cpp:85-108). */
void orc_pack_kernel(const float* src, int c_i, int c_o, int h_f, int w_f,
                     int c_ob, int c_ib, float* dst);
void orc_unpack_kernel(const float* src, int c_i, int c_o, int h_f, int w_f,
                       int c_ob, int c_ib, float* dst);

/* conv_oracle64 (reference.cpp:70-87): Alg. 1 loop order, fp64 accumulation,
 * rounded to fp32 once.  Dense CHW in/out, dense [C_i][C_o][H_f][W_f] kernel. */
void orc_conv_oracle64(const float* in, const float* k, int c_i, int c_o,
                       int h_i, int w_i, int h_f, int w_f, int stride,
                       float* out);

/* conv_naive (reference.cpp:34-52): same order, fp32 accumulation. */
void orc_conv_naive(const float* in, const float* k, int c_i, int c_o, int h_i,
                    int w_i, int h_f, int w_f, int stride, float* out);

/* conv_oracle64 evaluated directly on blocked buffers (same arithmetic, same
 * (i, n, m) summation order per output as reference.cpp:75-83), for big
 * parity cases: avoids the unpack.  in: [c_i/c_ib][h_i][w_i][c_ib] of one
 * image; k: blocked kernel; out: blocked [c_o/c_ob][h_o][w_o][c_ob] (padding
 * channels written as 0).  Output pixels restricted to rows [y0, y1). */
void orc_conv_oracle64_blocked(const float* in, const float* k, int c_i,
                               int c_o, int h_i, int w_i, int h_f, int w_f,
                               int stride, int c_ib, int c_ob, int y0, int y1,
                               float* out);

/* conv_direct restated from SPEC.md:306-358 and PAPER.md:326-363 (Alg. 3):
 *   j' (parallel, whole-block ownership) -> i' -> l -> k' -> n -> m -> ii ->
 *   kk -> jj, input index s*(k'*w_ob + kk) + m (SPEC.md:354 stride fix),
 *   output zero-initialised once, fp32 FMA.
 * `n_img` images are processed; parallel units are (image, j') pairs, run on
 * `threads` OpenMP threads (<=0: all).  Output fully written.
 * Returns 0, or -1 on a layout/parameter error. */
int orc_conv_direct(const float* in, const float* k, int n_img, int c_i,
                    int c_o, int h_i, int w_i, int h_f, int w_f, int stride,
                    int c_ib, int c_ob, int w_ob, int threads, float* out);

/* The same computation split into its parallel units (image, j', row band),
 * for an external scheduler: the reference's ThreadPool (thread_pool.cpp:64-97)
 * runs orc_direct_job_unit over [0, units) in oracle/ref_shim.cpp. */
typedef struct orc_direct_job {
  const float* in;
  const float* k;
  float* out;
  int n_img, c_i, c_o, h_i, w_i, h_f, w_f, s, c_ib, c_ob, w_ob, h_o, w_o;
  int ib_n, jb_n, bands, rows_per, units;
} orc_direct_job;
/* Returns the unit count (bands sized for `threads`), or -1 on a shape or
 * parameter error. */
int orc_direct_job_init(orc_direct_job* job, const float* in, const float* k, int n_img,
                        int c_i, int c_o, int h_i, int w_i, int h_f, int w_f, int stride,
                        int c_ib, int c_ob, int w_ob, int threads, float* out);
void orc_direct_job_unit(const orc_direct_job* job, int u);

/* The paper's literal Alg. 3 input index s*k'*w_ob + kk + m,
 * kept only for the mutation test of SPEC.md:622. */
int orc_conv_direct_literal_alg3(const float* in, const float* k, int c_i,
                                 int c_o, int h_i, int w_i, int h_f, int w_f,
                                 int stride, int c_ib, int c_ob, int w_ob,
                                 float* out);

/* relu_blocked: in place max(e, 0) over n floats. */
void orc_relu(float* x, int64_t n);
/* skip-add (not in the reference; "element-wise"): out = a + b. */
void orc_add(const float* a, const float* b, float* out, int64_t n);
/* 2x2 stride-2 max-pool on one blocked image [cb][h][w][c_b] -> [cb][h/2][w/2][c_b]
 * (not in the reference, SPEC.md:20 lists pooling out of scope there). */
void orc_maxpool2x2(const float* in, int n_cblk, int h, int w, int c_b,
                    float* out);

/* Counter-based uniform[-1,1) generator shared by tests and bench:
 * value i of stream (seed, stream) = splitmix64(seed ^ stream*K + i) -> 24-bit
 * mantissa.  Deterministic across platforms; see DESIGN.md "Synthetic data". */
void orc_fill_uniform(float* dst, int64_t n, uint64_t seed, uint64_t stream);

#ifdef __cplusplus
}
#endif
#endif
