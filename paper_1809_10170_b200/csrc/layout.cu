// layout.cu -- layout transforms and element-wise / pooling kernels in the
// blocked layout.  All are HBM-bound; each thread owns one (or four, vector)
// destination elements so stores are fully coalesced.
//
//   pack_kernel_dev   <- pack_kernel        tensor.cpp:85-95  (bit-exact)
//   unpack_kernel_dev <- unpack_kernel      tensor.cpp:97-108
//   pack_fm_dev       <- pack_feature_map   tensor.cpp:65-73  (+ optional halo)
//   unpack_fm_dev     <- unpack_feature_map tensor.cpp:75-83
//   relu / add        <- relu_blocked SPEC.md:326-334, skip layer PAPER.md:4-7
//   maxpool2x2        <- subsampling layer PAPER.md:9-10
#include "common.cuh"
#include "layout_kernels.h"

namespace dconv_dev {

namespace {

int grid_for(int64_t total, int per_thread = 1) {
  int64_t blocks = (total / per_thread + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  if (blocks < 1) blocks = 1;
  return (int)blocks;
}

struct PeerList {
  float* p[8];
  int n;
};

#define GRID_STRIDE(e, total)                                            \
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (total); \
       e += (int64_t)gridDim.x * blockDim.x)

__global__ void pack_kernel_dev(const float* __restrict__ src, int c_i, int c_o,
                                int h_f, int w_f, int c_ob, int c_ib,
                                int ib_n, int64_t total,
                                float* __restrict__ dst) {
  GRID_STRIDE(e, total) {
    int64_t t = e;
    const int jj = (int)(t % c_ob); t /= c_ob;
    const int ii = (int)(t % c_ib); t /= c_ib;
    const int m = (int)(t % w_f); t /= w_f;
    const int n = (int)(t % h_f); t /= h_f;
    const int ib = (int)(t % ib_n); t /= ib_n;
    const int jb = (int)t;
    const int i = ib * c_ib + ii, j = jb * c_ob + jj;
    dst[e] = (i < c_i && j < c_o)
                 ? src[(((int64_t)i * c_o + j) * h_f + n) * w_f + m]
                 : 0.0f;
  }
}

__global__ void unpack_kernel_dev(const float* __restrict__ src, int c_i,
                                  int c_o, int h_f, int w_f, int c_ob, int c_ib,
                                  int ib_n, int64_t total,
                                  float* __restrict__ dst) {
  GRID_STRIDE(e, total) {
    int64_t t = e;
    const int m = (int)(t % w_f); t /= w_f;
    const int n = (int)(t % h_f); t /= h_f;
    const int j = (int)(t % c_o); t /= c_o;
    const int i = (int)t;
    dst[e] = src[(((((int64_t)(j / c_ob) * ib_n + i / c_ib) * h_f + n) * w_f +
                   m) * c_ib + i % c_ib) * c_ob + j % c_ob];
  }
}

__global__ void pack_fm_dev(const float* __restrict__ src, int c, int h, int w,
                            int c_b, int halo, int nb, int64_t total,
                            float* __restrict__ dst) {
  const int hp = h + 2 * halo, wp = w + 2 * halo;
  GRID_STRIDE(e, total) {
    int64_t t = e;
    const int cc = (int)(t % c_b); t /= c_b;
    const int xp = (int)(t % wp); t /= wp;
    const int yp = (int)(t % hp); t /= hp;
    const int b = (int)(t % nb); t /= nb;
    const int img = (int)t;
    const int ch = b * c_b + cc, y = yp - halo, x = xp - halo;
    dst[e] = (ch < c && y >= 0 && y < h && x >= 0 && x < w)
                 ? src[(((int64_t)img * c + ch) * h + y) * w + x]
                 : 0.0f;
  }
}

// c_b = 8: one thread per output pencil (8 channel reads, each coalesced
// across x; two float4 stores), 32-bit index math per pencil.
__global__ void pack_fm8_dev(const float* __restrict__ src, int c, int h, int w, int halo,
                             int nb, int64_t pencils, float* __restrict__ dst) {
  const int hp = h + 2 * halo, wp = w + 2 * halo;
  GRID_STRIDE(e, pencils) {
    int64_t t = e;
    const int xp = (int)(t % wp); t /= wp;
    const int yp = (int)(t % hp); t /= hp;
    const int b = (int)(t % nb);
    const int img = (int)(t / nb);
    const int y = yp - halo, x = xp - halo;
    float v[8];
    const bool in = y >= 0 && y < h && x >= 0 && x < w;
    const float* s = src + (((int64_t)img * c + b * 8) * h + y) * w + x;
#pragma unroll
    for (int cc = 0; cc < 8; ++cc)
      v[cc] = (in && b * 8 + cc < c) ? __ldg(s + (int64_t)cc * h * w) : 0.0f;
    float4* d = reinterpret_cast<float4*>(dst + e * 8);
    d[0] = make_float4(v[0], v[1], v[2], v[3]);
    d[1] = make_float4(v[4], v[5], v[6], v[7]);
  }
}

// Space-to-depth + block packing of a dense image batch: output channel
// cs = (dy*f + dx)*c + ch of the s2d map is input (ch, s*ys + dy, s*xs + dx);
// [n][ceil(c*f*f/8)][hs][ws][8], zero outside the image and in pad channels.
__global__ void pack_s2d8_dev(const float* __restrict__ src, int c, int h, int w, int f,
                              int hs, int ws, int nb, int64_t pencils, float* __restrict__ dst) {
  const int cs_n = c * f * f;
  GRID_STRIDE(e, pencils) {
    int64_t t = e;
    const int xs = (int)(t % ws); t /= ws;
    const int ys = (int)(t % hs); t /= hs;
    const int b = (int)(t % nb);
    const int img = (int)(t / nb);
    float v[8];
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) {
      const int cs = b * 8 + cc;
      float x = 0.0f;
      if (cs < cs_n) {
        const int ch = cs % c, d = cs / c, dy = d / f, dx = d % f;
        const int y = ys * f + dy, xx = xs * f + dx;
        if (y < h && xx < w) x = __ldg(src + (((int64_t)img * c + ch) * h + y) * w + xx);
      }
      v[cc] = x;
    }
    float4* d4 = reinterpret_cast<float4*>(dst + e * 8);
    d4[0] = make_float4(v[0], v[1], v[2], v[3]);
    d4[1] = make_float4(v[4], v[5], v[6], v[7]);
  }
}

// The same pack for the 3-channel network input with a compile-time factor F:
// one thread per s2d output pixel (xs fastest across lanes) gathers all
// 3*F*F values -- per (channel, input row) F consecutive words, so a warp's
// loads cover one contiguous span of the input row -- with no index
// divisions, then writes its NB pencils (two 16-byte stores each).  The
// element-per-thread form above spends its time on the per-element index
// arithmetic (1.5 TB/s on the GoogLeNet stem at b64).
template <int F>
__global__ void pack_s2d3_dev(const float* __restrict__ src, int h, int w, int hs, int ws,
                              int64_t pixels, float* __restrict__ dst) {
  constexpr int C = 3, CS = C * F * F, NB = (CS + 7) / 8;
  GRID_STRIDE(e, pixels) {
    int64_t t = e;
    const int xs = (int)(t % ws); t /= ws;
    const int ys = (int)(t % hs);
    const int img = (int)(t / hs);
    float v[NB * 8];
#pragma unroll
    for (int i = CS; i < NB * 8; ++i) v[i] = 0.0f;
#pragma unroll
    for (int dy = 0; dy < F; ++dy) {
      const int y = ys * F + dy;
#pragma unroll
      for (int ch = 0; ch < C; ++ch) {
        const float* row = src + (((int64_t)img * C + ch) * h + y) * w;
#pragma unroll
        for (int dx = 0; dx < F; ++dx) {
          const int xx = xs * F + dx;
          v[(dy * F + dx) * C + ch] = (y < h && xx < w) ? __ldg(row + xx) : 0.0f;
        }
      }
    }
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      float4* d4 = reinterpret_cast<float4*>(
          dst + ((((int64_t)img * NB + b) * hs + ys) * ws + xs) * 8);
      d4[0] = make_float4(v[b * 8], v[b * 8 + 1], v[b * 8 + 2], v[b * 8 + 3]);
      d4[1] = make_float4(v[b * 8 + 4], v[b * 8 + 5], v[b * 8 + 6], v[b * 8 + 7]);
    }
  }
}

// Space-to-depth of a blocked map view (c_b = 8 in and out): output channel
// cs = (dy*f + dx)*c + ch at (ys, xs) is input channel ch at (f*ys+dy, f*xs+dx).
__global__ void s2d_blocked8_dev(const float* __restrict__ src, int64_t in_img, int64_t in_blk,
                                 int64_t in_row, int c, int h, int w, int f, int hs, int ws,
                                 int nb, int64_t pencils, float* __restrict__ dst) {
  const int cs_n = c * f * f;
  GRID_STRIDE(e, pencils) {
    int64_t t = e;
    const int xs = (int)(t % ws); t /= ws;
    const int ys = (int)(t % hs); t /= hs;
    const int b = (int)(t % nb);
    const int img = (int)(t / nb);
    float4* d4 = reinterpret_cast<float4*>(dst + e * 8);
    if ((c & 7) == 0) {
      // C a multiple of 8: an output pencil is one whole input pencil
      const int d = (b * 8) / c, ch0 = b * 8 - d * c, dy = d / f, dx = d % f;
      const int y = ys * f + dy, xx = xs * f + dx;
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f), q = a;
      if (y < h && xx < w) {
        const float4* sp = reinterpret_cast<const float4*>(
            src + img * in_img + (ch0 >> 3) * in_blk + y * in_row + (int64_t)xx * 8);
        a = __ldg(sp);
        q = __ldg(sp + 1);
      }
      d4[0] = a;
      d4[1] = q;
      continue;
    }
    float v[8];
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) {
      const int cs = b * 8 + cc;
      float x = 0.0f;
      if (cs < cs_n) {
        const int ch = cs % c, d = cs / c, dy = d / f, dx = d % f;
        const int y = ys * f + dy, xx = xs * f + dx;
        if (y < h && xx < w)
          x = __ldg(src + img * in_img + (ch >> 3) * in_blk + y * in_row + (int64_t)xx * 8 + (ch & 7));
      }
      v[cc] = x;
    }
    d4[0] = make_float4(v[0], v[1], v[2], v[3]);
    d4[1] = make_float4(v[4], v[5], v[6], v[7]);
  }
}

__global__ void unpack_fm_dev(const float* __restrict__ src, int c, int h,
                              int w, int c_b, int halo, int nb, int64_t total,
                              float* __restrict__ dst) {
  const int hp = h + 2 * halo, wp = w + 2 * halo;
  GRID_STRIDE(e, total) {
    int64_t t = e;
    const int x = (int)(t % w); t /= w;
    const int y = (int)(t % h); t /= h;
    const int ch = (int)(t % c); t /= c;
    const int img = (int)t;
    dst[e] = src[((((int64_t)img * nb + ch / c_b) * hp + y + halo) * wp + x +
                  halo) * c_b + ch % c_b];
  }
}

__global__ void relu4_dev(float4* x, int64_t n4) {
  GRID_STRIDE(e, n4) {
    float4 v = x[e];
    v.x = fmaxf(v.x, 0.f); v.y = fmaxf(v.y, 0.f);
    v.z = fmaxf(v.z, 0.f); v.w = fmaxf(v.w, 0.f);
    x[e] = v;
  }
}

__global__ void relu1_dev(float* x, int64_t n) {
  GRID_STRIDE(e, n) x[e] = fmaxf(x[e], 0.f);
}

__global__ void add4_dev(const float4* a, const float4* b, float4* o,
                         int64_t n4, int relu) {
  GRID_STRIDE(e, n4) {
    const float4 u = a[e], v = b[e];
    float4 r = make_float4(u.x + v.x, u.y + v.y, u.z + v.z, u.w + v.w);
    if (relu) {
      r.x = fmaxf(r.x, 0.f); r.y = fmaxf(r.y, 0.f);
      r.z = fmaxf(r.z, 0.f); r.w = fmaxf(r.w, 0.f);
    }
    o[e] = r;
  }
}

__global__ void add1_dev(const float* a, const float* b, float* o, int64_t n,
                         int relu) {
  GRID_STRIDE(e, n) {
    const float r = a[e] + b[e];
    o[e] = relu ? fmaxf(r, 0.f) : r;
  }
}

// one thread per output element of [img][blk][ho][wo][c_b]
__global__ void maxpool2x2_dev(const float* __restrict__ in, int n_blocks,
                               int h, int w, int c_b, int64_t total,
                               float* __restrict__ out, int64_t o_img,
                               int64_t o_blk, int64_t o_row) {
  const int ho = h / 2, wo = w / 2;
  GRID_STRIDE(e, total) {
    int64_t t = e;
    const int cc = (int)(t % c_b); t /= c_b;
    const int x = (int)(t % wo); t /= wo;
    const int y = (int)(t % ho); t /= ho;
    const int b = (int)(t % n_blocks); t /= n_blocks;
    const int img = (int)t;
    const float* p =
        in + ((((int64_t)img * n_blocks + b) * h + 2 * y) * w + 2 * x) * c_b + cc;
    float v = p[0];
    v = fmaxf(v, p[c_b]);
    v = fmaxf(v, p[(int64_t)w * c_b]);
    v = fmaxf(v, p[(int64_t)w * c_b + c_b]);
    out[(int64_t)img * o_img + (int64_t)b * o_blk + (int64_t)y * o_row +
        (int64_t)x * c_b + cc] = v;
  }
}

// c_b = 8: one thread per output pencil, 16-byte loads/stores (the pool is
// HBM-bound: 4 input pencils read, one written)
__device__ __forceinline__ float4 max4(float4 a, float4 b) {
  return make_float4(fmaxf(a.x, b.x), fmaxf(a.y, b.y), fmaxf(a.z, b.z), fmaxf(a.w, b.w));
}
__global__ void maxpool2x2_8_dev(const float* __restrict__ in, int n_blocks, int h, int w,
                                 int64_t pencils, float* __restrict__ out, int64_t o_img,
                                 int64_t o_blk, int64_t o_row) {
  const int ho = h / 2, wo = w / 2;
  GRID_STRIDE(e, pencils) {
    int64_t t = e;
    const int x = (int)(t % wo); t /= wo;
    const int y = (int)(t % ho); t /= ho;
    const int b = (int)(t % n_blocks);
    const int img = (int)(t / n_blocks);
    const float4* p = reinterpret_cast<const float4*>(
        in + ((((int64_t)img * n_blocks + b) * h + 2 * y) * w + 2 * x) * 8);
    const int64_t r4 = (int64_t)w * 2;  // one input row in float4 units
    const float4 a = max4(max4(__ldg(p), __ldg(p + 2)), max4(__ldg(p + r4), __ldg(p + r4 + 2)));
    const float4 c = max4(max4(__ldg(p + 1), __ldg(p + 3)),
                          max4(__ldg(p + r4 + 1), __ldg(p + r4 + 3)));
    float4* o = reinterpret_cast<float4*>(out + (int64_t)img * o_img + (int64_t)b * o_blk +
                                          (int64_t)y * o_row + (int64_t)x * 8);
    o[0] = a;
    o[1] = c;
  }
}

// fused C_o-shard gather of a first layer run on the TMA-store reader (which
// writes this rank's map only): the rank's blocks, one 32-byte pencil per
// thread, copied from its own map into every peer's copy at the same offset
// (NVLink stores).  The values are the reader's, so every rank's copy is
// bitwise the all-gathered map.
__global__ void copy_pencils_peers_dev(const float* __restrict__ src, int n_blocks, int h,
                                       int w, int64_t pencils, int64_t img_s, int64_t blk_s,
                                       int64_t row_s, PeerList peers) {
  GRID_STRIDE(e, pencils) {
    int64_t t = e;
    const int x = (int)(t % w); t /= w;
    const int y = (int)(t % h); t /= h;
    const int b = (int)(t % n_blocks);
    const int img = (int)(t / n_blocks);
    const int64_t off = (int64_t)img * img_s + (int64_t)b * blk_s + (int64_t)y * row_s +
                        (int64_t)x * 8;
    const float4 a = __ldg(reinterpret_cast<const float4*>(src + off));
    const float4 c = __ldg(reinterpret_cast<const float4*>(src + off + 4));
    for (int q = 0; q < peers.n; ++q) {
      float4* o = reinterpret_cast<float4*>(peers.p[q] + off);
      o[0] = a;
      o[1] = c;
    }
  }
}

}  // namespace

int launch_pack_kernel(const float* src, int c_i, int c_o, int h_f, int w_f,
                       int c_ob, int c_ib, float* dst, cudaStream_t st) {
  const int ib_n = (c_i + c_ib - 1) / c_ib, jb_n = (c_o + c_ob - 1) / c_ob;
  const int64_t total = (int64_t)jb_n * ib_n * h_f * w_f * c_ib * c_ob;
  pack_kernel_dev<<<grid_for(total), 256, 0, st>>>(src, c_i, c_o, h_f, w_f,
                                                   c_ob, c_ib, ib_n, total, dst);
  dconv_host::count_launch();
  return dconv_host::check_launch("pack_kernel_dev");
}

int launch_unpack_kernel(const float* src, int c_i, int c_o, int h_f, int w_f,
                         int c_ob, int c_ib, float* dst, cudaStream_t st) {
  const int ib_n = (c_i + c_ib - 1) / c_ib;
  const int64_t total = (int64_t)c_i * c_o * h_f * w_f;
  unpack_kernel_dev<<<grid_for(total), 256, 0, st>>>(
      src, c_i, c_o, h_f, w_f, c_ob, c_ib, ib_n, total, dst);
  dconv_host::count_launch();
  return dconv_host::check_launch("unpack_kernel_dev");
}

int launch_pack_fm(const float* src, int n, int c, int h, int w, int c_b,
                   int halo, float* dst, cudaStream_t st) {
  const int nb = (c + c_b - 1) / c_b;
  const int64_t total =
      (int64_t)n * nb * (h + 2 * halo) * (w + 2 * halo) * c_b;
  if (c_b == 8 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
    pack_fm8_dev<<<grid_for(total / 8), 256, 0, st>>>(src, c, h, w, halo, nb, total / 8, dst);
    dconv_host::count_launch();
    return dconv_host::check_launch("pack_fm8_dev");
  }
  pack_fm_dev<<<grid_for(total), 256, 0, st>>>(src, c, h, w, c_b, halo, nb,
                                               total, dst);
  dconv_host::count_launch();
  return dconv_host::check_launch("pack_fm_dev");
}

int launch_pack_s2d(const float* src, int n, int c, int h, int w, int f, float* dst,
                    cudaStream_t st) {
  const int hs = (h + f - 1) / f, ws = (w + f - 1) / f;
  const int nb = (c * f * f + 7) / 8;
  const int64_t pencils = (int64_t)n * nb * hs * ws;
  if (c == 3 && (f == 2 || f == 4) && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
    const int64_t pixels = (int64_t)n * hs * ws;
    if (f == 2)
      pack_s2d3_dev<2><<<grid_for(pixels), 256, 0, st>>>(src, h, w, hs, ws, pixels, dst);
    else
      pack_s2d3_dev<4><<<grid_for(pixels), 256, 0, st>>>(src, h, w, hs, ws, pixels, dst);
    dconv_host::count_launch();
    return dconv_host::check_launch("pack_s2d3_dev");
  }
  pack_s2d8_dev<<<grid_for(pencils), 256, 0, st>>>(src, c, h, w, f, hs, ws, nb, pencils, dst);
  dconv_host::count_launch();
  return dconv_host::check_launch("pack_s2d8_dev");
}

int launch_s2d_blocked(const float* src, int64_t in_img, int64_t in_blk, int64_t in_row, int n,
                       int c, int h, int w, int f, float* dst, cudaStream_t st) {
  const int hs = (h + f - 1) / f, ws = (w + f - 1) / f;
  const int nb = (c * f * f + 7) / 8;
  const int64_t pencils = (int64_t)n * nb * hs * ws;
  s2d_blocked8_dev<<<grid_for(pencils), 256, 0, st>>>(src, in_img, in_blk, in_row, c, h, w, f, hs,
                                                      ws, nb, pencils, dst);
  dconv_host::count_launch();
  return dconv_host::check_launch("s2d_blocked8_dev");
}

int launch_unpack_fm(const float* src, int n, int c, int h, int w, int c_b,
                     int halo, float* dst, cudaStream_t st) {
  const int nb = (c + c_b - 1) / c_b;
  const int64_t total = (int64_t)n * c * h * w;
  unpack_fm_dev<<<grid_for(total), 256, 0, st>>>(src, c, h, w, c_b, halo, nb,
                                                 total, dst);
  dconv_host::count_launch();
  return dconv_host::check_launch("unpack_fm_dev");
}

int launch_relu(float* x, int64_t count, cudaStream_t st) {
  if (count % 4 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0) {
    relu4_dev<<<grid_for(count / 4), 256, 0, st>>>(
        reinterpret_cast<float4*>(x), count / 4);
  } else {
    relu1_dev<<<grid_for(count), 256, 0, st>>>(x, count);
  }
  dconv_host::count_launch();
  return dconv_host::check_launch("relu_dev");
}

int launch_add(const float* a, const float* b, float* o, int64_t count,
               int relu, cudaStream_t st) {
  const bool vec = count % 4 == 0 &&
                   ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b) |
                     reinterpret_cast<uintptr_t>(o)) & 15) == 0;
  if (vec)
    add4_dev<<<grid_for(count / 4), 256, 0, st>>>(
        reinterpret_cast<const float4*>(a), reinterpret_cast<const float4*>(b),
        reinterpret_cast<float4*>(o), count / 4, relu);
  else
    add1_dev<<<grid_for(count), 256, 0, st>>>(a, b, o, count, relu);
  dconv_host::count_launch();
  return dconv_host::check_launch("add_dev");
}

int launch_copy_pencils_peers(const float* src, int n, int n_blocks, int h, int w,
                              int64_t img_s, int64_t blk_s, int64_t row_s,
                              float* const* peers, int n_peers, cudaStream_t st) {
  PeerList pl{};
  pl.n = n_peers;
  for (int q = 0; q < n_peers; ++q) pl.p[q] = peers[q];
  const int64_t pencils = (int64_t)n * n_blocks * h * w;
  copy_pencils_peers_dev<<<grid_for(pencils), 256, 0, st>>>(src, n_blocks, h, w, pencils, img_s,
                                                            blk_s, row_s, pl);
  dconv_host::count_launch();
  return dconv_host::check_launch("copy_pencils_peers_dev");
}

int launch_maxpool2x2(const float* in, int n, int n_blocks, int h, int w,
                      int c_b, float* out, int64_t o_img, int64_t o_blk,
                      int64_t o_row, cudaStream_t st) {
  const int64_t total = (int64_t)n * n_blocks * (h / 2) * (w / 2) * c_b;
  if (c_b == 8 && ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15) == 0 &&
      ((o_img | o_blk | o_row) & 3) == 0) {
    maxpool2x2_8_dev<<<grid_for(total / 8), 256, 0, st>>>(in, n_blocks, h, w, total / 8, out,
                                                          o_img, o_blk, o_row);
    dconv_host::count_launch();
    return dconv_host::check_launch("maxpool2x2_8_dev");
  }
  maxpool2x2_dev<<<grid_for(total), 256, 0, st>>>(in, n_blocks, h, w, c_b,
                                                  total, out, o_img, o_blk,
                                                  o_row);
  dconv_host::count_launch();
  return dconv_host::check_launch("maxpool2x2_dev");
}

}  // namespace dconv_dev
