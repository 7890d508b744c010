// Convolution-as-GEMM data movement and pooling for the CNN problems
// (LeNet / CIFAR-quick / AlexNet). The reference has no convolution
// (SPEC.md:67); these follow the conventions fixed in oracle/esgd_oracle.py
// (conv weights (out, in, kh, kw) row-major; im2col column order
// (ci, ky, kx); max-pool argmax = first max in (ky, kx) scan order).
//
// Backward passes use the gather form with a fixed (ky, kx) / (oy, ox)
// accumulation order, so they are deterministic and need no atomics; the
// order equals the oracle's sequential np.add.at order.
#include "esgd_common.cuh"

namespace esgd {
namespace {

__device__ __forceinline__ int64_t off4(const esgd_tensor4& t, int64_t n, int64_t c, int64_t h,
                                        int64_t w) {
  return n * t.sn + c * t.sc + h * t.sh + w * t.sw;
}

// im2col, col element (pix, k) at col[pix*col_sp + k*col_sk]. Threads walk
// the unit-stride side of the destination so stores coalesce: k-fastest for
// the row layout (col_sk == 1), pixel-fastest for the transposed layout the
// engine uses (col_sp == 1; reads then also coalesce along ox).
// 32-bit index math (host checks the sizes).
template <bool PIX_FAST>
__global__ void __launch_bounds__(256) k_im2col(float* __restrict__ col, int64_t col_sp, int64_t col_sk,
                                                int64_t col_sb, const float* __restrict__ x,
                                                esgd_tensor4 xd, int64_t x_sb, int kh, int kw,
                                                int stride, int pad, int oh, int ow) {
  const int z = blockIdx.y;
  const int np = xd.n * oh * ow, khw = kh * kw, kdim = xd.c * khw, ohw = oh * ow;
  const unsigned total = (unsigned)np * (unsigned)kdim;
  const float* xz = x + z * x_sb;
  float* cz = col + z * col_sb;
  for (unsigned e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    int pix, k;
    if (PIX_FAST) { k = (int)(e / (unsigned)np); pix = (int)(e - (unsigned)k * np); }
    else { pix = (int)(e / (unsigned)kdim); k = (int)(e - (unsigned)pix * kdim); }
    const int img = pix / ohw, p = pix - img * ohw;
    const int oy = p / ow, ox = p - oy * ow;
    const int ci = k / khw, r = k - ci * khw;
    const int ky = r / kw, kx = r - ky * kw;
    const int iy = oy * stride - pad + ky, ix = ox * stride - pad + kx;
    float v = 0.f;
    if (iy >= 0 && iy < xd.h && ix >= 0 && ix < xd.w)
      v = __ldg(xz + img * xd.sn + ci * xd.sc + iy * xd.sh + ix * xd.sw);
    cz[pix * col_sp + k * col_sk] = v;
  }
}

// col2im (gather form): dx(img, ci, y, x) = sum over (ky, kx) in fixed order
// of the dcol entries that im2col took from (y, x). Thread order is
// x-fastest, so both the dcol reads (transposed layout) and the dx writes of
// the CNHW engine layout coalesce.
__global__ void __launch_bounds__(256) k_col2im(float* __restrict__ dx, esgd_tensor4 xd,
                                                int64_t x_sb, const float* __restrict__ dcol,
                                                int64_t col_sp, int64_t col_sk, int64_t col_sb, int kh,
                                                int kw, int stride, int pad, int oh, int ow,
                                                const float* __restrict__ mask, int64_t mask_sb) {
  const int z = blockIdx.y;
  const unsigned total = (unsigned)xd.n * xd.c * xd.h * xd.w;
  const float* dz = dcol + z * col_sb;
  for (unsigned e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    unsigned t = e;
    const int xw = (int)(t % (unsigned)xd.w); t /= (unsigned)xd.w;
    const int yh = (int)(t % (unsigned)xd.h); t /= (unsigned)xd.h;
    const int img = (int)(t % (unsigned)xd.n);
    const int ci = (int)(t / (unsigned)xd.n);
    float acc = 0.f;
    for (int ky = 0; ky < kh; ++ky) {
      const int ny = yh + pad - ky;
      if (ny < 0 || ny % stride) continue;
      const int oy = ny / stride;
      if (oy >= oh) continue;
      for (int kx = 0; kx < kw; ++kx) {
        const int nx = xw + pad - kx;
        if (nx < 0 || nx % stride) continue;
        const int ox = nx / stride;
        if (ox >= ow) continue;
        const int pix = (img * oh + oy) * ow + ox;
        acc += __ldg(dz + pix * col_sp + ((ci * kh + ky) * kw + kx) * col_sk);
      }
    }
    const int64_t o = img * xd.sn + ci * xd.sc + yh * xd.sh + xw * xd.sw;
    if (mask) acc = __fmul_rn(acc, mask[z * mask_sb + o] > 0.f ? 1.f : 0.f);
    dx[z * x_sb + o] = acc;
  }
}

// ---- engine variants: thread <-> pixel of the whole batch (b*OH*OW), the
// pixel decomposition is done once and reused over a group of 16 k / channel
// values taken from blockIdx.y, so the inner loop is address math + one
// coalesced load and store (no per-element divisions) -------------------------
constexpr int kGroup = 16;

// channels / k values per thread: amortise the pixel decomposition over up to
// kGroup of them, but keep >= ~2 waves of threads (small LeNet layers)
inline int pick_group(int64_t pixels, int64_t count) {
  const int64_t want_threads = (int64_t)kNumSMs * 2048;
  int64_t g = (pixels * count) / want_threads;
  if (g < 1) g = 1;
  if (g > kGroup) g = kGroup;
  return (int)g;
}

// transposed im2col colT[k][pix]
__global__ void __launch_bounds__(256) k_im2col_t(float* __restrict__ col, int64_t col_sk, int64_t col_sb,
                                                  const float* __restrict__ x, esgd_tensor4 xd, int64_t x_sb,
                                                  int kh, int kw, int stride, int pad, int oh, int ow, int grp) {
  const int z = blockIdx.z;
  const int np = xd.n * oh * ow, kdim = xd.c * kh * kw, khw = kh * kw;
  const int pix = blockIdx.x * blockDim.x + threadIdx.x;
  if (pix >= np) return;
  const int ohw = oh * ow, img = pix / ohw, p = pix - img * ohw, oy = p / ow, ox = p - oy * ow;
  const int iy0 = oy * stride - pad, ix0 = ox * stride - pad;
  const float* xz = x + z * x_sb + img * xd.sn;
  float* cz = col + z * col_sb + pix;
  const int k0 = blockIdx.y * grp, k1 = min(kdim, k0 + grp);
  int ci = k0 / khw, r = k0 - ci * khw, ky = r / kw, kx = r - ky * kw;
  // all of the group's loads first (independent, up to kGroup in flight per
  // thread: the loop is latency-bound otherwise), then the coalesced stores
  float v[kGroup];
#pragma unroll
  for (int t = 0; t < kGroup; ++t) {
    v[t] = 0.f;
    if (k0 + t < k1) {
      const int iy = iy0 + ky, ix = ix0 + kx;
      if (iy >= 0 && iy < xd.h && ix >= 0 && ix < xd.w) v[t] = __ldg(xz + ci * xd.sc + iy * xd.sh + ix * xd.sw);
      if (++kx == kw) { kx = 0; if (++ky == kh) { ky = 0; ++ci; } }
    }
  }
#pragma unroll
  for (int t = 0; t < kGroup; ++t)
    if (k0 + t < k1) cz[(int64_t)(k0 + t) * col_sk] = v[t];
}

// transposed im2col for square KS x KS kernels over a unit-column-stride
// input (the engine's CNHW planes): thread <-> output pixel, a group of
// channels from blockIdx.y. Tap validity is two per-thread bit masks and the
// input/output pointers just advance, so an element costs one predicated load
// and one coalesced store (the generic kernel spent ~60 instructions on
// address math per element and was issue-bound at ~1.8 TB/s).
#ifndef ESGD_IM2COL_MINB
#define ESGD_IM2COL_MINB 6
#endif
#ifndef ESGD_COL2IM_MINB
#define ESGD_COL2IM_MINB 4
#endif
#ifndef ESGD_POOLF_MINB
#define ESGD_POOLF_MINB 8
#endif
template <int KS>
__global__ void __launch_bounds__(256, ESGD_IM2COL_MINB) k_im2col_sq(float* __restrict__ col, int64_t col_sk, int64_t col_sb,
                                                   const float* __restrict__ x, esgd_tensor4 xd, int64_t x_sb,
                                                   int stride, int pad, int oh, int ow, int cgrp) {
  const int z = blockIdx.z;
  const int ohw = oh * ow, np = xd.n * ohw;
  const int pix = blockIdx.x * blockDim.x + threadIdx.x;
  if (pix >= np) return;
  const int img = pix / ohw, p = pix - img * ohw, oy = p / ow, ox = p - oy * ow;
  const int iy0 = oy * stride - pad, ix0 = ox * stride - pad;
  uint32_t rowok = 0, colok = 0;
#pragma unroll
  for (int t = 0; t < KS; ++t) {
    rowok |= (uint32_t)(iy0 + t >= 0 && iy0 + t < xd.h) << t;
    colok |= (uint32_t)(ix0 + t >= 0 && ix0 + t < xd.w) << t;
  }
  const int c0 = blockIdx.y * cgrp, c1 = min(xd.c, c0 + cgrp);
  // (iy0, ix0) may lie in the padding: only valid taps are dereferenced
  const float* xp = x + z * x_sb + img * xd.sn + (int64_t)c0 * xd.sc + (int64_t)iy0 * xd.sh + ix0;
  float* cp = col + z * col_sb + (int64_t)c0 * KS * KS * col_sk + pix;
  for (int c = c0; c < c1; ++c, xp += xd.sc) {
#pragma unroll
    for (int ky = 0; ky < KS; ++ky) {
      const float* rp = xp + (int64_t)ky * xd.sh;
      const bool rok = (rowok >> ky) & 1u;
#pragma unroll
      for (int kx = 0; kx < KS; ++kx) {
        float v = 0.f;
        if (rok && ((colok >> kx) & 1u)) v = __ldg(rp + kx);
        *cp = v;
        cp += col_sk;
      }
    }
  }
}

// im2col for big square kernels with few channels (AlexNet conv1: 3 x 11 x 11,
// stride 4): one work item per (output pixel, channel, kernel row) — KS taps —
// so the 363-deep K of three channels spreads over 33x more threads than one
// pixel's full column (which left the launch at ~1.3 waves with long loops).
template <int KS>
__global__ void __launch_bounds__(256) k_im2col_rows(float* __restrict__ col, int64_t col_sk, int64_t col_sb,
                                                     const float* __restrict__ x, esgd_tensor4 xd, int64_t x_sb,
                                                     int stride, int pad, int oh, int ow) {
  const int z = blockIdx.z;
  const int ohw = oh * ow, np = xd.n * ohw;
  // grid x = (channel, kernel row), y = pixel block: the KS*C work items of
  // one pixel block run back to back, so the input rows their overlapping
  // windows share are still in L2 (x-fastest over pixels re-read the input
  // 2.1x from DRAM, r01_ncu_conv.md)
  const int pix = blockIdx.y * blockDim.x + threadIdx.x;
  if (pix >= np) return;
  const int c = blockIdx.x / KS, ky = blockIdx.x - c * KS;
  const int img = pix / ohw, p = pix - img * ohw, oy = p / ow, ox = p - oy * ow;
  const int iy = oy * stride - pad + ky, ix0 = ox * stride - pad;
  float* cp = col + z * col_sb + (int64_t)(c * KS * KS + ky * KS) * col_sk + pix;
  const bool rok = iy >= 0 && iy < xd.h;
  const float* rp = x + z * x_sb + img * xd.sn + (int64_t)c * xd.sc + (int64_t)iy * xd.sh + ix0;
  float v[KS];
#pragma unroll
  for (int kx = 0; kx < KS; ++kx) v[kx] = (rok && ix0 + kx >= 0 && ix0 + kx < xd.w) ? __ldg(rp + kx) : 0.f;
#pragma unroll
  for (int kx = 0; kx < KS; ++kx) cp[(int64_t)kx * col_sk] = v[kx];
}

// col2im from colT: thread <-> input pixel (img, y, x), channels of a group;
// (ky, kx) accumulation order fixed per element.
template <bool STRIDE1>
__global__ void __launch_bounds__(256) k_col2im_t(float* __restrict__ dx, esgd_tensor4 xd, int64_t x_sb,
                                                  const float* __restrict__ dcol, int64_t col_sk, int64_t col_sb,
                                                  int kh, int kw, int stride, int pad, int oh, int ow,
                                                  const float* __restrict__ mask, int64_t mask_sb, int grp) {
  const int z = blockIdx.z;
  const int hw = xd.h * xd.w, npin = xd.n * hw;
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= npin) return;
  const int img = q / hw, p = q - img * hw, yh = p / xd.w, xw = p - yh * xd.w;
  const float* dz = dcol + z * col_sb + (int64_t)img * oh * ow;
  const int c0 = blockIdx.y * grp, c1 = min(xd.c, c0 + grp);
  for (int ci = c0; ci < c1; ++ci) {
    const float* dc = dz + (int64_t)(ci * kh * kw) * col_sk;
    float acc = 0.f;
    for (int ky = 0; ky < kh; ++ky) {
      int oy = yh + pad - ky;
      if (oy < 0) continue;
      if (!STRIDE1) { if (oy % stride) continue; oy /= stride; }
      if (oy >= oh) continue;
      for (int kx = 0; kx < kw; ++kx) {
        int ox = xw + pad - kx;
        if (ox < 0) continue;
        if (!STRIDE1) { if (ox % stride) continue; ox /= stride; }
        if (ox >= ow) continue;
        acc += __ldg(dc + (int64_t)(ky * kw + kx) * col_sk + oy * ow + ox);
      }
    }
    const int64_t o = img * xd.sn + ci * xd.sc + yh * xd.sh + xw * xd.sw;
    if (mask) acc = __fmul_rn(acc, mask[z * mask_sb + o] > 0.f ? 1.f : 0.f);
    dx[z * x_sb + o] = acc;
  }
}

// col2im for square KS x KS stride-1 kernels (AlexNet conv2-5, LeNet): the
// KS*KS loads of a channel are issued together (predicated), then summed in
// the same (ky, kx) order as k_col2im_t, so results are identical. Capped at
// 64 registers (4 CTAs/SM) for every KS: at 3x3 the uncapped 75 registers
// allowed 3 (conv3-5 col2im 172 -> 156 us in total, tools/bench_conv.py).
template <int KS>
__global__ void __launch_bounds__(256, ESGD_COL2IM_MINB) k_col2im_sq(float* __restrict__ dx, esgd_tensor4 xd, int64_t x_sb,
                                                   const float* __restrict__ dcol, int64_t col_sk, int64_t col_sb,
                                                   int pad, int oh, int ow, const float* __restrict__ mask,
                                                   int64_t mask_sb, int grp) {
  const int z = blockIdx.z;
  const int hw = xd.h * xd.w, npin = xd.n * hw;
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= npin) return;
  const int img = q / hw, p = q - img * hw, yh = p / xd.w, xw = p - yh * xd.w;
  const float* dz = dcol + z * col_sb + (int64_t)img * oh * ow;
  // tap validity as row/column bit masks; the tap addresses walk from the
  // (0,0) tap's pixel (few registers: 4 CTAs of 256 threads per SM)
  uint32_t rowok = 0, colok = 0;
#pragma unroll
  for (int t = 0; t < KS; ++t) {
    rowok |= (uint32_t)(yh + pad - t >= 0 && yh + pad - t < oh) << t;
    colok |= (uint32_t)(xw + pad - t >= 0 && xw + pad - t < ow) << t;
  }
  const int base = (yh + pad) * ow + (xw + pad);
  const int c0 = blockIdx.y * grp, c1 = min(xd.c, c0 + grp);
#pragma unroll(KS <= 3 ? 2 : 1)
  for (int ci = c0; ci < c1; ++ci) {
    const float* dc = dz + (int64_t)(ci * KS * KS) * col_sk + base;
    float v[KS * KS];
#pragma unroll
    for (int ky = 0; ky < KS; ++ky) {
      const float* rp = dc + (int64_t)(ky * KS) * col_sk - ky * ow;
      const bool rk = (rowok >> ky) & 1u;
#pragma unroll
      for (int kx = 0; kx < KS; ++kx)
        v[ky * KS + kx] = (rk && ((colok >> kx) & 1u)) ? __ldg(rp + (int64_t)kx * col_sk - kx) : 0.f;
    }
    float acc = 0.f;
#pragma unroll
    for (int ky = 0; ky < KS; ++ky)
#pragma unroll
      for (int kx = 0; kx < KS; ++kx)
        if (((rowok >> ky) & 1u) && ((colok >> kx) & 1u)) acc += v[ky * KS + kx];
    const int64_t o = img * xd.sn + ci * xd.sc + yh * xd.sh + xw * xd.sw;
    if (mask) acc = __fmul_rn(acc, mask[z * mask_sb + o] > 0.f ? 1.f : 0.f);
    dx[z * x_sb + o] = acc;
  }
}

// max pooling, thread <-> output pixel of the batch, channels of a group
__global__ void __launch_bounds__(256) k_maxpool_fwd_t(float* __restrict__ y, esgd_tensor4 yd, int64_t y_sb,
                                                       int32_t* __restrict__ amax, const float* __restrict__ x,
                                                       esgd_tensor4 xd, int64_t x_sb, int k, int stride, int pad,
                                                       int grp) {
  const int z = blockIdx.z;
  const int ohw = yd.h * yd.w, np = yd.n * ohw;
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= np) return;
  const int img = q / ohw, p = q - img * ohw, oy = p / yd.w, ox = p - oy * yd.w;
  const int64_t ytotal = (int64_t)yd.n * yd.c * ohw;
  const int c0 = blockIdx.y * grp, c1 = min(yd.c, c0 + grp);
  for (int c = c0; c < c1; ++c) {
    const float* xp = x + z * x_sb + img * xd.sn + c * xd.sc;
    float best = -INFINITY;
    int bi = -1;
    for (int ky = 0; ky < k; ++ky) {
      const int iy = oy * stride - pad + ky;
      if (iy < 0 || iy >= xd.h) continue;
      for (int kx = 0; kx < k; ++kx) {
        const int ix = ox * stride - pad + kx;
        if (ix < 0 || ix >= xd.w) continue;
        const float v = __ldg(xp + iy * xd.sh + ix * xd.sw);
        if (bi < 0 || v > best) { best = v; bi = iy * xd.w + ix; }
      }
    }
    y[z * y_sb + img * yd.sn + c * yd.sc + oy * yd.sh + ox * yd.sw] = best;
    amax[z * ytotal + ((int64_t)img * yd.c + c) * ohw + p] = bi;
  }
}

// K x K max pooling over unit-column-stride planes: tap masks once per
// thread, the channel loop only walks pointers; K*K independent loads per
// channel, compared in (ky, kx) order with the generic kernel's tie rule
template <int K>
__global__ void __launch_bounds__(256, ESGD_POOLF_MINB) k_maxpool_fwd_sq(float* __restrict__ y, esgd_tensor4 yd, int64_t y_sb,
                                                        int32_t* __restrict__ amax, const float* __restrict__ x,
                                                        esgd_tensor4 xd, int64_t x_sb, int stride, int pad, int grp) {
  const int z = blockIdx.z;
  const int ohw = yd.h * yd.w, np = yd.n * ohw;
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= np) return;
  const int img = q / ohw, p = q - img * ohw, oy = p / yd.w, ox = p - oy * yd.w;
  const int iy0 = oy * stride - pad, ix0 = ox * stride - pad;
  bool ok[K * K];
  int idx[K * K];
#pragma unroll
  for (int ky = 0; ky < K; ++ky)
#pragma unroll
    for (int kx = 0; kx < K; ++kx) {
      ok[ky * K + kx] = iy0 + ky >= 0 && iy0 + ky < xd.h && ix0 + kx >= 0 && ix0 + kx < xd.w;
      idx[ky * K + kx] = (iy0 + ky) * xd.w + ix0 + kx;
    }
  const int c0 = blockIdx.y * grp, c1 = min(yd.c, c0 + grp);
  const float* xp = x + z * x_sb + img * xd.sn + (int64_t)c0 * xd.sc + (int64_t)iy0 * xd.sh + ix0;
  float* yp = y + z * y_sb + img * yd.sn + (int64_t)c0 * yd.sc + oy * yd.sh + ox * yd.sw;
  int32_t* ap = amax + z * ((int64_t)yd.n * yd.c * ohw) + ((int64_t)img * yd.c + c0) * ohw + p;
#pragma unroll 2
  for (int c = c0; c < c1; ++c) {
    float v[K * K];
#pragma unroll
    for (int ky = 0; ky < K; ++ky)
#pragma unroll
      for (int kx = 0; kx < K; ++kx) v[ky * K + kx] = ok[ky * K + kx] ? __ldg(xp + ky * xd.sh + kx) : 0.f;
    float best = -INFINITY;
    int bi = -1;
#pragma unroll
    for (int t = 0; t < K * K; ++t)
      if (ok[t] && (bi < 0 || v[t] > best)) { best = v[t]; bi = idx[t]; }
    *yp = best;
    *ap = bi;
    xp += xd.sc;
    yp += yd.sc;
    ap += ohw;
  }
}

// max-pool backward for K x K / stride 2 / pad 0 (AlexNet 3/2, LeNet 2/2):
// thread <-> a 2x2 block of input pixels (2a..2a+1, 2b..2b+1), whose covering
// windows are outputs (a-1..a, b-1..b) for K = 3 and (a, b) for K = 2, so one
// thread loads 4 argmax + 4 dy values per channel for 4 outputs (the per-pixel
// gather loads 8 per pixel). Each pixel still sums its windows in (oy, ox)
// order, so results equal k_maxpool_bwd_t's.
// GATE fuses the relu backward of the pool's input: 1 = the input itself
// (gsrc laid out as dx) > 0; 2 = the pooled output (laid out as dy) > 0 of a
// window that selected the pixel — that window's max is the pixel's own
// value, and a pixel gets a nonzero sum only through such a window, so 2
// gives 1's bits while reading the 4x smaller output. Every load of a channel
// is issued before any is used, two channels per iteration: the kernel is
// load-latency bound otherwise (ncu: 17% of DRAM bandwidth with the gate
// loads issued behind the argmax compares).
#ifndef ESGD_POOL_MINB
#define ESGD_POOL_MINB 4
#endif
#ifndef ESGD_POOL_UNROLL
#define ESGD_POOL_UNROLL 2
#endif
constexpr int kPoolUnroll = ESGD_POOL_UNROLL;
template <int K, int GATE>
__global__ void __launch_bounds__(256, ESGD_POOL_MINB) k_maxpool_bwd_s2(float* __restrict__ dx, esgd_tensor4 xd, int64_t x_sb,
                                                        const float* __restrict__ dy, esgd_tensor4 yd, int64_t y_sb,
                                                        const int32_t* __restrict__ amax,
                                                        const float* __restrict__ gsrc, int64_t g_sb, int grp) {
  const int z = blockIdx.z;
  const int bh = (xd.h + 1) / 2, bw = (xd.w + 1) / 2, nb = bh * bw, ohw = yd.h * yd.w;
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= xd.n * nb) return;
  const int img = q / nb, r = q - img * nb, a = r / bw, b = r - a * bw;
  // window slots t = (ti, tj): output (a - 1 + ti, b - 1 + tj); K = 2 uses slot 3 only
  bool wok[4];
  int wo[4], yo[4];
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int oy = a - 1 + (t >> 1), ox = b - 1 + (t & 1);
    wok[t] = (K == 3 || t == 3) && oy >= 0 && oy < yd.h && ox >= 0 && ox < yd.w;
    wo[t] = oy * yd.w + ox;
    yo[t] = oy * yd.sh + ox * yd.sw;
  }
  // block pixels i = (di, dj): input (2a + di, 2b + dj)
  const int iy0 = 2 * a, ix0 = 2 * b;
  const bool pok[4] = {true, ix0 + 1 < xd.w, iy0 + 1 < xd.h, iy0 + 1 < xd.h && ix0 + 1 < xd.w};
  const int64_t xo[4] = {0, xd.sw, xd.sh, xd.sh + xd.sw};
  const int p00 = iy0 * xd.w + ix0;
  const int pidx[4] = {p00, p00 + 1, p00 + xd.w, p00 + xd.w + 1};
  const int c0 = blockIdx.y * grp, c1 = min(xd.c, c0 + grp);
  const int32_t* ap = amax + z * ((int64_t)yd.n * yd.c * ohw) + ((int64_t)img * yd.c + c0) * ohw;
  const int64_t yoff = img * yd.sn + (int64_t)c0 * yd.sc;
  const float* dyp = dy + z * y_sb + yoff;
  const int64_t o0 = img * xd.sn + (int64_t)c0 * xd.sc + iy0 * xd.sh + ix0 * xd.sw;
  float* dxp = dx + z * x_sb + o0;
  const float* gp = GATE == 1 ? gsrc + z * g_sb + o0 : GATE == 2 ? gsrc + z * g_sb + yoff : nullptr;
  const int64_t gstep = GATE == 1 ? xd.sc : yd.sc;
#pragma unroll kPoolUnroll
  for (int c = c0; c < c1; ++c) {
    int am[4];
    float d[4], gv[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      am[t] = wok[t] ? __ldg(ap + wo[t]) : -1;
      d[t] = wok[t] ? __ldg(dyp + yo[t]) : 0.f;
      if (GATE == 2) gv[t] = wok[t] ? __ldg(gp + yo[t]) : 0.f;
      if (GATE == 1) gv[t] = pok[t] ? __ldg(gp + xo[t]) : 0.f;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float acc = 0.f;
      bool pos = false;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        // slot t's window covers pixel i iff di <= ti and dj <= tj (K = 3)
        const bool cov = K == 3 ? ((i >> 1) <= (t >> 1) && (i & 1) <= (t & 1)) : t == 3;
        if (cov && am[t] == pidx[i]) {
          acc += d[t];
          if (GATE == 2) pos = pos || gv[t] > 0.f;
        }
      }
      if (GATE == 1) acc = __fmul_rn(acc, gv[i] > 0.f ? 1.f : 0.f);
      if (GATE == 2) acc = __fmul_rn(acc, pos ? 1.f : 0.f);
      if (pok[i]) dxp[xo[i]] = acc;
    }
    ap += ohw;
    dyp += yd.sc;
    dxp += xd.sc;
    if (GATE) gp += gstep;
  }
}

__global__ void __launch_bounds__(256) k_maxpool_bwd_t(float* __restrict__ dx, esgd_tensor4 xd, int64_t x_sb,
                                                       const float* __restrict__ dy, esgd_tensor4 yd, int64_t y_sb,
                                                       const int32_t* __restrict__ amax,
                                                       const float* __restrict__ mask, int64_t mask_sb,
                                                       const float* __restrict__ ymask, int64_t ym_sb, int k,
                                                       int stride, int pad, int grp) {
  const int z = blockIdx.z;
  const int hw = xd.h * xd.w, npin = xd.n * hw, ohw = yd.h * yd.w;
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= npin) return;
  const int img = q / hw, p = q - img * hw, iy = p / xd.w, ix = p - iy * xd.w;
  const int64_t ytotal = (int64_t)yd.n * yd.c * ohw;
  int oy_lo = iy + pad - k + 1;
  oy_lo = oy_lo <= 0 ? 0 : (oy_lo + stride - 1) / stride;
  int oy_hi = (iy + pad) / stride;
  if (oy_hi > yd.h - 1) oy_hi = yd.h - 1;
  int ox_lo = ix + pad - k + 1;
  ox_lo = ox_lo <= 0 ? 0 : (ox_lo + stride - 1) / stride;
  int ox_hi = (ix + pad) / stride;
  if (ox_hi > yd.w - 1) ox_hi = yd.w - 1;
  const int c0 = blockIdx.y * grp, c1 = min(xd.c, c0 + grp);
  if (oy_hi - oy_lo < 2 && ox_hi - ox_lo < 2) {
    // <= 2x2 windows cover this pixel (k <= 2*stride, AlexNet 3/2, LeNet 2/2):
    // issue the four argmax/dy loads together, sum in (oy, ox) order
    const bool v01 = ox_lo + 1 <= ox_hi, v10 = oy_lo + 1 <= oy_hi;
    const bool ok[4] = {oy_lo <= oy_hi && ox_lo <= ox_hi, oy_lo <= oy_hi && v01, v10 && ox_lo <= ox_hi, v10 && v01};
    const int wo[4] = {oy_lo * yd.w + ox_lo, oy_lo * yd.w + ox_lo + 1, (oy_lo + 1) * yd.w + ox_lo,
                       (oy_lo + 1) * yd.w + ox_lo + 1};
    const int yo[4] = {oy_lo * yd.sh + ox_lo * yd.sw, oy_lo * yd.sh + (ox_lo + 1) * yd.sw,
                       (oy_lo + 1) * yd.sh + ox_lo * yd.sw, (oy_lo + 1) * yd.sh + (ox_lo + 1) * yd.sw};
    const int32_t* ap = amax + z * ytotal + ((int64_t)img * yd.c + c0) * ohw;
    const float* dyp = dy + z * y_sb + img * yd.sn + (int64_t)c0 * yd.sc;
    const int64_t o0 = z * x_sb + img * xd.sn + (int64_t)c0 * xd.sc + iy * xd.sh + ix * xd.sw;
    float* dxp = dx + o0;
    const float* mp = mask ? mask + z * mask_sb + (o0 - z * x_sb) : nullptr;
    const float* ymp = ymask ? ymask + z * ym_sb + img * yd.sn + (int64_t)c0 * yd.sc : nullptr;
#pragma unroll 2
    for (int c = c0; c < c1; ++c) {
      int a[4];
      float d[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        a[t] = ok[t] ? __ldg(ap + wo[t]) : -1;
        d[t] = ok[t] ? __ldg(dyp + yo[t]) : 0.f;
      }
      float acc = 0.f, g = 0.f;
#pragma unroll
      for (int t = 0; t < 4; ++t)
        if (a[t] == p) {
          acc += d[t];
          if (ymp && __ldg(ymp + yo[t]) > 0.f) g = 1.f;
        }
      if (mp) {
        acc = __fmul_rn(acc, *mp > 0.f ? 1.f : 0.f);
        mp += xd.sc;
      }
      if (ymp) {
        acc = __fmul_rn(acc, g);
        ymp += yd.sc;
      }
      *dxp = acc;
      ap += ohw;
      dyp += yd.sc;
      dxp += xd.sc;
    }
    return;
  }
  for (int c = c0; c < c1; ++c) {
    const int32_t* ap = amax + z * ytotal + ((int64_t)img * yd.c + c) * ohw;
    const float* dyp = dy + z * y_sb + img * yd.sn + c * yd.sc;
    float acc = 0.f, g = 0.f;
    for (int oy = oy_lo; oy <= oy_hi; ++oy)
      for (int ox = ox_lo; ox <= ox_hi; ++ox)
        if (ap[oy * yd.w + ox] == p) {
          acc += __ldg(dyp + oy * yd.sh + ox * yd.sw);
          if (ymask && __ldg(ymask + z * ym_sb + img * yd.sn + c * yd.sc + oy * yd.sh + ox * yd.sw) > 0.f) g = 1.f;
        }
    const int64_t o = img * xd.sn + c * xd.sc + iy * xd.sh + ix * xd.sw;
    if (mask) acc = __fmul_rn(acc, mask[z * mask_sb + o] > 0.f ? 1.f : 0.f);
    if (ymask) acc = __fmul_rn(acc, g);
    dx[z * x_sb + o] = acc;
  }
}

__global__ void __launch_bounds__(256) k_copy4(float* __restrict__ dst, esgd_tensor4 dd,
                                               int64_t d_sb, const float* __restrict__ src,
                                               esgd_tensor4 sd, int64_t s_sb) {
  const int z = blockIdx.y;
  const unsigned total = (unsigned)dd.n * dd.c * dd.h * dd.w;
  for (unsigned e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    unsigned t = e;
    const int w = (int)(t % (unsigned)dd.w); t /= (unsigned)dd.w;
    const int h = (int)(t % (unsigned)dd.h); t /= (unsigned)dd.h;
    const int c = (int)(t % (unsigned)dd.c);
    const int n = (int)(t / (unsigned)dd.c);
    dst[z * d_sb + off4(dd, n, c, h, w)] = __ldg(src + z * s_sb + off4(sd, n, c, h, w));
  }
}

bool valid4(const esgd_tensor4& t) {
  return t.n >= 1 && t.c >= 1 && t.h >= 1 && t.w >= 1 &&
         (int64_t)t.n * t.c * t.h * t.w < (int64_t(1) << 31);
}

// Row sums: out[z*out_sb + r] = sum_{j < cols} x[z*x_sb + r*ld + j] (conv bias
// gradients over the channel-major activation rows). Pass 1: CTA per (row,
// chunk), 4 independent partials per thread + fixed-order block tree.
// VEC: 16-B loads (rows 16-B aligned, chunk a multiple of 4): four float4
// loads in flight per thread instead of four floats (the bias gradients of
// AlexNet's convolutions read ~250 MB per round)
template <bool VEC>
__global__ void __launch_bounds__(256) k_rowsum_partial(float* part, const float* __restrict__ x, int64_t ld,
                                                        int64_t x_sb, int cols, int chunk, float* out,
                                                        int64_t out_sb, int direct) {
  __shared__ float red[256];
  const int r = blockIdx.x, ch = blockIdx.y, z = blockIdx.z;
  const float* row = x + z * x_sb + r * ld;
  const int j0 = ch * chunk, j1 = min(cols, j0 + chunk);
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
  if (VEC) {
    const float4* r4 = reinterpret_cast<const float4*>(row);
    const int q1 = j1 >> 2;
    int q = (j0 >> 2) + threadIdx.x;
    for (; q + 768 < q1; q += 1024) {
      const float4 a = __ldg(r4 + q), b = __ldg(r4 + q + 256), c = __ldg(r4 + q + 512), d = __ldg(r4 + q + 768);
      s0 += (a.x + a.y) + (a.z + a.w); s1 += (b.x + b.y) + (b.z + b.w);
      s2 += (c.x + c.y) + (c.z + c.w); s3 += (d.x + d.y) + (d.z + d.w);
    }
    for (; q < q1; q += 256) {
      const float4 a = __ldg(r4 + q);
      s0 += (a.x + a.y) + (a.z + a.w);
    }
    for (int j = (q1 << 2) + threadIdx.x; j < j1; j += 256) s1 += __ldg(row + j);  // (cols % 4 tail)
  } else {
    int j = j0 + threadIdx.x;
    for (; j + 768 < j1; j += 1024) {
      s0 += __ldg(row + j); s1 += __ldg(row + j + 256); s2 += __ldg(row + j + 512); s3 += __ldg(row + j + 768);
    }
    for (; j < j1; j += 256) s0 += __ldg(row + j);
  }
  red[threadIdx.x] = (s0 + s1) + (s2 + s3);
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (direct) out[z * out_sb + r] = red[0];
    else part[((int64_t)z * gridDim.x + r) * gridDim.y + ch] = red[0];
  }
}
__global__ void k_rowsum_final(float* out, int64_t out_sb, const float* part, int rows, int nchunk, int batch) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows * batch) return;
  const int z = i / rows, r = i % rows;
  const float* p = part + ((int64_t)z * rows + r) * nchunk;
  float t = 0.f;
  for (int k = 0; k < nchunk; ++k) t += p[k];
  out[z * out_sb + r] = t;
}

}  // namespace
}  // namespace esgd

using namespace esgd;
#define ESGD_STREAM(s) reinterpret_cast<cudaStream_t>(s)

extern "C" int esgd_im2col_f32(float* col, int64_t col_sp, int64_t col_sk, int64_t col_sb,
                               const float* x, esgd_tensor4 xd, int64_t x_sb, int32_t kh, int32_t kw,
                               int32_t stride, int32_t pad, int32_t oh, int32_t ow, int32_t batch,
                               esgd_stream_t stream) {
  ESGD_REQUIRE(valid4(xd) && kh >= 1 && kw >= 1 && stride >= 1 && pad >= 0 && oh >= 1 &&
                   ow >= 1 && batch >= 1,
               ESGD_ERR_SHAPE, "im2col: bad geometry");
  const int64_t np = (int64_t)xd.n * oh * ow, kdim = (int64_t)xd.c * kh * kw;
  ESGD_REQUIRE(np * kdim < (int64_t(1) << 31), ESGD_ERR_UNSUPPORTED, "im2col: more than 2^31 elements");
  ESGD_REQUIRE((col_sk == 1 && col_sp >= kdim) || (col_sp == 1 && col_sk >= np), ESGD_ERR_SHAPE,
               "im2col: col strides must be (>=K, 1) or (1, >=pixels)");
  ESGD_REQUIRE(batch <= 65535, ESGD_ERR_UNSUPPORTED, "im2col: batch > 65535");
  ESGD_REQUIRE(col && x, ESGD_ERR_INPUT, "im2col: null buffer");
  if (col_sp == 1 && kh == kw && (kh == 3 || kh == 5 || kh == 11) && xd.sw == 1) {
    const int gc = pick_group(np * batch * kh * kw / kGroup, xd.c);
    dim3 g2((unsigned)((np + 255) / 256), (unsigned)((xd.c + gc - 1) / gc), batch);
    if (kh == 3)
      k_im2col_sq<3><<<g2, 256, 0, ESGD_STREAM(stream)>>>(col, col_sk, col_sb, x, xd, x_sb, stride, pad, oh, ow, gc);
    else if (kh == 5)
      k_im2col_sq<5><<<g2, 256, 0, ESGD_STREAM(stream)>>>(col, col_sk, col_sb, x, xd, x_sb, stride, pad, oh, ow, gc);
    else if ((np + 255) / 256 <= 65535) {
      dim3 g3((unsigned)(xd.c * kh), (unsigned)((np + 255) / 256), batch);
      k_im2col_rows<11><<<g3, 256, 0, ESGD_STREAM(stream)>>>(col, col_sk, col_sb, x, xd, x_sb, stride, pad, oh, ow);
    } else
      k_im2col_sq<11><<<g2, 256, 0, ESGD_STREAM(stream)>>>(col, col_sk, col_sb, x, xd, x_sb, stride, pad, oh, ow, gc);
    return check_launch("esgd_im2col_f32");
  }
  const int gi = pick_group(np * batch, kdim);
  if (col_sp == 1 && (kdim + gi - 1) / gi <= 65535) {
    dim3 g2((unsigned)((np + 255) / 256), (unsigned)((kdim + gi - 1) / gi), batch);
    k_im2col_t<<<g2, 256, 0, ESGD_STREAM(stream)>>>(col, col_sk, col_sb, x, xd, x_sb, kh, kw, stride, pad, oh, ow, gi);
    return check_launch("esgd_im2col_f32");
  }
  dim3 grid(stride_grid(np * kdim, 256, 16), batch);
  if (col_sp == 1)
    k_im2col<true><<<grid, 256, 0, ESGD_STREAM(stream)>>>(col, col_sp, col_sk, col_sb, x, xd, x_sb, kh, kw, stride, pad, oh, ow);
  else
    k_im2col<false><<<grid, 256, 0, ESGD_STREAM(stream)>>>(col, col_sp, col_sk, col_sb, x, xd, x_sb, kh, kw, stride, pad, oh, ow);
  return check_launch("esgd_im2col_f32");
}

extern "C" int esgd_col2im_f32(float* dx, esgd_tensor4 xd, int64_t x_sb, const float* dcol,
                               int64_t col_sp, int64_t col_sk, int64_t col_sb, int32_t kh, int32_t kw,
                               int32_t stride, int32_t pad, int32_t oh, int32_t ow, const float* mask,
                               int64_t mask_sb, int32_t batch, esgd_stream_t stream) {
  ESGD_REQUIRE(valid4(xd) && kh >= 1 && kw >= 1 && stride >= 1 && pad >= 0 && oh >= 1 &&
                   ow >= 1 && batch >= 1,
               ESGD_ERR_SHAPE, "col2im: bad geometry");
  const int64_t np = (int64_t)xd.n * oh * ow, kdim = (int64_t)xd.c * kh * kw;
  ESGD_REQUIRE((col_sk == 1 && col_sp >= kdim) || (col_sp == 1 && col_sk >= np), ESGD_ERR_SHAPE,
               "col2im: col strides must be (>=K, 1) or (1, >=pixels)");
  ESGD_REQUIRE(np * kdim < (int64_t(1) << 31), ESGD_ERR_UNSUPPORTED, "col2im: more than 2^31 elements");
  ESGD_REQUIRE(batch <= 65535, ESGD_ERR_UNSUPPORTED, "col2im: batch > 65535");
  ESGD_REQUIRE(dx && dcol, ESGD_ERR_INPUT, "col2im: null buffer");
  const int gc = pick_group((int64_t)xd.n * xd.h * xd.w * batch, xd.c);
  if (col_sp == 1 && (xd.c + gc - 1) / gc <= 65535) {
    dim3 g2((unsigned)(((int64_t)xd.n * xd.h * xd.w + 255) / 256), (unsigned)((xd.c + gc - 1) / gc), batch);
    dim3 b2(256);
    if (stride == 1 && kh == kw && kh == 3)
      k_col2im_sq<3><<<g2, b2, 0, ESGD_STREAM(stream)>>>(dx, xd, x_sb, dcol, col_sk, col_sb, pad, oh, ow, mask, mask_sb, gc);
    else if (stride == 1 && kh == kw && kh == 5)
      k_col2im_sq<5><<<g2, b2, 0, ESGD_STREAM(stream)>>>(dx, xd, x_sb, dcol, col_sk, col_sb, pad, oh, ow, mask, mask_sb, gc);
    else if (stride == 1)
      k_col2im_t<true><<<g2, b2, 0, ESGD_STREAM(stream)>>>(dx, xd, x_sb, dcol, col_sk, col_sb, kh, kw, stride, pad, oh, ow, mask, mask_sb, gc);
    else
      k_col2im_t<false><<<g2, b2, 0, ESGD_STREAM(stream)>>>(dx, xd, x_sb, dcol, col_sk, col_sb, kh, kw, stride, pad, oh, ow, mask, mask_sb, gc);
    return check_launch("esgd_col2im_f32");
  }
  int64_t total = (int64_t)xd.n * xd.c * xd.h * xd.w;
  dim3 grid(stride_grid(total, 256, 16), batch);
  k_col2im<<<grid, 256, 0, ESGD_STREAM(stream)>>>(dx, xd, x_sb, dcol, col_sp, col_sk, col_sb, kh, kw, stride, pad, oh, ow, mask, mask_sb);
  return check_launch("esgd_col2im_f32");
}

extern "C" int esgd_rowsum_f32(float* out, int64_t out_sb, const float* x, int64_t ld, int64_t x_sb,
                               int32_t rows, int64_t cols, int32_t batch, float* scratch,
                               esgd_stream_t stream) {
  ESGD_REQUIRE(rows >= 1 && cols >= 1 && batch >= 1 && ld >= cols && cols < (int64_t(1) << 31),
               ESGD_ERR_SHAPE, "rowsum: bad shape");
  ESGD_REQUIRE(out && x, ESGD_ERR_INPUT, "rowsum: null buffer");
  ESGD_REQUIRE(rows <= 65535 && batch <= 65535, ESGD_ERR_UNSUPPORTED, "rowsum: grid too large");
  // ~8 CTAs per SM overall (the row sums are latency-bound at fewer), chunks
  // of >= 4096 elements
  int64_t nchunk = (8 * kNumSMs + (int64_t)rows - 1) / (int64_t)rows;  // batch-independent order
  int64_t maxc = (cols + 4095) / 4096;
  if (nchunk > maxc) nchunk = maxc;
  if (nchunk > 64) nchunk = 64;
  if (nchunk < 1) nchunk = 1;
  const bool vec = (ld & 3) == 0 && (x_sb & 3) == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0;
  int64_t chunk = (cols + nchunk - 1) / nchunk;
  if (vec) chunk = (chunk + 3) & ~int64_t(3);  // chunk starts 16-B aligned
  nchunk = (cols + chunk - 1) / chunk;
  ESGD_REQUIRE(nchunk == 1 || scratch, ESGD_ERR_INPUT, "rowsum: scratch required");
  cudaStream_t st = ESGD_STREAM(stream);
  dim3 grid(rows, (unsigned)nchunk, batch);
  if (vec)
    k_rowsum_partial<true><<<grid, 256, 0, st>>>(scratch, x, ld, x_sb, (int)cols, (int)chunk, out, out_sb, nchunk == 1);
  else
    k_rowsum_partial<false><<<grid, 256, 0, st>>>(scratch, x, ld, x_sb, (int)cols, (int)chunk, out, out_sb, nchunk == 1);
  if (nchunk > 1) {
    int tot = rows * batch;
    k_rowsum_final<<<(tot + 255) / 256, 256, 0, st>>>(out, out_sb, scratch, rows, (int)nchunk, batch);
  }
  return check_launch("esgd_rowsum_f32");
}

extern "C" int esgd_maxpool_fwd_f32(float* y, esgd_tensor4 yd, int64_t y_sb, int32_t* argmax,
                                    const float* x, esgd_tensor4 xd, int64_t x_sb, int32_t k,
                                    int32_t stride, int32_t pad, int32_t batch,
                                    esgd_stream_t stream) {
  ESGD_REQUIRE(valid4(xd) && valid4(yd) && k >= 1 && stride >= 1 && pad >= 0 && pad < k &&
                   batch >= 1 && yd.n == xd.n && yd.c == xd.c,
               ESGD_ERR_SHAPE, "maxpool_fwd: bad geometry");
  ESGD_REQUIRE(batch <= 65535, ESGD_ERR_UNSUPPORTED, "maxpool: batch > 65535");
  ESGD_REQUIRE(y && argmax && x, ESGD_ERR_INPUT, "maxpool_fwd: null buffer");
  {
    const int gp = pick_group((int64_t)yd.n * yd.h * yd.w * batch, yd.c);
    dim3 g2((unsigned)(((int64_t)yd.n * yd.h * yd.w + 255) / 256), (unsigned)((yd.c + gp - 1) / gp), batch);
    dim3 b2(256);
    if (xd.sw == 1 && k == 3)
      k_maxpool_fwd_sq<3><<<g2, b2, 0, ESGD_STREAM(stream)>>>(y, yd, y_sb, argmax, x, xd, x_sb, stride, pad, gp);
    else if (xd.sw == 1 && k == 2)
      k_maxpool_fwd_sq<2><<<g2, b2, 0, ESGD_STREAM(stream)>>>(y, yd, y_sb, argmax, x, xd, x_sb, stride, pad, gp);
    else
      k_maxpool_fwd_t<<<g2, b2, 0, ESGD_STREAM(stream)>>>(y, yd, y_sb, argmax, x, xd, x_sb, k, stride, pad, gp);
    return check_launch("esgd_maxpool_fwd_f32");
  }
}

static int maxpool_bwd(float* dx, esgd_tensor4 xd, int64_t x_sb, const float* dy, esgd_tensor4 yd, int64_t y_sb,
                       const int32_t* argmax, const float* mask, int64_t mask_sb, const float* ymask,
                       int64_t ym_sb, int32_t k, int32_t stride, int32_t pad, int32_t batch,
                       esgd_stream_t stream) {
  ESGD_REQUIRE(valid4(xd) && valid4(yd) && k >= 1 && stride >= 1 && pad >= 0 && batch >= 1 &&
                   yd.n == xd.n && yd.c == xd.c,
               ESGD_ERR_SHAPE, "maxpool_bwd: bad geometry");
  ESGD_REQUIRE(batch <= 65535, ESGD_ERR_UNSUPPORTED, "maxpool: batch > 65535");
  ESGD_REQUIRE(dx && dy && argmax, ESGD_ERR_INPUT, "maxpool_bwd: null buffer");
  if (stride == 2 && pad == 0 && (k == 2 || k == 3) && (yd.h - 1) * 2 + k <= xd.h + 1 &&
      (yd.w - 1) * 2 + k <= xd.w + 1) {
    const int64_t nblk = (int64_t)xd.n * ((xd.h + 1) / 2) * ((xd.w + 1) / 2);
    const int gp = pick_group(nblk * batch, xd.c);
    dim3 g2((unsigned)((nblk + 255) / 256), (unsigned)((xd.c + gp - 1) / gp), batch);
    const float* gs = ymask ? ymask : mask;
    const int64_t gsb = ymask ? ym_sb : mask_sb;
    const int gate = ymask ? 2 : mask ? 1 : 0;
    cudaStream_t st = ESGD_STREAM(stream);
#define ESGD_POOL_S2(KK, GG) \
  k_maxpool_bwd_s2<KK, GG><<<g2, 256, 0, st>>>(dx, xd, x_sb, dy, yd, y_sb, argmax, gs, gsb, gp)
    if (k == 3) {
      if (gate == 2) ESGD_POOL_S2(3, 2);
      else if (gate == 1) ESGD_POOL_S2(3, 1);
      else ESGD_POOL_S2(3, 0);
    } else {
      if (gate == 2) ESGD_POOL_S2(2, 2);
      else if (gate == 1) ESGD_POOL_S2(2, 1);
      else ESGD_POOL_S2(2, 0);
    }
#undef ESGD_POOL_S2
    return check_launch("esgd_maxpool_bwd_f32");
  }
  const int gp = pick_group((int64_t)xd.n * xd.h * xd.w * batch, xd.c);
  dim3 g2((unsigned)(((int64_t)xd.n * xd.h * xd.w + 255) / 256), (unsigned)((xd.c + gp - 1) / gp), batch);
  k_maxpool_bwd_t<<<g2, 256, 0, ESGD_STREAM(stream)>>>(dx, xd, x_sb, dy, yd, y_sb, argmax, mask, mask_sb, ymask,
                                                       ym_sb, k, stride, pad, gp);
  return check_launch("esgd_maxpool_bwd_f32");
}

extern "C" int esgd_maxpool_bwd_f32(float* dx, esgd_tensor4 xd, int64_t x_sb, const float* dy,
                                    esgd_tensor4 yd, int64_t y_sb, const int32_t* argmax,
                                    const float* mask, int64_t mask_sb, int32_t k, int32_t stride,
                                    int32_t pad, int32_t batch, esgd_stream_t stream) {
  return maxpool_bwd(dx, xd, x_sb, dy, yd, y_sb, argmax, mask, mask_sb, nullptr, 0, k, stride, pad, batch, stream);
}

extern "C" int esgd_maxpool_bwd_relu_f32(float* dx, esgd_tensor4 xd, int64_t x_sb, const float* dy,
                                         esgd_tensor4 yd, int64_t dy_sb, const int32_t* argmax, const float* y,
                                         int64_t y_sb, int32_t k, int32_t stride, int32_t pad, int32_t batch,
                                         esgd_stream_t stream) {
  ESGD_REQUIRE(y, ESGD_ERR_INPUT, "maxpool_bwd_relu: null pooled output");
  return maxpool_bwd(dx, xd, x_sb, dy, yd, dy_sb, argmax, nullptr, 0, y, y_sb, k, stride, pad, batch, stream);
}

extern "C" int esgd_copy4_f32(float* dst, esgd_tensor4 dd, int64_t d_sb, const float* src,
                              esgd_tensor4 sd, int64_t s_sb, int32_t batch, esgd_stream_t stream) {
  ESGD_REQUIRE(valid4(dd) && dd.n == sd.n && dd.c == sd.c && dd.h == sd.h && dd.w == sd.w &&
                   batch >= 1,
               ESGD_ERR_SHAPE, "copy4: shape mismatch");
  ESGD_REQUIRE(batch <= 65535, ESGD_ERR_UNSUPPORTED, "copy4: batch > 65535");
  ESGD_REQUIRE(dst && src, ESGD_ERR_INPUT, "copy4: null buffer");
  int64_t total = (int64_t)dd.n * dd.c * dd.h * dd.w;
  dim3 grid(stride_grid(total, 256, 16), batch);
  k_copy4<<<grid, 256, 0, ESGD_STREAM(stream)>>>(dst, dd, d_sb, src, sd, s_sb);
  return check_launch("esgd_copy4_f32");
}
