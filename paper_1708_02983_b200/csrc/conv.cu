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

// one thread per column element; consecutive threads walk a column row
__global__ void __launch_bounds__(256) k_im2col(float* __restrict__ col, int64_t ldc,
                                                int64_t col_sb, const float* __restrict__ x,
                                                esgd_tensor4 xd, int64_t x_sb, int kh, int kw,
                                                int stride, int pad, int oh, int ow) {
  const int z = blockIdx.y;
  const int64_t rows = (int64_t)xd.n * oh * ow;
  const int64_t total = rows * ldc;
  const int kdim = xd.c * kh * kw;
  const float* xz = x + z * x_sb;
  float* cz = col + z * col_sb;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = e / ldc;
    const int k = (int)(e - row * ldc);
    float v = 0.f;
    if (k < kdim) {
      const int img = (int)(row / ((int64_t)oh * ow));
      const int pix = (int)(row - (int64_t)img * oh * ow);
      const int oy = pix / ow, ox = pix - oy * ow;
      const int ci = k / (kh * kw), r = k - ci * kh * kw;
      const int ky = r / kw, kx = r - ky * kw;
      const int iy = oy * stride - pad + ky, ix = ox * stride - pad + kx;
      if (iy >= 0 && iy < xd.h && ix >= 0 && ix < xd.w) v = __ldg(xz + off4(xd, img, ci, iy, ix));
    }
    cz[e] = v;
  }
}

__global__ void __launch_bounds__(256) k_col2im(float* __restrict__ dx, esgd_tensor4 xd,
                                                int64_t x_sb, const float* __restrict__ dcol,
                                                int64_t ldc, int64_t col_sb, int kh, int kw,
                                                int stride, int pad, int oh, int ow,
                                                const float* __restrict__ mask) {
  const int z = blockIdx.y;
  const int64_t total = (int64_t)xd.n * xd.c * xd.h * xd.w;
  const float* dz = dcol + z * col_sb;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    // canonical (img, ci, y, x) order of the element
    int64_t t = e;
    const int xw = (int)(t % xd.w); t /= xd.w;
    const int yh = (int)(t % xd.h); t /= xd.h;
    const int ci = (int)(t % xd.c);
    const int img = (int)(t / xd.c);
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
        const int64_t row = ((int64_t)img * oh + oy) * ow + ox;
        acc += __ldg(dz + row * ldc + (ci * kh + ky) * kw + kx);
      }
    }
    const int64_t o = z * x_sb + off4(xd, img, ci, yh, xw);
    if (mask) acc = __fmul_rn(acc, mask[o] > 0.f ? 1.f : 0.f);
    dx[o] = acc;
  }
}

__global__ void __launch_bounds__(256) k_maxpool_fwd(float* __restrict__ y, esgd_tensor4 yd,
                                                     int64_t y_sb, int32_t* __restrict__ amax,
                                                     const float* __restrict__ x, esgd_tensor4 xd,
                                                     int64_t x_sb, int k, int stride, int pad) {
  const int z = blockIdx.y;
  const int64_t total = (int64_t)yd.n * yd.c * yd.h * yd.w;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t t = e;
    const int ox = (int)(t % yd.w); t /= yd.w;
    const int oy = (int)(t % yd.h); t /= yd.h;
    const int c = (int)(t % yd.c);
    const int img = (int)(t / yd.c);
    float best = -INFINITY;
    int bi = -1;
    for (int ky = 0; ky < k; ++ky) {
      const int iy = oy * stride - pad + ky;
      if (iy < 0 || iy >= xd.h) continue;
      for (int kx = 0; kx < k; ++kx) {
        const int ix = ox * stride - pad + kx;
        if (ix < 0 || ix >= xd.w) continue;
        const float v = __ldg(x + z * x_sb + off4(xd, img, c, iy, ix));
        if (bi < 0 || v > best) { best = v; bi = iy * xd.w + ix; }
      }
    }
    y[z * y_sb + off4(yd, img, c, oy, ox)] = best;
    amax[z * total + e] = bi;
  }
}

__global__ void __launch_bounds__(256) k_maxpool_bwd(float* __restrict__ dx, esgd_tensor4 xd,
                                                     int64_t x_sb, const float* __restrict__ dy,
                                                     esgd_tensor4 yd, int64_t y_sb,
                                                     const int32_t* __restrict__ amax,
                                                     const float* __restrict__ mask, int k,
                                                     int stride, int pad) {
  const int z = blockIdx.y;
  const int64_t total = (int64_t)xd.n * xd.c * xd.h * xd.w;
  const int64_t ytotal = (int64_t)yd.n * yd.c * yd.h * yd.w;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t t = e;
    const int ix = (int)(t % xd.w); t /= xd.w;
    const int iy = (int)(t % xd.h); t /= xd.h;
    const int c = (int)(t % xd.c);
    const int img = (int)(t / xd.c);
    const int me = iy * xd.w + ix;
    // windows covering iy: oy*stride - pad <= iy <= oy*stride - pad + k - 1
    int oy_lo = iy + pad - k + 1;
    oy_lo = oy_lo <= 0 ? 0 : (oy_lo + stride - 1) / stride;
    int oy_hi = (iy + pad) / stride;
    if (oy_hi > yd.h - 1) oy_hi = yd.h - 1;
    int ox_lo = ix + pad - k + 1;
    ox_lo = ox_lo <= 0 ? 0 : (ox_lo + stride - 1) / stride;
    int ox_hi = (ix + pad) / stride;
    if (ox_hi > yd.w - 1) ox_hi = yd.w - 1;
    float acc = 0.f;
    for (int oy = oy_lo; oy <= oy_hi; ++oy)
      for (int ox = ox_lo; ox <= ox_hi; ++ox) {
        const int64_t ye = (((int64_t)img * yd.c + c) * yd.h + oy) * yd.w + ox;
        if (amax[z * ytotal + ye] == me) acc += __ldg(dy + z * y_sb + off4(yd, img, c, oy, ox));
      }
    const int64_t o = z * x_sb + off4(xd, img, c, iy, ix);
    if (mask) acc = __fmul_rn(acc, mask[o] > 0.f ? 1.f : 0.f);
    dx[o] = acc;
  }
}

__global__ void __launch_bounds__(256) k_copy4(float* __restrict__ dst, esgd_tensor4 dd,
                                               int64_t d_sb, const float* __restrict__ src,
                                               esgd_tensor4 sd, int64_t s_sb) {
  const int z = blockIdx.y;
  const int64_t total = (int64_t)dd.n * dd.c * dd.h * dd.w;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t t = e;
    const int w = (int)(t % dd.w); t /= dd.w;
    const int h = (int)(t % dd.h); t /= dd.h;
    const int c = (int)(t % dd.c);
    const int n = (int)(t / dd.c);
    dst[z * d_sb + off4(dd, n, c, h, w)] = __ldg(src + z * s_sb + off4(sd, n, c, h, w));
  }
}

bool valid4(const esgd_tensor4& t) { return t.n >= 1 && t.c >= 1 && t.h >= 1 && t.w >= 1; }

}  // namespace
}  // namespace esgd

using namespace esgd;
#define ESGD_STREAM(s) reinterpret_cast<cudaStream_t>(s)

extern "C" int esgd_im2col_f32(float* col, int64_t ldc, int64_t col_sb, const float* x,
                               esgd_tensor4 xd, int64_t x_sb, int32_t kh, int32_t kw,
                               int32_t stride, int32_t pad, int32_t oh, int32_t ow, int32_t batch,
                               esgd_stream_t stream) {
  ESGD_REQUIRE(valid4(xd) && kh >= 1 && kw >= 1 && stride >= 1 && pad >= 0 && oh >= 1 &&
                   ow >= 1 && batch >= 1,
               ESGD_ERR_SHAPE, "im2col: bad geometry");
  ESGD_REQUIRE(ldc >= (int64_t)xd.c * kh * kw, ESGD_ERR_SHAPE, "im2col: ldc < C*kh*kw");
  ESGD_REQUIRE(batch <= 65535, ESGD_ERR_UNSUPPORTED, "im2col: batch > 65535");
  ESGD_REQUIRE(col && x, ESGD_ERR_INPUT, "im2col: null buffer");
  int64_t total = (int64_t)xd.n * oh * ow * ldc;
  dim3 grid(stride_grid(total, 256, 16), batch);
  k_im2col<<<grid, 256, 0, ESGD_STREAM(stream)>>>(col, ldc, col_sb, x, xd, x_sb, kh, kw, stride, pad, oh, ow);
  return check_launch("esgd_im2col_f32");
}

extern "C" int esgd_col2im_f32(float* dx, esgd_tensor4 xd, int64_t x_sb, const float* dcol,
                               int64_t ldc, int64_t col_sb, int32_t kh, int32_t kw, int32_t stride,
                               int32_t pad, int32_t oh, int32_t ow, const float* mask,
                               int32_t batch, esgd_stream_t stream) {
  ESGD_REQUIRE(valid4(xd) && kh >= 1 && kw >= 1 && stride >= 1 && pad >= 0 && oh >= 1 &&
                   ow >= 1 && batch >= 1,
               ESGD_ERR_SHAPE, "col2im: bad geometry");
  ESGD_REQUIRE(ldc >= (int64_t)xd.c * kh * kw, ESGD_ERR_SHAPE, "col2im: ldc < C*kh*kw");
  ESGD_REQUIRE(batch <= 65535, ESGD_ERR_UNSUPPORTED, "col2im: batch > 65535");
  ESGD_REQUIRE(dx && dcol, ESGD_ERR_INPUT, "col2im: null buffer");
  int64_t total = (int64_t)xd.n * xd.c * xd.h * xd.w;
  dim3 grid(stride_grid(total, 256, 16), batch);
  k_col2im<<<grid, 256, 0, ESGD_STREAM(stream)>>>(dx, xd, x_sb, dcol, ldc, col_sb, kh, kw, stride, pad, oh, ow, mask);
  return check_launch("esgd_col2im_f32");
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
  int64_t total = (int64_t)yd.n * yd.c * yd.h * yd.w;
  dim3 grid(stride_grid(total, 256, 16), batch);
  k_maxpool_fwd<<<grid, 256, 0, ESGD_STREAM(stream)>>>(y, yd, y_sb, argmax, x, xd, x_sb, k, stride, pad);
  return check_launch("esgd_maxpool_fwd_f32");
}

extern "C" int esgd_maxpool_bwd_f32(float* dx, esgd_tensor4 xd, int64_t x_sb, const float* dy,
                                    esgd_tensor4 yd, int64_t y_sb, const int32_t* argmax,
                                    const float* mask, int32_t k, int32_t stride, int32_t pad,
                                    int32_t batch, esgd_stream_t stream) {
  ESGD_REQUIRE(valid4(xd) && valid4(yd) && k >= 1 && stride >= 1 && pad >= 0 && batch >= 1 &&
                   yd.n == xd.n && yd.c == xd.c,
               ESGD_ERR_SHAPE, "maxpool_bwd: bad geometry");
  ESGD_REQUIRE(batch <= 65535, ESGD_ERR_UNSUPPORTED, "maxpool: batch > 65535");
  ESGD_REQUIRE(dx && dy && argmax, ESGD_ERR_INPUT, "maxpool_bwd: null buffer");
  int64_t total = (int64_t)xd.n * xd.c * xd.h * xd.w;
  dim3 grid(stride_grid(total, 256, 16), batch);
  k_maxpool_bwd<<<grid, 256, 0, ESGD_STREAM(stream)>>>(dx, xd, x_sb, dy, yd, y_sb, argmax, mask, k, stride, pad);
  return check_launch("esgd_maxpool_bwd_f32");
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
