// Dense-layer kernels for the per-worker gradient (trainers/problems.py:42-47):
// a strided/batched fp32 FFMA GEMM for the small contractions (LeNet/MLP
// shapes are launch-latency bound), activations, the fused
// softmax cross-entropy (kernels.py:85-106), row argmax and deterministic
// column sums (bias gradients, network.py:195).
#include "esgd_common.cuh"

#include <stdlib.h>

#include <math.h>

namespace esgd {
namespace {

// ---- activations (kernels.py:30-70) ----------------------------------------

__device__ __forceinline__ float act_apply(float z, int act) {
  switch (act) {
    case ESGD_ACT_RELU: return fmaxf(z, 0.f);
    case ESGD_ACT_TANH: return tanhf(z);
    case ESGD_ACT_SIGMOID:
      if (z >= 0.f) return 1.f / (1.f + expf(-z));
      else { float e = expf(z); return e / (1.f + e); }
    default: return z;
  }
}

// d * act'(z), kernels.py:34-66 (relu_grad is (z > 0) as 0/1)
__device__ __forceinline__ float act_grad_mul(float d, float z, int act) {
  switch (act) {
    case ESGD_ACT_RELU: return __fmul_rn(d, z > 0.f ? 1.f : 0.f);
    case ESGD_ACT_TANH: { float t = tanhf(z); return d * (1.f - t * t); }
    case ESGD_ACT_SIGMOID: { float s = act_apply(z, ESGD_ACT_SIGMOID); return d * (s * (1.f - s)); }
    default: return d;
  }
}

// ---- strided batched FFMA GEMM ---------------------------------------------
// TBM x TBN output tile per 256-thread CTA (16x16 threads, (TBM/16)x(TBN/16)
// per thread), BK=16 slabs staged through shared memory (A transposed so the
// inner loop reads contiguous rows). 64x64 for large outputs, 32x32 when the
// output is skinny (weight gradients of small layers) so more CTAs share the
// split-K reduction.
constexpr int BK = 16;
#ifndef ESGD_REDUCE8_MIN
#define ESGD_REDUCE8_MIN 16
#endif

__device__ __forceinline__ float epilogue(const esgd_gemm_desc& d, float acc, int z, int gm, int gn,
                                          float* C, float* Cp, int64_t off) {
  const float* bias = d.bias ? d.bias + z * d.bias_sb : nullptr;
  const float* mask = d.mask ? d.mask + z * d.mask_sb : nullptr;
  float v = acc;
  if (d.accumulate) v = __fadd_rn(C[off], v);
  if (bias) v = __fadd_rn(v, bias[gn]);
  if (Cp) Cp[off] = v;
  v = act_apply(v, d.act);
  if (mask) v = __fmul_rn(v, mask[(int64_t)gm * d.mask_sm + (int64_t)gn * d.mask_sn] > 0.f ? 1.f : 0.f);
  return v;
}

// splits > 1: blockIdx.z = batch * splits + slice; each slice reduces its own
// k range and writes raw partials to ws[z][slice][m][n]; k_gemm_reduce
// combines slices in order and applies the epilogue.
template <int TBM, int TBN>
__global__ void __launch_bounds__(256) k_gemm(esgd_gemm_desc d, int splits, int kchunk) {
  constexpr int MI = TBM / 16, NI = TBN / 16, LA = TBM * BK / 256, LB = TBN * BK / 256;
  __shared__ __align__(16) float As[2][BK][TBM + 4];
  __shared__ __align__(16) float Bs[2][BK][TBN + 4];
  const int z = blockIdx.z / splits, slice = blockIdx.z % splits;
  const int kbeg = slice * kchunk, kend = min(d.k, kbeg + kchunk);
  const float* A = d.a + z * d.a_sb;
  const float* B = d.b + z * d.b_sb;
  const int m0 = blockIdx.y * TBM, n0 = blockIdx.x * TBN;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const bool a_kfast = (d.a_sk == 1);
  const bool b_nfast = (d.b_sn == 1);

  float acc[MI][NI];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) acc[i][j] = 0.f;

  float ra[LA], rb[LB];
  auto load_regs = [&](int k0) {
#pragma unroll
    for (int j = 0; j < LA; ++j) {
      int e = tid + j * 256;
      int mm, kk;
      if (a_kfast) { mm = e / BK; kk = e % BK; } else { mm = e % TBM; kk = e / TBM; }
      int gm = m0 + mm, gk = k0 + kk;
      ra[j] = (gm < d.m && gk < kend) ? __ldg(A + (int64_t)gm * d.a_sm + (int64_t)gk * d.a_sk) : 0.f;
    }
#pragma unroll
    for (int j = 0; j < LB; ++j) {
      int e = tid + j * 256;
      int nn, kb;
      if (b_nfast) { nn = e % TBN; kb = e / TBN; } else { nn = e / BK; kb = e % BK; }
      int gn = n0 + nn, gkb = k0 + kb;
      rb[j] = (gn < d.n && gkb < kend) ? __ldg(B + (int64_t)gkb * d.b_sk + (int64_t)gn * d.b_sn) : 0.f;
    }
  };
  auto store_smem = [&](int buf) {
#pragma unroll
    for (int j = 0; j < LA; ++j) {
      int e = tid + j * 256;
      int mm, kk;
      if (a_kfast) { mm = e / BK; kk = e % BK; } else { mm = e % TBM; kk = e / TBM; }
      As[buf][kk][mm] = ra[j];
    }
#pragma unroll
    for (int j = 0; j < LB; ++j) {
      int e = tid + j * 256;
      int nn, kb;
      if (b_nfast) { nn = e % TBN; kb = e / TBN; } else { nn = e / BK; kb = e % BK; }
      Bs[buf][kb][nn] = rb[j];
    }
  };

  const int nk = (kend - kbeg + BK - 1) / BK;
  load_regs(kbeg);
  store_smem(0);
  __syncthreads();
  for (int t = 0; t < nk; ++t) {
    const int buf = t & 1;
    if (t + 1 < nk) load_regs(kbeg + (t + 1) * BK);  // prefetch next slab into registers
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float av[MI], bv[NI];
#pragma unroll
      for (int i = 0; i < MI; ++i) av[i] = As[buf][kk][ty * MI + i];
#pragma unroll
      for (int j = 0; j < NI; ++j) bv[j] = Bs[buf][kk][tx * NI + j];
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    if (t + 1 < nk) store_smem(buf ^ 1);
    __syncthreads();
  }

  if (splits > 1) {
    float* P = d.ws + ((int64_t)z * splits + slice) * d.m * d.n;
#pragma unroll
    for (int i = 0; i < MI; ++i) {
      int gm = m0 + ty * MI + i;
      if (gm >= d.m) continue;
#pragma unroll
      for (int j = 0; j < NI; ++j) {
        int gn = n0 + tx * NI + j;
        if (gn < d.n) P[(int64_t)gm * d.n + gn] = acc[i][j];
      }
    }
    return;
  }
  float* C = d.c + z * d.c_sb;
  float* Cp = d.c_pre ? d.c_pre + z * d.c_sb : nullptr;
#pragma unroll
  for (int i = 0; i < MI; ++i) {
    int gm = m0 + ty * MI + i;
    if (gm >= d.m) continue;
#pragma unroll
    for (int j = 0; j < NI; ++j) {
      int gn = n0 + tx * NI + j;
      if (gn >= d.n) continue;
      int64_t off = (int64_t)gm * d.c_sm + (int64_t)gn * d.c_sn;
      C[off] = epilogue(d, acc[i][j], z, gm, gn, C, Cp, off);
    }
  }
}

__global__ void __launch_bounds__(256) k_gemm_reduce(esgd_gemm_desc d, int splits) {
  const int64_t mn = (int64_t)d.m * d.n;
  const int z = blockIdx.y;
  float* C = d.c + z * d.c_sb;
  float* Cp = d.c_pre ? d.c_pre + z * d.c_sb : nullptr;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < mn; e += (int64_t)gridDim.x * blockDim.x) {
    const float* P = d.ws + (int64_t)z * splits * mn + e;
    float v0 = 0.f, v1 = 0.f, v2 = 0.f, v3 = 0.f;
    int s = 0;
    for (; s + 3 < splits; s += 4) {  // four loads in flight per thread, fixed combine order
      v0 += P[s * mn]; v1 += P[(s + 1) * mn]; v2 += P[(s + 2) * mn]; v3 += P[(s + 3) * mn];
    }
    for (; s < splits; ++s) v0 += P[s * mn];
    const float v = (v0 + v1) + (v2 + v3);
    const int gm = (int)(e / d.n), gn = (int)(e % d.n);
    const int64_t off = (int64_t)gm * d.c_sm + (int64_t)gn * d.c_sn;
    C[off] = epilogue(d, v, z, gm, gn, C, Cp, off);
  }
}

// Wide split-K combine: 8 threads per output element, thread j summing
// slices j, j+8, ... (four loads in flight), then a fixed xor-shuffle tree —
// deterministic, and the splits' loads spread over 8x more threads than
// k_gemm_reduce (LeNet's 20 x 25 weight gradient is 128 slices deep: one
// thread per element walked all of them)
__global__ void __launch_bounds__(256) k_gemm_reduce8(esgd_gemm_desc d, int splits) {
  const int64_t mn = (int64_t)d.m * d.n;
  const int z = blockIdx.y;
  const int sub = threadIdx.x & 7;
  float* C = d.c + z * d.c_sb;
  float* Cp = d.c_pre ? d.c_pre + z * d.c_sb : nullptr;
  const int64_t stride = ((int64_t)gridDim.x * blockDim.x) >> 3;
  // e0 is warp-uniform (4 elements per warp), so every lane reaches the shuffles
  for (int64_t e0 = (blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31)) >> 3; e0 < mn; e0 += stride) {
    const int64_t e = e0 + ((threadIdx.x & 31) >> 3);
    float v0 = 0.f, v1 = 0.f, v2 = 0.f, v3 = 0.f;
    if (e < mn) {
      const float* P = d.ws + (int64_t)z * splits * mn + e;
      int s = sub;
      for (; s + 24 < splits; s += 32) {
        v0 += P[s * mn]; v1 += P[(s + 8) * mn]; v2 += P[(s + 16) * mn]; v3 += P[(s + 24) * mn];
      }
      for (; s < splits; s += 8) v0 += P[s * mn];
    }
    float v = (v0 + v1) + (v2 + v3);
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    v += __shfl_xor_sync(0xffffffffu, v, 2);
    v += __shfl_xor_sync(0xffffffffu, v, 4);
    if (sub == 0 && e < mn) {
      const int gm = (int)(e / d.n), gn = (int)(e % d.n);
      const int64_t off = (int64_t)gm * d.c_sm + (int64_t)gn * d.c_sn;
      C[off] = epilogue(d, v, z, gm, gn, C, Cp, off);
    }
  }
}

__global__ void k_act_fwd(float* y, const float* z, int64_t n, int act) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = act_apply(z[i], act);
}
__global__ void k_act_bwd(float* dd, const float* z, int64_t n, int act) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dd[i] = act_grad_mul(dd[i], z[i], act);
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// softmax_cross_entropy (kernels.py:85-106): one warp per row.
__global__ void __launch_bounds__(128) k_softmax_xent(float* dl, float* row_loss, const float* lg,
                                                      int64_t ld, int64_t zs, const int32_t* labels,
                                                      int64_t lzs, int rows, int cols,
                                                      int32_t* bad) {
  const int z = blockIdx.y;
  const int row = blockIdx.x * 4 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const float* x = lg + z * zs + (int64_t)row * ld;
  float* o = dl + z * zs + (int64_t)row * ld;
  const int label = labels[z * lzs + row];
  const bool ok = label >= 0 && label < cols;
  float m = -INFINITY;
  for (int j = lane; j < cols; j += 32) m = fmaxf(m, x[j]);
  m = warp_max(m);
  float s = 0.f;
  for (int j = lane; j < cols; j += 32) s += expf(x[j] - m);
  s = warp_sum(s);
  float picked = 0.f;
  for (int j = lane; j < cols; j += 32) {
    float p = expf(x[j] - m) / s;
    if (j == label) picked = p;
    float g = (j == label) ? __fsub_rn(p, 1.f) : p;
    o[j] = ok ? __fdiv_rn(g, (float)rows) : 0.f;
  }
  picked = warp_sum(picked);
  if (lane == 0) {
    if (row_loss) row_loss[z * rows + row] = ok ? -logf(picked) : NAN;
    if (!ok && bad) *bad = 1;
  }
}

__global__ void __launch_bounds__(128) k_argmax(int32_t* out, const float* x, int64_t ld, int rows,
                                                int cols) {
  const int row = blockIdx.x * 4 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const float* r = x + (int64_t)row * ld;
  float best = -INFINITY;
  int bi = 0x7fffffff;
  for (int j = lane; j < cols; j += 32) {
    float v = r[j];
    if (v > best || (v == best && j < bi)) { best = v; bi = j; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    float ov = __shfl_xor_sync(0xffffffffu, best, o);
    int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
  }
  if (lane == 0) out[row] = bi == 0x7fffffff ? 0 : bi;
}

// Column sums, pass 1: CTA = 32 columns x 8 row-lanes over one row chunk;
// every thread keeps 4 independent partial sums (loads in flight instead of a
// serial dependency chain), combined in a fixed order, one partial per
// (chunk, col).
__global__ void __launch_bounds__(256) k_colsum_partial(float* part, const float* __restrict__ x, int64_t ld,
                                                        int64_t x_sb, int64_t rows, int cols,
                                                        int64_t chunk, float* out, int64_t out_sb,
                                                        int direct) {
  __shared__ float red[8][33];
  const int z = blockIdx.z, c = blockIdx.x * 32 + threadIdx.x, ty = threadIdx.y;
  const int64_t r0 = blockIdx.y * chunk, r1 = min(rows, r0 + chunk);
  const float* xz = x + z * x_sb;
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
  if (c < cols) {
    int64_t r = r0 + ty;
    for (; r + 24 < r1; r += 32) {
      s0 += __ldg(xz + r * ld + c);
      s1 += __ldg(xz + (r + 8) * ld + c);
      s2 += __ldg(xz + (r + 16) * ld + c);
      s3 += __ldg(xz + (r + 24) * ld + c);
    }
    for (; r < r1; r += 8) s0 += __ldg(xz + r * ld + c);
  }
  red[ty][threadIdx.x] = (s0 + s1) + (s2 + s3);
  __syncthreads();
  if (ty == 0 && c < cols) {
    float t = red[0][threadIdx.x];
#pragma unroll
    for (int k = 1; k < 8; ++k) t += red[k][threadIdx.x];
    if (direct) out[z * out_sb + c] = t;
    else part[((int64_t)z * gridDim.y + blockIdx.y) * cols + c] = t;
  }
}
__global__ void k_colsum_final(float* out, int64_t out_sb, const float* part, int nchunk, int cols,
                               int batch) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cols * batch) return;
  int z = i / cols, c = i % cols;
  const float* p = part + (int64_t)z * nchunk * cols + c;
  float t0 = 0.f, t1 = 0.f;
  int k = 0;
  for (; k + 1 < nchunk; k += 2) { t0 += p[(int64_t)k * cols]; t1 += p[(int64_t)(k + 1) * cols]; }
  if (k < nchunk) t0 += p[(int64_t)k * cols];
  out[z * out_sb + c] = t0 + t1;
}

// batched 2-D transpose through a padded 32x33 smem tile (both sides coalesced)
__global__ void __launch_bounds__(256) k_transpose(float* __restrict__ dst, int64_t ldd, int64_t d_sb,
                                                   const float* __restrict__ src, int64_t lds, int64_t s_sb,
                                                   int rows, int cols) {
  __shared__ float tile[32][33];
  const int z = blockIdx.z;
  const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
  const float* sz = src + z * s_sb;
  float* dz = dst + z * d_sb;
#pragma unroll
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int r = r0 + i, c = c0 + threadIdx.x;
    tile[i][threadIdx.x] = (r < rows && c < cols) ? __ldg(sz + (int64_t)r * lds + c) : 0.f;
  }
  __syncthreads();
#pragma unroll
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int c = c0 + i, r = r0 + threadIdx.x;
    if (c < cols && r < rows) dz[(int64_t)c * ldd + r] = tile[threadIdx.x][i];
  }
}

}  // namespace
}  // namespace esgd

using namespace esgd;
#define ESGD_STREAM(s) reinterpret_cast<cudaStream_t>(s)

namespace esgd {
namespace {
// Tile and K split of one FFMA GEMM. The split depends on the per-replica
// problem only (never on `batch` or the workspace size): replicas compute
// bit-identical results whatever the launch groups them with. A NULL
// workspace means "do not split"; one that is too small is an error.
struct FfmaPlan {
  bool small;
  int splits, kchunk;
};
FfmaPlan ffma_plan(const esgd_gemm_desc* d) {
  // tuning knobs (read once): ESGD_FFMA_TILE = 32 / 64 forces the tile,
  // ESGD_FFMA_MAXSPLIT caps the K split
  static const int force_tile = getenv("ESGD_FFMA_TILE") ? atoi(getenv("ESGD_FFMA_TILE")) : 0;
  static const int max_split = getenv("ESGD_FFMA_MAXSPLIT") ? atoi(getenv("ESGD_FFMA_MAXSPLIT")) : 128;
  FfmaPlan p;
  // 32x32 tiles only for outputs that are <= 32 wide on one side (a 64-wide
  // tile would be mostly padding); measured per LeNet GEMM: conv1 fwd
  // (N = 20) 17.1 -> 12.7 us, conv2 fwd / wgrad 30.9 -> 24.7 / 35.1 -> 23.4 us
  p.small = force_tile ? force_tile == 32 : (d->m <= 32 || d->n <= 32);
  const int TM = p.small ? 32 : 64, TN = TM;
  const int tiles = ((d->n + TN - 1) / TN) * ((d->m + TM - 1) / TM);
  int splits = 1;
  if (d->ws && tiles < 2 * kNumSMs && d->k >= 4 * BK * 4) {
    // enough slices to give ~2 CTAs per SM, each slice at least 4 slabs deep
    int want = (2 * kNumSMs + tiles - 1) / tiles;
    int maxs = d->k / (4 * BK);
    splits = want < maxs ? want : maxs;
    if (splits > max_split) splits = max_split;
    if (splits < 1) splits = 1;
  }
  p.kchunk = ((d->k + splits - 1) / splits + BK - 1) / BK * BK;
  p.splits = splits > 1 ? (d->k + p.kchunk - 1) / p.kchunk : 1;
  return p;
}
}  // namespace
}  // namespace esgd

extern "C" int esgd_gemm_ws_floats(const esgd_gemm_desc* d, int64_t* floats) {
  using namespace esgd;
  ESGD_REQUIRE(d && floats, ESGD_ERR_INPUT, "gemm_ws_floats: null argument");
  *floats = 0;
  if (d->m <= 0 || d->n <= 0 || d->batch <= 0 || d->k <= 0) return ESGD_OK;
  esgd_gemm_desc q = *d;
  if (!q.ws) q.ws = reinterpret_cast<float*>(uintptr_t(256));
  const FfmaPlan p = ffma_plan(&q);
  *floats = p.splits > 1 ? (int64_t)p.splits * d->m * d->n * d->batch : 0;
  return ESGD_OK;
}

extern "C" int esgd_gemm_f32(const esgd_gemm_desc* d, esgd_stream_t stream) {
  ESGD_REQUIRE(d, ESGD_ERR_INPUT, "gemm: null descriptor");
  ESGD_REQUIRE(d->m >= 0 && d->n >= 0 && d->k >= 0 && d->batch >= 0, ESGD_ERR_SHAPE,
               "gemm shape mismatch: m=%d n=%d k=%d batch=%d", d->m, d->n, d->k, d->batch);
  ESGD_REQUIRE(d->act >= 0 && d->act <= 3, ESGD_ERR_INPUT, "gemm: unknown activation %d", d->act);
  if (d->m == 0 || d->n == 0 || d->batch == 0) return ESGD_OK;
  ESGD_REQUIRE(d->c && (d->k == 0 || (d->a && d->b)), ESGD_ERR_INPUT, "gemm: null operand");
  ESGD_REQUIRE(d->batch <= 65535, ESGD_ERR_UNSUPPORTED, "gemm: batch > 65535");
  const esgd::FfmaPlan p = esgd::ffma_plan(d);
  const int splits = p.splits, kchunk = p.kchunk;
  const int TM = p.small ? 32 : 64, TN = TM;
  if (splits > 1) {
    const int64_t need = (int64_t)splits * d->m * d->n * d->batch;
    ESGD_REQUIRE(need <= d->ws_floats, ESGD_ERR_UNSUPPORTED,
                 "gemm: split-K workspace too small (need %lld floats, have %lld; size it with "
                 "esgd_gemm_ws_floats)", (long long)need, (long long)d->ws_floats);
    ESGD_REQUIRE((int64_t)d->batch * splits <= 65535, ESGD_ERR_UNSUPPORTED, "gemm: batch x K split > 65535");
  }
  dim3 grid((d->n + TN - 1) / TN, (d->m + TM - 1) / TM, d->batch * splits);
  ESGD_REQUIRE(grid.y <= 65535, ESGD_ERR_UNSUPPORTED, "gemm: m too large for the FFMA path");
  if (p.small) k_gemm<32, 32><<<grid, 256, 0, ESGD_STREAM(stream)>>>(*d, splits, kchunk);
  else k_gemm<64, 64><<<grid, 256, 0, ESGD_STREAM(stream)>>>(*d, splits, kchunk);
  if (splits > 1) {
    // deep splits over small outputs: 8 threads per element (k_gemm_reduce8)
    if (splits >= ESGD_REDUCE8_MIN) {
      dim3 rgrid(stride_grid((int64_t)d->m * d->n * 8, 256, 4), d->batch);
      k_gemm_reduce8<<<rgrid, 256, 0, ESGD_STREAM(stream)>>>(*d, splits);
    } else {
      dim3 rgrid(stride_grid((int64_t)d->m * d->n, 256, 4), d->batch);
      k_gemm_reduce<<<rgrid, 256, 0, ESGD_STREAM(stream)>>>(*d, splits);
    }
  }
  return check_launch("esgd_gemm_f32");
}

extern "C" int esgd_act_fwd_f32(float* y, const float* z, int64_t n, int32_t act,
                                esgd_stream_t stream) {
  ESGD_REQUIRE(act >= 0 && act <= 3, ESGD_ERR_INPUT, "unknown activation %d", act);
  if (n <= 0) return n == 0 ? ESGD_OK : ESGD_ERR_SHAPE;
  k_act_fwd<<<stride_grid(n, 256), 256, 0, ESGD_STREAM(stream)>>>(y, z, n, act);
  return check_launch("esgd_act_fwd_f32");
}

extern "C" int esgd_act_bwd_f32(float* dd, const float* z, int64_t n, int32_t act,
                                esgd_stream_t stream) {
  ESGD_REQUIRE(act >= 0 && act <= 3, ESGD_ERR_INPUT, "unknown activation %d", act);
  if (n <= 0) return n == 0 ? ESGD_OK : ESGD_ERR_SHAPE;
  k_act_bwd<<<stride_grid(n, 256), 256, 0, ESGD_STREAM(stream)>>>(dd, z, n, act);
  return check_launch("esgd_act_bwd_f32");
}

extern "C" int esgd_softmax_xent_f32(float* dlogits, float* row_loss, const float* logits,
                                     int64_t ld, int64_t z_stride, const int32_t* labels,
                                     int64_t label_z_stride, int32_t rows, int32_t cols,
                                     int32_t batch, int32_t* bad_label, esgd_stream_t stream) {
  ESGD_REQUIRE(rows >= 1 && cols >= 1 && batch >= 1 && ld >= cols, ESGD_ERR_SHAPE,
               "softmax_xent: bad shape rows=%d cols=%d ld=%lld", rows, cols, (long long)ld);
  ESGD_REQUIRE(dlogits && logits && labels, ESGD_ERR_INPUT, "softmax_xent: null buffer");
  dim3 grid((rows + 3) / 4, batch);
  k_softmax_xent<<<grid, 128, 0, ESGD_STREAM(stream)>>>(dlogits, row_loss, logits, ld, z_stride,
                                                        labels, label_z_stride, rows, cols, bad_label);
  return check_launch("esgd_softmax_xent_f32");
}

extern "C" int esgd_argmax_rows_f32(int32_t* out, const float* x, int64_t ld, int32_t rows,
                                    int32_t cols, esgd_stream_t stream) {
  ESGD_REQUIRE(rows >= 0 && cols >= 1 && ld >= cols, ESGD_ERR_SHAPE, "argmax: bad shape");
  if (rows == 0) return ESGD_OK;
  k_argmax<<<(rows + 3) / 4, 128, 0, ESGD_STREAM(stream)>>>(out, x, ld, rows, cols);
  return check_launch("esgd_argmax_rows_f32");
}

extern "C" int esgd_colsum_f32(float* out, int64_t out_sb, const float* x, int64_t ld,
                               int64_t x_sb, int64_t rows, int32_t cols, int32_t batch,
                               float* scratch, esgd_stream_t stream) {
  ESGD_REQUIRE(rows >= 1 && cols >= 1 && batch >= 1 && ld >= cols, ESGD_ERR_SHAPE,
               "colsum: bad shape");
  ESGD_REQUIRE(out && x, ESGD_ERR_INPUT, "colsum: null buffer");
  // ~2 CTAs per SM per batch entry, chunks of >= 128 rows (batch-independent
  // chunking keeps each entry's sum order fixed)
  int64_t col_groups = (cols + 31) / 32;
  int64_t nchunk = (rows + 127) / 128;
  int64_t cap = (2 * kNumSMs + col_groups - 1) / col_groups;
  if (nchunk > cap) nchunk = cap;
  if (nchunk > 256) nchunk = 256;
  if (nchunk < 1) nchunk = 1;
  int64_t chunk = (rows + nchunk - 1) / nchunk;
  nchunk = (rows + chunk - 1) / chunk;
  ESGD_REQUIRE(nchunk == 1 || scratch, ESGD_ERR_INPUT, "colsum: scratch required for %lld rows",
               (long long)rows);
  dim3 grid((cols + 31) / 32, (unsigned)nchunk, batch), block(32, 8);
  cudaStream_t st = ESGD_STREAM(stream);
  k_colsum_partial<<<grid, block, 0, st>>>(scratch, x, ld, x_sb, rows, cols, chunk, out, out_sb,
                                           nchunk == 1);
  if (nchunk > 1) {
    int tot = cols * batch;
    k_colsum_final<<<(tot + 255) / 256, 256, 0, st>>>(out, out_sb, scratch, (int)nchunk, cols, batch);
  }
  return check_launch("esgd_colsum_f32");
}

extern "C" int esgd_transpose_f32(float* dst, int64_t ldd, int64_t d_sb, const float* src, int64_t lds,
                                  int64_t s_sb, int32_t rows, int32_t cols, int32_t batch,
                                  esgd_stream_t stream) {
  ESGD_REQUIRE(rows >= 0 && cols >= 0 && batch >= 1 && lds >= cols && ldd >= rows, ESGD_ERR_SHAPE,
               "transpose: bad shape");
  if (rows == 0 || cols == 0) return ESGD_OK;
  ESGD_REQUIRE(dst && src, ESGD_ERR_INPUT, "transpose: null buffer");
  ESGD_REQUIRE((rows + 31) / 32 <= 65535 && batch <= 65535, ESGD_ERR_UNSUPPORTED, "transpose: grid too large");
  dim3 grid((cols + 31) / 32, (rows + 31) / 32, batch), block(32, 8);
  k_transpose<<<grid, block, 0, ESGD_STREAM(stream)>>>(dst, ldd, d_sb, src, lds, s_sb, rows, cols);
  return check_launch("esgd_transpose_f32");
}
