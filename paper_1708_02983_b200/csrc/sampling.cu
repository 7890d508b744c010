// Counter-based SplitMix64 draws (rng.py) and with-replacement minibatch
// sampling (datasets.py:166-171) on the device, plus the quadratic problem's
// gradient (trainers/problems.py:95-96).
//
// Integer work: uint64 wrap-around arithmetic is bit-identical to the
// reference's numpy uint64 path, so drawn indices match exactly.
#include "esgd_common.cuh"

namespace esgd {
namespace {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;  // rng.py:30

// rng.py:44-49 (_mix64_vec)
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// CounterRng._raw_block draw i (0-based) of a stream at `counter` (rng.py:66-70)
__device__ __forceinline__ uint64_t draw(uint64_t seed, uint64_t counter, uint64_t i) {
  return mix64(seed + (counter + i + 1) * kGolden);
}

__global__ void k_randint(int64_t* out, uint64_t seed, uint64_t counter, int64_t count,
                          uint64_t upper) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int64_t)(draw(seed, counter, (uint64_t)i) % upper);
}

// One CTA per (sample, row chunk, replica): draw the row index, copy the
// chunk (128-bit when the row pitch allows, kUnroll independent loads in
// flight per thread), chunk 0 writes the label. The last CTA of a replica to
// finish advances that replica's counter by b so the launch is replayable.
constexpr int kSampleThreads = 256, kSampleUnroll = 4;
constexpr int64_t kSampleChunk = kSampleThreads * kSampleUnroll;  // vectors per CTA

template <int V>
__global__ void __launch_bounds__(kSampleThreads) k_sample_batch(float* __restrict__ xo, int64_t ldx_rep,
                                                                 int32_t* __restrict__ yo, int64_t* idx_out,
                                                                 const float* __restrict__ X,
                                                                 const int32_t* __restrict__ labels,
                                                                 int64_t n, int64_t d, uint64_t* rng_state,
                                                                 int32_t* ticket, int b) {
  const int i = blockIdx.x, r = blockIdx.z;
  const uint64_t seed = rng_state[2 * r], counter = rng_state[2 * r + 1];
  const int64_t row = (int64_t)(draw(seed, counter, (uint64_t)i) % (uint64_t)n);
  const int64_t nv = d / V, v0 = blockIdx.y * kSampleChunk;
  if (V == 4) {
    const float4* s4 = reinterpret_cast<const float4*>(X + row * d);
    float4* d4 = reinterpret_cast<float4*>(xo + r * ldx_rep + (int64_t)i * d);
    float4 t[kSampleUnroll];
#pragma unroll
    for (int u = 0; u < kSampleUnroll; ++u) {
      const int64_t j = v0 + u * kSampleThreads + threadIdx.x;
      if (j < nv) t[u] = __ldg(s4 + j);
    }
#pragma unroll
    for (int u = 0; u < kSampleUnroll; ++u) {
      const int64_t j = v0 + u * kSampleThreads + threadIdx.x;
      if (j < nv) d4[j] = t[u];
    }
  } else {
    const float* src = X + row * d;
    float* dst = xo + r * ldx_rep + (int64_t)i * d;
    for (int64_t j = v0 + threadIdx.x; j < min(nv, v0 + kSampleChunk); j += kSampleThreads) dst[j] = __ldg(src + j);
  }
  if (threadIdx.x == 0 && blockIdx.y == 0) {
    yo[r * b + i] = labels[row];
    if (idx_out) idx_out[r * b + i] = row;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const int t = atomicAdd(ticket + r, 1);
    if (t == b * (int)gridDim.y - 1) {  // every CTA of this replica has read the counter
      rng_state[2 * r + 1] = counter + (uint64_t)b;
      ticket[r] = 0;
      __threadfence();
    }
  }
}

template <int V>
__global__ void __launch_bounds__(256) k_quad_grad(float* G, int64_t ldg, const float* W,
                                                   int64_t ldw, int nrep,
                                                   const float* __restrict__ target,
                                                   const float* __restrict__ curv, int64_t n) {
  // curvature * (weights - target)
  int64_t nv = n / V;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (V == 4) {
      float4 t = __ldg(reinterpret_cast<const float4*>(target) + i);
      float4 c = __ldg(reinterpret_cast<const float4*>(curv) + i);
      for (int r = 0; r < nrep; ++r) {
        float4 w = reinterpret_cast<const float4*>(W + r * ldw)[i], g;
        g.x = __fmul_rn(c.x, __fsub_rn(w.x, t.x));
        g.y = __fmul_rn(c.y, __fsub_rn(w.y, t.y));
        g.z = __fmul_rn(c.z, __fsub_rn(w.z, t.z));
        g.w = __fmul_rn(c.w, __fsub_rn(w.w, t.w));
        reinterpret_cast<float4*>(G + r * ldg)[i] = g;
      }
    } else {
      for (int r = 0; r < nrep; ++r)
        G[r * ldg + i] = __fmul_rn(curv[i], __fsub_rn(W[r * ldw + i], target[i]));
    }
  }
  if (V == 4 && blockIdx.x == 0 && threadIdx.x < (n & 3)) {
    int64_t j = (n & ~int64_t(3)) + threadIdx.x;
    for (int r = 0; r < nrep; ++r)
      G[r * ldg + j] = __fmul_rn(curv[j], __fsub_rn(W[r * ldw + j], target[j]));
  }
}

}  // namespace
}  // namespace esgd

using namespace esgd;
#define ESGD_STREAM(s) reinterpret_cast<cudaStream_t>(s)

extern "C" int esgd_randint_u64(int64_t* out, uint64_t seed, uint64_t counter, int64_t count,
                                uint64_t upper, esgd_stream_t stream) {
  ESGD_REQUIRE(upper > 0, ESGD_ERR_INPUT, "upper bound must be positive, got %llu",
               (unsigned long long)upper);
  ESGD_REQUIRE(count >= 0, ESGD_ERR_SHAPE, "randint: negative count");
  if (count == 0) return ESGD_OK;
  ESGD_REQUIRE(out, ESGD_ERR_INPUT, "randint: null buffer");
  k_randint<<<stride_grid(count, 256), 256, 0, ESGD_STREAM(stream)>>>(out, seed, counter, count, upper);
  return check_launch("esgd_randint_u64");
}

extern "C" int esgd_sample_batch_f32(float* x_out, int64_t ldx_rep, int32_t* y_out,
                                     int64_t* idx_out, const float* X, const int32_t* labels,
                                     int64_t n, int64_t d, uint64_t* rng_state, int32_t* ticket,
                                     int32_t b, int32_t nrep, esgd_stream_t stream) {
  ESGD_REQUIRE(b >= 1 && b <= n, ESGD_ERR_INPUT, "batch size %d out of range [1, %lld]", b,
               (long long)n);
  ESGD_REQUIRE(d >= 1 && nrep >= 1, ESGD_ERR_SHAPE, "sample_batch: bad shape");
  ESGD_REQUIRE(nrep == 1 || ldx_rep >= (int64_t)b * d, ESGD_ERR_SHAPE,
               "sample_batch: replica pitch shorter than b*d");
  ESGD_REQUIRE(b <= 65535 * 64 && nrep <= 65535, ESGD_ERR_UNSUPPORTED, "sample_batch: grid too large");
  ESGD_REQUIRE(x_out && y_out && X && labels && rng_state && ticket, ESGD_ERR_INPUT,
               "sample_batch: null buffer");
  bool v4 = (d & 3) == 0 && aligned16(x_out) && aligned16(X) && (ldx_rep & 3) == 0;
  const int64_t nchunk = ((v4 ? d / 4 : d) + kSampleChunk - 1) / kSampleChunk;
  ESGD_REQUIRE(nchunk <= 65535 && (int64_t)b * nchunk < (int64_t(1) << 31), ESGD_ERR_UNSUPPORTED,
               "sample_batch: rows too long");
  dim3 grid(b, (unsigned)nchunk, nrep);
  if (v4)
    k_sample_batch<4><<<grid, kSampleThreads, 0, ESGD_STREAM(stream)>>>(x_out, ldx_rep, y_out, idx_out, X, labels, n, d, rng_state, ticket, b);
  else
    k_sample_batch<1><<<grid, kSampleThreads, 0, ESGD_STREAM(stream)>>>(x_out, ldx_rep, y_out, idx_out, X, labels, n, d, rng_state, ticket, b);
  return check_launch("esgd_sample_batch_f32");
}

extern "C" int esgd_gather_rows_h2d(void* dst, int64_t dst_pitch, const void* src, int64_t src_pitch,
                                    const int64_t* rows, int32_t nrows, int64_t row_bytes, int64_t src_rows,
                                    esgd_stream_t stream) {
  ESGD_REQUIRE(nrows >= 0 && row_bytes >= 0 && dst_pitch >= row_bytes && src_pitch >= row_bytes, ESGD_ERR_SHAPE,
               "gather_rows_h2d: bad geometry");
  if (nrows == 0 || row_bytes == 0) return ESGD_OK;
  ESGD_REQUIRE(dst && src && rows, ESGD_ERR_INPUT, "gather_rows_h2d: null pointer");
  cudaStream_t st = ESGD_STREAM(stream);
  char* d = static_cast<char*>(dst);
  const char* s = static_cast<const char*>(src);
  for (int32_t i = 0; i < nrows;) {
    const int64_t r = rows[i];
    ESGD_REQUIRE(r >= 0 && r < src_rows, ESGD_ERR_INPUT, "gather_rows_h2d: row %lld out of range [0, %lld)",
                 (long long)r, (long long)src_rows);
    int32_t run = 1;  // merge consecutive source rows into one transfer when the pitches allow
    while (i + run < nrows && rows[i + run] == r + run && dst_pitch == src_pitch) ++run;
    const cudaError_t e = cudaMemcpyAsync(d + (int64_t)i * dst_pitch, s + r * src_pitch,
                                          (size_t)((run - 1) * src_pitch + row_bytes), cudaMemcpyHostToDevice, st);
    ESGD_REQUIRE(e == cudaSuccess, ESGD_ERR_CUDA, "gather_rows_h2d: %s", cudaGetErrorString(e));
    i += run;
  }
  return ESGD_OK;
}

extern "C" int esgd_quadratic_grad_f32(float* G, int64_t ldg, const float* W, int64_t ldw,
                                       int32_t nrep, const float* target, const float* curvature,
                                       int64_t n, esgd_stream_t stream) {
  ESGD_REQUIRE(n >= 0 && nrep >= 1, ESGD_ERR_SHAPE, "quadratic_grad: bad shape");
  ESGD_REQUIRE(nrep == 1 || (ldw >= n && ldg >= n), ESGD_ERR_SHAPE, "quadratic_grad: pitch < n");
  if (n == 0) return ESGD_OK;
  ESGD_REQUIRE(G && W && target && curvature, ESGD_ERR_INPUT, "quadratic_grad: null buffer");
  bool v4 = aligned16(G) && aligned16(W) && aligned16(target) && aligned16(curvature) &&
            (nrep == 1 || ((ldw & 3) == 0 && (ldg & 3) == 0));
  if (v4)
    k_quad_grad<4><<<stride_grid(n / 4 + 1, 256), 256, 0, ESGD_STREAM(stream)>>>(G, ldg, W, ldw, nrep, target, curvature, n);
  else
    k_quad_grad<1><<<stride_grid(n, 256), 256, 0, ESGD_STREAM(stream)>>>(G, ldg, W, ldw, nrep, target, curvature, n);
  return check_launch("esgd_quadratic_grad_f32");
}
