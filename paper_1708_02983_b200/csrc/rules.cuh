// Shared device helpers of the update kernels (updates.cu, nvls.cu): the
// reference's scalar rules in its exact fp32 operation order (explicit RN
// intrinsics, so ptxas cannot contract a multiply-add) and the binomial
// tree-sum association of fabric/collectives.py.
#pragma once
#include "esgd_common.cuh"

namespace esgd {
namespace {

// ---- scalar rules (reference operation order) -----------------------------

// updates.py:93  (w - eta*grad) - (eta*rho)*(w - center)
__device__ __forceinline__ float worker_rule(float w, float g, float c, float eta, float er) {
  return __fsub_rn(__fsub_rn(w, __fmul_rn(eta, g)), __fmul_rn(er, __fsub_rn(w, c)));
}
// updates.py:119  center + (eta*rho)*(weight_sum - num_workers*center)
__device__ __forceinline__ float center_rule(float c, float s, float p, float er) {
  return __fadd_rn(c, __fmul_rn(er, __fsub_rn(s, __fmul_rn(p, c))));
}
// updates.py:131  center + (eta*rho)*(worker - center)
__device__ __forceinline__ float incr_rule(float c, float w, float er) {
  return __fadd_rn(c, __fmul_rn(er, __fsub_rn(w, c)));
}
// updates.py:139  v' = mu*v - eta*grad
__device__ __forceinline__ float momentum_rule(float v, float g, float mu, float eta) {
  return __fsub_rn(__fmul_rn(mu, v), __fmul_rn(eta, g));
}
// updates.py:140  (w + v') - (eta*rho)*(w - center)
__device__ __forceinline__ float measgd_rule(float w, float vn, float c, float er) {
  return __fsub_rn(__fadd_rn(w, vn), __fmul_rn(er, __fsub_rn(w, c)));
}

__device__ __forceinline__ float4 ld4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ float4 ld4rw(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }

// tree_sum (fabric/collectives.py:25-32): partial[pos] += partial[pos+distance]
// for distance = 1, 2, 4, ... — the same association as the reference, kept in
// registers (fully unrolled over the compile-time bound).
template <int MAXP>
__device__ __forceinline__ float binomial_sum(float (&v)[MAXP], int p) {
#pragma unroll
  for (int d = 1; d < MAXP; d <<= 1) {
#pragma unroll
    for (int pos = 0; pos + d < MAXP; pos += 2 * d)
      if (pos + d < p) v[pos] = __fadd_rn(v[pos], v[pos + d]);
  }
  return v[0];
}

}  // namespace
}  // namespace esgd
