// Elastic-averaging update rules (updates.py) and the replica reduction
// (fabric/collectives.py tree_sum) as HBM-streaming sm_100a kernels.
//
// All rules are pure elementwise streams: one 128-bit load per operand per
// four parameters, grid-stride over 148 SMs x 8 resident CTAs, no shared
// memory (nothing is reused). Arithmetic is the reference's exact fp32
// operation order with explicit round-to-nearest intrinsics so ptxas cannot
// contract a multiply-add: results are bitwise equal to the float32
// reference (SURVEY.md §8c "Bit-exactness available").
#include "esgd_common.cuh"
#include "rules.cuh"

namespace esgd {
namespace {

// ---- worker / center rules ------------------------------------------------
// (outputs are not __restrict__: the in-place callers pass wo == w)

template <int V>
__global__ void __launch_bounds__(256) k_worker_step(float* wo, const float* w,
                                                     const float* __restrict__ g,
                                                     const float* __restrict__ c, int64_t n,
                                                     float eta, float er) {
  int64_t nv = n / V;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (V == 4) {
      float4 a = ld4rw(w + 4 * i), b = ld4(g + 4 * i), d = ld4(c + 4 * i), r;
      r.x = worker_rule(a.x, b.x, d.x, eta, er);
      r.y = worker_rule(a.y, b.y, d.y, eta, er);
      r.z = worker_rule(a.z, b.z, d.z, eta, er);
      r.w = worker_rule(a.w, b.w, d.w, eta, er);
      st4(wo + 4 * i, r);
    } else {
      wo[i] = worker_rule(w[i], g[i], c[i], eta, er);
    }
  }
  if (V == 4 && blockIdx.x == 0 && threadIdx.x < (n & 3)) {
    int64_t j = (n & ~int64_t(3)) + threadIdx.x;
    wo[j] = worker_rule(w[j], g[j], c[j], eta, er);
  }
}

template <int V>
__global__ void __launch_bounds__(256) k_center_from_sum(float* co, const float* c,
                                                         const float* __restrict__ s, int64_t n,
                                                         float er, float p) {
  int64_t nv = n / V;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (V == 4) {
      float4 a = ld4rw(c + 4 * i), b = ld4(s + 4 * i), r;
      r.x = center_rule(a.x, b.x, p, er);
      r.y = center_rule(a.y, b.y, p, er);
      r.z = center_rule(a.z, b.z, p, er);
      r.w = center_rule(a.w, b.w, p, er);
      st4(co + 4 * i, r);
    } else {
      co[i] = center_rule(c[i], s[i], p, er);
    }
  }
  if (V == 4 && blockIdx.x == 0 && threadIdx.x < (n & 3)) {
    int64_t j = (n & ~int64_t(3)) + threadIdx.x;
    co[j] = center_rule(c[j], s[j], p, er);
  }
}

// Fused synchronous round (trainers/synchronous.py:57-64): every local
// replica's worker step against the pre-update center, then the full-sum
// center step, in one pass. C and S are read once for all replicas.
template <int V>
__global__ void __launch_bounds__(256) k_sync_update(float* W, int64_t ldw,
                                                     const float* __restrict__ G, int64_t ldg,
                                                     int nrep, float* C,
                                                     const float* __restrict__ S, int64_t n,
                                                     float eta, float er, float p) {
  int64_t nv = n / V;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (V == 4) {
      float4 c = ld4rw(C + 4 * i), s = ld4(S + 4 * i);
      for (int r = 0; r < nrep; ++r) {
        float* wp = W + r * ldw + 4 * i;
        float4 w = ld4rw(wp), g = ld4(G + r * ldg + 4 * i), o;
        o.x = worker_rule(w.x, g.x, c.x, eta, er);
        o.y = worker_rule(w.y, g.y, c.y, eta, er);
        o.z = worker_rule(w.z, g.z, c.z, eta, er);
        o.w = worker_rule(w.w, g.w, c.w, eta, er);
        st4(wp, o);
      }
      float4 o;
      o.x = center_rule(c.x, s.x, p, er);
      o.y = center_rule(c.y, s.y, p, er);
      o.z = center_rule(c.z, s.z, p, er);
      o.w = center_rule(c.w, s.w, p, er);
      st4(C + 4 * i, o);
    } else {
      float c = C[i], s = S[i];
      for (int r = 0; r < nrep; ++r) {
        float* wp = W + r * ldw + i;
        *wp = worker_rule(*wp, G[r * ldg + i], c, eta, er);
      }
      C[i] = center_rule(c, s, p, er);
    }
  }
  if (V == 4 && blockIdx.x == 0 && threadIdx.x < (n & 3)) {
    int64_t j = (n & ~int64_t(3)) + threadIdx.x;
    float c = C[j], s = S[j];
    for (int r = 0; r < nrep; ++r) {
      float* wp = W + r * ldw + j;
      *wp = worker_rule(*wp, G[r * ldg + j], c, eta, er);
    }
    C[j] = center_rule(c, s, p, er);
  }
}

template <int V>
__global__ void __launch_bounds__(256) k_measgd(float* w, float* v, const float* __restrict__ g,
                                                const float* __restrict__ c, int64_t n, float eta,
                                                float mu, float er) {
  int64_t nv = n / V;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (V == 4) {
      float4 a = ld4rw(w + 4 * i), b = ld4rw(v + 4 * i), gg = ld4(g + 4 * i), cc = ld4(c + 4 * i);
      float4 vn, wn;
      vn.x = momentum_rule(b.x, gg.x, mu, eta);
      vn.y = momentum_rule(b.y, gg.y, mu, eta);
      vn.z = momentum_rule(b.z, gg.z, mu, eta);
      vn.w = momentum_rule(b.w, gg.w, mu, eta);
      wn.x = measgd_rule(a.x, vn.x, cc.x, er);
      wn.y = measgd_rule(a.y, vn.y, cc.y, er);
      wn.z = measgd_rule(a.z, vn.z, cc.z, er);
      wn.w = measgd_rule(a.w, vn.w, cc.w, er);
      st4(v + 4 * i, vn);
      st4(w + 4 * i, wn);
    } else {
      float vn = momentum_rule(v[i], g[i], mu, eta);
      w[i] = measgd_rule(w[i], vn, c[i], er);
      v[i] = vn;
    }
  }
  if (V == 4 && blockIdx.x == 0 && threadIdx.x < (n & 3)) {
    int64_t j = (n & ~int64_t(3)) + threadIdx.x;
    float vn = momentum_rule(v[j], g[j], mu, eta);
    w[j] = measgd_rule(w[j], vn, c[j], er);
    v[j] = vn;
  }
}

template <int V>
__global__ void __launch_bounds__(256) k_center_incr(float* co, const float* c,
                                                     const float* __restrict__ w, int64_t n,
                                                     float er) {
  int64_t nv = n / V;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (V == 4) {
      float4 a = ld4rw(c + 4 * i), b = ld4(w + 4 * i), r;
      r.x = incr_rule(a.x, b.x, er);
      r.y = incr_rule(a.y, b.y, er);
      r.z = incr_rule(a.z, b.z, er);
      r.w = incr_rule(a.w, b.w, er);
      st4(co + 4 * i, r);
    } else {
      co[i] = incr_rule(c[i], w[i], er);
    }
  }
  if (V == 4 && blockIdx.x == 0 && threadIdx.x < (n & 3)) {
    int64_t j = (n & ~int64_t(3)) + threadIdx.x;
    co[j] = incr_rule(c[j], w[j], er);
  }
}

// sgd_step (updates.py:74): w - eta*grad ; msgd_step (:80-82)
template <int V>
__global__ void __launch_bounds__(256) k_sgd(float* w, const float* __restrict__ g, int64_t n,
                                             float eta) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    w[i] = __fsub_rn(w[i], __fmul_rn(eta, g[i]));
}
template <int V>
__global__ void __launch_bounds__(256) k_msgd(float* w, float* v, const float* __restrict__ g,
                                              int64_t n, float eta, float mu) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float vn = momentum_rule(v[i], g[i], mu, eta);
    w[i] = __fadd_rn(w[i], vn);
    v[i] = vn;
  }
}

// Lock-free elastic apply (fabric/engine.py:156-166 + trainers/hogwild.py:180):
// delta = etarho*(w - snap) computed per element, then a 128-bit vector
// reduction into the shared center (RED.E.ADD.F32x4 on sm_90+); concurrent
// streams interleave at element granularity exactly like the reference's
// unsynchronised numpy += (no tearing within a float).
template <int V>
__global__ void __launch_bounds__(256) k_hogwild(float* center, const float* __restrict__ w,
                                                 const float* __restrict__ snap, int64_t n,
                                                 float er) {
  int64_t nv = n / V;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (V == 4) {
      float4 a = ld4(w + 4 * i), b = ld4(snap + 4 * i), d;
      d.x = __fmul_rn(er, __fsub_rn(a.x, b.x));
      d.y = __fmul_rn(er, __fsub_rn(a.y, b.y));
      d.z = __fmul_rn(er, __fsub_rn(a.z, b.z));
      d.w = __fmul_rn(er, __fsub_rn(a.w, b.w));
      atomicAdd(reinterpret_cast<float4*>(center + 4 * i), d);
    } else {
      atomicAdd(center + i, __fmul_rn(er, __fsub_rn(w[i], snap[i])));
    }
  }
  if (V == 4 && blockIdx.x == 0 && threadIdx.x < (n & 3)) {
    int64_t j = (n & ~int64_t(3)) + threadIdx.x;
    atomicAdd(center + j, __fmul_rn(er, __fsub_rn(w[j], snap[j])));
  }
}

template <int V>
__global__ void __launch_bounds__(256) k_hogwild_axpy(float* center, const float* __restrict__ g,
                                                      int64_t n, float scale) {
  int64_t nv = n / V;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (V == 4) {
      float4 a = ld4(g + 4 * i), d;
      d.x = __fmul_rn(scale, a.x);
      d.y = __fmul_rn(scale, a.y);
      d.z = __fmul_rn(scale, a.z);
      d.w = __fmul_rn(scale, a.w);
      atomicAdd(reinterpret_cast<float4*>(center + 4 * i), d);
    } else {
      atomicAdd(center + i, __fmul_rn(scale, g[i]));
    }
  }
  if (V == 4 && blockIdx.x == 0 && threadIdx.x < (n & 3)) {
    int64_t j = (n & ~int64_t(3)) + threadIdx.x;
    atomicAdd(center + j, __fmul_rn(scale, g[j]));
  }
}

// Original EASGD step (trainers/roundrobin.py:120-124): worker step against
// the center snapshot and the incremental center step with the worker's
// pre-update weights, both from the same old (w, c), in place.
template <int V>
__global__ void __launch_bounds__(256) k_exchange(float* w, const float* __restrict__ g, float* c,
                                                  int64_t n, float eta, float er) {
  int64_t nv = n / V;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (V == 4) {
      float4 a = ld4rw(w + 4 * i), gg = ld4(g + 4 * i), cc = ld4rw(c + 4 * i), wn, cn;
      wn.x = worker_rule(a.x, gg.x, cc.x, eta, er); cn.x = incr_rule(cc.x, a.x, er);
      wn.y = worker_rule(a.y, gg.y, cc.y, eta, er); cn.y = incr_rule(cc.y, a.y, er);
      wn.z = worker_rule(a.z, gg.z, cc.z, eta, er); cn.z = incr_rule(cc.z, a.z, er);
      wn.w = worker_rule(a.w, gg.w, cc.w, eta, er); cn.w = incr_rule(cc.w, a.w, er);
      st4(w + 4 * i, wn);
      st4(c + 4 * i, cn);
    } else {
      float a = w[i], cc = c[i];
      w[i] = worker_rule(a, g[i], cc, eta, er);
      c[i] = incr_rule(cc, a, er);
    }
  }
  if (V == 4 && blockIdx.x == 0 && threadIdx.x < (n & 3)) {
    int64_t j = (n & ~int64_t(3)) + threadIdx.x;
    float a = w[j], cc = c[j];
    w[j] = worker_rule(a, g[j], cc, eta, er);
    c[j] = incr_rule(cc, a, er);
  }
}

template <int MAXP>
__global__ void __launch_bounds__(256) k_tree_sum(float* __restrict__ S, const float* __restrict__ W,
                                                  int64_t ldw, int p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float v[MAXP];
#pragma unroll
    for (int r = 0; r < MAXP; ++r) v[r] = r < p ? __ldg(W + r * ldw + i) : 0.f;
    S[i] = binomial_sum<MAXP>(v, p);
  }
}

template <int MAXP>
__global__ void __launch_bounds__(256) k_tree_sum4(float* __restrict__ S, const float* __restrict__ W,
                                                   int64_t ldw, int p, int64_t n) {
  int64_t nv = n / 4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv;
       i += (int64_t)gridDim.x * blockDim.x) {
    float vx[MAXP], vy[MAXP], vz[MAXP], vw[MAXP];
#pragma unroll
    for (int r = 0; r < MAXP; ++r) {
      float4 a = r < p ? ld4(W + r * ldw + 4 * i) : make_float4(0.f, 0.f, 0.f, 0.f);
      vx[r] = a.x; vy[r] = a.y; vz[r] = a.z; vw[r] = a.w;
    }
    float4 o;
    o.x = binomial_sum<MAXP>(vx, p);
    o.y = binomial_sum<MAXP>(vy, p);
    o.z = binomial_sum<MAXP>(vz, p);
    o.w = binomial_sum<MAXP>(vw, p);
    st4(S + 4 * i, o);
  }
  if (blockIdx.x == 0 && threadIdx.x < (n & 3)) {
    int64_t j = (n & ~int64_t(3)) + threadIdx.x;
    float v[MAXP];
#pragma unroll
    for (int r = 0; r < MAXP; ++r) v[r] = r < p ? W[r * ldw + j] : 0.f;
    S[j] = binomial_sum<MAXP>(v, p);
  }
}

inline bool vec_ok(std::initializer_list<const void*> ps) {
  for (const void* p : ps)
    if (!aligned16(p)) return false;
  return true;
}

}  // namespace
}  // namespace esgd

using namespace esgd;

#define ESGD_STREAM(s) reinterpret_cast<cudaStream_t>(s)

extern "C" int esgd_worker_step_f32(float* w_out, const float* w, const float* g, const float* c,
                                    int64_t n, float eta, float etarho, esgd_stream_t stream) {
  ESGD_REQUIRE(n >= 0, ESGD_ERR_SHAPE, "worker_step: negative length %lld", (long long)n);
  if (n == 0) return ESGD_OK;
  ESGD_REQUIRE(w_out && w && g && c, ESGD_ERR_INPUT, "worker_step: null buffer");
  if (vec_ok({w_out, w, g, c}))
    k_worker_step<4><<<stride_grid(n / 4 + 1, 256), 256, 0, ESGD_STREAM(stream)>>>(w_out, w, g, c, n, eta, etarho);
  else
    k_worker_step<1><<<stride_grid(n, 256), 256, 0, ESGD_STREAM(stream)>>>(w_out, w, g, c, n, eta, etarho);
  return check_launch("esgd_worker_step_f32");
}

// The round update of k_sync_update plus the NEXT round's local replica sum:
// S_next = tree_sum(W_r(t+1)) in the reference's binomial order, from the
// registers that hold the new replicas — the separate replica-sum pass
// (8 B/param at P_local = 1) disappears. S_next may alias S (each element is
// read before it is written, by the same thread). 28 B/param at nrep = 1.
template <int MAXP>
__global__ void __launch_bounds__(256) k_sync_update_sum4(float* W, int64_t ldw, const float* __restrict__ G,
                                                          int64_t ldg, int nrep, float* C, const float* S,
                                                          float* S_next, int64_t n, float eta, float er,
                                                          float p) {
  const int64_t nv = n / 4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float4 c = ld4rw(C + 4 * i), s = ld4rw(S + 4 * i);
    float vx[MAXP], vy[MAXP], vz[MAXP], vw[MAXP];
#pragma unroll
    for (int r = 0; r < MAXP; ++r) {
      if (r < nrep) {
        float* wp = W + r * ldw + 4 * i;
        const float4 w = ld4rw(wp), g = ld4(G + r * ldg + 4 * i);
        float4 o;
        o.x = worker_rule(w.x, g.x, c.x, eta, er);
        o.y = worker_rule(w.y, g.y, c.y, eta, er);
        o.z = worker_rule(w.z, g.z, c.z, eta, er);
        o.w = worker_rule(w.w, g.w, c.w, eta, er);
        st4(wp, o);
        vx[r] = o.x; vy[r] = o.y; vz[r] = o.z; vw[r] = o.w;
      } else {
        vx[r] = vy[r] = vz[r] = vw[r] = 0.f;
      }
    }
    float4 o;
    o.x = center_rule(c.x, s.x, p, er);
    o.y = center_rule(c.y, s.y, p, er);
    o.z = center_rule(c.z, s.z, p, er);
    o.w = center_rule(c.w, s.w, p, er);
    st4(C + 4 * i, o);
    float4 t;
    t.x = binomial_sum<MAXP>(vx, nrep);
    t.y = binomial_sum<MAXP>(vy, nrep);
    t.z = binomial_sum<MAXP>(vz, nrep);
    t.w = binomial_sum<MAXP>(vw, nrep);
    st4(S_next + 4 * i, t);
  }
  if (blockIdx.x == 0 && threadIdx.x < (n & 3)) {
    const int64_t j = (n & ~int64_t(3)) + threadIdx.x;
    const float c = C[j], s = S[j];
    float v[MAXP];
#pragma unroll
    for (int r = 0; r < MAXP; ++r) {
      if (r < nrep) {
        float* wp = W + r * ldw + j;
        *wp = v[r] = worker_rule(*wp, G[r * ldg + j], c, eta, er);
      } else {
        v[r] = 0.f;
      }
    }
    C[j] = center_rule(c, s, p, er);
    S_next[j] = binomial_sum<MAXP>(v, nrep);
  }
}

// One worker in total (P = 1): the round's sum S = tree_sum([W]) is W(t)
// itself, so the update reads W, G, C and writes W, C — 20 B/param instead
// of the 28 of k_sync_update_sum4 (no S read, no S_next write). Bitwise the
// reference's round: center_rule(c, w(t), 1, er) with the pre-update w.
__global__ void __launch_bounds__(256) k_sync_update_solo4(float* W, const float* __restrict__ G, float* C,
                                                           int64_t n, float eta, float er) {
  const int64_t nv = n / 4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float4 c = ld4rw(C + 4 * i), w = ld4rw(W + 4 * i), g = ld4(G + 4 * i);
    float4 o, q;
    o.x = worker_rule(w.x, g.x, c.x, eta, er);
    o.y = worker_rule(w.y, g.y, c.y, eta, er);
    o.z = worker_rule(w.z, g.z, c.z, eta, er);
    o.w = worker_rule(w.w, g.w, c.w, eta, er);
    q.x = center_rule(c.x, w.x, 1.f, er);
    q.y = center_rule(c.y, w.y, 1.f, er);
    q.z = center_rule(c.z, w.z, 1.f, er);
    q.w = center_rule(c.w, w.w, 1.f, er);
    st4(W + 4 * i, o);
    st4(C + 4 * i, q);
  }
  if (blockIdx.x == 0 && threadIdx.x < (n & 3)) {
    const int64_t j = (n & ~int64_t(3)) + threadIdx.x;
    const float c = C[j], w = W[j];
    W[j] = worker_rule(w, G[j], c, eta, er);
    C[j] = center_rule(c, w, 1.f, er);
  }
}

extern "C" int esgd_sync_update_solo_f32(float* W, const float* G, float* C, int64_t n, float eta,
                                         float etarho, esgd_stream_t stream) {
  ESGD_REQUIRE(n >= 0, ESGD_ERR_SHAPE, "sync_update_solo: negative length");
  if (n == 0) return ESGD_OK;
  ESGD_REQUIRE(W && G && C, ESGD_ERR_INPUT, "sync_update_solo: null buffer");
  ESGD_REQUIRE(vec_ok({W, G, C}), ESGD_ERR_UNSUPPORTED, "sync_update_solo: buffers must be 16-B aligned");
  k_sync_update_solo4<<<stride_grid(n / 4 + 1, 256), 256, 0, ESGD_STREAM(stream)>>>(W, G, C, n, eta, etarho);
  return check_launch("esgd_sync_update_solo_f32");
}

// Snapshot form of the center step (updates.py:96-110) in the reference's
// exact order: total = sum over workers (fixed order) of (W_i - C), then
// C + (eta*rho)*total — bitwise the reference's fp32 arithmetic.
__global__ void __launch_bounds__(256) k_center_snapshots(float* co, const float* c, const float* __restrict__ S,
                                                          int64_t lds, int P, int64_t n, float er) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float ci = c[i];
    float t = 0.f;
    for (int r = 0; r < P; ++r) t = __fadd_rn(t, __fsub_rn(S[r * lds + i], ci));
    co[i] = __fadd_rn(ci, __fmul_rn(er, t));
  }
}

extern "C" int esgd_center_step_snapshots_f32(float* c_out, const float* c, const float* snaps, int64_t lds,
                                              int32_t num_workers, int64_t n, float etarho, esgd_stream_t stream) {
  ESGD_REQUIRE(n >= 0 && num_workers >= 1 && (num_workers == 1 || lds >= n), ESGD_ERR_SHAPE,
               "center_step_snapshots: bad sizes");
  if (n == 0) return ESGD_OK;
  ESGD_REQUIRE(c_out && c && snaps, ESGD_ERR_INPUT, "center_step_snapshots: null buffer");
  k_center_snapshots<<<stride_grid(n, 256), 256, 0, ESGD_STREAM(stream)>>>(c_out, c, snaps, lds, num_workers, n,
                                                                          etarho);
  return check_launch("esgd_center_step_snapshots_f32");
}

extern "C" int esgd_center_step_from_sum_f32(float* c_out, const float* c, const float* s,
                                             int64_t n, float etarho, int32_t num_workers,
                                             esgd_stream_t stream) {
  ESGD_REQUIRE(n >= 0, ESGD_ERR_SHAPE, "center_step_from_sum: negative length");
  ESGD_REQUIRE(num_workers >= 1, ESGD_ERR_INPUT, "num_workers must be >= 1");
  if (n == 0) return ESGD_OK;
  ESGD_REQUIRE(c_out && c && s, ESGD_ERR_INPUT, "center_step_from_sum: null buffer");
  float p = (float)num_workers;
  if (vec_ok({c_out, c, s}))
    k_center_from_sum<4><<<stride_grid(n / 4 + 1, 256), 256, 0, ESGD_STREAM(stream)>>>(c_out, c, s, n, etarho, p);
  else
    k_center_from_sum<1><<<stride_grid(n, 256), 256, 0, ESGD_STREAM(stream)>>>(c_out, c, s, n, etarho, p);
  return check_launch("esgd_center_step_from_sum_f32");
}

extern "C" int esgd_sync_update_f32(float* W, int64_t ldw, const float* G, int64_t ldg,
                                    int32_t nrep, float* C, const float* S, int64_t n, float eta,
                                    float etarho, int32_t num_workers, esgd_stream_t stream) {
  ESGD_REQUIRE(n >= 0 && nrep >= 0, ESGD_ERR_SHAPE, "sync_update: negative size");
  ESGD_REQUIRE(num_workers >= 1, ESGD_ERR_INPUT, "num_workers must be >= 1");
  ESGD_REQUIRE(nrep <= 1 || (ldw >= n && ldg >= n), ESGD_ERR_SHAPE,
               "sync_update: replica pitch (%lld, %lld) shorter than n=%lld", (long long)ldw,
               (long long)ldg, (long long)n);
  if (n == 0) return ESGD_OK;
  ESGD_REQUIRE(C && S && (nrep == 0 || (W && G)), ESGD_ERR_INPUT, "sync_update: null buffer");
  float p = (float)num_workers;
  bool v4 = vec_ok({W, G, C, S}) && (nrep <= 1 || ((ldw & 3) == 0 && (ldg & 3) == 0));
  if (v4)
    k_sync_update<4><<<stride_grid(n / 4 + 1, 256), 256, 0, ESGD_STREAM(stream)>>>(W, ldw, G, ldg, nrep, C, S, n, eta, etarho, p);
  else
    k_sync_update<1><<<stride_grid(n, 256), 256, 0, ESGD_STREAM(stream)>>>(W, ldw, G, ldg, nrep, C, S, n, eta, etarho, p);
  return check_launch("esgd_sync_update_f32");
}

extern "C" int esgd_sync_update_sum_f32(float* W, int64_t ldw, const float* G, int64_t ldg,
                                        int32_t nrep, float* C, const float* S, float* S_next, int64_t n,
                                        float eta, float etarho, int32_t num_workers, esgd_stream_t stream) {
  ESGD_REQUIRE(n >= 0 && nrep >= 1, ESGD_ERR_SHAPE, "sync_update_sum: bad size");
  ESGD_REQUIRE(nrep <= 8, ESGD_ERR_UNSUPPORTED, "sync_update_sum: at most 8 local replicas, got %d", nrep);
  ESGD_REQUIRE(num_workers >= 1, ESGD_ERR_INPUT, "num_workers must be >= 1");
  ESGD_REQUIRE(nrep == 1 || (ldw >= n && ldg >= n), ESGD_ERR_SHAPE,
               "sync_update_sum: replica pitch (%lld, %lld) shorter than n=%lld", (long long)ldw,
               (long long)ldg, (long long)n);
  if (n == 0) return ESGD_OK;
  ESGD_REQUIRE(W && G && C && S && S_next, ESGD_ERR_INPUT, "sync_update_sum: null buffer");
  ESGD_REQUIRE(vec_ok({W, G, C, S, S_next}) && (nrep == 1 || ((ldw & 3) == 0 && (ldg & 3) == 0)),
               ESGD_ERR_UNSUPPORTED, "sync_update_sum: buffers and pitches must be 16-B aligned");
  const float p = (float)num_workers;
  const int grid = stride_grid(n / 4 + 1, 256);
  cudaStream_t st = ESGD_STREAM(stream);
  if (nrep == 1) k_sync_update_sum4<1><<<grid, 256, 0, st>>>(W, ldw, G, ldg, nrep, C, S, S_next, n, eta, etarho, p);
  else if (nrep == 2) k_sync_update_sum4<2><<<grid, 256, 0, st>>>(W, ldw, G, ldg, nrep, C, S, S_next, n, eta, etarho, p);
  else if (nrep <= 4) k_sync_update_sum4<4><<<grid, 256, 0, st>>>(W, ldw, G, ldg, nrep, C, S, S_next, n, eta, etarho, p);
  else k_sync_update_sum4<8><<<grid, 256, 0, st>>>(W, ldw, G, ldg, nrep, C, S, S_next, n, eta, etarho, p);
  return check_launch("esgd_sync_update_sum_f32");
}

extern "C" int esgd_measgd_update_f32(float* w, float* v, const float* g, const float* c,
                                      int64_t n, float eta, float mu, float etarho,
                                      esgd_stream_t stream) {
  ESGD_REQUIRE(n >= 0, ESGD_ERR_SHAPE, "measgd_update: negative length");
  if (n == 0) return ESGD_OK;
  ESGD_REQUIRE(w && v && g && c, ESGD_ERR_INPUT, "measgd_update: null buffer");
  if (vec_ok({w, v, g, c}))
    k_measgd<4><<<stride_grid(n / 4 + 1, 256), 256, 0, ESGD_STREAM(stream)>>>(w, v, g, c, n, eta, mu, etarho);
  else
    k_measgd<1><<<stride_grid(n, 256), 256, 0, ESGD_STREAM(stream)>>>(w, v, g, c, n, eta, mu, etarho);
  return check_launch("esgd_measgd_update_f32");
}

extern "C" int esgd_center_incr_f32(float* c_out, const float* c, const float* w, int64_t n,
                                    float etarho, esgd_stream_t stream) {
  ESGD_REQUIRE(n >= 0, ESGD_ERR_SHAPE, "center_incr: negative length");
  if (n == 0) return ESGD_OK;
  ESGD_REQUIRE(c_out && c && w, ESGD_ERR_INPUT, "center_incr: null buffer");
  if (vec_ok({c_out, c, w}))
    k_center_incr<4><<<stride_grid(n / 4 + 1, 256), 256, 0, ESGD_STREAM(stream)>>>(c_out, c, w, n, etarho);
  else
    k_center_incr<1><<<stride_grid(n, 256), 256, 0, ESGD_STREAM(stream)>>>(c_out, c, w, n, etarho);
  return check_launch("esgd_center_incr_f32");
}

extern "C" int esgd_sgd_step_f32(float* w, const float* g, int64_t n, float eta,
                                 esgd_stream_t stream) {
  ESGD_REQUIRE(n >= 0, ESGD_ERR_SHAPE, "sgd_step: negative length");
  if (n == 0) return ESGD_OK;
  ESGD_REQUIRE(w && g, ESGD_ERR_INPUT, "sgd_step: null buffer");
  k_sgd<1><<<stride_grid(n, 256), 256, 0, ESGD_STREAM(stream)>>>(w, g, n, eta);
  return check_launch("esgd_sgd_step_f32");
}

extern "C" int esgd_msgd_step_f32(float* w, float* v, const float* g, int64_t n, float eta,
                                  float mu, esgd_stream_t stream) {
  ESGD_REQUIRE(n >= 0, ESGD_ERR_SHAPE, "msgd_step: negative length");
  if (n == 0) return ESGD_OK;
  ESGD_REQUIRE(w && v && g, ESGD_ERR_INPUT, "msgd_step: null buffer");
  k_msgd<1><<<stride_grid(n, 256), 256, 0, ESGD_STREAM(stream)>>>(w, v, g, n, eta, mu);
  return check_launch("esgd_msgd_step_f32");
}

extern "C" int esgd_hogwild_apply_f32(float* center, const float* w, const float* snap, int64_t n,
                                      float etarho, esgd_stream_t stream) {
  ESGD_REQUIRE(n >= 0, ESGD_ERR_SHAPE, "hogwild_apply: negative length");
  if (n == 0) return ESGD_OK;
  ESGD_REQUIRE(center && w && snap, ESGD_ERR_INPUT, "hogwild_apply: null buffer");
  if (vec_ok({center, w, snap}))
    k_hogwild<4><<<stride_grid(n / 4 + 1, 256), 256, 0, ESGD_STREAM(stream)>>>(center, w, snap, n, etarho);
  else
    k_hogwild<1><<<stride_grid(n, 256), 256, 0, ESGD_STREAM(stream)>>>(center, w, snap, n, etarho);
  return check_launch("esgd_hogwild_apply_f32");
}

extern "C" int esgd_hogwild_axpy_f32(float* center, const float* g, int64_t n, float scale,
                                     esgd_stream_t stream) {
  ESGD_REQUIRE(n >= 0, ESGD_ERR_SHAPE, "hogwild_axpy: negative length");
  if (n == 0) return ESGD_OK;
  ESGD_REQUIRE(center && g, ESGD_ERR_INPUT, "hogwild_axpy: null buffer");
  if (vec_ok({center, g}))
    k_hogwild_axpy<4><<<stride_grid(n / 4 + 1, 256), 256, 0, ESGD_STREAM(stream)>>>(center, g, n, scale);
  else
    k_hogwild_axpy<1><<<stride_grid(n, 256), 256, 0, ESGD_STREAM(stream)>>>(center, g, n, scale);
  return check_launch("esgd_hogwild_axpy_f32");
}

extern "C" int esgd_replica_tree_sum_f32(float* S, const float* W, int64_t ldw, int32_t nrep,
                                         int64_t n, esgd_stream_t stream) {
  ESGD_REQUIRE(n >= 0, ESGD_ERR_SHAPE, "tree_sum: negative length");
  ESGD_REQUIRE(nrep >= 1, ESGD_ERR_INPUT, "tree_sum needs at least one buffer");
  ESGD_REQUIRE(nrep <= 64, ESGD_ERR_UNSUPPORTED, "tree_sum: at most 64 local replicas, got %d", nrep);
  ESGD_REQUIRE(nrep == 1 || ldw >= n, ESGD_ERR_SHAPE, "tree_sum: replica pitch shorter than n");
  if (n == 0) return ESGD_OK;
  ESGD_REQUIRE(S && W, ESGD_ERR_INPUT, "tree_sum: null buffer");
  cudaStream_t st = ESGD_STREAM(stream);
  // four-wide only while the per-replica register arrays stay small
  bool v4 = vec_ok({S, W}) && (nrep == 1 || (ldw & 3) == 0) && nrep <= 8;
  int g4 = stride_grid(n / 4 + 1, 256), g1 = stride_grid(n, 256);
#define ESGD_TREE(MAXP)                                                              \
  if (v4) k_tree_sum4<MAXP><<<g4, 256, 0, st>>>(S, W, ldw, nrep, n);                 \
  else k_tree_sum<MAXP><<<g1, 256, 0, st>>>(S, W, ldw, nrep, n);
  if (nrep <= 1) { ESGD_TREE(1) }
  else if (nrep <= 2) { ESGD_TREE(2) }
  else if (nrep <= 4) { ESGD_TREE(4) }
  else if (nrep <= 8) { ESGD_TREE(8) }
  else if (nrep <= 16) { ESGD_TREE(16) }
  else if (nrep <= 32) { ESGD_TREE(32) }
  else { ESGD_TREE(64) }
#undef ESGD_TREE
  return check_launch("esgd_replica_tree_sum_f32");
}

extern "C" int esgd_exchange_update_f32(float* w, const float* g, float* c, int64_t n, float eta,
                                        float etarho, esgd_stream_t stream) {
  ESGD_REQUIRE(n >= 0, ESGD_ERR_SHAPE, "exchange_update: negative length");
  if (n == 0) return ESGD_OK;
  ESGD_REQUIRE(w && g && c, ESGD_ERR_INPUT, "exchange_update: null buffer");
  if (vec_ok({w, g, c}))
    k_exchange<4><<<stride_grid(n / 4 + 1, 256), 256, 0, ESGD_STREAM(stream)>>>(w, g, c, n, eta, etarho);
  else
    k_exchange<1><<<stride_grid(n, 256), 256, 0, ESGD_STREAM(stream)>>>(w, g, c, n, eta, etarho);
  return check_launch("esgd_exchange_update_f32");
}
