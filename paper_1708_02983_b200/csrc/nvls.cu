// Multi-GPU Sync-EASGD round update fused with its collective over NVLink
// SHARP (NVLS) multicast — replaces "ncclAllReduce(S) then update" (the
// reference's tree_sum + center step, fabric/collectives.py:18-32 and
// trainers/synchronous.py:57-64) by ONE kernel per round:
//
//   * center slice (this rank's 1/world of the packed buffer): the sum of the
//     workers' replica sums S is read through the multicast address with
//     multimem.ld_reduce (the NVSwitch adds the world copies in flight), the
//     center step is applied and the new center slice is broadcast to every
//     GPU with multimem.st — each rank owns a slice, every rank ends with the
//     identical full center;
//   * workers (full buffer, local HBM): the elastic worker step against the
//     pre-update center, plus the next round's local replica sum (binomial
//     tree order) from registers.
//
// Double-buffered symmetric buffers S[2], C[2] (round parity p): round t
// reads S[p] (all ranks) and C[p], writes C[p^1] (all ranks, multicast) and
// S[p^1] (local). One cross-GPU barrier per round (esgd_nvls_barrier, before
// the update) orders round t-1's writes before round t's reads and round
// t-1's reads before round t's overwrites.
#include "esgd_common.cuh"
#include "rules.cuh"
#include <algorithm>

namespace esgd {
namespace {

__device__ __forceinline__ float4 mc_ld_reduce4(const float* mc) {
  float4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(mc)
               : "memory");
  return v;
}
__device__ __forceinline__ void mc_st4(float* mc, float4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w)
               : "memory");
}

template <int MAXP>
__global__ void __launch_bounds__(256) k_sync_update_nvls(float* W, int64_t ldw, const float* __restrict__ G,
                                                          int64_t ldg, int nrep, const float* __restrict__ C_old,
                                                          const float* S_mc, float* C_new_mc, float* S_next,
                                                          int64_t nv, int64_t lo, int64_t hi, float eta, float er,
                                                          float p) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
  // center slice [lo, hi) (float4 units): NVSwitch-reduced sum -> center step -> broadcast
  for (int64_t i = lo + tid; i < hi; i += nth) {
    const float4 s = mc_ld_reduce4(S_mc + 4 * i), c = ld4(C_old + 4 * i);
    float4 o;
    o.x = center_rule(c.x, s.x, p, er);
    o.y = center_rule(c.y, s.y, p, er);
    o.z = center_rule(c.z, s.z, p, er);
    o.w = center_rule(c.w, s.w, p, er);
    mc_st4(C_new_mc + 4 * i, o);
  }
  // local replicas: worker step against the pre-update center + next local sum
  for (int64_t i = tid; i < nv; i += nth) {
    const float4 c = ld4(C_old + 4 * i);
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
    float4 t;
    t.x = binomial_sum<MAXP>(vx, nrep);
    t.y = binomial_sum<MAXP>(vy, nrep);
    t.z = binomial_sum<MAXP>(vz, nrep);
    t.w = binomial_sum<MAXP>(vw, nrep);
    st4(S_next + 4 * i, t);
  }
}

// Center slice only (the overlapped variant): runs on a side stream
// concurrently with the round's forward/backward, which never touches S or C.
// Sized to fit NEXT TO a persistent tcgen05 GEMM CTA on the same SM (that
// kernel leaves ~8K registers and 2 KB of shared memory free): 128 threads x
// <= 40 registers, no shared memory — so the GEMM's CTAs are never held back
// by the collective (measured: a 256 x 58-register version delayed them).
// Two float4 NVLS loads in flight per thread hide the NVLink round trip.
__global__ void __launch_bounds__(128, 12) k_center_nvls(const float* __restrict__ C_old, const float* S_mc,
                                                         float* C_new_mc, int64_t lo, int64_t hi, float er, float p) {
  constexpr int U = 2;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = lo + tid; i0 < hi; i0 += U * nth) {
    float4 s[U], c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * nth;
      if (i < hi) {
        s[u] = mc_ld_reduce4(S_mc + 4 * i);
        c[u] = ld4(C_old + 4 * i);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * nth;
      if (i < hi) {
        float4 o;
        o.x = center_rule(c[u].x, s[u].x, p, er);
        o.y = center_rule(c[u].y, s[u].y, p, er);
        o.z = center_rule(c[u].z, s[u].z, p, er);
        o.w = center_rule(c[u].w, s[u].w, p, er);
        mc_st4(C_new_mc + 4 * i, o);
      }
    }
  }
}

// Worker step of every local replica against C plus the next round's local
// replica sum (binomial order) — the local half of the overlapped variant.
template <int MAXP>
__global__ void __launch_bounds__(256) k_worker_step_sum(float* W, int64_t ldw, const float* __restrict__ G,
                                                         int64_t ldg, int nrep, const float* __restrict__ C,
                                                         float* S_next, int64_t nv, float eta, float er) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 c = ld4(C + 4 * i);
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
    float4 t;
    t.x = binomial_sum<MAXP>(vx, nrep);
    t.y = binomial_sum<MAXP>(vy, nrep);
    t.z = binomial_sum<MAXP>(vz, nrep);
    t.w = binomial_sum<MAXP>(vw, nrep);
    st4(S_next + 4 * i, t);
  }
}

// Cross-GPU barrier over a symmetric int32 flag array: thread j marks this
// rank's arrival in rank j's flags (slot `rank`) and waits for rank j's mark
// in its own. The epoch lives in device memory so graph replays advance it.
__global__ void k_nvls_barrier(int32_t* const* peer_flags, int world, int rank, int32_t* epoch) {
  __shared__ int32_t ep;
  if (threadIdx.x == 0) {
    ep = *epoch + 1;
    *epoch = ep;
  }
  __syncthreads();
  const int j = threadIdx.x;
  if (j < world) {
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    int32_t* remote = peer_flags[j] + rank;
    asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(remote), "r"(ep) : "memory");
    const int32_t* mine = peer_flags[rank] + j;
    int32_t v;
    do {
      asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(mine) : "memory");
    } while (v < ep);
  }
  __syncthreads();
}

}  // namespace
}  // namespace esgd

using namespace esgd;

extern "C" int esgd_nvls_barrier(int32_t* const* peer_flags, int32_t world, int32_t rank, int32_t* epoch,
                                 esgd_stream_t stream) {
  ESGD_REQUIRE(world >= 1 && world <= 64 && rank >= 0 && rank < world, ESGD_ERR_INPUT,
               "nvls_barrier: bad world/rank (%d, %d)", world, rank);
  ESGD_REQUIRE(peer_flags && epoch, ESGD_ERR_INPUT, "nvls_barrier: null pointer");
  k_nvls_barrier<<<1, 64, 0, reinterpret_cast<cudaStream_t>(stream)>>>(peer_flags, world, rank, epoch);
  return check_launch("esgd_nvls_barrier");
}

extern "C" int esgd_sync_update_nvls_f32(float* W, int64_t ldw, const float* G, int64_t ldg, int32_t nrep,
                                         const float* C_old, const float* S_mc, float* C_new_mc, float* S_next,
                                         int64_t n4, int32_t world, int32_t rank, float eta, float etarho,
                                         int32_t num_workers, esgd_stream_t stream) {
  ESGD_REQUIRE(n4 >= 0 && (n4 & 3) == 0, ESGD_ERR_SHAPE, "sync_update_nvls: length %lld must be a multiple of 4",
               (long long)n4);
  ESGD_REQUIRE(nrep >= 1 && nrep <= 8, ESGD_ERR_UNSUPPORTED, "sync_update_nvls: 1..8 local replicas, got %d", nrep);
  ESGD_REQUIRE(world >= 1 && rank >= 0 && rank < world && num_workers >= 1, ESGD_ERR_INPUT,
               "sync_update_nvls: bad world/rank/workers");
  ESGD_REQUIRE(nrep == 1 || (ldw >= n4 && ldg >= n4 && (ldw & 3) == 0 && (ldg & 3) == 0), ESGD_ERR_SHAPE,
               "sync_update_nvls: replica pitch");
  if (n4 == 0) return ESGD_OK;
  ESGD_REQUIRE(W && G && C_old && S_mc && C_new_mc && S_next, ESGD_ERR_INPUT, "sync_update_nvls: null pointer");
  ESGD_REQUIRE(aligned16(W) && aligned16(G) && aligned16(C_old) && aligned16(S_mc) && aligned16(C_new_mc) &&
                   aligned16(S_next),
               ESGD_ERR_INPUT, "sync_update_nvls: buffers must be 16-B aligned");
  const int64_t nv = n4 / 4;
  // this rank's center slice, whole float4 vectors
  const int64_t per = (nv + world - 1) / world;
  const int64_t lo = std::min<int64_t>(nv, per * rank), hi = std::min<int64_t>(nv, lo + per);
  const int grid = stride_grid(nv + 1, 256);
  const float p = (float)num_workers;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
#define ESGD_NVLS(MP)                                                                                            \
  k_sync_update_nvls<MP><<<grid, 256, 0, st>>>(W, ldw, G, ldg, nrep, C_old, S_mc, C_new_mc, S_next, nv, lo, hi, \
                                               eta, etarho, p)
  if (nrep == 1) ESGD_NVLS(1);
  else if (nrep == 2) ESGD_NVLS(2);
  else if (nrep <= 4) ESGD_NVLS(4);
  else ESGD_NVLS(8);
#undef ESGD_NVLS
  return check_launch("esgd_sync_update_nvls_f32");
}

// Dedicated-SM variant (ctas < 0 in esgd_center_step_nvls_f32): -ctas CTAs
// of 512 threads, four float4 NVLS loads in flight per thread, each CTA
// asking for 16 KB of (unused) shared memory so that it cannot share an SM
// with a persistent GEMM CTA: the GEMMs run on the other SMs
// (esgd_set_sm_reserve) instead of being slowed where a center CTA sits next
// to one (a co-resident center CTA slows its SM's GEMM CTA, and with static
// tile assignment the whole GEMM waits for that SM).
__global__ void __launch_bounds__(512) k_center_nvls_wide(const float* __restrict__ C_old, const float* S_mc,
                                                          float* C_new_mc, int64_t lo, int64_t hi, float er,
                                                          float p) {
  constexpr int U = 4;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = lo + tid; i0 < hi; i0 += U * nth) {
    float4 s[U], c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * nth;
      if (i < hi) {
        s[u] = mc_ld_reduce4(S_mc + 4 * i);
        c[u] = ld4(C_old + 4 * i);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * nth;
      if (i < hi) {
        float4 o;
        o.x = center_rule(c[u].x, s[u].x, p, er);
        o.y = center_rule(c[u].y, s[u].y, p, er);
        o.z = center_rule(c[u].z, s[u].z, p, er);
        o.w = center_rule(c[u].w, s[u].w, p, er);
        mc_st4(C_new_mc + 4 * i, o);
      }
    }
  }
}

extern "C" int esgd_center_step_nvls_f32(const float* C_old, const float* S_mc, float* C_new_mc, int64_t n4,
                                         int32_t world, int32_t rank, float etarho, int32_t num_workers,
                                         int32_t ctas, esgd_stream_t stream) {
  ESGD_REQUIRE(n4 >= 0 && (n4 & 3) == 0, ESGD_ERR_SHAPE, "center_step_nvls: length must be a multiple of 4");
  ESGD_REQUIRE(world >= 1 && rank >= 0 && rank < world && num_workers >= 1, ESGD_ERR_INPUT,
               "center_step_nvls: bad world/rank/workers");
  if (n4 == 0) return ESGD_OK;
  ESGD_REQUIRE(C_old && S_mc && C_new_mc && aligned16(C_old) && aligned16(S_mc) && aligned16(C_new_mc),
               ESGD_ERR_INPUT, "center_step_nvls: null or misaligned pointer");
  const int64_t nv = n4 / 4, per = (nv + world - 1) / world;
  const int64_t lo = std::min<int64_t>(nv, per * rank), hi = std::min<int64_t>(nv, lo + per);
  if (ctas < 0) {  // dedicated SMs
    k_center_nvls_wide<<<-ctas, 512, 16384, reinterpret_cast<cudaStream_t>(stream)>>>(C_old, S_mc, C_new_mc, lo,
                                                                                      hi, etarho,
                                                                                      (float)num_workers);
    return check_launch("esgd_center_step_nvls_f32");
  }
  const int grid = ctas > 0 ? ctas : kNumSMs;
  k_center_nvls<<<grid, 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(C_old, S_mc, C_new_mc, lo, hi, etarho,
                                                                          (float)num_workers);
  return check_launch("esgd_center_step_nvls_f32");
}

// Copy-engine variant of the center slice (ESGD_NVLS=ce): the ranks' slices
// of S arrive in local buffers through cudaMemcpyAsync over NVLink (copy
// engines: no SM time taken from the forward / backward running beside it),
// are summed here in binomial rank order, and the center step is applied;
// the caller then copies the new slice to every peer.
__global__ void __launch_bounds__(256) k_center_sum(const float* __restrict__ C_old,
                                                    const float* const* __restrict__ src, int nsrc,
                                                    float* __restrict__ C_new, int64_t nv, float er, float p) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.x * blockDim.x) {
    float vx[8], vy[8], vz[8], vw[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      if (r < nsrc) {
        const float4 v = ld4(src[r] + 4 * i);
        vx[r] = v.x; vy[r] = v.y; vz[r] = v.z; vw[r] = v.w;
      } else {
        vx[r] = vy[r] = vz[r] = vw[r] = 0.f;
      }
    }
    const float4 c = ld4(C_old + 4 * i);
    float4 o;
    o.x = center_rule(c.x, binomial_sum<8>(vx, nsrc), p, er);
    o.y = center_rule(c.y, binomial_sum<8>(vy, nsrc), p, er);
    o.z = center_rule(c.z, binomial_sum<8>(vz, nsrc), p, er);
    o.w = center_rule(c.w, binomial_sum<8>(vw, nsrc), p, er);
    st4(C_new + 4 * i, o);
  }
}

extern "C" int esgd_center_step_sum_f32(const float* C_old, const float* const* srcs, int32_t nsrc, float* C_new,
                                        int64_t n4, float etarho, int32_t num_workers, esgd_stream_t stream) {
  ESGD_REQUIRE(n4 >= 0 && (n4 & 3) == 0, ESGD_ERR_SHAPE, "center_step_sum: length must be a multiple of 4");
  ESGD_REQUIRE(nsrc >= 1 && nsrc <= 8 && num_workers >= 1, ESGD_ERR_INPUT, "center_step_sum: 1..8 sources");
  if (n4 == 0) return ESGD_OK;
  ESGD_REQUIRE(C_old && srcs && C_new && aligned16(C_old) && aligned16(C_new), ESGD_ERR_INPUT,
               "center_step_sum: null or misaligned pointer");
  const int64_t nv = n4 / 4;
  k_center_sum<<<stride_grid(nv, 256), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      C_old, srcs, nsrc, C_new, nv, etarho, (float)num_workers);
  return check_launch("esgd_center_step_sum_f32");
}

// stream-ordered device copy (peer pointers of symmetric memory included):
// the copy engines move the CE variant's slices
extern "C" int esgd_copy_async(void* dst, const void* src, int64_t bytes, esgd_stream_t stream) {
  ESGD_REQUIRE(bytes >= 0, ESGD_ERR_SHAPE, "copy_async: negative size");
  if (bytes == 0) return ESGD_OK;
  ESGD_REQUIRE(dst && src, ESGD_ERR_INPUT, "copy_async: null pointer");
  cudaError_t e = cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToDevice,
                                  reinterpret_cast<cudaStream_t>(stream));
  ESGD_REQUIRE(e == cudaSuccess, ESGD_ERR_CUDA, "copy_async: %s", cudaGetErrorString(e));
  return ESGD_OK;
}

extern "C" int esgd_worker_step_sum_f32(float* W, int64_t ldw, const float* G, int64_t ldg, int32_t nrep,
                                        const float* C, float* S_next, int64_t n4, float eta, float etarho,
                                        esgd_stream_t stream) {
  ESGD_REQUIRE(n4 >= 0 && (n4 & 3) == 0, ESGD_ERR_SHAPE, "worker_step_sum: length must be a multiple of 4");
  ESGD_REQUIRE(nrep >= 1 && nrep <= 8, ESGD_ERR_UNSUPPORTED, "worker_step_sum: 1..8 local replicas, got %d", nrep);
  ESGD_REQUIRE(nrep == 1 || (ldw >= n4 && ldg >= n4 && (ldw & 3) == 0 && (ldg & 3) == 0), ESGD_ERR_SHAPE,
               "worker_step_sum: replica pitch");
  if (n4 == 0) return ESGD_OK;
  ESGD_REQUIRE(W && G && C && S_next && aligned16(W) && aligned16(G) && aligned16(C) && aligned16(S_next),
               ESGD_ERR_INPUT, "worker_step_sum: null or misaligned pointer");
  const int64_t nv = n4 / 4;
  const int grid = stride_grid(nv + 1, 256);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (nrep == 1) k_worker_step_sum<1><<<grid, 256, 0, st>>>(W, ldw, G, ldg, nrep, C, S_next, nv, eta, etarho);
  else if (nrep == 2) k_worker_step_sum<2><<<grid, 256, 0, st>>>(W, ldw, G, ldg, nrep, C, S_next, nv, eta, etarho);
  else if (nrep <= 4) k_worker_step_sum<4><<<grid, 256, 0, st>>>(W, ldw, G, ldg, nrep, C, S_next, nv, eta, etarho);
  else k_worker_step_sum<8><<<grid, 256, 0, st>>>(W, ldw, G, ldg, nrep, C, S_next, nv, eta, etarho);
  return check_launch("esgd_worker_step_sum_f32");
}
