// Device-side parameter server for the asynchronous elastic schedules
// (reference trainers/asynchronous.py:170-264, the threaded master; FCFS
// queue fabric/engine.py:125-148): no host in the loop.
//
//   worker stream, per cycle:  post  ->  gradient  ->  wait  ->  elastic step
//   master (one persistent kernel on the center's GPU): serve tickets in order
//
// * post (1 thread, worker stream): takes the next ticket with an atomic on
//   the control block (FCFS = ticket order; simultaneous arrivals are ordered
//   by the atomic), enqueues the worker id under it and publishes the ticket.
//   The worker's W is final at this point (its previous step is done), so the
//   exchange overlaps the worker's next forward/backward, as in the reference
//   (the worker ships W; :121-132).
// * master: for ticket t = 0, 1, ...: wait until published, then — the sole
//   writer of the center, all CTAs on slices — snap_w = C (the reply: the
//   pre-update center) and C = C + eta*rho*(W_w - C) (easgd_center_incremental,
//   updates.py:122-131) reading W_w from the worker's GPU over NVLink (peer
//   access) and writing the snapshot into the worker's GPU; then, after a grid
//   barrier, served[w] += 1.
// * wait (1 thread, worker stream): spin until served[w] reaches the worker's
//   own post count; the stream then applies the (momentum) elastic step
//   against snap_w (updates.py:134-140).
// Spins give up after 20 s without progress and raise the control block's
// error flag instead of hanging the device.
#include "esgd_common.cuh"
#include "rules.cuh"

namespace esgd {
namespace {

constexpr unsigned long long kTimeoutNs = 20ull * 1000 * 1000 * 1000;  // 20 s without progress

// control block (int32): [0] ticket, [1] error, [2] barrier count, [3] barrier
// generation, [16, 16+Q) queue, [16+Q, 16+2Q) published, [16+2Q, 16+2Q+P) served
__device__ __forceinline__ int* q_of(int* ctl) { return ctl + 16; }

__device__ __forceinline__ unsigned long long now_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__global__ void k_async_post(int* ctl, int Q, int worker, int* my_posts) {
  const int t = atomicAdd(ctl, 1);
  ctl[16 + t % Q] = worker;
  __threadfence_system();
  st_release(ctl + 16 + Q + t % Q, t + 1);
  *my_posts += 1;
}

__global__ void k_async_wait(int* ctl, int Q, int worker, const int* my_posts) {
  const int want = *my_posts;
  const int* served = ctl + 16 + 2 * Q + worker;
  const unsigned long long t0 = now_ns();
  while (ld_acquire(served) < want) {
    if (ld_acquire(ctl + 1)) return;  // the master gave up
    if (now_ns() - t0 > kTimeoutNs) {
      atomicExch(ctl + 1, 2);
      return;
    }
    __nanosleep(200);
  }
}

// grid-wide barrier on the control block (generation counting)
__device__ __forceinline__ bool grid_barrier(int* ctl, int nblocks) {
  __syncthreads();
  bool ok = true;
  if (threadIdx.x == 0) {
    const int gen = ld_acquire(ctl + 3);
    __threadfence();
    if (atomicAdd(ctl + 2, 1) == nblocks - 1) {
      ctl[2] = 0;
      __threadfence();
      st_release(ctl + 3, gen + 1);
    } else {
      const unsigned long long t0 = now_ns();
      while (ld_acquire(ctl + 3) == gen) {
        if (now_ns() - t0 > kTimeoutNs) {
          atomicExch(ctl + 1, 3);
          ok = false;
          break;
        }
      }
    }
  }
  __syncthreads();
  return ok;
}

__global__ void __launch_bounds__(128) k_async_master(float* C, int64_t n, const float* const* W,
                                                      float* const* snap, int* ctl, int Q, int P,
                                                      int64_t services, float er) {
  __shared__ int s_worker;
  const int64_t nv = n / 4;
  for (int64_t t = 0; t < services; ++t) {
    if (threadIdx.x == 0) {
      const int* pub = ctl + 16 + Q + t % Q;
      const unsigned long long t0 = now_ns();
      int w = -1;
      while (ld_acquire(pub) != (int)(t + 1)) {
        if (ld_acquire(ctl + 1) || now_ns() - t0 > kTimeoutNs) {
          atomicExch(ctl + 1, ld_acquire(ctl + 1) ? ld_acquire(ctl + 1) : 1);
          break;
        }
      }
      if (!ld_acquire(ctl + 1)) w = q_of(ctl)[t % Q];
      s_worker = w;
    }
    __syncthreads();
    const int w = s_worker;
    if (w < 0 || w >= P) return;
    const float* Ww = W[w];
    float* sw = snap[w];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.x * blockDim.x) {
      // W_w changes between services of this long-lived kernel (the worker's
      // steps): uncached loads, never the non-coherent path
      float4 x;
      asm volatile("ld.global.cv.v4.f32 {%0, %1, %2, %3}, [%4];"
                   : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w) : "l"(Ww + 4 * i));
      const float4 c = ld4rw(C + 4 * i);
      st4(sw + 4 * i, c);  // the reply: the pre-update center
      float4 o;
      o.x = incr_rule(c.x, x.x, er);
      o.y = incr_rule(c.y, x.y, er);
      o.z = incr_rule(c.z, x.z, er);
      o.w = incr_rule(c.w, x.w, er);
      st4(C + 4 * i, o);
    }
    if (blockIdx.x == 0 && threadIdx.x < (n & 3)) {
      const int64_t j = (n & ~int64_t(3)) + threadIdx.x;
      const float c = C[j];
      float x;
      asm volatile("ld.global.cv.f32 %0, [%1];" : "=f"(x) : "l"(Ww + j));
      sw[j] = c;
      C[j] = incr_rule(c, x, er);
    }
    __threadfence_system();
    if (!grid_barrier(ctl, gridDim.x)) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      int* served = ctl + 16 + 2 * Q + w;
      st_release(served, *served + 1);
    }
  }
}

}  // namespace
}  // namespace esgd

using namespace esgd;
#define ESGD_STREAM(s) reinterpret_cast<cudaStream_t>(s)

extern "C" int esgd_async_ctl_ints(int32_t workers) { return 16 + 4 * workers + workers; }

// CUDA loads kernels lazily at their first launch, and a load can wait for
// running kernels — a spinning master would then wait for a post kernel that
// waits for its own load. Load the protocol's kernels up front (current device).
extern "C" int esgd_async_preload(void) {
  cudaFuncAttributes a;
  cudaError_t e = cudaFuncGetAttributes(&a, k_async_post);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, k_async_wait);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, k_async_master);
  ESGD_REQUIRE(e == cudaSuccess, ESGD_ERR_CUDA, "async preload: %s", cudaGetErrorString(e));
  return ESGD_OK;
}

extern "C" int esgd_enable_peer_access(int32_t device, int32_t peer) {
  if (device == peer) return ESGD_OK;
  int can = 0;
  cudaError_t e = cudaDeviceCanAccessPeer(&can, device, peer);
  ESGD_REQUIRE(e == cudaSuccess && can, ESGD_ERR_UNSUPPORTED, "peer access %d -> %d unavailable", device, peer);
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(device);
  e = cudaDeviceEnablePeerAccess(peer, 0);
  cudaSetDevice(cur);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return ESGD_OK;
  }
  ESGD_REQUIRE(e == cudaSuccess, ESGD_ERR_CUDA, "enable peer access %d -> %d: %s", device, peer,
               cudaGetErrorString(e));
  return ESGD_OK;
}

extern "C" int esgd_async_master_f32(float* C, int64_t n, const float* const* w_ptrs, float* const* snap_ptrs,
                                     int32_t* ctl, int32_t workers, int64_t services, float etarho,
                                     int32_t ctas, esgd_stream_t stream) {
  ESGD_REQUIRE(n >= 0 && workers >= 1 && services >= 0, ESGD_ERR_SHAPE, "async_master: bad sizes");
  ESGD_REQUIRE(C && w_ptrs && snap_ptrs && ctl, ESGD_ERR_INPUT, "async_master: null buffer");
  ESGD_REQUIRE(aligned16(C), ESGD_ERR_UNSUPPORTED, "async_master: center must be 16-B aligned");
  if (services == 0) return ESGD_OK;
  const int g = ctas > 0 ? (ctas < 64 ? ctas : 64) : 8;
  // few small CTAs without shared memory: they co-reside with the workers'
  // kernels on this GPU (every CTA of the persistent master stays resident)
  k_async_master<<<g, 128, 0, ESGD_STREAM(stream)>>>(C, n, w_ptrs, snap_ptrs, ctl, 2 * workers, workers,
                                                      services, etarho);
  return check_launch("esgd_async_master_f32");
}

extern "C" int esgd_async_post(int32_t* ctl, int32_t workers, int32_t worker, int32_t* my_posts,
                               esgd_stream_t stream) {
  ESGD_REQUIRE(ctl && my_posts && worker >= 0 && worker < workers, ESGD_ERR_INPUT, "async_post: bad arguments");
  k_async_post<<<1, 1, 0, ESGD_STREAM(stream)>>>(ctl, 2 * workers, worker, my_posts);
  return check_launch("esgd_async_post");
}

extern "C" int esgd_async_wait(int32_t* ctl, int32_t workers, int32_t worker, const int32_t* my_posts,
                               esgd_stream_t stream) {
  ESGD_REQUIRE(ctl && my_posts && worker >= 0 && worker < workers, ESGD_ERR_INPUT, "async_wait: bad arguments");
  k_async_wait<<<1, 1, 0, ESGD_STREAM(stream)>>>(ctl, 2 * workers, worker, my_posts);
  return check_launch("esgd_async_wait");
}
