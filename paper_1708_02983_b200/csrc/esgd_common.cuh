// Shared launch/error plumbing for the libesgd C-ABI (include/esgd.h).
//
// Every exported entry point validates its arguments on the host, launches
// on the caller's stream and returns an esgd status code; the message of the
// last failure on the calling thread is available from esgd_last_error().
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdarg.h>

#include "../../include/esgd.h"

namespace esgd {

void set_error(const char* fmt, ...);

inline int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: CUDA launch failed: %s", what, cudaGetErrorString(e));
    return ESGD_ERR_CUDA;
  }
  return ESGD_OK;
}

#define ESGD_REQUIRE(cond, code, ...)      \
  do {                                     \
    if (!(cond)) {                         \
      ::esgd::set_error(__VA_ARGS__);      \
      return (code);                       \
    }                                      \
  } while (0)

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

constexpr int kNumSMs = 148;

// SMs the persistent tensor-core kernels leave free for a concurrently
// running collective (esgd_set_sm_reserve; 0 by default). Only the grid size
// changes — tile plans and split-K counts use kNumSMs, so results do not.
int sm_reserve();

// Grid for a grid-stride elementwise kernel over `work` items: enough CTAs for
// `per_sm` resident blocks on each of the 148 SMs, never more than the work.
inline int stride_grid(int64_t work, int threads, int per_sm = 8) {
  int64_t blocks = (work + threads - 1) / threads;
  int64_t cap = (int64_t)kNumSMs * per_sm;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  return (int)blocks;
}

}  // namespace esgd
