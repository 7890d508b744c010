// Library-level C-ABI: error reporting and device checks (include/esgd.h).
#include "esgd_common.cuh"

#include <string.h>

#include <atomic>

namespace esgd {

static std::atomic<int> g_sm_reserve{0};
int sm_reserve() { return g_sm_reserve.load(std::memory_order_relaxed); }

static thread_local char g_last_error[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
}

}  // namespace esgd

extern "C" const char* esgd_last_error(void) { return esgd::g_last_error; }

extern "C" int esgd_abi_version(void) { return 1; }

extern "C" int esgd_set_sm_reserve(int32_t sms) {
  ESGD_REQUIRE(sms >= 0 && sms <= esgd::kNumSMs - 16, ESGD_ERR_INPUT, "set_sm_reserve: 0..%d SMs, got %d",
               esgd::kNumSMs - 16, sms);
  esgd::g_sm_reserve.store(sms & ~1, std::memory_order_relaxed);  // (even: CTA pairs keep whole TPCs)
  return ESGD_OK;
}

extern "C" int esgd_device_ok(int device) {
  cudaDeviceProp prop;
  cudaError_t e = cudaGetDeviceProperties(&prop, device);
  if (e != cudaSuccess) {
    esgd::set_error("esgd_device_ok: %s", cudaGetErrorString(e));
    cudaGetLastError();
    return 0;
  }
  if (prop.major != 10 || prop.minor != 0) {
    esgd::set_error("libesgd is built for sm_100a; device %d is sm_%d%d", device, prop.major,
                    prop.minor);
    return 0;
  }
  return 1;
}
