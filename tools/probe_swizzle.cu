// Probe: byte layout that TMA produces for one 32(MN) x 32(K) fp32 box with
// CU_TENSOR_MAP_SWIZZLE_128B vs CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B — dumps
// shared memory linearly so the swizzle can be read off (tools/probe_swizzle.py).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__global__ void k_dump(const __grid_constant__ CUtensorMap map, float* out) {
  __shared__ __align__(1024) float tile[1024];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(tile), b = (uint32_t)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 4096;" ::"r"(b) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(s),
        "l"(reinterpret_cast<uint64_t>(&map)), "r"(b), "r"(0), "r"(0)
        : "memory");
  }
  uint32_t done = 0;
  while (!done) {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(b) : "memory");
  }
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) out[i] = tile[i];
}

extern "C" int probe_swizzle(float* out_dev, const float* src_dev, int atom32) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess) return 1;
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  CUtensorMap map;
  cuuint64_t dims[2] = {32, 32};
  cuuint64_t strides[1] = {32 * 4};
  cuuint32_t box[2] = {32, 32}, estr[2] = {1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(src_dev), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE,
                   atom32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return 2;
  k_dump<<<1, 128>>>(map, out_dev);
  return cudaDeviceSynchronize() == cudaSuccess ? 0 : 3;
}
