// Tensor-core issue-rate probe: cycles per tcgen05.mma.kind::tf32 (M=128,
// K=8) as a function of N, with A from shared memory (SS) or from TMEM (TS).
// One CTA per SM, one thread issues `iters` x 4 MMAs into a single TMEM
// accumulator, commit + wait, clock64 around it. Operand values are zeros;
// only the rate is measured. INTF adds concurrent traffic from 4 other warps
// (1 shared-memory copy, 2 tcgen05.st into TMEM, 3 tcgen05.ld from TMEM) to
// see which resource the MMA shares.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/probe_mma tools/probe_mma_rate.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__host__ __device__ constexpr uint32_t idesc(int m, int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

// REAL: random operand values, and the GEMM's exact 3xTF32 issue pattern
// (alo.bh, ahi.bl, ahi.bh per 8-K step, 4 rotating TMEM A slots, a commit
// per 32-K block)
template <int N, bool TS, int INTF, bool REAL = false, int EXTRA = 0>
__global__ void __launch_bounds__(448, 1) probe(int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar, bar2, bar3, ring_empty[4], ring_split[4];
  __shared__ uint32_t slot;
  __shared__ volatile int stop;
  if (threadIdx.x == 0) stop = 0;
  for (int i = threadIdx.x; i < (96 * 1024) / 4; i += blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u;
    h ^= h >> 15;
    ((float*)base)[i] = REAL ? (float)(int)(h & 0xFFFF) / 32768.f - 1.f : 0.f;
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar2)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar3)));
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&bar3)) : "memory");
    for (int i = 0; i < 4; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&ring_empty[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 4;" ::"r"(su32(&ring_split[i])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  if (REAL && threadIdx.x < 128) {  // random A hi/lo in 4 slots of 64 columns at 256..511
    uint32_t v[8];
    for (int c = 256; c < 512; c += 8) {
      for (int j = 0; j < 8; ++j) v[j] = __float_as_uint((float)((threadIdx.x * 7 + c + j * 13) % 97) / 50.f - 0.97f);
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                       tmem + ((uint32_t)((threadIdx.x >> 5) * 32) << 16) + c),
                   "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]) : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (REAL && threadIdx.x == 0) {
    const uint32_t b_s = su32(base + 16384), bl_s = su32(base + 16384 + 32768);
    constexpr uint32_t id = idesc(128, N);
    long long t0 = clock64();
    for (int g = 0; g < iters; ++g) {
      if (EXTRA & 8) {
        uint32_t ok = 0;
        while (!ok)
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                       "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(su32(&ring_split[g % 4])), "r"((g / 4) & 1) : "memory");
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      }
      if (EXTRA & 2) {
        uint32_t ok = 0;
        while (!ok)
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                       "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(su32(&bar3)) : "memory");
      }
      if (EXTRA & 1) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t so = (EXTRA & 4) ? (g % 2) * 8192 : 0;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t bh = desc_sw128(b_s + so + kk * 32), bl = desc_sw128(bl_s + so + kk * 32);
        const uint32_t ahi = tmem + 256 + (g % 4) * 64 + kk * 8, alo = ahi + 32;
        const uint32_t acc = tmem + ((g / 2) % 2) * (N <= 128 ? N : 0);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, {%5, %5, %5, %5}, p;\n\t}" ::"r"(acc),
            "r"(alo), "l"(bh), "r"(id), "r"((g % 2 || kk) ? 1u : 0u), "r"(0u));
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, {%5, %5, %5, %5}, p;\n\t}" ::"r"(acc),
            "r"(ahi), "l"(bl), "r"(id), "r"(1u), "r"(0u));
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, {%5, %5, %5, %5}, p;\n\t}" ::"r"(acc),
            "r"(ahi), "l"(bh), "r"(id), "r"(1u), "r"(0u));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       su32((EXTRA & 8) ? &ring_empty[g % 4] : &bar2)) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar))
                 : "memory");
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                   "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"(su32(&bar)) : "memory");
    out[blockIdx.x] = (clock64() - t0) / 3;  // 12 MMAs per block: report per 4
    stop = 1;
  } else if (threadIdx.x == 0) {
    const uint32_t a_s = su32(base), b_s = su32(base + 16384);
    constexpr uint32_t id = idesc(128, N);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t bd = desc_sw128(b_s + kk * 32);
        if (TS) {
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, {%5, %5, %5, %5}, p;\n\t}" ::"r"(tmem),
              "r"(tmem + 256 + kk * 8), "l"(bd), "r"(id), "r"(1u), "r"(0u));
        } else {
          const uint64_t ad = desc_sw128(a_s + kk * 32);
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
              "l"(ad), "l"(bd), "r"(id), "r"(1u));
        }
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar))
                 : "memory");
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                   "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"(su32(&bar)) : "memory");
    out[blockIdx.x] = clock64() - t0;
    stop = 1;
  } else if ((EXTRA & 8) && threadIdx.x >= 128 && threadIdx.x < 256) {  // 4 "split" warps
    for (int g = 0; g < iters; ++g) {
      if (g >= 4) {
        uint32_t ok = 0;
        while (!ok)
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                       "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(su32(&ring_empty[g % 4])), "r"(((g / 4) - 1) & 1) : "memory");
      }
      __syncwarp();
      if ((threadIdx.x & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&ring_split[g % 4])) : "memory");
    }
  } else if (INTF >= 5 && threadIdx.x >= 128 && threadIdx.x < 256) {  // 4 warps: proxy fence every ~T ns
    while (!stop) {
      __nanosleep(INTF == 5 ? 500 : 2000);
      if (INTF == 7) asm volatile("fence.acq_rel.cta;" ::: "memory");
      else asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
  } else if (INTF == 4 && threadIdx.x >= 32) {  // 13 warps polling an mbarrier (like idle roles)
    uint32_t ok = 0;
    while (!ok && !stop)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 1;\n\t"
                   "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(su32(&bar3)) : "memory");
  } else if (threadIdx.x >= 128 && INTF) {
    const int w = (threadIdx.x >> 5) & 3, l = threadIdx.x & 31;
    if (INTF == 1) {  // smem: read 16 B + write 16 B per thread per iteration, 48 KB region
      float4* src = (float4*)(base + 49152);
      for (int it = 0; !stop; ++it) {
        const int i = (it * 128 + threadIdx.x - 128) & 1023;
        float4 v = src[i];
        v.x += 1.f;
        src[(i + 1536) & 3071] = v;
      }
    } else {
      const uint32_t ta = tmem + ((uint32_t)(w * 32) << 16) + 384 + (INTF == 3 ? 0 : 64);
      uint32_t v[8] = {0, 0, 0, 0, 0, 0, 0, (uint32_t)l};
      while (!stop) {
        if (INTF == 2)
          asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n\t"
                       "tcgen05.wait::st.sync.aligned;" ::"r"(ta), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]),
                       "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]) : "memory");
        else
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n\t"
                       "tcgen05.wait::ld.sync.aligned;" : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]),
                       "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]) : "r"(ta) : "memory");
      }
      if (v[0] == 12345) out[0] = 0;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

template <int N, bool TS, int INTF = 0, bool REAL = false, int EXTRA = 0>
void run(long long* d, int grid, int iters = 4096) {
  const int smem = 96 * 1024 + 1024;
  cudaFuncSetAttribute(probe<N, TS, INTF, REAL, EXTRA>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<N, TS, INTF, REAL, EXTRA><<<grid, 448, smem>>>(64, d);
  probe<N, TS, INTF, REAL, EXTRA><<<grid, 448, smem>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(long long) * grid, cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < grid; ++i) s += h[i];
  const double cyc = s / grid / (iters * 4.0);
  printf("%s%s x%d intf=%d N=%3d grid=%3d: %6.1f cycles/MMA (floor %5.1f) -> %5.1f%% of floor  %s\n", TS ? "TS" : "SS", REAL ? "-3x" : "", EXTRA, INTF, N, grid,
         cyc, N / 2.0, 100.0 * (N / 2.0) / cyc, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  run<64, false>(d, 1); run<128, false>(d, 1); run<192, false>(d, 1); run<256, false>(d, 1);
  run<64, true>(d, 1); run<128, true>(d, 1); run<192, true>(d, 1); run<256, true>(d, 1);
  run<128, true, 1>(d, 1); run<192, true, 1>(d, 1); run<256, true, 1>(d, 1); run<128, false, 1>(d, 1);
  run<128, true, 2>(d, 1); run<192, true, 2>(d, 1); run<256, true, 2>(d, 1);
  run<128, true, 3>(d, 1); run<192, true, 3>(d, 1); run<256, true, 3>(d, 1);
  run<128, true, 0, true>(d, 1); run<192, true, 0, true>(d, 1); run<128, true, 0, true>(d, 148);
  run<192, true, 0, true>(d, 148); run<128, true, 1, true>(d, 148);
  run<128, true, 0, true, 1>(d, 148); run<128, true, 0, true, 2>(d, 148); run<128, true, 0, true, 4>(d, 148);
  run<128, true, 0, true, 7>(d, 148); run<128, true, 4, true, 7>(d, 148); run<128, true, 4, true, 0>(d, 148);
  run<128, true, 0, true, 8>(d, 148); run<192, true, 0, true, 8>(d, 148); run<128, true, 0, true, 15>(d, 148);
  return 0;
}
