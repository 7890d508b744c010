// Tensor-core GEMM for the conv-as-GEMM and FC contractions (sm_100a).
//
//   C[z] (m x n) = act( A[z] (m x k, K-major) . B[z] (n x k, K-major)^T + bias )
//
// Blackwell-native structure (one 128 x BN output tile per CTA):
//   warp 0      : TMA producer — cp.async.bulk.tensor 3-D loads of raw fp32
//                 A/B tiles (128-byte swizzle) into a multi-stage smem ring,
//                 completion tracked by mbarrier transaction counts.
//   warps 2..5  : split warps — for 3xTF32 they write A's rows as tf32 hi/lo
//                 (hi = x & 0xffffe000, lo = x - hi) into TMEM, and B's
//                 lo = x - hi into a twin smem buffer of identical (swizzled)
//                 layout (the raw B tile already is B_hi to the tensor core,
//                 which ignores the low 13 mantissa bits), then
//                 fence.proxy.async and arrive.
//   warp 1      : TMEM allocation and the single-thread tcgen05.mma issuer,
//                 kind::tf32, M=128, N=BN, K=8 per instruction, into one of
//                 two TMEM accumulators per kChunkKB*32-deep K chunk;
//                 tcgen05.commit frees smem slots and hands finished chunks
//                 to the drain.
//   warps 6..13 : drain/epilogue, two warps per TMEM lane quadrant (half the
//                 columns each) — tcgen05.ld each chunk's partial sums and add
//                 them into fp32 registers with RN adds (the tensor-core
//                 accumulator alone loses ~1e-8*K relative), then bias/act/
//                 mask and the smem-staged TMA store.
//
// 3xTF32: a.b ~= hi_a.hi_b + hi_a.lo_b + lo_a.hi_b, accumulated in fp32 in
// TMEM — fp32-grade products (relative error ~2^-21), which the parity gate
// (1e-5 relative, BASELINE.json north_star) requires; plain TF32 (~1e-3)
// would not pass it.
#include "esgd_common.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <stdlib.h>
#include <string.h>

namespace esgd {
namespace tc {

constexpr int BM = 128;
constexpr int BK = 32;                  // 32 fp32 = 128 B = one swizzle atom row
constexpr int kThreads = 448;           // 14 warps: TMA, MMA, 4 split, 8 drain/epilogue (BN = 192)
// split warps per CTA: 4 (one per TMEM lane quadrant). The kernel also runs
// with 8 (two per quadrant, each half of the 32 K columns; ESGD_SPLIT_WARPS=8
// at build time, BN <= 128, 96 registers per thread): measured no faster on
// the AlexNet shapes (conv2 dgrad 0.34 -> 0.37 ms, conv4 dgrad 0.19 -> 0.18 ms)
// — the split warps are not short of issue slots but of TMEM / smem bandwidth
#ifndef ESGD_SPLIT_WARPS
#define ESGD_SPLIT_WARPS 4
#endif
__host__ __device__ constexpr int split_warps(int bn, bool split) {
  return (split && bn <= 128 && ESGD_SPLIT_WARPS == 8) ? 8 : 4;
}
__host__ __device__ constexpr int cta_threads(int bn, bool split) { return 32 * (10 + split_warps(bn, split)); }
constexpr int kDrainWarps = 8;         // two per TMEM lane quadrant, each owning half of the BN columns
// K-blocks (x32) per TMEM accumulation before promotion into fp32 registers.
// 4 (128-deep chunks) measured ~8% faster on the AlexNet shapes (the drain's
// TMEM reads compete with the TS-mode A operand) but doubles the tensor-core
// accumulation error, and a 3-round multi-replica CNN run then drifted 2e-3
// from the oracle (tests/test_gpu_sync.py); 2 keeps every parity test green.
#ifndef ESGD_CHUNK_KB
#define ESGD_CHUNK_KB 2
#endif
constexpr int kChunkKB = ESGD_CHUNK_KB;
// output-tile waves a split-K GEMM is cut into (weight gradients)
#ifndef ESGD_SPLIT_WAVES
#define ESGD_SPLIT_WAVES 1
#endif
constexpr int kTileBytesA = BM * BK * 4;  // 16 KB

template <int BN, bool SPLIT, bool PAIR = false, int EXTRA = 0>
struct Cfg {
  // PAIR (cta_group::2): the CTA pair computes a 256 x BN tile; each CTA holds
  // its own 128 A rows and half of B's BN rows in shared memory, and a 128 x BN
  // accumulator in its own TMEM
  static constexpr int kRowsB = PAIR ? BN / 2 : BN;
  static constexpr int kTileBytesB = kRowsB * BK * 4;
  // stage layout: [lo spill | A raw | B raw], every tile 1024-B aligned.
  // In 3xTF32 mode A never gets a lo twin in smem: the split warps write the
  // tf32 hi/lo rows of A straight into TMEM and the MMAs read A from there —
  // so once they have read the A tile, B's lo twin is written over it,
  // starting at the stage base; the spill is the part of B lo that does not
  // fit in A's 16 KB (8 KB at BN = 192). 48 KB stages at BN = 192 give a
  // fourth ring stage (three covered TMA latency + split + MMA per stage
  // only partly), 32 KB at BN = 128 six.
  static constexpr int kLoSpill = (SPLIT && kTileBytesB > kTileBytesA) ? kTileBytesB - kTileBytesA : 0;
  static constexpr int kOffA = kLoSpill;
  static constexpr int kOffB = kOffA + kTileBytesA;
  static constexpr int kOffBLo = 0;
  static constexpr int kStageBytes = kLoSpill + kTileBytesA + kTileBytesB;
  // EXTRA: bytes after the barriers (the gathered-B row table of GM = 2)
  static constexpr int kStages =
      (192 * 1024 - EXTRA) / kStageBytes > 8 ? 8 : (192 * 1024 - EXTRA) / kStageBytes;
#ifndef ESGD_ACC_BUFS128
#define ESGD_ACC_BUFS128 2
#endif
  // TMEM accumulator buffers (chunks in flight between the MMA and the drain)
  static constexpr int kAccBufs = (BN == 128 && SPLIT) ? ESGD_ACC_BUFS128 : 2;
  static constexpr int kACol0 = kAccBufs * BN;  // TMEM columns of the A regions (64 per slot: hi 32 | lo 32)
  // TMEM A slots (a ring of its own): as many as the 512 columns leave next to
  // the two BN-wide accumulators — 4 at BN <= 128, 2 at BN = 192
  static constexpr int kASlots = SPLIT ? ((512 - kACol0) / 64 < kStages ? (512 - kACol0) / 64 : kStages) : 1;
  static constexpr int kTmemCols = SPLIT ? 512 : (2 * BN < 32 ? 32 : 2 * BN);
  static_assert(!SPLIT || (kASlots >= 2 && kACol0 + 64 * kASlots <= 512), "TMEM budget");
  static constexpr int kStageOutBytes = 32768;  // epilogue staging: 128 rows x 64 cols fp32
  static constexpr int kSmemBytes =
      kStages * kStageBytes + kStageOutBytes + 1024 /*align*/ + 256 /*barriers*/ + EXTRA;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                            int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
// TMA im2col load (4-D NHWC source, c innermost): `pixels` consecutive output
// positions of the map's traversal starting at (w, h, n), channels c0.., each
// read at that position + (off_w, off_h) — one k-block of an implicit GEMM
__device__ __forceinline__ void tma_load_im2col(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int w,
                                                int h, int n, int off_w, int off_h) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(w), "r"(h), "r"(n),
      "h"((unsigned short)off_w), "h"((unsigned short)off_h)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// K-major, 128-byte swizzle canonical layout: rows of 128 B, 8-row atoms
// 1024 B apart (SBO), LBO = 1 (unused for swizzled K-major), version 1.
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
// MN-major tf32 operands: UMMA accepts only the "128B swizzle with 32-byte
// atomicity" layout (SWIZZLE_128B_BASE32B; CUTLASS sm100 builder: "for
// mn-major tf32 operands, SW128_32B is the only available smem layout"),
// loaded by TMA with CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B. Atoms are 32 MN
// elements (128 B) x 4 K rows; each TMA box of 32(MN) x 32(K) lands as 4 KB,
// so K-atoms are SBO = 512 B apart and MN-atoms LBO = 4096 B.
__device__ __forceinline__ uint64_t desc_sw128_mn(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)(4096 >> 4) << 16;
  d |= (uint64_t)(512 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)1 << 61;  // SWIZZLE_128B_BASE32B
  return d;
}
// instruction descriptor: kind::tf32, fp32 accumulate, A/B major per flag
__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n, bool a_mn, bool b_mn) {
  return (1u << 4)                      // c_format = F32
         | (2u << 7)                    // a_format = TF32
         | (2u << 10)                   // b_format = TF32
         | ((a_mn ? 1u : 0u) << 15)     // a_major: 1 = MN-major
         | ((b_mn ? 1u : 0u) << 16)     // b_major
         | ((uint32_t)(n >> 3) << 17)   // N >> 3
         | ((uint32_t)(m >> 4) << 24);  // M >> 4
}
__device__ __forceinline__ void mma_tf32(uint32_t tmem_c, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_c),
      "l"(a), "l"(b), "r"(idesc), "r"(accum));
}
// A operand from TMEM ("TS"): K-major rows = TMEM lanes, 8 tf32 columns per MMA
__device__ __forceinline__ void mma_tf32_ts(uint32_t tmem_c, uint32_t tmem_a, uint64_t b, uint32_t idesc,
                                            uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, {%5, %5, %5, %5}, p;\n\t}" ::"r"(tmem_c),
      "r"(tmem_a), "l"(b), "r"(idesc), "r"(accum), "r"(0u));
}
// cta_group::2 (leader CTA issues for the pair; D / A rows 0-127 in the
// leader's TMEM, 128-255 in the peer's; B halves in both CTAs' shared memory)
__device__ __forceinline__ void mma_tf32_ts_pair(uint32_t tmem_c, uint32_t tmem_a, uint64_t b, uint32_t idesc,
                                              uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, {%5, %5, %5, %5, %5, %5, %5, %5}, p;\n\t}" ::"r"(tmem_c),
      "r"(tmem_a), "l"(b), "r"(idesc), "r"(accum), "r"(0u));
}
__device__ __forceinline__ void mma_tf32_pair(uint32_t tmem_c, uint64_t a, uint64_t b, uint32_t idesc,
                                           uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, {%5, %5, %5, %5, %5, %5, %5, %5}, p;\n\t}" ::"r"(tmem_c),
      "l"(a), "l"(b), "r"(idesc), "r"(accum), "r"(0u));
}
// commit the pair's outstanding MMAs to the barrier at the same offset in both CTAs
__device__ __forceinline__ void mma_commit_pair(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
      "h"((uint16_t)3)
      : "memory");
}
// arrive on the barrier at the same offset in CTA 0 of the cluster (the leader)
__device__ __forceinline__ void mbar_arrive_leader(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\t"
      "mapa.shared::cluster.u32 ra, %0, 0;\n\t"
      "mbarrier.arrive.shared::cluster.b64 _, [ra];\n\t}" ::"r"(bar)
      : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint32_t bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
      "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
      "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
// 32 columns of the warp's 32 TMEM lanes, no wait (pair with tmem_wait_ld)
__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

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

struct Epi {
  float* c; int64_t c_sm, c_sn, c_sb;
  const float* bias; int64_t bias_sb;
  const float* mask; int64_t mask_sm, mask_sn, mask_sb;
  int act, accumulate, m, n, k;
  float* ws;        // split-K partials [batch][splits][m][n]
  int splits, kb_per_split, batch;
  int out_mode;     // 0 direct stores (via smem staging), 1 TMA store M-contiguous C, 2 TMA store N-contiguous C
  int m_fast;       // rasterise units m-fastest (M-contiguous output) else n-fastest
};

// Implicit-GEMM operand gathered by the split warps straight from a CNHW
// activation tensor (channel planes of `plane` floats, each plane [n][y][x]
// of images SH x SW), instead of a materialised im2col matrix:
//   GM = 1 (conv forward / data gradient): A[m][k], m a pixel of the MH x MW
//     grid (n, r, c), k = (ch, kh, kw) in the packed weight order;
//   GM = 2 (weight gradient): B[n][k], n = (ch, kh, kw), k a pixel.
// value = S[z*sb + ch*plane + n*SH*SW + y*SW + x] with
//   y = r*stride + yoff + sgn*kh, x = c*stride + xoff + sgn*kw,
// zero outside the image (padding) and for pixels / k beyond the problem.
// sgn = +1 is the convolution's own window (forward, weight gradient); sgn =
// -1 with stride 1 and offset +pad is the transposed window of the data
// gradient (dx[ci][pix] = sum_{co,kh,kw} W[co][ci][kh][kw] d[co][pix+pad-k]).
struct Gather {
  const float* src;
  int64_t sb;      // replica (batch) stride
  int plane;       // channel plane pitch
  int nstride;     // image stride (SH*SW for CNHW planes, C*SH*SW for NCHW rows)
  int SH, SW;      // source image
  int MH, MW;      // pixel grid of the gathered side
  int stride, yoff, xoff, sgn;
  int KH, KW;      // window
  int npix;        // pixels of the grid over the whole batch of images
  int kdim;        // channels * KH * KW
  int hpitch;      // GM = 3: floats per channel of the smem halo
};

// GM = 4 / 5 (TMA im2col, NHWC source of SH x SW images, C = kdim / (KH*KW)
// channels, K ordered (kh, kw, c)): the traversal position (w, h, n) of grid
// pixel p (image n, row r, column c of the MH x MW grid) is
// (c*stride + xoff, r*stride + yoff, n); yoff = xoff = -pad
__device__ __forceinline__ void im2col_pos(const Gather& g, int p, int& w, int& h, int& n) {
  const int hw = g.MH * g.MW;
  n = p / hw;
  const int r = p - n * hw, y = r / g.MW;
  h = y * g.stride + g.yoff;
  w = (r - y * g.MW) * g.stride + g.xoff;
}

// GM = 3 (halo): the source rows a unit's 128 pixels touch, as flattened
// (image, y) rows of the channel planes, clamped to the planes
__device__ __forceinline__ void halo_rows(const Gather& g, int m0, int& r_lo, int& r_hi) {
  const int hw = g.MH * g.MW, last = min(m0 + BM, g.npix) - 1;
  const int n0 = m0 / hw, y0 = ((m0 - n0 * hw) / g.MW) * g.stride + g.yoff;
  const int n1 = last / hw, y1 = ((last - n1 * hw) / g.MW) * g.stride + g.yoff;
  const int reach = g.sgn * (g.KH - 1);
  r_lo = max(0, n0 * g.SH + y0 + min(0, reach));
  r_hi = min(g.npix / hw * g.SH - 1, n1 * g.SH + y1 + max(0, reach));
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const float* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

// (koff, kh | kw << 16) of packed k = (ch, kh, kw); an out-of-range k gets kh
// = 0x7fff so every bounds test fails
__device__ __forceinline__ void gather_k(const Gather& g, int k, int& koff, int& khkw) {
  if (k >= g.kdim) {
    koff = 0;
    khkw = 0x7fff;
    return;
  }
  const int kk = g.KH * g.KW;
  const int ch = k / kk, t = k - ch * kk, kh = t / g.KW, kw = t - kh * g.KW;
  koff = ch * g.plane + g.sgn * (kh * g.SW + kw);
  khkw = kh | (kw << 16);
}
// pixel p of the grid -> offset of its window origin and the origin itself;
// a pixel beyond the grid gets an origin far outside the image
__device__ __forceinline__ void gather_pix(const Gather& g, int p, int& pbase, int& y0, int& x0) {
  if (p >= g.npix) {
    pbase = 0;
    y0 = x0 = -(1 << 28);
    return;
  }
  const int hw = g.MH * g.MW;
  const int n = p / hw, rem = p - n * hw, r = rem / g.MW, c = rem - r * g.MW;
  y0 = r * g.stride + g.yoff;
  x0 = c * g.stride + g.xoff;
  pbase = n * g.nstride + y0 * g.SW + x0;
}
__device__ __forceinline__ float gather_ld(const Gather& g, const float* zs, int pbase, int y0, int x0, int koff,
                                           int khkw) {
  const int y = y0 + g.sgn * (khkw & 0xffff), x = x0 + g.sgn * (khkw >> 16);
  return ((unsigned)y < (unsigned)g.SH && (unsigned)x < (unsigned)g.SW) ? __ldg(zs + (pbase + koff)) : 0.f;
}

__device__ __forceinline__ void cp_async4(uint32_t dst, const float* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(valid ? 4 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_arrive(uint32_t bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
}
// cp.async of one gathered element (zero-filled when outside the image)
__device__ __forceinline__ void gather_cp(const Gather& g, const float* zs, int pbase, int y0, int x0, int koff,
                                          int khkw, uint32_t dst) {
  const int y = y0 + g.sgn * (khkw & 0xffff), x = x0 + g.sgn * (khkw >> 16);
  const bool ok = (unsigned)y < (unsigned)g.SH && (unsigned)x < (unsigned)g.SW;
  cp_async4(dst, ok ? zs + (pbase + koff) : zs, ok);
}

// epilogue value without the read-modify-write of accumulate (TMA-store path)
__device__ __forceinline__ float epi_value(const Epi& ep, float x, int z, int row, int col) {
  if (ep.bias && col < ep.n) x = __fadd_rn(x, ep.bias[z * ep.bias_sb + col]);
  x = act_apply(x, ep.act);
  if (ep.mask && row < ep.m && col < ep.n)
    x = __fmul_rn(x, ep.mask[z * ep.mask_sb + (int64_t)row * ep.mask_sm + (int64_t)col * ep.mask_sn] > 0.f ? 1.f : 0.f);
  return x;
}

__device__ __forceinline__ float epi_apply(const Epi& ep, float x, int z, int row, int col, int64_t off,
                                           const float* cz) {
  const float* bz = ep.bias ? ep.bias + z * ep.bias_sb : nullptr;
  const float* mz = ep.mask ? ep.mask + z * ep.mask_sb : nullptr;
  if (ep.accumulate) x = __fadd_rn(cz[off], x);
  if (bz) x = __fadd_rn(x, bz[col]);
  x = act_apply(x, ep.act);
  if (mz) x = __fmul_rn(x, mz[(int64_t)row * ep.mask_sm + (int64_t)col * ep.mask_sn] > 0.f ? 1.f : 0.f);
  return x;
}

// TMA of one operand tile for k-block kb: K-major = one box (32 K x rows);
// MN-major = rows/32 boxes of (32 MN x 32 K), 4 KB apart.
template <bool MN, int ROWS>
__device__ __forceinline__ void load_operand(uint32_t dst, const CUtensorMap* map, uint32_t bar, int kb,
                                             int r0, int z) {
  if (!MN) {
    tma_load_3d(dst, map, bar, kb * BK, r0, z);
  } else {
#pragma unroll
    for (int j = 0; j < ROWS / 32; ++j) tma_load_3d(dst + j * 4096, map, bar, r0 + 32 * j, kb * BK, z);
  }
}

template <bool MN>
__device__ __forceinline__ uint64_t op_desc(uint32_t tile, int kk) {
  return MN ? desc_sw128_mn(tile + kk * 1024) : desc_sw128(tile + kk * 32);
}

// split one landed tile: hi = tf32-truncated x (in place), lo = x - hi.
// Shared-window addresses with explicit ld/st.shared.v4 (a generic pointer
// here costs an address-space check and L1TEX latency per access), eight
// 16-B loads in flight per thread before any store.
__device__ __forceinline__ float4 lds4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts4(uint32_t a, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

template <int BYTES, int NT = 128>
__device__ __forceinline__ void split_tile(uint32_t raw, uint32_t lo, int tid) {
  constexpr int kVec = BYTES / 16, kPer = kVec / NT;
  constexpr int kBatch = kPer <= 8 ? kPer : (kPer % 8 == 0 ? 8 : (kPer % 6 == 0 ? 6 : 4));
  static_assert(kVec % NT == 0 && kPer % kBatch == 0, "tile must split evenly over the threads");
#pragma unroll
  for (int b0 = 0; b0 < kPer; b0 += kBatch) {
    float4 x[kBatch];
#pragma unroll
    for (int j = 0; j < kBatch; ++j) x[j] = lds4(raw + 16 * (tid + NT * (b0 + j)));
#pragma unroll
    for (int j = 0; j < kBatch; ++j) {
      const uint32_t off = 16 * (tid + NT * (b0 + j));
      float4 h, l;
      h.x = tf32_hi(x[j].x); h.y = tf32_hi(x[j].y); h.z = tf32_hi(x[j].z); h.w = tf32_hi(x[j].w);
      l.x = __fsub_rn(x[j].x, h.x); l.y = __fsub_rn(x[j].y, h.y);
      l.z = __fsub_rn(x[j].z, h.z); l.w = __fsub_rn(x[j].w, h.w);
      // the hi part is NOT written back: kind::tf32 MMAs ignore the low 13
      // mantissa bits of an fp32 operand (measured bit-exact against
      // pre-truncated operands, tools/probe_tf32.py), so the raw tile already
      // is B_hi to the tensor core — one 16 KB smem write less per k-block
      sts4(lo + off, l);
    }
  }
}

// Work unit = (n tile, m tile, batch z, K slice); units are dealt to the
// persistent CTAs round-robin. Every role walks the same unit sequence, so the
// smem-stage ring (global k-block counter) and the TMEM-accumulator ring
// (global chunk counter) stay in lockstep across units: the TMA of unit u+1
// overlaps the MMAs of unit u, and the epilogue of unit u overlaps both.
struct Unit {
  int n0, m0, z, slice, kb0, nkb;
};
__device__ __forceinline__ Unit unit_of(int u, const Epi& ep, int ntn, int ntm, int nkb_all, int BN_,
                                       int BM_ = BM) {
  Unit w;
  const int per_z = ntn * ntm * ep.splits;
  w.z = u / per_z;
  int r = u - w.z * per_z;
  w.slice = r / (ntn * ntm);
  r -= w.slice * ntn * ntm;
  // Concurrent CTAs take neighbouring tiles along the output's contiguous
  // dimension, so their stores (and the operand loads) stay within a few
  // 2-MB pages: n-fastest ordering on an M-contiguous 600-MB output scattered
  // 148 tiles over every page and throttled the stores to ~220 GB/s (TLB).
  if (ep.m_fast) {
    w.n0 = (r / ntm) * BN_;
    w.m0 = (r % ntm) * BM_;
  } else {
    w.m0 = (r / ntn) * BM_;
    w.n0 = (r % ntn) * BN_;
  }
  w.kb0 = w.slice * ep.kb_per_split;
  w.nkb = max(0, min(nkb_all - w.kb0, ep.kb_per_split));
  return w;
}

// staged-quarter smem address of (row r, column j) of a 32-column quarter:
// mode 1 (M-contiguous C): [32 cols][128 rows]; mode 2 (N-contiguous C): 128-B
// rows with the 128B swizzle the TMA store map expects
template <int MODE>
__device__ __forceinline__ uint32_t stage_addr(uint32_t sb, int r, int j) {
  return MODE == 1 ? sb + (j * 128 + r) * 4 : sb + r * 128 + ((((j >> 2) ^ (r & 7))) << 4) + (j & 3) * 4;
}

// registers -> smem for the thread's local quarter lq (columns col0..col0+31
// of the tile row); FAST applies bias + identity/relu
template <int NACC, int MODE, bool FAST>
__device__ __forceinline__ void stage_quarter(const float (&racc)[NACC], int lq, uint32_t sb, int r,
                                              const float* bz, bool relu, int col0, int n) {
#pragma unroll
  for (int jj = 0; jj < 32; jj += 4) {
    const int j = lq * 32 + jj;
    float v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float x = racc[j + e];
      if (FAST) {
        if (bz) x = __fadd_rn(x, col0 + jj + e < n ? __ldg(bz + col0 + jj + e) : 0.f);
        if (relu) x = fmaxf(x, 0.f);
      }
      v[e] = x;
    }
    if (MODE == 1) {
#pragma unroll
      for (int e = 0; e < 4; ++e)
        asm volatile("st.shared.f32 [%0], %1;" ::"r"(stage_addr<1>(sb, r, jj + e)), "f"(v[e]) : "memory");
    } else {
      sts4(stage_addr<2>(sb, r, jj), make_float4(v[0], v[1], v[2], v[3]));
    }
  }
}

// general epilogue over the thread's own staged row (raw sums in mode-1 or
// mode-2 layout): bias, activation, mask; mode 0 stores straight to C
// (accumulate / strides the TMA store cannot express)
__device__ __forceinline__ void general_quarter(const Epi& ep, uint32_t sb, int r, int row, int z, int col0) {
  float* cz = ep.c + z * ep.c_sb;
#pragma unroll 1
  for (int j = 0; j < 32; ++j) {
    const uint32_t addr = ep.out_mode == 2 ? stage_addr<2>(sb, r, j) : stage_addr<1>(sb, r, j);
    float x;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x) : "r"(addr) : "memory");
    const int col = col0 + j;
    if (ep.out_mode == 0) {
      if (row < ep.m && col < ep.n) {
        const int64_t off = (int64_t)row * ep.c_sm + (int64_t)col * ep.c_sn;
        cz[off] = epi_apply(ep, x, z, row, col, off, cz);
      }
    } else {
      x = epi_value(ep, x, z, row, col);
      asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(x) : "memory");
    }
  }
}

// Diagnostic builds only (tools/build_variant.sh; never in libesgd.so):
// ESGD_TRACE stamps CTA 0's role timeline; ESGD_X_{NOTMA,NOAST,NOSPLITB,
// NODRAIN,NOEPI} switch one role's work off (wrong results, timing only) to
// attribute the gap between the MMA issue rate and the tensor-core floor.
#ifdef ESGD_TRACE
// clock64 stamps of CTA 0's roles (tools/trace_gemm.py)
constexpr int kTraceN = 4096;
__device__ unsigned long long g_trace[8][kTraceN];
#define TRACE(row, idx)                                                          \
  do {                                                                           \
    if (blockIdx.x == 0 && (idx) < kTraceN) g_trace[row][idx] = clock64();       \
  } while (0)
#else
#define TRACE(row, idx) \
  do {                  \
  } while (0)
#endif

// PAIR = false: one CTA per 128 x BN output tile (cta_group::1).
// PAIR = true: a cluster of two CTAs (one TPC) per 256 x BN tile
// (cta_group::2): each CTA loads and splits its own 128 A rows and half of
// B's rows, so every CTA's shared memory serves only half of B to the tensor
// cores (the per-SM shared-memory traffic per MMA-cycle, which bounds the
// 1-CTA kernel at BN = 128 / 192, drops by a third); the leader CTA's
// single thread issues the pair's MMAs, whose commits arrive on both CTAs'
// barriers (multicast); the peer's split and drain warps arrive on the
// leader's barriers across the cluster.
template <int BN, bool SPLIT, bool AMN, bool BMN, bool PAIR, int GM = 0>
__global__ void __launch_bounds__(cta_threads(BN, SPLIT), 1)
    k_tc_gemm(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
              const __grid_constant__ CUtensorMap map_c, Epi ep, Gather ga) {
  using C = Cfg<BN, SPLIT, PAIR>;
  static_assert(GM == 0 || (SPLIT && !AMN && (GM == 5 ? BMN : !BMN)),
                "gathered operands: 3xTF32, K-major A; im2col B (GM = 5) is MN-major");
  constexpr int NS = split_warps(BN, SPLIT);   // split warps (warps 2 .. 1+NS)
  constexpr int KC = 32 / (NS / 4);            // K columns of an A row per split thread
  constexpr int D0 = 2 + NS;                   // first drain warp
  constexpr int kCtas = PAIR ? 2 : 1;
  constexpr int BMU = BM * kCtas;  // output rows per unit
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stage_out = smem + C::kStages * C::kStageBytes;  // 32 KB, 1024-aligned
  uint64_t* bars = reinterpret_cast<uint64_t*>(stage_out + C::kStageOutBytes);
  // bars: full[S], split[S], empty[S], acc_full[2], acc_empty[2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * C::kStages + 2 * C::kAccBufs);
  const uint32_t full0 = smem_u32(bars), split0 = smem_u32(bars + C::kStages),
                 empty0 = smem_u32(bars + 2 * C::kStages), afull0 = smem_u32(bars + 3 * C::kStages),
                 aempty0 = afull0 + 8 * C::kAccBufs;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = PAIR ? cluster_rank() : 0u;
  const int ubase = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int ustep = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  const int ntn = (ep.n + BN - 1) / BN, ntm = (ep.m + BMU - 1) / BMU;
  const int nkb_all = (ep.k + BK - 1) / BK;
  const int nunits = ntn * ntm * ep.splits * ep.batch;
  const int arow = (int)rank * BM;          // this CTA's first row inside a unit
  const int brow = (int)rank * C::kRowsB;   // this CTA's first B row inside a unit

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(full0 + 8 * s, (GM == 1 || GM == 2) ? 1 + 32 * NS : 1);  // + the gathering threads (cp.async arrive)
      mbar_init(split0 + 8 * s, NS * kCtas);  // one arrive per split warp (of both CTAs: the leader's is used)
      mbar_init(empty0 + 8 * s, 1);
    }
    for (int b = 0; b < C::kAccBufs; ++b) {
      mbar_init(afull0 + 8 * b, 1);   // tcgen05.commit
      mbar_init(aempty0 + 8 * b, kDrainWarps * kCtas);  // one arrive per drain warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(C::kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(C::kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  if (PAIR) cluster_sync_all();  // both CTAs' barriers initialised before any remote arrive
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer (each CTA its own A rows and B half)
      uint32_t g = 0;  // global k-block counter (stage ring position)
      for (int u = ubase; u < nunits; u += ustep) {
        const Unit w = unit_of(u, ep, ntn, ntm, nkb_all, BN, BMU);
        for (int kb = 0; kb < w.nkb; ++kb, ++g) {
          const int s = g % C::kStages;
          if (g >= (uint32_t)C::kStages) mbar_wait(empty0 + 8 * s, ((g / C::kStages) - 1) & 1);
          TRACE(0, g);
          uint8_t* st = smem + s * C::kStageBytes;
#ifdef ESGD_X_NOTMA
          if (g >= (uint32_t)C::kStages) { mbar_arrive(full0 + 8 * s); continue; }
#endif
          if (GM == 3) {  // halo: the channels this k-block touches, rows of the unit, one bulk copy each
            int r_lo, r_hi;
            halo_rows(ga, w.m0 + arow, r_lo, r_hi);
            const int k0 = (w.kb0 + kb) * BK, kk = ga.KH * ga.KW;
            const int c_lo = k0 / kk, c_hi = min(k0 + BK, ga.kdim) / kk - ((min(k0 + BK, ga.kdim) % kk) ? 0 : 1);
            const int e0 = r_lo * ga.SW, e0a = e0 & ~3;
            const int len = min((e0 - e0a + (r_hi - r_lo + 1) * ga.SW + 3) & ~3, ga.plane - e0a);
            mbar_expect_tx(full0 + 8 * s, C::kTileBytesB + (uint32_t)(c_hi - c_lo + 1) * len * 4);
            const float* zs = ga.src + (int64_t)w.z * ga.sb;
            for (int c = c_lo; c <= c_hi; ++c)
              bulk_g2s(smem_u32(st + C::kOffA) + (c - c_lo) * ga.hpitch * 4, zs + (int64_t)c * ga.plane + e0a,
                       len * 4, full0 + 8 * s);
          } else {
            mbar_expect_tx(full0 + 8 * s, (GM == 1 ? 0 : kTileBytesA) + (GM == 2 ? 0 : C::kTileBytesB));
          }
          if (GM == 0 || GM == 2 || GM == 5)
            load_operand<AMN, BM>(smem_u32(st + C::kOffA), &map_a, full0 + 8 * s, w.kb0 + kb, w.m0 + arow, w.z);
          if (GM == 4) {  // A = 128 grid pixels x 32 channels of one window tap
            const int k0 = (w.kb0 + kb) * BK, cin = ga.kdim / (ga.KH * ga.KW);
            const int tap = k0 / cin, c0 = k0 - tap * cin;
            int iw, ih, in;
            im2col_pos(ga, w.m0 + arow, iw, ih, in);
            tma_load_im2col(smem_u32(st + C::kOffA), &map_a, full0 + 8 * s, c0, iw, ih,
                            in + w.z * (ga.npix / (ga.MH * ga.MW)), tap % ga.KW, tap / ga.KW);
          }
          if (GM == 5) {  // B = 32 grid pixels (K) x 32 channels (N) boxes, one tap each, MN-major
            const int cin = ga.kdim / (ga.KH * ga.KW);
            int iw, ih, in;
            im2col_pos(ga, (w.kb0 + kb) * BK, iw, ih, in);
            in += w.z * (ga.npix / (ga.MH * ga.MW));
#pragma unroll
            for (int j = 0; j < C::kRowsB / 32; ++j) {
              const int n = min(w.n0 + brow + 32 * j, ga.kdim - 32), tap = n / cin;
              tma_load_im2col(smem_u32(st + C::kOffB) + j * 4096, &map_b, full0 + 8 * s, n - tap * cin, iw, ih, in,
                              tap % ga.KW, tap / ga.KW);
            }
          }
          if (GM != 2 && GM != 5)
            load_operand<BMN, C::kRowsB>(smem_u32(st + C::kOffB), &map_b, full0 + 8 * s, w.kb0 + kb,
                                         w.n0 + brow, w.z);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {  // ---- MMA issuer: one K-chunk per TMEM accumulator buffer
      constexpr uint32_t idesc = idesc_tf32(BMU, BN, AMN, BMN);
      constexpr uint32_t idesc_ts = idesc_tf32(BMU, BN, false, BMN);  // A from TMEM is K-major
      uint32_t g = 0, c = 0;
      for (int u = ubase; u < nunits; u += ustep) {
        const Unit w = unit_of(u, ep, ntn, ntm, nkb_all, BN, BMU);
        for (int kc = 0; kc < w.nkb; kc += kChunkKB, ++c) {
          const int buf = c % C::kAccBufs;
          if (c >= (uint32_t)C::kAccBufs) {
            if (PAIR) mbar_wait_cluster(aempty0 + 8 * buf, ((c / C::kAccBufs) - 1) & 1);
            else mbar_wait(aempty0 + 8 * buf, ((c / C::kAccBufs) - 1) & 1);
          }
          TRACE(2, c);
          tc_fence_after();
          const uint32_t acc = tmem + buf * BN;
          const int kend = min(w.nkb, kc + kChunkKB);
          for (int kb = kc; kb < kend; ++kb, ++g) {
            const int s = g % C::kStages;
            const uint32_t ph = (g / C::kStages) & 1;
            if (SPLIT) {
              if (PAIR) mbar_wait_cluster(split0 + 8 * s, ph);
              else mbar_wait(split0 + 8 * s, ph);
            } else {
              mbar_wait(full0 + 8 * s, ph);
            }
            TRACE(1, g);
            tc_fence_after();
            const uint32_t st = smem_u32(smem + s * C::kStageBytes);
#ifndef ESGD_X_NOMMA
#pragma unroll
            for (int kk = 0; kk < BK / 8; ++kk) {
              // K-major: 8 tf32 = 32 B along K inside the swizzle atom;
              // MN-major: one 8-row K slab (1024 B) per instruction
              const uint64_t bh = op_desc<BMN>(st + C::kOffB, kk);
              const uint32_t acc0 = (kb > kc || kk > 0) ? 1u : 0u;
              if (SPLIT) {
                const uint64_t bl = op_desc<BMN>(st + C::kOffBLo, kk);
                const uint32_t ahi = tmem + C::kACol0 + (g % C::kASlots) * 64 + kk * 8, alo = ahi + 32;
                if (PAIR) {
                  mma_tf32_ts_pair(acc, alo, bh, idesc_ts, acc0);  // small terms first
                  mma_tf32_ts_pair(acc, ahi, bl, idesc_ts, 1u);
                  mma_tf32_ts_pair(acc, ahi, bh, idesc_ts, 1u);
                } else {
                  mma_tf32_ts(acc, alo, bh, idesc_ts, acc0);  // small terms first
                  mma_tf32_ts(acc, ahi, bl, idesc_ts, 1u);
                  mma_tf32_ts(acc, ahi, bh, idesc_ts, 1u);
                }
              } else {
                if (PAIR) mma_tf32_pair(acc, op_desc<AMN>(st + C::kOffA, kk), bh, idesc, acc0);
                else mma_tf32(acc, op_desc<AMN>(st + C::kOffA, kk), bh, idesc, acc0);
              }
            }
#endif
            if (PAIR) mma_commit_pair(empty0 + 8 * s);  // slot reusable (in both CTAs) once these MMAs retire
            else mma_commit(empty0 + 8 * s);
          }
          if (PAIR) mma_commit_pair(afull0 + 8 * buf);  // this chunk's partial sum is complete
          else mma_commit(afull0 + 8 * buf);
        }
      }
    }
  } else if (warp < D0) {
    if (SPLIT) {
      // ---- split warps: A row r (= TMEM lane) -> tf32 hi / lo in TMEM;
      //      B tile -> hi in place + lo twin in smem
      const int et = threadIdx.x - 64;  // 0 .. 32*NS-1
      const int q = warp & 3, r = q * 32 + lane;
      const int c0 = ((warp - 2) >> 2) * KC;  // this thread's K columns of row r: [c0, c0 + KC)
      uint32_t g = 0;
      // Gathered operand (GM): the split warps also produce it, kAhead
      // k-blocks ahead of the split, with 4-byte cp.async (zero-fill for the
      // padding) into the stage's raw tile in the TMA layout (K-major SW128),
      // arriving on the stage's full barrier — loads in flight without
      // holding registers. GM = 1: row r = pixel (lane-consecutive pixels:
      // coalesced), 32 k; GM = 2: B rows n of this CTA, lane = pixel.
      constexpr int kAhead = (GM == 1 || GM == 2) ? (C::kStages - 2 < 3 ? C::kStages - 2 : 3) : 0;
      int gu = ubase, gkb = 0;  // gather cursor: unit, k-block in unit
      uint32_t gg = 0;          // global k-block counter of the cursor
      Unit gw = unit_of(gu < nunits ? gu : 0, ep, ntn, ntm, nkb_all, BN, BMU);
      int gpb = 0, gy0 = 0, gx0 = 0;  // GM = 1: this thread's pixel in the cursor's unit
      // GM = 2: (koff, kh|kw) of the warp's B rows i = warp-2 + 4j, j = lane and lane + 32
      int gk[2] = {0, 0}, gkk[2] = {0, 0};
      auto unit_rows = [&]() {
        if (GM == 1) gather_pix(ga, gw.m0 + arow + r, gpb, gy0, gx0);
        if (GM == 2) {
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            const int i = warp - 2 + NS * (lane + 32 * h2), n = gw.n0 + brow + i;
            gather_k(ga, (i < C::kRowsB && n < ep.n) ? n : ga.kdim, gk[h2], gkk[h2]);
          }
        }
      };
      if ((GM == 1 || GM == 2) && gu < nunits) unit_rows();
      auto gather_next = [&]() {
        if (gu >= nunits) return;
        const int s2 = gg % C::kStages;
        if (gg >= (uint32_t)C::kStages) mbar_wait(empty0 + 8 * s2, ((gg / C::kStages) - 1) & 1);
        const uint32_t st2 = smem_u32(smem + s2 * C::kStageBytes);
        const float* zs = ga.src + (int64_t)gw.z * ga.sb;
        if (GM == 1) {
          int ko, kk;
          gather_k(ga, (gw.kb0 + gkb) * BK + lane, ko, kk);
          const uint32_t row = st2 + C::kOffA + r * 128;
#pragma unroll
          for (int jj = 0; jj < KC; ++jj) {
            const int j = c0 + jj;
            gather_cp(ga, zs, gpb, gy0, gx0, __shfl_sync(0xffffffffu, ko, j), __shfl_sync(0xffffffffu, kk, j),
                      row + ((((j >> 2) ^ (r & 7))) << 4) + ((j & 3) << 2));
          }
        } else {
          int pb2, y02, x02;
          gather_pix(ga, (gw.kb0 + gkb) * BK + lane, pb2, y02, x02);
          const uint32_t col = (lane & 3) << 2;
#pragma unroll
          for (int j = 0; j < C::kRowsB / NS; ++j) {
            const int i = warp - 2 + NS * j;
            const int ko = __shfl_sync(0xffffffffu, gk[j >> 5], j & 31);
            const int kk = __shfl_sync(0xffffffffu, gkk[j >> 5], j & 31);
            gather_cp(ga, zs, pb2, y02, x02, ko, kk,
                      st2 + C::kOffB + i * 128 + ((((lane >> 2) ^ (i & 7))) << 4) + col);
          }
        }
        cp_async_arrive(full0 + 8 * s2);
        ++gg;
        if (++gkb >= gw.nkb) {
          gkb = 0;
          gu += ustep;
          if (gu < nunits) {
            gw = unit_of(gu, ep, ntn, ntm, nkb_all, BN, BMU);
            unit_rows();
          }
        }
      };
      if (GM == 1 || GM == 2)
        for (int d = 0; d < kAhead; ++d) gather_next();
      for (int u = ubase; u < nunits; u += ustep) {
        const Unit w = unit_of(u, ep, ntn, ntm, nkb_all, BN, BMU);
        int hb = 0, hy0 = 0, hx0 = 0;  // GM = 3: this thread's pixel inside the unit's halo
        if (GM == 3) {
          int r_lo, r_hi, pb_unused;
          halo_rows(ga, w.m0 + arow, r_lo, r_hi);
          gather_pix(ga, w.m0 + arow + r, pb_unused, hy0, hx0);
          const int m = w.m0 + arow + r, hw = ga.MH * ga.MW;
          hb = ((r_lo * ga.SW) & 3) + ((m / hw) * ga.SH + hy0 - r_lo) * ga.SW + hx0;
        }
        for (int kb = 0; kb < w.nkb; ++kb, ++g) {
          const int s = g % C::kStages;
          if (GM == 1 || GM == 2) gather_next();  // k-block g + kAhead
          mbar_wait(full0 + 8 * s, (g / C::kStages) & 1);
          if (warp == 2 && lane == 0) TRACE(3, g);
          const uint32_t st = smem_u32(smem + s * C::kStageBytes);
          const uint32_t sa = st + C::kOffA;
          uint32_t hi[KC], lo[KC];
          if (GM == 3) {  // A row r read from the halo: lane-consecutive pixels -> consecutive words
            const int k0 = (w.kb0 + kb) * BK, c_lo = k0 / (ga.KH * ga.KW);
            int ko, kk;
            gather_k(ga, k0 + lane, ko, kk);
            if (k0 + lane < ga.kdim) {  // channel-local offset inside the halo
              const int ch = (k0 + lane) / (ga.KH * ga.KW);
              ko = (ch - c_lo) * ga.hpitch + ga.sgn * ((kk & 0xffff) * ga.SW + (kk >> 16));
            }
#pragma unroll
            for (int jj = 0; jj < KC; ++jj) {
              const int j = c0 + jj;
              const int koj = __shfl_sync(0xffffffffu, ko, j), kkj = __shfl_sync(0xffffffffu, kk, j);
              const int y = hy0 + ga.sgn * (kkj & 0xffff), x = hx0 + ga.sgn * (kkj >> 16);
              float v = 0.f;
              if ((unsigned)y < (unsigned)ga.SH && (unsigned)x < (unsigned)ga.SW)
                asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(sa + 4 * (hb + koj)));
              const float h = tf32_hi(v);
              hi[jj] = __float_as_uint(h);
              lo[jj] = __float_as_uint(__fsub_rn(v, h));
            }
          } else if (!AMN || GM == 1) {  // K-major SW128 tile: row r at r*128 B, 16-B chunk c at (c ^ r%8)
#pragma unroll
            for (int cc = 0; cc < KC / 4; ++cc) {
              const int c = c0 / 4 + cc;
              const float4 x = lds4(sa + r * 128 + ((c ^ (r & 7)) << 4));
              const float xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float h = tf32_hi(xs[e]);
                hi[4 * cc + e] = __float_as_uint(h);
                lo[4 * cc + e] = __float_as_uint(__fsub_rn(xs[e], h));
              }
            }
          } else {  // MN-major SW128 boxes of 32(M) x 32(K): 4 KB per box, 16-B chunk (m%32)/4 ^ k%8
            const uint32_t base = sa + (r >> 5) * 4096 + ((r & 3) << 2);
            const int c4 = (r & 31) >> 2;
#pragma unroll
            for (int kk2 = 0; kk2 < KC; ++kk2) {
              const int k = c0 + kk2;
              float x;
              asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x) : "r"(base + k * 128 + ((c4 ^ (k & 7)) << 4)));
              const float h = tf32_hi(x);
              hi[kk2] = __float_as_uint(h);
              lo[kk2] = __float_as_uint(__fsub_rn(x, h));
            }
          }
          // TMEM A slot g % kASlots: free once the MMAs of k-block g - kASlots
          // retired (their commit completes that k-block's smem-stage phase)
          if (C::kASlots < C::kStages && g >= (uint32_t)C::kASlots) {
            const uint32_t gp = g - C::kASlots;
            mbar_wait(empty0 + 8 * (gp % C::kStages), (gp / C::kStages) & 1);
            tc_fence_after();
          }
          const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + C::kACol0 + (g % C::kASlots) * 64;
#ifndef ESGD_X_NOAST
          if constexpr (KC == 32) {
            tmem_st32(ta, *reinterpret_cast<const uint32_t(*)[32]>(hi));
            tmem_st32(ta + 32, *reinterpret_cast<const uint32_t(*)[32]>(lo));
          } else {
            tmem_st16(ta + c0, hi);
            tmem_st16(ta + 32 + c0, lo);
          }
#endif
          // every split thread has read its A row: B lo may overwrite the tile
          named_bar_sync(3, 32 * NS);
#ifndef ESGD_X_NOSPLITB
          {
            split_tile<C::kTileBytesB, 32 * NS>(st + C::kOffB, st + C::kOffBLo, et);
          }
#endif
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (PAIR) mbar_arrive_leader(split0 + 8 * s);
            else mbar_arrive(split0 + 8 * s);
          }
          if (warp == 2 && lane == 0) TRACE(4, g);
        }
      }
    }
  } else {
    // ---- drain + epilogue warps 6..13: warp w owns TMEM lanes 32*(w%4)..+31
    // and columns [h*BN/2, (h+1)*BN/2) of each tile, h = (w-6)/4. Each
    // K-chunk's TMEM partial is added into fp32 registers with round-to-
    // nearest adds (promotion): the tensor-core accumulator only ever sums
    // kChunkKB*32 products, which keeps the long-K error fp32-grade. Two warps
    // per lane quadrant halve the registers per thread, so a 32-column slab is
    // loaded per TMEM wait (the drain is bound by the TMEM load latency).
    constexpr int HB = BN / 2;  // columns per drain warp
    const int q = warp & 3, h = (warp - D0) >> 2;
    const int issuer = 32 * D0 + h * 128;  // lane 0 of the first drain warp of each half: bulk-store issue
    uint32_t c = 0;
    for (int u = ubase; u < nunits; u += ustep) {
      const Unit w = unit_of(u, ep, ntn, ntm, nkb_all, BN, BMU);
      float racc[HB];
#pragma unroll
      for (int j = 0; j < HB; ++j) racc[j] = 0.f;
      for (int kc = 0; kc < w.nkb; kc += kChunkKB, ++c) {
        const int buf = c % C::kAccBufs;
        mbar_wait(afull0 + 8 * buf, (c / C::kAccBufs) & 1);
        if (warp == D0 && lane == 0) TRACE(5, c);
        tc_fence_after();
#ifndef ESGD_X_NODRAIN
        if (HB <= 64 && NS == 4) {  // (the 8-split-warp CTA keeps 96 registers: 16-column loads)
#pragma unroll
          for (int c0 = 0; c0 < HB; c0 += 32) {
            uint32_t v[32];
            tmem_ld32_nowait(tmem + ((uint32_t)(q * 32) << 16) + buf * BN + h * HB + c0, v);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 32; ++j) racc[c0 + j] = __fadd_rn(racc[c0 + j], __uint_as_float(v[j]));
          }
        } else {  // BN = 192 (96 accumulators per thread), or the 8-split-warp CTA at 96 registers: 16-column loads
#pragma unroll
          for (int c0 = 0; c0 < HB; c0 += 16) {
            float v[16];
            tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + buf * BN + h * HB + c0, v);
#pragma unroll
            for (int j = 0; j < 16; ++j) racc[c0 + j] = __fadd_rn(racc[c0 + j], v[j]);
          }
        }
#endif
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (PAIR) mbar_arrive_leader(aempty0 + 8 * buf);
          else mbar_arrive(aempty0 + 8 * buf);
        }
        if (warp == D0 && lane == 0) TRACE(6, c);
      }
      const int m0 = w.m0 + arow;  // this CTA's rows of the unit
      const int row = m0 + q * 32 + lane;
      const int n0 = w.n0 + h * HB;  // first column of this warp's half
#ifdef ESGD_X_NOEPI
      if (row == -1) {
#else
      if (ep.splits > 1) {
#endif  // raw partial of this K slice; k_tc_reduce applies the epilogue
        if (row < ep.m) {
          float* P = ep.ws + ((int64_t)w.z * ep.splits + w.slice) * ep.m * ep.n + (int64_t)row * ep.n;
#pragma unroll
          for (int j = 0; j < HB; ++j)
            if (n0 + j < ep.n) P[n0 + j] = racc[j];
        }
      } else {
        // 32 columns (16 KB) at a time through this half's 16 KB smem slot;
        // the two halves stage and store concurrently. The register->smem
        // staging is the only unrolled code (one variant per layout; the fast
        // variant fuses bias + relu); the general epilogue (mask/tanh/sigmoid,
        // or accumulate / strided direct stores in mode 0) is a rolled pass
        // over the thread's own staged row, so the kernel's code stays small
        // enough for the instruction cache (an unrolled general epilogue
        // measured 26% of warp samples in no_instruction stalls).
        const uint32_t sb = smem_u32(stage_out) + h * 16384;
        const bool fast = ep.mask == nullptr && (ep.act == ESGD_ACT_NONE || ep.act == ESGD_ACT_RELU) &&
                          ep.out_mode != 0;
        const bool relu = ep.act == ESGD_ACT_RELU;
        const float* bz = ep.bias ? ep.bias + w.z * ep.bias_sb : nullptr;
        const int r = q * 32 + lane;
#pragma unroll
        for (int lq = 0; lq < HB / 32; ++lq) {
          const int col0 = n0 + lq * 32;
          // slot free? (this half's previous bulk store has read it)
          if (threadIdx.x == issuer) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          named_bar_sync(1 + h, 128);
          if (ep.out_mode == 2) {
            if (fast) stage_quarter<HB, 2, true>(racc, lq, sb, r, bz, relu, col0, ep.n);
            else stage_quarter<HB, 2, false>(racc, lq, sb, r, bz, relu, col0, ep.n);
          } else {
            if (fast) stage_quarter<HB, 1, true>(racc, lq, sb, r, bz, relu, col0, ep.n);
            else stage_quarter<HB, 1, false>(racc, lq, sb, r, bz, relu, col0, ep.n);
          }
          if (!fast) general_quarter(ep, sb, r, row, w.z, col0);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          named_bar_sync(1 + h, 128);
          if (threadIdx.x == issuer && ep.out_mode != 0) {
            if (ep.out_mode == 1)
              asm volatile(
                  "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                      reinterpret_cast<uint64_t>(&map_c)),
                  "r"(m0), "r"(col0), "r"(w.z), "r"(sb)
                  : "memory");
            else
              asm volatile(
                  "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                      reinterpret_cast<uint64_t>(&map_c)),
                  "r"(col0), "r"(m0), "r"(w.z), "r"(sb)
                  : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        }
      }
    }
    if ((ep.out_mode == 1 || ep.out_mode == 2) && threadIdx.x == issuer)
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  tc_fence_before();
  if (PAIR) cluster_sync_all();  // the peer's remote arrives / the leader's commits are done
  else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::kTmemCols));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::kTmemCols));
  }
}

// combine split-K partials in slice order (deterministic), then the epilogue
__global__ void __launch_bounds__(256) k_tc_reduce(Epi ep) {
  const int64_t mn = (int64_t)ep.m * ep.n;
  const int z = blockIdx.y;
  float* cz = ep.c + z * ep.c_sb;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < mn; e += (int64_t)gridDim.x * blockDim.x) {
    const float* P = ep.ws + (int64_t)z * ep.splits * mn + e;
    float v0 = 0.f, v1 = 0.f, v2 = 0.f, v3 = 0.f;
    int s = 0;
    for (; s + 3 < ep.splits; s += 4) {
      v0 = __fadd_rn(v0, P[s * mn]); v1 = __fadd_rn(v1, P[(s + 1) * mn]);
      v2 = __fadd_rn(v2, P[(s + 2) * mn]); v3 = __fadd_rn(v3, P[(s + 3) * mn]);
    }
    for (; s < ep.splits; ++s) v0 = __fadd_rn(v0, P[s * mn]);
    const int row = (int)(e / ep.n), col = (int)(e % ep.n);
    const int64_t off = (int64_t)row * ep.c_sm + (int64_t)col * ep.c_sn;
    cz[off] = epi_apply(ep, __fadd_rn(__fadd_rn(v0, v1), __fadd_rn(v2, v3)), z, row, col, off, cz);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

typedef CUresult (*PFN_encodeIm2col)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                     const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t,
                                     const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                     CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
PFN_encodeIm2col get_encode_im2col() {
  static PFN_encodeIm2col fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeIm2col>(p);
  }
  return fn;
}

// im2col map over an NHWC source (c innermost) of nimg images, for GM = 4 /
// 5: boxes of `pixels` traversal positions x 32 channels. The traversal box
// per image runs from lower = (xoff, yoff) = -pad to (SW - 1, SH - 1) + upper,
// upper = pad - (K - 1), in steps of the conv stride — the output grid
// (CUTLASS make_im2col_tma_copy_desc uses the same corners).
int make_im2col_map(CUtensorMap* map, const Gather& g, int64_t nimg, int pixels, bool atom32) {
  auto enc = get_encode_im2col();
  ESGD_REQUIRE(enc, ESGD_ERR_CUDA, "tc_conv_tma: cuTensorMapEncodeIm2col unavailable");
  const int cin = g.kdim / (g.KH * g.KW);
  cuuint64_t dims[4] = {(cuuint64_t)cin, (cuuint64_t)g.SW, (cuuint64_t)g.SH, (cuuint64_t)nimg};
  cuuint64_t strides[3] = {(cuuint64_t)cin * 4, (cuuint64_t)g.SW * cin * 4, (cuuint64_t)g.SH * g.SW * cin * 4};
  int lower[2] = {g.xoff, g.yoff};
  int upper[2] = {-g.xoff - (g.KW - 1), -g.yoff - (g.KH - 1)};
  cuuint32_t estr[4] = {1, (cuuint32_t)g.stride, (cuuint32_t)g.stride, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(g.src), dims, strides, lower, upper,
                   32, (cuuint32_t)pixels, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   atom32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  ESGD_REQUIRE(r == CUDA_SUCCESS, ESGD_ERR_CUDA, "tc_conv_tma: cuTensorMapEncodeIm2col failed (%d)", (int)r);
  // drivers <= 13.1 encode a bit that breaks im2col loads from tensors under
  // 128 KB (CUTLASS clears it the same way)
  int drv = 0;
  if (cudaDriverGetVersion(&drv) == cudaSuccess && drv <= 13010 && (int64_t)nimg * strides[2] < 131072)
    reinterpret_cast<uint64_t*>(map)[1] &= ~(1ull << 21);
  return ESGD_OK;
}

// 3-D map over an operand. K-major: dims (k, rows, batch), box (32, box_rows, 1).
// MN-major: dims (rows, k, batch) with rows contiguous, box (32, 32, 1).
int make_map(CUtensorMap* map, const float* base, int64_t k, int64_t rows, int64_t ld,
             int64_t batch, int64_t sb, int box_rows, bool mn_major, bool atom32 = true) {
  auto enc = get_encode();
  ESGD_REQUIRE(enc, ESGD_ERR_CUDA, "tc_gemm: cuTensorMapEncodeTiled unavailable");
  const int64_t inner = mn_major ? rows : k, outer = mn_major ? k : rows;
  cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)outer, (cuuint64_t)batch};
  int64_t bstride = batch > 1 ? sb : ld * outer;
  bstride = (bstride + 3) & ~int64_t(3);
  cuuint64_t strides[2] = {(cuuint64_t)(ld * 4), (cuuint64_t)(bstride * 4)};
  cuuint32_t box[3] = {32, (cuuint32_t)(mn_major ? BK : box_rows), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   (mn_major && atom32) ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  ESGD_REQUIRE(r == CUDA_SUCCESS, ESGD_ERR_CUDA, "tc_gemm: cuTensorMapEncodeTiled failed (%d)", (int)r);
  return ESGD_OK;
}

// N tile width. 192-wide tiles (3 smem stages, 2 TMEM A slots) read the
// TS-mode A operand from TMEM once per 192 instead of 128 output columns, so
// they win wherever they add little padding and there are enough M tiles to
// fill the SMs (measured: conv2 fwd N=192 0.34 -> 0.25 ms, conv3 fwd N=384
// 0.154 -> 0.143, conv4 dgrad N=3456 0.201 -> 0.189); with a single M tile
// (the FC layers, M = batch) 128 stays faster.
inline int64_t padded(int64_t n, int bn) { return ((n + bn - 1) / bn) * bn; }
inline int pick_bn(int64_t m, int64_t n, bool split) {
  static const int force = getenv("ESGD_TC_BN") ? atoi(getenv("ESGD_TC_BN")) : 0;  // tuning runs
  if (force == 64 || force == 128 || (force == 192 && split)) return force;
  if (n <= 64) return 64;
  if (!split) return 128;
  if (padded(n, 192) < padded(n, 128)) return 192;
  // with >= 16 M tiles 192 also wins at up to ~4% more padding: conv2's data
  // gradient (N = 1600: 1728 vs 1664 columns) 0.338 -> 0.318 ms, because A is
  // loaded and split once per 192 instead of 128 output columns (the FC weight
  // gradients at N = 4096 are neutral)
  return (padded(n, 192) * 100 <= padded(n, 128) * 104 && m >= 16 * BM) ? 192 : 128;
}
// CTA-pair mode (cta_group::2, 256-row units) for the 3xTF32 path when M has
// enough rows that 256-row tiles add little padding (ESGD_TC_PAIR=0/1 forces
// it off / on for tuning runs)
inline bool use_pair(int64_t m, bool split) {
  static const int force = getenv("ESGD_TC_PAIR") ? atoi(getenv("ESGD_TC_PAIR")) : -1;
  if (!split || m <= BM) return false;
  if (force >= 0) return force == 1;
  return m >= 8 * 256 && padded(m, 256) * 8 <= padded(m, BM) * 9;
}
// padded MMA area of an orientation (M tiled by 128 or 256, N by the chosen width)
inline int64_t padded_cost(int64_t m, int64_t n, bool split) {
  return padded(m, use_pair(m, split) ? 2 * BM : BM) * padded(n, pick_bn(m, n, split));
}

// Launch plan of one GEMM: orientation (C^T = B.A^T when it needs less padded
// tensor-core work), tile width and K split.
struct Plan {
  esgd_tc_gemm_desc d;  // the oriented problem
  int bn, splits, kbps;
  bool pair;            // cta_group::2, 256-row units
};

inline Plan make_plan(const esgd_tc_gemm_desc* d0, bool allow_swap = true) {
  Plan p;
  p.d = *d0;
  const bool split = d0->precision == 3;
  // Orientation: C^T = B . A^T is the same GEMM with the operands' roles
  // swapped; take it when it needs less padded tensor-core work (M is tiled
  // by 128: a 64- or 192-row M wastes half / a quarter of every MMA). Only
  // without a per-column bias (the epilogue applies bias along N).
  static const int force_swap = getenv("ESGD_TC_SWAP") ? atoi(getenv("ESGD_TC_SWAP")) : -1;  // tuning runs
  const bool swap = force_swap >= 0 ? force_swap == 1
                                    : padded_cost(d0->n, d0->m, split) < padded_cost(d0->m, d0->n, split);
  if (allow_swap && !d0->bias && swap) {
    esgd_tc_gemm_desc& sw = p.d;
    sw.m = d0->n; sw.n = d0->m;
    sw.a = d0->b; sw.lda = d0->ldb; sw.a_sb = d0->b_sb; sw.a_major = d0->b_major;
    sw.b = d0->a; sw.ldb = d0->lda; sw.b_sb = d0->a_sb; sw.b_major = d0->a_major;
    sw.c_sm = d0->c_sn; sw.c_sn = d0->c_sm;
    sw.mask_sm = d0->mask_sn; sw.mask_sn = d0->mask_sm;
  }
  const esgd_tc_gemm_desc* d = &p.d;
  p.bn = pick_bn(d->m, d->n, split);
  p.pair = use_pair(d->m, split);
  const int bmu = p.pair ? 2 * BM : BM, units_per_wave = p.pair ? kNumSMs / 2 : kNumSMs;
  const int nkb = (d->k + BK - 1) / BK;
  // The K split depends on the per-replica problem only, never on `batch` or
  // on the workspace size: a replica computes bit-identical results however
  // many replicas share the launch, so runs are reproducible across GPU
  // counts. Split when the output tiles cannot fill the 148 SMs (weight
  // gradients reduce over every pixel of the batch): ~1 wave, >= 2 chunks per
  // slice (2 waves: conv2.wgrad 0.30 vs 0.28 ms and a ~2% slower round - twice
  // the partials for k_tc_reduce; 3-4 far worse). A NULL workspace means "do
  // not split"; a workspace that is too small is an error (esgd_tc_gemm_f32
  // returns ESGD_ERR_UNSUPPORTED; size it with esgd_tc_gemm_ws_floats).
  const int tiles_z = ((d->n + p.bn - 1) / p.bn) * ((d->m + bmu - 1) / bmu);
  int splits = 1;
  if (d->ws && tiles_z < units_per_wave && nkb >= 2 * kChunkKB) {
    splits = (ESGD_SPLIT_WAVES * units_per_wave) / tiles_z;
    splits = std::min(splits, nkb / (2 * kChunkKB));
    splits = std::min(splits, 128);
    if (splits < 1) splits = 1;
  }
  int kbps = (nkb + splits - 1) / splits;
  kbps = (kbps + kChunkKB - 1) / kChunkKB * kChunkKB;
  p.splits = (nkb + kbps - 1) / kbps;
  p.kbps = kbps;
  return p;
}

inline int64_t ws_need(const Plan& p) {
  return p.splits > 1 ? (int64_t)p.splits * p.d.m * p.d.n * p.d.batch : 0;
}

template <int BN, bool SPLIT, bool AMN, bool BMN, bool PAIR, int GM = 0>
int launch(const Plan& p, cudaStream_t st, const Gather& ga = Gather{}) {
  using C = Cfg<BN, SPLIT, PAIR>;
  constexpr int BMU = PAIR ? 2 * BM : BM;
  const esgd_tc_gemm_desc* d = &p.d;
  // per-device attribute; cheap, and legal while a stream is being captured
  cudaError_t e = cudaFuncSetAttribute(k_tc_gemm<BN, SPLIT, AMN, BMN, PAIR, GM>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
  ESGD_REQUIRE(e == cudaSuccess, ESGD_ERR_CUDA, "tc_gemm: smem attribute: %s", cudaGetErrorString(e));
  CUtensorMap ma, mb;
  // 3xTF32: A is read by the split warps (not by UMMA), plain 128B swizzle
  memset(&ma, 0, sizeof(ma));
  memset(&mb, 0, sizeof(mb));
  int rc = ESGD_OK;
  const int64_t nimg_all = (int64_t)(ga.npix / std::max(1, ga.MH * ga.MW)) * d->batch;
  if (GM == 0 || GM == 2 || GM == 5) {  // (a gathered operand has no tensor map)
    rc = make_map(&ma, d->a, d->k, d->m, d->lda, d->batch, d->a_sb, BM, AMN, /*atom32=*/!SPLIT);
    if (rc) return rc;
  }
  if (GM == 4) {
    rc = make_im2col_map(&ma, ga, nimg_all, BM, /*atom32=*/false);
    if (rc) return rc;
  }
  if (GM == 5) {
    rc = make_im2col_map(&mb, ga, nimg_all, 32, /*atom32=*/true);
    if (rc) return rc;
  }
  if (GM != 2 && GM != 5) {
    rc = make_map(&mb, d->b, d->k, d->n, d->ldb, d->batch, d->b_sb, C::kRowsB, BMN);
    if (rc) return rc;
  }
  const int splits = p.splits, kbps = p.kbps;
  const int tiles = ((d->n + BN - 1) / BN) * ((d->m + BMU - 1) / BMU) * d->batch;
  // output: TMA store when one C stride is unit and the other 16-B aligned
  int out_mode = 0;
  CUtensorMap mc;
  memset(&mc, 0, sizeof(mc));
  if (splits == 1 && !d->accumulate && aligned16(d->c) && (d->batch == 1 || (d->c_sb & 3) == 0)) {
    if (d->c_sm == 1 && (d->c_sn & 3) == 0 && d->c_sn >= d->m) out_mode = 1;
    else if (d->c_sn == 1 && (d->c_sm & 3) == 0 && d->c_sm >= d->n) out_mode = 2;
  }
  if (out_mode) {
    auto enc = get_encode();
    const bool mcont = out_mode == 1;
    const int64_t inner = mcont ? d->m : d->n, outer = mcont ? d->n : d->m;
    const int64_t ld = mcont ? d->c_sn : d->c_sm;
    int64_t bstride = d->batch > 1 ? d->c_sb : ld * outer;
    bstride = (bstride + 3) & ~int64_t(3);
    cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)outer, (cuuint64_t)d->batch};
    cuuint64_t strides[2] = {(cuuint64_t)(ld * 4), (cuuint64_t)(bstride * 4)};
    cuuint32_t box[3] = {mcont ? 128u : 32u, mcont ? 32u : 128u, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(&mc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d->c, dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, mcont ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) out_mode = 0;
  }
  const int m_fast = 0;  // (measured: m-fastest rasterisation was slower on every shape)
  Epi ep{d->c, d->c_sm, d->c_sn, d->c_sb, d->bias, d->bias_sb, d->mask, d->mask_sm, d->mask_sn,
         d->mask_sb, d->act, d->accumulate, d->m, d->n, d->k, d->ws, splits, kbps, d->batch, out_mode,
         m_fast};
  // persistent: one CTA per SM (smem-limited), units dealt round-robin (to
  // CTA pairs in PAIR mode: clusters of 2 on one TPC)
  const int64_t units = (int64_t)tiles * splits;
  if (PAIR) {
    const int pairs = (int)std::min<int64_t>(units, (kNumSMs - sm_reserve()) / 2);
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof(cfg));
    cfg.gridDim = dim3(2 * pairs);
    cfg.blockDim = dim3(cta_threads(BN, SPLIT));
    cfg.dynamicSmemBytes = C::kSmemBytes;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, k_tc_gemm<BN, SPLIT, AMN, BMN, true, GM>, ma, mb, mc, ep, ga);
    ESGD_REQUIRE(e == cudaSuccess, ESGD_ERR_CUDA, "tc_gemm: cluster launch: %s", cudaGetErrorString(e));
  } else {
    const int grid = (int)std::min<int64_t>(units, kNumSMs - sm_reserve());
    k_tc_gemm<BN, SPLIT, AMN, BMN, false, GM><<<grid, cta_threads(BN, SPLIT), C::kSmemBytes, st>>>(ma, mb, mc, ep, ga);
  }
  if (splits > 1) {
    dim3 rg(stride_grid((int64_t)d->m * d->n, 256, 8), d->batch);
    k_tc_reduce<<<rg, 256, 0, st>>>(ep);
  }
  return check_launch("esgd_tc_gemm_f32");
}

template <int BN, bool SPLIT, bool PAIR>
int launch_major(const Plan& p, cudaStream_t st) {
  const esgd_tc_gemm_desc* d = &p.d;
  if (d->a_major)
    return d->b_major ? launch<BN, SPLIT, true, true, PAIR>(p, st) : launch<BN, SPLIT, true, false, PAIR>(p, st);
  return d->b_major ? launch<BN, SPLIT, false, true, PAIR>(p, st) : launch<BN, SPLIT, false, false, PAIR>(p, st);
}
template <int BN>
int launch_split(const Plan& p, cudaStream_t st) {
  return p.pair ? launch_major<BN, true, true>(p, st) : launch_major<BN, true, false>(p, st);
}
// implicit-GEMM convolutions: GM = 1 gathers A (K-major B), GM = 2 gathers B (K-major A),
// GM = 3 reads A from a per-k-block halo of source rows
template <int BN, int GM>
int launch_gather(const Plan& p, cudaStream_t st, const Gather& ga) {
  return p.pair ? launch<BN, true, false, false, true, GM>(p, st, ga) : launch<BN, true, false, false, false, GM>(p, st, ga);
}

// TMA-im2col convolutions: GM = 4 loads A (K-major B), GM = 5 loads B (MN-major; K-major A)
template <int BN, int GM>
int launch_im2col(const Plan& p, cudaStream_t st, const Gather& ga) {
  if (GM == 5)
    return p.pair ? launch<BN, true, false, true, true, 5>(p, st, ga) : launch<BN, true, false, true, false, 5>(p, st, ga);
  return p.pair ? launch<BN, true, false, false, true, 4>(p, st, ga) : launch<BN, true, false, false, false, 4>(p, st, ga);
}

int validate(const esgd_tc_gemm_desc* d) {
  ESGD_REQUIRE(d, ESGD_ERR_INPUT, "tc_gemm: null descriptor");
  ESGD_REQUIRE(d->m >= 0 && d->n >= 0 && d->k >= 0 && d->batch >= 0, ESGD_ERR_SHAPE,
               "tc_gemm shape mismatch: m=%d n=%d k=%d", d->m, d->n, d->k);
  ESGD_REQUIRE(d->precision == 1 || d->precision == 3, ESGD_ERR_INPUT,
               "tc_gemm: precision must be 1 (tf32) or 3 (3xtf32)");
  ESGD_REQUIRE(d->act >= 0 && d->act <= 3, ESGD_ERR_INPUT, "tc_gemm: unknown activation");
  return ESGD_OK;
}

}  // namespace tc
}  // namespace esgd

extern "C" int esgd_tc_gemm_ws_floats(const esgd_tc_gemm_desc* d, int64_t* floats) {
  using namespace esgd;
  ESGD_REQUIRE(floats, ESGD_ERR_INPUT, "tc_gemm_ws_floats: null output");
  *floats = 0;
  if (int rc = tc::validate(d)) return rc;
  if (d->m == 0 || d->n == 0 || d->batch == 0 || d->k == 0) return ESGD_OK;
  esgd_tc_gemm_desc q = *d;
  if (!q.ws) q.ws = reinterpret_cast<float*>(uintptr_t(256));  // ask: how much would it use
  *floats = tc::ws_need(tc::make_plan(&q));
  return ESGD_OK;
}

extern "C" int esgd_tc_gemm_f32(const esgd_tc_gemm_desc* d, esgd_stream_t stream) {
  using namespace esgd;
  if (int rc = tc::validate(d)) return rc;
  if (d->m == 0 || d->n == 0 || d->batch == 0) return ESGD_OK;
  ESGD_REQUIRE(d->k >= 1 && d->a && d->b && d->c, ESGD_ERR_INPUT, "tc_gemm: null operand");
  ESGD_REQUIRE(d->lda >= (d->a_major ? d->m : d->k) && d->ldb >= (d->b_major ? d->n : d->k) &&
                   (d->lda & 3) == 0 && (d->ldb & 3) == 0,
               ESGD_ERR_SHAPE, "tc_gemm: lda/ldb must cover the contiguous dim and be multiples of 4 (TMA 16-B strides)");
  ESGD_REQUIRE(aligned16(d->a) && aligned16(d->b), ESGD_ERR_INPUT, "tc_gemm: A/B must be 16-B aligned");
  ESGD_REQUIRE(d->batch == 1 || ((d->a_sb & 3) == 0 && (d->b_sb & 3) == 0), ESGD_ERR_SHAPE,
               "tc_gemm: batch strides must be multiples of 4");
  ESGD_REQUIRE((int64_t)((d->m + tc::BM - 1) / tc::BM) * ((d->n + 63) / 64) * d->batch < (int64_t(1) << 30),
               ESGD_ERR_UNSUPPORTED, "tc_gemm: too many tiles");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const bool split = d->precision == 3;
  const tc::Plan p = tc::make_plan(d);
  const int64_t need = tc::ws_need(p);
  ESGD_REQUIRE(need <= d->ws_floats, ESGD_ERR_UNSUPPORTED,
               "tc_gemm: split-K workspace too small (need %lld floats, have %lld; size it with "
               "esgd_tc_gemm_ws_floats)", (long long)need, (long long)d->ws_floats);
  if (p.bn == 64) return split ? tc::launch_split<64>(p, st) : tc::launch_major<64, false, false>(p, st);
  if (p.bn == 192) return tc::launch_split<192>(p, st);
  return split ? tc::launch_split<128>(p, st) : tc::launch_major<128, false, false>(p, st);
}

extern "C" int esgd_tc_conv_f32(const esgd_tc_gemm_desc* d, const esgd_conv_gather* cg, int32_t side,
                                esgd_stream_t stream) {
  using namespace esgd;
  if (int rc = tc::validate(d)) return rc;
  ESGD_REQUIRE(cg && (side == 1 || side == 2), ESGD_ERR_INPUT, "tc_conv: gather descriptor and side 1|2 required");
  ESGD_REQUIRE(d->precision == 3, ESGD_ERR_UNSUPPORTED, "tc_conv: 3xTF32 only");
  if (d->m == 0 || d->n == 0 || d->batch == 0) return ESGD_OK;
  const int64_t kdim = (int64_t)cg->channels * cg->kh * cg->kw;
  ESGD_REQUIRE(cg->src && cg->kh >= 1 && cg->kw >= 1 && cg->channels >= 1 && cg->stride >= 1 &&
                   (cg->sgn == 1 || cg->sgn == -1) && cg->src_h >= 1 && cg->src_w >= 1 && cg->grid_h >= 1 &&
                   cg->grid_w >= 1 && cg->npix >= 1 && cg->npix % (cg->grid_h * cg->grid_w) == 0 &&
                   cg->img_stride >= 0,
               ESGD_ERR_INPUT, "tc_conv: bad gather geometry");
  if ((cg->img_stride == 0 || cg->img_stride == cg->src_h * cg->src_w) && cg->channels > 1)  // CNHW planes
    ESGD_REQUIRE((int64_t)cg->plane >= (int64_t)(cg->npix / (cg->grid_h * cg->grid_w)) * cg->src_h * cg->src_w,
                 ESGD_ERR_INPUT, "tc_conv: channel plane shorter than its images");
  ESGD_REQUIRE((int64_t)cg->plane * cg->channels < (int64_t(1) << 31) && kdim < (int64_t(1) << 30),
               ESGD_ERR_UNSUPPORTED, "tc_conv: source tensor too large for 32-bit offsets");
  if (side == 1) {
    ESGD_REQUIRE(d->m == cg->npix && d->k == kdim, ESGD_ERR_SHAPE,
                 "tc_conv: gathered A is npix x channels*kh*kw (m=%d k=%d vs %d x %lld)", d->m, d->k, cg->npix,
                 (long long)kdim);
    ESGD_REQUIRE(d->b && d->b_major == 0 && (d->ldb & 3) == 0 && d->ldb >= d->k && aligned16(d->b),
                 ESGD_ERR_SHAPE, "tc_conv: B must be K-major with a 16-B aligned pitch");
  } else {
    ESGD_REQUIRE(d->n == kdim && d->k == cg->npix, ESGD_ERR_SHAPE,
                 "tc_conv: gathered B is channels*kh*kw x npix (n=%d k=%d vs %lld x %d)", d->n, d->k,
                 (long long)kdim, cg->npix);
    ESGD_REQUIRE(d->a && d->a_major == 0 && (d->lda & 3) == 0 && d->lda >= d->k && aligned16(d->a),
                 ESGD_ERR_SHAPE, "tc_conv: A must be K-major with a 16-B aligned pitch");
  }
  ESGD_REQUIRE(d->c, ESGD_ERR_INPUT, "tc_conv: null output");
  ESGD_REQUIRE(d->batch == 1 || ((d->a_sb & 3) == 0 && (d->b_sb & 3) == 0), ESGD_ERR_SHAPE,
               "tc_conv: batch strides must be multiples of 4");
  const int nstride = cg->img_stride ? cg->img_stride : cg->src_h * cg->src_w;
  // a single-channel source: its "plane" (the halo copies' bound) is all its images
  const int plane = (cg->channels == 1 && nstride == cg->src_h * cg->src_w)
                        ? ((cg->npix / (cg->grid_h * cg->grid_w)) * cg->src_h * cg->src_w + 3) & ~3
                        : cg->plane;
  tc::Gather ga{cg->src, cg->src_sb, plane, nstride, cg->src_h, cg->src_w, cg->grid_h, cg->grid_w,
                cg->stride, cg->yoff, cg->xoff, cg->sgn, cg->kh, cg->kw, cg->npix, (int)kdim, 0};
  // side 1: the source rows of each 128-pixel tile staged once per k-block as
  // a halo (one bulk copy per channel the k-block touches) when they fit in
  // the A tile's 16 KB — the split warps then read A from shared memory;
  // otherwise (AlexNet conv1's 224-wide rows) per-element cp.async gathers
  bool halo = false;
  if (side == 1 && nstride == cg->src_h * cg->src_w && !getenv("ESGD_NO_HALO")) {  // (CNHW planes)
    const int hw = cg->grid_h * cg->grid_w, reach = cg->sgn * (cg->kh - 1);
    const int nimg = cg->npix / hw;
    int64_t lmax = 0;
    for (int m0 = 0; m0 < cg->npix; m0 += tc::BM) {
      const int last = std::min(m0 + tc::BM, cg->npix) - 1;
      const int n0 = m0 / hw, y0 = ((m0 - n0 * hw) / cg->grid_w) * cg->stride + cg->yoff;
      const int n1 = last / hw, y1 = ((last - n1 * hw) / cg->grid_w) * cg->stride + cg->yoff;
      const int r_lo = std::max(0, n0 * cg->src_h + y0 + std::min(0, reach));
      const int r_hi = std::min(nimg * cg->src_h - 1, n1 * cg->src_h + y1 + std::max(0, reach));
      const int64_t e0 = (int64_t)r_lo * cg->src_w;
      const int64_t len = (e0 - (e0 & ~int64_t(3)) + (int64_t)(r_hi - r_lo + 1) * cg->src_w + 3) & ~int64_t(3);
      lmax = std::max(lmax, len);
    }
    const int kk = cg->kh * cg->kw;
    const int hchan = (tc::BK - 1) / kk + 2;
    ga.hpitch = (int)((lmax + 3) & ~int64_t(3));
    halo = (int64_t)hchan * ga.hpitch * 4 <= tc::kTileBytesA;
  }
  const tc::Plan p = tc::make_plan(d, /*allow_swap=*/false);
  const int64_t need = tc::ws_need(p);
  ESGD_REQUIRE(need <= d->ws_floats, ESGD_ERR_UNSUPPORTED,
               "tc_conv: split-K workspace too small (need %lld floats, have %lld; size it with "
               "esgd_tc_conv_ws_floats)", (long long)need, (long long)d->ws_floats);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (side == 1 && halo) {
    if (p.bn == 64) return tc::launch_gather<64, 3>(p, st, ga);
    if (p.bn == 192) return tc::launch_gather<192, 3>(p, st, ga);
    return tc::launch_gather<128, 3>(p, st, ga);
  }
  if (side == 1) {
    if (p.bn == 64) return tc::launch_gather<64, 1>(p, st, ga);
    if (p.bn == 192) return tc::launch_gather<192, 1>(p, st, ga);
    return tc::launch_gather<128, 1>(p, st, ga);
  }
  if (p.bn == 64) return tc::launch_gather<64, 2>(p, st, ga);
  if (p.bn == 192) return tc::launch_gather<192, 2>(p, st, ga);
  return tc::launch_gather<128, 2>(p, st, ga);
}

extern "C" int esgd_tc_conv_tma_f32(const esgd_tc_gemm_desc* d, const esgd_conv_gather* cg, int32_t side,
                                    esgd_stream_t stream) {
  using namespace esgd;
  if (int rc = tc::validate(d)) return rc;
  ESGD_REQUIRE(cg && (side == 1 || side == 2), ESGD_ERR_INPUT, "tc_conv_tma: gather descriptor and side 1|2 required");
  ESGD_REQUIRE(d->precision == 3, ESGD_ERR_UNSUPPORTED, "tc_conv_tma: 3xTF32 only");
  if (d->m == 0 || d->n == 0 || d->batch == 0) return ESGD_OK;
  const int64_t kdim = (int64_t)cg->channels * cg->kh * cg->kw;
  const int hw = cg->grid_h * cg->grid_w;
  ESGD_REQUIRE(cg->src && cg->kh >= 1 && cg->kw >= 1 && cg->stride >= 1 && cg->stride <= 8 && cg->sgn == 1 &&
                   cg->src_h >= 1 && cg->src_w >= 1 && hw >= 1 && cg->npix >= 1 && cg->npix % hw == 0 &&
                   aligned16(cg->src),
               ESGD_ERR_INPUT, "tc_conv_tma: bad gather geometry");
  ESGD_REQUIRE(cg->channels % 32 == 0, ESGD_ERR_UNSUPPORTED,
               "tc_conv_tma: channels must be a multiple of 32 (one k-block = 32 channels of one tap)");
  // the traversal grid the map's corners define must be the conv's output grid
  const int gw = (cg->src_w - 2 * cg->xoff - cg->kw) / cg->stride + 1;
  const int gh = (cg->src_h - 2 * cg->yoff - cg->kh) / cg->stride + 1;
  ESGD_REQUIRE(cg->xoff <= 0 && cg->yoff <= 0 && -cg->xoff < cg->kw && -cg->yoff < cg->kh && gw == cg->grid_w &&
                   gh == cg->grid_h && cg->kw <= 128 && cg->kh <= 128,
               ESGD_ERR_SHAPE, "tc_conv_tma: grid %dx%d is not the window's output grid %dx%d", cg->grid_h,
               cg->grid_w, gh, gw);
  const int64_t nimg = cg->npix / hw;
  ESGD_REQUIRE(d->batch == 1 || cg->src_sb == nimg * cg->src_h * cg->src_w * cg->channels, ESGD_ERR_SHAPE,
               "tc_conv_tma: replica NHWC sources must be contiguous (src_sb = images*H*W*C)");
  if (side == 1) {
    ESGD_REQUIRE(d->m == cg->npix && d->k == kdim, ESGD_ERR_SHAPE,
                 "tc_conv_tma: im2col A is npix x kh*kw*channels (m=%d k=%d)", d->m, d->k);
    ESGD_REQUIRE(d->b && d->b_major == 0 && (d->ldb & 3) == 0 && d->ldb >= d->k && aligned16(d->b),
                 ESGD_ERR_SHAPE, "tc_conv_tma: B must be K-major with a 16-B aligned pitch");
  } else {
    ESGD_REQUIRE(d->n == kdim && d->k == cg->npix, ESGD_ERR_SHAPE,
                 "tc_conv_tma: im2col B is kh*kw*channels x npix (n=%d k=%d)", d->n, d->k);
    ESGD_REQUIRE(d->a && d->a_major == 0 && (d->lda & 3) == 0 && d->lda >= d->k && aligned16(d->a),
                 ESGD_ERR_SHAPE, "tc_conv_tma: A must be K-major with a 16-B aligned pitch");
  }
  ESGD_REQUIRE(d->c, ESGD_ERR_INPUT, "tc_conv_tma: null output");
  ESGD_REQUIRE(d->batch == 1 || ((d->a_sb & 3) == 0 && (d->b_sb & 3) == 0), ESGD_ERR_SHAPE,
               "tc_conv_tma: batch strides must be multiples of 4");
  tc::Gather ga{cg->src, cg->src_sb, 0, cg->src_h * cg->src_w * cg->channels, cg->src_h, cg->src_w, cg->grid_h,
                cg->grid_w, cg->stride, cg->yoff, cg->xoff, 1, cg->kh, cg->kw, cg->npix, (int)kdim, 0};
  const tc::Plan p = tc::make_plan(d, /*allow_swap=*/false);
  const int64_t need = tc::ws_need(p);
  ESGD_REQUIRE(need <= d->ws_floats, ESGD_ERR_UNSUPPORTED,
               "tc_conv_tma: split-K workspace too small (need %lld floats, have %lld; size it with "
               "esgd_tc_conv_ws_floats)", (long long)need, (long long)d->ws_floats);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (side == 1) {
    if (p.bn == 64) return tc::launch_im2col<64, 4>(p, st, ga);
    if (p.bn == 192) return tc::launch_im2col<192, 4>(p, st, ga);
    return tc::launch_im2col<128, 4>(p, st, ga);
  }
  if (p.bn == 64) return tc::launch_im2col<64, 5>(p, st, ga);
  if (p.bn == 192) return tc::launch_im2col<192, 5>(p, st, ga);
  return tc::launch_im2col<128, 5>(p, st, ga);
}

extern "C" int esgd_tc_conv_ws_floats(const esgd_tc_gemm_desc* d, int64_t* floats) {
  using namespace esgd;
  ESGD_REQUIRE(floats, ESGD_ERR_INPUT, "tc_conv_ws_floats: null output");
  *floats = 0;
  if (int rc = tc::validate(d)) return rc;
  if (d->m == 0 || d->n == 0 || d->batch == 0 || d->k == 0) return ESGD_OK;
  esgd_tc_gemm_desc q = *d;
  if (!q.ws) q.ws = reinterpret_cast<float*>(uintptr_t(256));
  *floats = tc::ws_need(tc::make_plan(&q, /*allow_swap=*/false));
  return ESGD_OK;
}

#ifdef ESGD_TRACE
extern "C" int esgd_trace_copy(void* dst) {
  return cudaMemcpyFromSymbol(dst, esgd::tc::g_trace, sizeof(esgd::tc::g_trace)) == cudaSuccess ? 0 : 1;
}
#endif
