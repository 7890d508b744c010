/*
 * esgd.h — C-ABI of libesgd, the B200 (sm_100a) kernels behind the
 * elastic-averaging SGD trainers of arXiv 1708.02983.
 *
 * Plain pointers, sizes and scalars only (no torch types). All buffers are
 * caller-owned DEVICE memory unless noted; every call is stream-ordered on
 * `stream` (a cudaStream_t passed as void*; NULL = legacy default stream) and
 * returns ESGD_OK or an error code, with a message in esgd_last_error().
 * Nothing here allocates device memory or synchronizes the device.
 *
 * Each entry point names the reference interface it replaces
 * (paths relative to /root/reference/pkg/src/elasticsgd/).
 *
 * Numerics: the update rules evaluate exactly the reference's fp32 operation
 * sequence with round-to-nearest and no FMA contraction, so their results are
 * bitwise equal to the reference run with a float32 ModelSpec.
 */
#ifndef ESGD_H_
#define ESGD_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ESGD_OK 0
#define ESGD_ERR_SHAPE 1  /* maps to elasticsgd.errors.ShapeError  */
#define ESGD_ERR_INPUT 2  /* maps to elasticsgd.errors.InputError  */
#define ESGD_ERR_CUDA 3   /* CUDA runtime / launch failure          */
#define ESGD_ERR_UNSUPPORTED 4

#define ESGD_ACT_NONE 0
#define ESGD_ACT_RELU 1
#define ESGD_ACT_TANH 2
#define ESGD_ACT_SIGMOID 3

typedef void* esgd_stream_t;
typedef void* esgd_comm_t; /* an NCCL communicator (ncclComm_t) */
#define ESGD_NCCL_ID_BYTES 128

/* ---- library ----------------------------------------------------------- */
const char* esgd_last_error(void);
int esgd_abi_version(void);

/* SMs the persistent tcgen05 GEMM / conv kernels leave free (grid = 148 -
 * sms, rounded down to even) for a collective that runs beside them on
 * dedicated SMs (esgd_center_step_nvls_f32 with ctas < 0). Process-wide,
 * default 0; the tile plan and split-K counts (so the results) do not change. */
int esgd_set_sm_reserve(int32_t sms);
/* 1 if the library was built for sm_100a and a device of that class is present */
int esgd_device_ok(int device);

/* ---- update rules: updates.py ------------------------------------------ */

/* easgd_worker_step, updates.py:85-93:
 *   w_out = (w - eta*g) - etarho*(w - c);  w_out may alias w.            */
int esgd_worker_step_f32(float* w_out, const float* w, const float* g, const float* c,
                         int64_t n, float eta, float etarho, esgd_stream_t stream);

/* easgd_center_step_from_sum, updates.py:113-119:
 *   c_out = c + etarho*(s - P*c);  c_out may alias c.                      */
int esgd_center_step_from_sum_f32(float* c_out, const float* c, const float* s, int64_t n,
                                  float etarho, int32_t num_workers, esgd_stream_t stream);
/* Snapshot form, updates.py:96-110: C' = C + etarho * sum_i (W_i - C) with the
 * sum in worker order (rows of `snaps`, pitch lds floats) — bitwise the
 * reference's fp32 arithmetic (the from-sum form differs by rounding).      */
int esgd_center_step_snapshots_f32(float* c_out, const float* c, const float* snaps, int64_t lds,
                                   int32_t num_workers, int64_t n, float etarho, esgd_stream_t stream);

/* _sync_round, trainers/synchronous.py:57-64 (fused, in place):
 * for every local replica r < nrep:
 *   W[r] = (W[r] - eta*G[r]) - etarho*(W[r] - C)
 * then C = C + etarho*(S - P*C), all against the pre-update C.
 * W/G rows are ldw/ldg floats apart. 24 B/param algorithmic at nrep=1.      */
int esgd_sync_update_f32(float* W, int64_t ldw, const float* G, int64_t ldg, int32_t nrep,
                         float* C, const float* S, int64_t n, float eta, float etarho,
                         int32_t num_workers, esgd_stream_t stream);

/* esgd_sync_update_f32 plus the next round's local replica sum (the
 * tree_sum of fabric/collectives.py:18-32 over the updated replicas, same
 * binomial order): S_next = sum_r W_r(t+1). S_next may alias S. 1 <= nrep
 * <= 8, 16-B aligned buffers/pitches. 28 B/param at nrep = 1.              */
int esgd_sync_update_sum_f32(float* W, int64_t ldw, const float* G, int64_t ldg, int32_t nrep,
                             float* C, const float* S, float* S_next, int64_t n, float eta,
                             float etarho, int32_t num_workers, esgd_stream_t stream);

/* Sync-EASGD round update for a run with ONE worker in total (P = 1, one
 * process): the sum S = tree_sum([W]) (fabric/collectives.py:18-32) is W(t)
 * itself, so W <- worker_step(W, G, C), C <- center_step_from_sum(C, W(t), 1)
 * read W, G, C and write W, C (20 B/param; esgd_sync_update_sum_f32 moves 28).
 * Bitwise equal to the reference round (trainers/synchronous.py:57-64, P=1). */
int esgd_sync_update_solo_f32(float* W, const float* G, float* C, int64_t n, float eta, float etarho,
                              esgd_stream_t stream);

/* Multi-GPU round update fused with its collective over NVLink SHARP
 * (NVLS) multicast (replaces ncclAllReduce(S) + esgd_sync_update_sum_f32):
 * this rank's 1/world slice of the center is updated from the NVSwitch-
 * reduced sum of every rank's S (multimem.ld_reduce on S_mc) and broadcast
 * to all ranks (multimem.st to C_new_mc); all local replicas take the worker
 * step against C_old and S_next = their binomial tree sum. S_mc / C_new_mc
 * are multicast addresses of symmetric buffers (torch symmetric memory);
 * C_old, S_next local. n4 = padded length (multiple of 4, zero padding).
 * Call esgd_nvls_barrier first (orders the previous round's writes/reads). */
int esgd_sync_update_nvls_f32(float* W, int64_t ldw, const float* G, int64_t ldg, int32_t nrep,
                              const float* C_old, const float* S_mc, float* C_new_mc, float* S_next,
                              int64_t n4, int32_t world, int32_t rank, float eta, float etarho,
                              int32_t num_workers, esgd_stream_t stream);

/* The same round split for overlap (what the engine runs): the center
 * slice (NVLS ld_reduce -> center step -> multicast broadcast) on a side
 * stream concurrently with the forward/backward (ctas = grid size of small
 * CTAs that sit next to the GEMM's, 0 = one per SM; ctas < 0: -ctas wide
 * CTAs that take whole SMs, for use with esgd_set_sm_reserve), and the local
 * worker step + next replica sum after it.                                  */
int esgd_center_step_nvls_f32(const float* C_old, const float* S_mc, float* C_new_mc, int64_t n4,
                              int32_t world, int32_t rank, float etarho, int32_t num_workers, int32_t ctas,
                              esgd_stream_t stream);
/* Copy-engine variant of the center slice: C_new = center step of C_old with
 * sum(srcs[0..nsrc)) (device array of nsrc <= 8 slice pointers, summed in
 * binomial order), all over n4 floats; the slices are moved between GPUs by
 * esgd_copy_async (cudaMemcpyAsync: copy engines over NVLink).              */
int esgd_center_step_sum_f32(const float* C_old, const float* const* srcs, int32_t nsrc, float* C_new,
                             int64_t n4, float etarho, int32_t num_workers, esgd_stream_t stream);
int esgd_copy_async(void* dst, const void* src, int64_t bytes, esgd_stream_t stream);
int esgd_worker_step_sum_f32(float* W, int64_t ldw, const float* G, int64_t ldg, int32_t nrep,
                             const float* C, float* S_next, int64_t n4, float eta, float etarho,
                             esgd_stream_t stream);

/* Cross-GPU barrier on the device: peer_flags = device array of world
 * pointers to each rank's symmetric int32 flag array (>= world entries,
 * zero-initialised); epoch = this rank's device counter (graph-replayable). */
int esgd_nvls_barrier(int32_t* const* peer_flags, int32_t world, int32_t rank, int32_t* epoch,
                      esgd_stream_t stream);

/* ---- collective (no torch.distributed) ----------------------------------- */
/* The cross-GPU replica sum of the Sync round as an in-place NCCL allreduce,
 * for hosts that drive libesgd directly (SURVEY.md §8(b) esgd_nccl_init_all /
 * esgd_allreduce_sum_f32 / esgd_nccl_destroy; replaces the reference's
 * tree_sum over workers, fabric/collectives.py:18-32, across processes). NCCL
 * is dlopen'ed (libnccl.so.2); without it these return ESGD_ERR_UNSUPPORTED.
 * Rank 0 creates the id, the host ships its 128 bytes to every rank, each
 * rank (with its GPU current) calls esgd_nccl_init. The sum order is NCCL's
 * (bitwise equal to the binomial tree at world = 2).                       */
int esgd_nccl_available(void);
int esgd_nccl_unique_id(void* id_out /* ESGD_NCCL_ID_BYTES */);
int esgd_nccl_init(esgd_comm_t* comm, const void* id, int32_t world, int32_t rank);
int esgd_allreduce_sum_f32(esgd_comm_t comm, float* buf, int64_t n, esgd_stream_t stream);
int esgd_nccl_destroy(esgd_comm_t comm);

/* measgd_worker_step, updates.py:134-140 (in place):
 *   v = mu*v - eta*g;  w = (w + v) - etarho*(w - c).  24 B/param.          */
int esgd_measgd_update_f32(float* w, float* v, const float* g, const float* c, int64_t n,
                           float eta, float mu, float etarho, esgd_stream_t stream);

/* easgd_center_incremental, updates.py:122-131: c_out = c + etarho*(w - c) */
int esgd_center_incr_f32(float* c_out, const float* c, const float* w, int64_t n,
                         float etarho, esgd_stream_t stream);

/* original EASGD round (trainers/roundrobin.py:120-124), fused, in place:
 * from the same old (w, c):  w = (w - eta*g) - etarho*(w - c);
 *                            c = c + etarho*(w_old - c).   20 B/param.      */
int esgd_exchange_update_f32(float* w, const float* g, float* c, int64_t n, float eta,
                             float etarho, esgd_stream_t stream);

/* sgd_step / msgd_step, updates.py:71-82 (in place) */
int esgd_sgd_step_f32(float* w, const float* g, int64_t n, float eta, esgd_stream_t stream);
int esgd_msgd_step_f32(float* w, float* v, const float* g, int64_t n, float eta, float mu,
                       esgd_stream_t stream);

/* hogwild_apply, fabric/engine.py:156-166 with the elastic delta of
 * trainers/hogwild.py:180:  center += etarho*(w - snap), lock-free
 * (vector red.global.add), racing other streams by design.                  */
int esgd_hogwild_apply_f32(float* center, const float* w, const float* snap, int64_t n,
                           float etarho, esgd_stream_t stream);
/* hogwild-sgd delta (trainers/hogwild.py:190): center += scale*g, lock-free */
int esgd_hogwild_axpy_f32(float* center, const float* g, int64_t n, float scale,
                          esgd_stream_t stream);

/* tree_sum, fabric/collectives.py:18-32, over nrep local replicas (rows of
 * W, ldw apart) in the reference's fixed binomial order. nrep <= 64.       */
int esgd_replica_tree_sum_f32(float* S, const float* W, int64_t ldw, int32_t nrep, int64_t n,
                              esgd_stream_t stream);

/* ---- counter RNG + sampling: rng.py, datasets.py ------------------------ */

/* CounterRng.randint_block, rng.py:87-91: out[i] = mix64(seed + (counter+i+1)*GOLDEN) % upper */
int esgd_randint_u64(int64_t* out, uint64_t seed, uint64_t counter, int64_t count,
                     uint64_t upper, esgd_stream_t stream);

/* sample_batch, datasets.py:166-171, for nrep replicas in one launch.
 * rng_state[2r] = seed, rng_state[2r+1] = counter of replica r (device
 * memory; the counter is advanced by b on the device, so the call can be
 * replayed from a CUDA graph). ticket: nrep int32 zeros (scratch).
 * x_out[r] = rows of X (n x d, row-major) at the drawn indices, row pitch ldx;
 * y_out[r] = labels (int32) ; idx_out (optional) = the indices.             */
int esgd_sample_batch_f32(float* x_out, int64_t ldx_rep, int32_t* y_out, int64_t* idx_out,
                          const float* X, const int32_t* labels, int64_t n, int64_t d,
                          uint64_t* rng_state, int32_t* ticket, int32_t b, int32_t nrep,
                          esgd_stream_t stream);

/* Host data path (the e2e loader): copy rows[i] of a PINNED host matrix
 * (src, row pitch src_pitch bytes, src_rows rows) to dst + i*dst_pitch on
 * the device with DMA (cudaMemcpyAsync per row run, no SMs used, no host
 * gather). rows: host array of nrows indices. Asynchronous on `stream`.    */
int esgd_gather_rows_h2d(void* dst, int64_t dst_pitch, const void* src, int64_t src_pitch,
                         const int64_t* rows, int32_t nrows, int64_t row_bytes, int64_t src_rows,
                         esgd_stream_t stream);

/* QuadraticProblem.gradient, trainers/problems.py:95-96:
 *   G[r] = curvature*(W[r] - target) for nrep replicas.                    */
int esgd_quadratic_grad_f32(float* G, int64_t ldg, const float* W, int64_t ldw, int32_t nrep,
                            const float* target, const float* curvature, int64_t n,
                            esgd_stream_t stream);

/* ---- dense layers: kernels.py, network.py ------------------------------ */

/* C[z] (m x n) = act( A[z](m x k) . B[z](k x n) + bias[z] ) with arbitrary
 * element strides (row/col/batch) for every operand; optional epilogue mask
 * multiplies by (mask > 0) (relu-grad), optional c_pre keeps the
 * pre-activation; accumulate adds into C. fp32 FFMA, for the small GEMMs.
 * When the output has few tiles and k is long (weight gradients reduce over
 * every pixel of the batch) the reduction is split across CTAs into `ws`
 * (ws_floats floats of device scratch, may be NULL) and combined in a fixed
 * order, so results stay deterministic.
 * (network.py:166-171 forward, :194-199 backward, kernels.py:22-26)        */
typedef struct {
  int32_t m, n, k, batch;
  const float* a; int64_t a_sm, a_sk, a_sb;
  const float* b; int64_t b_sk, b_sn, b_sb;
  float* c; int64_t c_sm, c_sn, c_sb;
  const float* bias; int64_t bias_sb;
  const float* mask; int64_t mask_sm, mask_sn, mask_sb;
  float* c_pre;
  int32_t act;
  int32_t accumulate;
  float* ws;
  int64_t ws_floats;
} esgd_gemm_desc;
int esgd_gemm_f32(const esgd_gemm_desc* desc, esgd_stream_t stream);
/* floats of `ws` esgd_gemm_f32 needs for this problem (0: no K split). The
 * split depends on the per-replica shape only, so results never depend on
 * `batch` or the workspace; a smaller `ws` fails with ESGD_ERR_UNSUPPORTED. */
int esgd_gemm_ws_floats(const esgd_gemm_desc* desc, int64_t* floats);

/* Tensor-core GEMM (tcgen05.mma kind::tf32, TMA-fed, accumulator in TMEM)
 * with 3xTF32 error compensation (hi*hi + hi*lo + lo*hi) and per-128-K
 * promotion of the TMEM partial sums into fp32 registers: fp32-grade
 * results. C[z] = A[z] . B[z] (+bias, act, mask), C (m x n) with strides
 * (c_sm, c_sn). Operand layouts (fp32):
 *   a_major 0: A[m*lda + k] (K-major)   1: A[k*lda + m] (M-major)
 *   b_major 0: B[n*ldb + k] (K-major)   1: B[k*ldb + n] (N-major)
 * lda/ldb multiples of 4, A/B 16-B aligned (TMA). Batched over `batch` with
 * element strides a_sb, b_sb, c_sb. With `ws` (ws_floats floats of device
 * scratch) small-output / long-K problems split K across CTAs and combine
 * the partials in a fixed order (deterministic).                           */
typedef struct {
  int32_t m, n, k, batch;
  const float* a; int64_t lda, a_sb;
  const float* b; int64_t ldb, b_sb;
  float* c; int64_t c_sm, c_sn, c_sb;
  const float* bias; int64_t bias_sb;
  const float* mask; int64_t mask_sm, mask_sn, mask_sb;
  int32_t act;
  int32_t accumulate;
  int32_t precision; /* 3 = 3xTF32 (fp32-grade, default), 1 = plain TF32 */
  int32_t a_major, b_major;
  float* ws;
  int64_t ws_floats;
} esgd_tc_gemm_desc;
int esgd_tc_gemm_f32(const esgd_tc_gemm_desc* desc, esgd_stream_t stream);
/* floats of `ws` esgd_tc_gemm_f32 needs for this problem (0: no K split);
 * same contract as esgd_gemm_ws_floats.                                    */
int esgd_tc_gemm_ws_floats(const esgd_tc_gemm_desc* desc, int64_t* floats);

/* Implicit-GEMM convolution on the tensor cores (same 3xTF32 kernel): one
 * GEMM operand is gathered by the kernel straight from a CNHW activation
 * tensor (channel planes of `plane` floats, each [n][y][x] of src_h x
 * src_w images) instead of an im2col matrix; the other operand, the output
 * and the epilogue are those of `desc` (its `a` or `b` is ignored).
 *   side 1 (forward / data gradient): A[m][k], m = pixel (n, r, c) of the
 *     grid_h x grid_w grid (npix = images * grid_h * grid_w = desc->m),
 *     k = (ch, kh, kw) in the packed weight order (desc->k = channels*kh*kw);
 *   side 2 (weight gradient): B[n][k], n = (ch, kh, kw) (desc->n), k = pixel
 *     (desc->k = npix).
 * value = src[z*src_sb + ch*plane + n*img_stride + y*src_w + x] with
 * y = r*stride + yoff + sgn*kh, x = c*stride + xoff + sgn*kw, zero outside the
 * image (zero padding). Convolution window (forward, weight gradient): sgn =
 * +1, yoff = xoff = -pad. Data gradient of a stride-1 convolution: sgn = -1,
 * yoff = xoff = +pad, src = the output gradient.
 * (replaces network.py's dense contractions for the CNN layers the reference
 * lacks — SPEC.md:67; oracle: oracle/esgd_oracle.py _im2col / _col2im)      */
typedef struct {
  const float* src; int64_t src_sb;
  int32_t plane;      /* channel stride (floats) */
  int32_t img_stride; /* image stride: 0 = src_h*src_w (CNHW planes); c*h*w for NCHW rows */
  int32_t src_h, src_w;
  int32_t grid_h, grid_w;
  int32_t stride, yoff, xoff, sgn;
  int32_t kh, kw;
  int32_t npix;
  int32_t channels;
} esgd_conv_gather;
int esgd_tc_conv_f32(const esgd_tc_gemm_desc* desc, const esgd_conv_gather* gather, int32_t side,
                     esgd_stream_t stream);
/* The same implicit GEMM with the gathered operand loaded by TMA in im2col
 * mode (cp.async.bulk.tensor...im2col) from an NHWC source: src is [n][y][x][c]
 * (c innermost; replicas stacked along n: src_sb = images*src_h*src_w*c),
 * `channels` a multiple of 32, K ordered (kh, kw, c) — one k-block is 32
 * channels of one window tap, so the tile lands in the same 128-B-swizzled
 * layout as a TMA-tiled operand. Forward window only: sgn = 1, yoff = xoff =
 * -pad, grid = the window's output grid at `stride` (<= 8). side 1: A[m][k]
 * (m = grid pixel; forward, or a stride-1 data gradient as the forward conv
 * of the NHWC output gradient with pad' = k-1-pad and flipped weights);
 * side 2: B[n][k] (n = (kh, kw, c), k = grid pixel; weight gradient).
 * plane / img_stride are unused. Split-K workspace: esgd_tc_conv_ws_floats. */
int esgd_tc_conv_tma_f32(const esgd_tc_gemm_desc* desc, const esgd_conv_gather* gather, int32_t side,
                         esgd_stream_t stream);
/* split-K workspace floats esgd_tc_conv_f32 needs for `desc` (0: no split). */
int esgd_tc_conv_ws_floats(const esgd_tc_gemm_desc* desc, int64_t* floats);

/* activation forward/backward, kernels.py:30-70.
 * act_fwd: y = act(z); act_bwd: d = d * act'(z) (in place).                 */
int esgd_act_fwd_f32(float* y, const float* z, int64_t n, int32_t act, esgd_stream_t stream);
int esgd_act_bwd_f32(float* d, const float* z, int64_t n, int32_t act, esgd_stream_t stream);

/* softmax_cross_entropy, kernels.py:85-106, per batch z of rows x cols logits
 * (row pitch ld): dlogits = (softmax - onehot)/rows (may alias logits),
 * row_loss[z*rows + i] = -log(softmax[i, label]) (optional).
 * Labels out of range -> ESGD_ERR_INPUT is reported via *bad_label (device
 * int32, optional; set to 1 on a bad label).                               */
int esgd_softmax_xent_f32(float* dlogits, float* row_loss, const float* logits, int64_t ld,
                          int64_t z_stride, const int32_t* labels, int64_t label_z_stride,
                          int32_t rows, int32_t cols, int32_t batch, int32_t* bad_label,
                          esgd_stream_t stream);

/* batched transpose: dst[z][c*ldd + r] = src[z][r*lds + c], r < rows, c < cols
 * (operand re-layout so no tensor-core GEMM needs two MN-major operands).   */
int esgd_transpose_f32(float* dst, int64_t ldd, int64_t d_sb, const float* src, int64_t lds,
                       int64_t s_sb, int32_t rows, int32_t cols, int32_t batch, esgd_stream_t stream);

/* argmax per row (ties -> lowest index), records.py:92-101 */
int esgd_argmax_rows_f32(int32_t* out, const float* x, int64_t ld, int32_t rows, int32_t cols,
                         esgd_stream_t stream);

/* column sums over rows: out[z*out_sb + j] = sum_i x[z][i*ld + j] (bias grad,
 * network.py:195). Deterministic fixed-order two-pass reduction.
 * scratch: >= 256*cols*batch floats.                                         */
int esgd_colsum_f32(float* out, int64_t out_sb, const float* x, int64_t ld, int64_t x_sb,
                    int64_t rows, int32_t cols, int32_t batch, float* scratch,
                    esgd_stream_t stream);

/* ---- convolution / pooling (CNN problems; no reference counterpart:
 *      SPEC.md:67, conventions follow network.py) ------------------------- */

/* activation tensors are described by element strides (n, c, h, w) so NCHW
 * (dataset rows) and NHWC (internal) both work.                             */
typedef struct {
  int32_t n, c, h, w;
  int64_t sn, sc, sh, sw;
} esgd_tensor4;

/* im2col: the column element (pix, k), pix = (img*OH + oh)*OW + ow and
 * k = (ci*kh + ky)*kw + kx, is col[pix*col_sp + k*col_sk] =
 * x(img, ci, oh*stride - pad + ky, ow*stride - pad + kx) (0 outside).
 * Layouts: (col_sp, col_sk) = (>=K, 1) row-major, or (1, >=pixels)
 * transposed (the engine's; TMA-friendly for the weight-gradient GEMM).
 * Batched over `batch` (x_sb, col_sb).                                     */
int esgd_im2col_f32(float* col, int64_t col_sp, int64_t col_sk, int64_t col_sb, const float* x,
                    esgd_tensor4 xd, int64_t x_sb, int32_t kh, int32_t kw, int32_t stride,
                    int32_t pad, int32_t oh, int32_t ow, int32_t batch, esgd_stream_t stream);

/* col2im (adjoint of im2col, gather form, fixed (ky, kx) order): dx(img,ci,y,x)
 * = sum of the dcol entries im2col took from (y,x); optional mask multiplies
 * the result by (mask>0); mask has dx's layout within a batch entry and its
 * own batch stride mask_sb (relu-grad from the producer's activation).     */
int esgd_col2im_f32(float* dx, esgd_tensor4 xd, int64_t x_sb, const float* dcol, int64_t col_sp,
                    int64_t col_sk, int64_t col_sb, int32_t kh, int32_t kw, int32_t stride,
                    int32_t pad, int32_t oh, int32_t ow, const float* mask, int64_t mask_sb,
                    int32_t batch, esgd_stream_t stream);

/* row sums: out[z*out_sb + r] = sum_{j<cols} x[z*x_sb + r*ld + j] (conv bias
 * gradients over channel-major activations; network.py:195 generalised).
 * Deterministic fixed-order reduction; scratch >= 64*rows*batch floats.     */
int esgd_rowsum_f32(float* out, int64_t out_sb, const float* x, int64_t ld, int64_t x_sb,
                    int32_t rows, int64_t cols, int32_t batch, float* scratch, esgd_stream_t stream);

/* max pooling kxk/stride/pad; argmax (flat h*W+w of the input plane, first
 * max in (ky,kx) scan order) kept for backward.                             */
int esgd_maxpool_fwd_f32(float* y, esgd_tensor4 yd, int64_t y_sb, int32_t* argmax,
                         const float* x, esgd_tensor4 xd, int64_t x_sb, int32_t k,
                         int32_t stride, int32_t pad, int32_t batch, esgd_stream_t stream);
/* dx = sum of dy routed to argmax (gather form), optional relu mask (x>0)
 * with dx's layout and batch stride mask_sb.                                */
int esgd_maxpool_bwd_f32(float* dx, esgd_tensor4 xd, int64_t x_sb, const float* dy,
                         esgd_tensor4 yd, int64_t y_sb, const int32_t* argmax,
                         const float* mask, int64_t mask_sb, int32_t k, int32_t stride,
                         int32_t pad, int32_t batch, esgd_stream_t stream);

/* the same with the relu backward of the pool's input fused, gated by the
 * pooled output y (stride y_sb between replicas) of a window that selected
 * the pixel — that window's max is the pixel's own value, so the result is
 * bitwise the mask=input form while reading the pooled output instead of the
 * input. Replaces network.py:197-199's act' for conv->relu->pool stacks.     */
int esgd_maxpool_bwd_relu_f32(float* dx, esgd_tensor4 xd, int64_t x_sb, const float* dy,
                              esgd_tensor4 yd, int64_t dy_sb, const int32_t* argmax, const float* y,
                              int64_t y_sb, int32_t k, int32_t stride, int32_t pad, int32_t batch,
                              esgd_stream_t stream);

/* strided 4-D copy (layout change, e.g. NHWC -> NCHW flatten for the FC
 * head and back), optional relu mask on the source (src>0 of mask).         */
int esgd_copy4_f32(float* dst, esgd_tensor4 dd, int64_t d_sb, const float* src, esgd_tensor4 sd,
                   int64_t s_sb, int32_t batch, esgd_stream_t stream);


/* ---- device-side parameter server: trainers/asynchronous.py:170-264 ------
 * Asynchronous EASGD / MEASGD with the master as ONE persistent kernel on the
 * center's GPU, FCFS by ticket (fabric/engine.py:125-148), no host in the
 * loop. Per worker cycle on the worker's stream: esgd_async_post (takes a
 * ticket; W is final), the gradient, esgd_async_wait (until the master has
 * served this worker's post), then the elastic step against the snapshot.
 * The master (esgd_async_master_f32) serves `services` tickets in order:
 * snap_w = C (the pre-update center), C += etarho*(W_w - C)
 * (updates.py:122-131), over NVLink for workers on other GPUs (peer access:
 * esgd_enable_peer_access both ways). ctl: esgd_async_ctl_ints(workers)
 * zeroed int32 on the master GPU; ctl[1] != 0 after a 20 s stall (error).   */
int esgd_async_ctl_ints(int32_t workers);
/* load the protocol's kernels on the current device before the master runs
 * (a lazy load at first launch can wait on the running master)             */
int esgd_async_preload(void);
int esgd_enable_peer_access(int32_t device, int32_t peer);
int esgd_async_master_f32(float* center, int64_t n, const float* const* w_ptrs, float* const* snap_ptrs,
                          int32_t* ctl, int32_t workers, int64_t services, float etarho, int32_t ctas,
                          esgd_stream_t stream);
int esgd_async_post(int32_t* ctl, int32_t workers, int32_t worker, int32_t* my_posts, esgd_stream_t stream);
int esgd_async_wait(int32_t* ctl, int32_t workers, int32_t worker, const int32_t* my_posts,
                    esgd_stream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* ESGD_H_ */
