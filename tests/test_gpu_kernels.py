"""Kernel-level parity on the B200: libesgd vs the reference's own outputs
(golden fixtures) and the pinned oracle. Update rules, the tree sum and the
sampled indices are bitwise; GEMMs are checked against float64."""

import ctypes as C

import numpy as np
import pytest
import torch

from oracle import esgd_oracle as O
from paper_1708_02983_b200 import _lib, updates as U
from paper_1708_02983_b200.fabric import collectives, engine
from paper_1708_02983_b200.device import stream_ptr
from _gpu_util import dev, host, rel_err

pytestmark = pytest.mark.gpu


def test_library_on_b200():
    lib = _lib.load()
    assert lib.esgd_device_ok(0) == 1, _lib.last_error()


def test_update_rules_bitwise_vs_reference(golden):
    g = golden("updates")
    eta, rho, mu, P = (float(x) for x in g["scalars"])
    w, v, gr, c, s = (dev(a) for a in g["float32_in"])
    assert np.array_equal(host(U.easgd_worker_step(w, gr, c, eta, rho)), g["float32_worker"])
    assert np.array_equal(host(U.easgd_center_step_from_sum(c, s, int(P), eta, rho)),
                          g["float32_center_from_sum"])
    assert np.array_equal(host(U.easgd_center_incremental(c, w, eta, rho)), g["float32_center_incr"])
    mw, mv = U.measgd_worker_step(w, v, gr, c, eta, mu, rho)
    assert np.array_equal(host(mw), g["float32_measgd_w"])
    assert np.array_equal(host(mv), g["float32_measgd_v"])
    assert np.array_equal(host(U.sgd_step(w, gr, eta)), g["float32_sgd"])
    a, b = U.msgd_step(w, v, gr, eta, mu)
    assert np.array_equal(host(a), g["float32_msgd_w"]) and np.array_equal(host(b), g["float32_msgd_v"])


@pytest.mark.parametrize("p", [1, 2, 3, 5, 8, 13])
def test_tree_sum_bitwise_vs_reference(golden, p):
    g = golden("updates")
    bufs = [dev(x) for x in g[f"float32_tree_in_{p}"]]
    assert np.array_equal(host(collectives.tree_sum(bufs)), g[f"float32_tree_out_{p}"])


@pytest.mark.parametrize("n", [0, 1, 3, 4, 1029, 65536 + 7])
@pytest.mark.parametrize("offset", [0, 1])
def test_fused_sync_update_bitwise(n, offset):
    """fused worker+center kernel == reference op sequence, incl. unaligned
    (offset) and tail sizes, for 1..3 local replicas."""
    rng = np.random.default_rng(n + offset)
    for nrep in (1, 3):
        ld = n + 64 + offset
        W0 = rng.standard_normal((nrep, ld)).astype(np.float32)
        G0 = rng.standard_normal((nrep, ld)).astype(np.float32)
        C0 = rng.standard_normal(ld).astype(np.float32)
        S0 = rng.standard_normal(ld).astype(np.float32)
        hy = U.HyperParams(eta=0.05, rho=0.25)
        W, G, Cc, S = dev(W0), dev(G0), dev(C0), dev(S0)
        Wv, Gv = W[:, offset:], G[:, offset:]
        _lib.call("esgd_sync_update_f32", Wv.data_ptr(), ld, Gv.data_ptr(), ld, nrep,
                  Cc[offset:].data_ptr(), S[offset:].data_ptr(), n, hy.eta32, hy.etarho32, 4, stream_ptr())
        ew = [O.easgd_worker_step(W0[r, offset:offset + n], G0[r, offset:offset + n],
                                  C0[offset:offset + n], 0.05, 0.25) for r in range(nrep)]
        ec = O.easgd_center_step_from_sum(C0[offset:offset + n], S0[offset:offset + n], 4, 0.05, 0.25)
        for r in range(nrep):
            assert np.array_equal(host(W)[r, offset:offset + n], ew[r])
            assert np.array_equal(host(W)[r, offset + n:], W0[r, offset + n:])  # untouched
        assert np.array_equal(host(Cc)[offset:offset + n], ec)


def test_hogwild_single_stream_exact():
    rng = np.random.default_rng(1)
    n = 4099
    c0, w0, s0 = (rng.standard_normal(n).astype(np.float32) for _ in range(3))
    c, wd, sd = dev(c0), dev(w0), dev(s0)
    engine.hogwild_elastic_apply(c, wd, sd, float(np.float32(0.05 * 0.25)))
    expect = c0.copy()
    O.hogwild_apply(expect, (0.05 * 0.25) * (w0 - s0))
    assert np.array_equal(host(c), expect)


def test_hogwild_concurrent_streams_commutative():
    """many streams racing on one center: the sum of integer-valued deltas is
    exact regardless of interleaving (fabric/engine.py:156-166 contract)."""
    n = 1 << 20
    c = torch.zeros(n, device="cuda")
    deltas = [torch.full((n,), float(k + 1), device="cuda") for k in range(16)]
    streams = [torch.cuda.Stream() for _ in range(16)]
    torch.cuda.synchronize()
    for k, s in enumerate(streams):
        with torch.cuda.stream(s):
            engine.hogwild_apply(c, deltas[k])
    torch.cuda.synchronize()
    assert torch.all(c == float(sum(range(1, 17))))


def test_sampled_indices_bitwise_vs_reference(golden):
    g = golden("rng")
    seed = O.stream_seed(3, 2)
    out = torch.empty(256, dtype=torch.int64, device="cuda")
    _lib.call("esgd_randint_u64", out.data_ptr(), seed, 0, 256, 60000, stream_ptr())
    assert np.array_equal(host(out), g["randint_60000"])


def test_sample_batch_gathers_and_advances_counter():
    rng = np.random.default_rng(0)
    n, d, b, nrep = 1000, 36, 17, 3
    X = rng.standard_normal((n, d)).astype(np.float32)
    Y = rng.integers(0, 10, n).astype(np.int32)
    seeds = [O.stream_seed(9, w) for w in range(nrep)]
    state = torch.tensor(np.array([[s, 5] for s in seeds], dtype=np.uint64).view(np.int64), device="cuda")
    ticket = torch.zeros(nrep, dtype=torch.int32, device="cuda")
    xo = torch.zeros((nrep, b * d), device="cuda")
    yo = torch.zeros((nrep, b), dtype=torch.int32, device="cuda")
    Xd, Yd = dev(X), dev(Y, torch.int32)  # keep alive: launches are asynchronous
    for rnd in range(2):
        _lib.call("esgd_sample_batch_f32", xo.data_ptr(), xo.stride(0), yo.data_ptr(), None,
                  Xd.data_ptr(), Yd.data_ptr(), n, d, state.data_ptr(),
                  ticket.data_ptr(), b, nrep, stream_ptr())
        torch.cuda.synchronize()
        for r in range(nrep):
            o = O.CounterRng(seeds[r], 5 + rnd * b)
            xs, ys = O.sample_batch(X, Y, b, o)
            assert np.array_equal(host(xo[r]).reshape(b, d), xs)
            assert np.array_equal(host(yo[r]), ys)
    assert np.all(host(state)[:, 1] == 5 + 2 * b)


def test_softmax_xent_vs_reference(golden):
    g = golden("net")
    logits = g["xent_logits"].astype(np.float32)
    labels = g["xent_labels"].astype(np.int32)
    rows, cols = logits.shape
    lg = dev(logits)
    dl = torch.empty_like(lg)
    rl = torch.empty(rows, device="cuda")
    lab = dev(labels, torch.int32)
    _lib.call("esgd_softmax_xent_f32", dl.data_ptr(), rl.data_ptr(), lg.data_ptr(), cols, rows * cols,
              lab.data_ptr(), rows, rows, cols, 1, None, stream_ptr())
    assert rel_err(host(dl), g["xent_dlogits"]) < 1e-6
    assert abs(float(host(rl).astype(np.float64).mean()) - g["xent_loss"][0]) < 1e-6


def _gemm_ref(A, B):
    return A.astype(np.float64) @ B.astype(np.float64)


@pytest.mark.parametrize("m,n,k,batch", [(1, 1, 1, 1), (64, 10, 500, 2), (130, 70, 33, 3), (257, 500, 800, 1),
                                         (20, 25, 36864, 2), (50, 500, 4096, 1)])
@pytest.mark.parametrize("split", [False, True])
def test_ffma_gemm_strided(m, n, k, batch, split):
    rng = np.random.default_rng(m * n + k)
    A = rng.standard_normal((batch, m, k)).astype(np.float32)
    B = rng.standard_normal((batch, n, k)).astype(np.float32)  # stored N x K -> B(k,n) stride (1, k)
    bias = rng.standard_normal((batch, n)).astype(np.float32)
    Ad, Bd, bd = dev(A), dev(B), dev(bias)
    Cd = torch.zeros((batch, m, n), device="cuda")
    ws = torch.zeros(1 << 20, device="cuda")
    d = _lib.GemmDesc(m, n, k, batch, Ad.data_ptr(), k, 1, m * k, Bd.data_ptr(), 1, k, n * k,
                      Cd.data_ptr(), n, 1, m * n, bd.data_ptr(), n, None, 0, 0, 0, None, 1, 0,
                      ws.data_ptr() if split else None, ws.numel() if split else 0)
    _lib.check(_lib.load().esgd_gemm_f32(C.byref(d), stream_ptr()))
    for z in range(batch):
        ref = np.maximum(_gemm_ref(A[z], B[z].T) + bias[z], 0)
        # sequential fp32 accumulation: error grows ~sqrt(k) without split-K
        assert rel_err(host(Cd[z]), ref) < (2e-6 if (split or k <= 1024) else 1e-5)


@pytest.mark.parametrize("m,n,k,batch", [(128, 64, 32, 1), (300, 50, 500, 2), (1024, 192, 1600, 1),
                                         (4096, 128, 363, 1), (257, 1000, 4096, 1), (129, 20, 25, 3)])
@pytest.mark.parametrize("precision,tol", [(3, 3e-6), (1, 5e-3)])
def test_tcgen05_gemm(m, n, k, batch, precision, tol):
    """tcgen05 kind::tf32 GEMM: 3xTF32 reaches fp32-grade error; plain TF32 ~1e-3."""
    rng = np.random.default_rng(m + n + k)
    kp = (k + 3) // 4 * 4
    A = np.zeros((batch, m, kp), np.float32)
    B = np.zeros((batch, n, kp), np.float32)
    A[:, :, :k] = rng.standard_normal((batch, m, k))
    B[:, :, :k] = rng.standard_normal((batch, n, k))
    bias = rng.standard_normal((batch, n)).astype(np.float32)
    Ad, Bd, bd = dev(A), dev(B), dev(bias)
    Cd = torch.zeros((batch, m, n), device="cuda")
    d = _lib.TcGemmDesc(m, n, k, batch, Ad.data_ptr(), kp, m * kp, Bd.data_ptr(), kp, n * kp,
                        Cd.data_ptr(), n, 1, m * n, bd.data_ptr(), n, None, 0, 0, 0, 0, 0, precision,
                        0, 0, None, 0)
    _lib.check(_lib.load().esgd_tc_gemm_f32(C.byref(d), stream_ptr()))
    torch.cuda.synchronize()
    for z in range(batch):
        ref = _gemm_ref(A[z, :, :k], B[z, :, :k].T) + bias[z]
        assert rel_err(host(Cd[z]), ref) < tol, (z, rel_err(host(Cd[z]), ref))


def test_im2col_col2im_adjoint_and_oracle():
    rng = np.random.default_rng(3)
    n, c, h, w, k, s, p = 2, 3, 13, 11, 5, 2, 2
    oh, ow = (h + 2 * p - k) // s + 1, (w + 2 * p - k) // s + 1
    x = rng.standard_normal((n, c, h, w)).astype(np.float32)
    K = c * k * k
    kp = (K + 3) // 4 * 4
    col = torch.zeros((n * oh * ow, kp), device="cuda")
    xd = dev(x)
    _lib.call("esgd_im2col_f32", col.data_ptr(), kp, 1, 0, xd.data_ptr(), _lib.nchw(n, c, h, w), 0,
              k, k, s, p, oh, ow, 1, stream_ptr())
    ref, _, _ = O._im2col(x, k, s, p)
    assert np.array_equal(host(col)[:, :K], ref)
    dcol = rng.standard_normal((n * oh * ow, kp)).astype(np.float32)
    dx = torch.zeros((n, c, h, w), device="cuda")
    dcd = dev(dcol)
    _lib.call("esgd_col2im_f32", dx.data_ptr(), _lib.nchw(n, c, h, w), 0, dcd.data_ptr(), kp, 1, 0,
              k, k, s, p, oh, ow, None, 0, 1, stream_ptr())
    exp = O._col2im(dcol[:, :K].copy(), (n, c, h, w), k, s, p, oh, ow)
    assert np.array_equal(host(dx), exp)


def test_maxpool_fwd_bwd_vs_oracle():
    rng = np.random.default_rng(4)
    n, c, h, w, k, s, p = 2, 4, 15, 15, 3, 2, 1
    oh, ow = (h + 2 * p - k) // s + 1, (w + 2 * p - k) // s + 1
    x = rng.standard_normal((n, c, h, w)).astype(np.float32)
    x[0, 0, :4, :4] = 1.0  # ties: first max in scan order wins
    y = torch.zeros((n, c, oh, ow), device="cuda")
    am = torch.zeros((n, c, oh, ow), dtype=torch.int32, device="cuda")
    xd = dev(x)
    _lib.call("esgd_maxpool_fwd_f32", y.data_ptr(), _lib.nchw(n, c, oh, ow), 0, am.data_ptr(), xd.data_ptr(),
              _lib.nchw(n, c, h, w), 0, k, s, p, 1, stream_ptr())
    ey, ea = O._maxpool(x, k, s, p)
    assert np.array_equal(host(y), ey) and np.array_equal(host(am), ea)
    dy = rng.standard_normal((n, c, oh, ow)).astype(np.float32)
    dx = torch.zeros((n, c, h, w), device="cuda")
    dyd = dev(dy)
    _lib.call("esgd_maxpool_bwd_f32", dx.data_ptr(), _lib.nchw(n, c, h, w), 0, dyd.data_ptr(),
              _lib.nchw(n, c, oh, ow), 0, am.data_ptr(), None, 0, k, s, p, 1, stream_ptr())
    assert np.array_equal(host(dx), O._maxpool_bwd(dy, ea, (n, c, h, w)))


@pytest.mark.parametrize("a_major,b_major", [(0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("m,n,k,batch", [(200, 96, 300, 2), (64, 363, 38720, 1), (9216 // 8, 4096 // 8, 128, 1)])
def test_tcgen05_gemm_mn_major_and_split_k(a_major, b_major, m, n, k, batch):
    """MN-major operands (weight-gradient / N-major weight layouts) and the
    deterministic split-K path (long reductions over pixels)."""
    rng = np.random.default_rng(m * 7 + n + k)
    A = rng.standard_normal((batch, m, k)).astype(np.float32)
    B = rng.standard_normal((batch, n, k)).astype(np.float32)
    As = np.ascontiguousarray(A.transpose(0, 2, 1)) if a_major else A
    Bs = np.ascontiguousarray(B.transpose(0, 2, 1)) if b_major else B
    lda = m if a_major else k
    ldb = n if b_major else k
    if lda % 4 or ldb % 4:
        pytest.skip("TMA needs 16-B pitches")
    Ad, Bd = dev(As), dev(Bs)
    Cd = torch.zeros((batch, m, n), device="cuda")
    ws = torch.zeros(1 << 24, device="cuda")
    d = _lib.TcGemmDesc(m, n, k, batch, Ad.data_ptr(), lda, m * k, Bd.data_ptr(), ldb, n * k,
                        Cd.data_ptr(), n, 1, m * n, None, 0, None, 0, 0, 0, 0, 0, 3,
                        a_major, b_major, ws.data_ptr(), ws.numel())
    _lib.check(_lib.load().esgd_tc_gemm_f32(C.byref(d), stream_ptr()))
    torch.cuda.synchronize()
    for z in range(batch):
        ref = _gemm_ref(A[z], B[z].T)
        assert rel_err(host(Cd[z]), ref) < 3e-6, (z, rel_err(host(Cd[z]), ref))
    # determinism of the split-K combine
    C2 = torch.zeros_like(Cd)
    d.c = C2.data_ptr()
    _lib.check(_lib.load().esgd_tc_gemm_f32(C.byref(d), stream_ptr()))
    assert torch.equal(Cd, C2)


def test_transposed_im2col_cnhw_and_rowsum():
    """the engine's layouts: CNHW input planes, transposed colT[K][pixels]."""
    rng = np.random.default_rng(5)
    n, c, h, w, k, s, p = 3, 4, 9, 10, 3, 2, 1
    oh, ow = (h + 2 * p - k) // s + 1, (w + 2 * p - k) // s + 1
    npix = n * oh * ow
    np4 = (npix + 3) // 4 * 4
    x = rng.standard_normal((n, c, h, w)).astype(np.float32)
    plane = (n * h * w + 3) // 4 * 4
    xc = np.zeros((c, plane), np.float32)
    xc[:, :n * h * w] = x.transpose(1, 0, 2, 3).reshape(c, -1)
    K = c * k * k
    colT = torch.zeros((K, np4), device="cuda")
    xcd = dev(xc)
    _lib.call("esgd_im2col_f32", colT.data_ptr(), 1, np4, 0, xcd.data_ptr(), _lib.cnhw(n, c, h, w, plane), 0,
              k, k, s, p, oh, ow, 1, stream_ptr())
    ref, _, _ = O._im2col(x, k, s, p)
    assert np.array_equal(host(colT)[:, :npix].T, ref)
    dcolT = np.zeros((K, np4), np.float32)
    dcolT[:, :npix] = rng.standard_normal((K, npix))
    dd = dev(dcolT)
    dx = torch.zeros((c, plane), device="cuda")
    _lib.call("esgd_col2im_f32", dx.data_ptr(), _lib.cnhw(n, c, h, w, plane), 0, dd.data_ptr(), 1, np4, 0,
              k, k, s, p, oh, ow, None, 0, 1, stream_ptr())
    exp = O._col2im(dcolT[:, :npix].T.copy(), (n, c, h, w), k, s, p, oh, ow)
    assert np.array_equal(host(dx)[:, :n * h * w].reshape(c, n, h, w).transpose(1, 0, 2, 3), exp)
    rows = rng.standard_normal((7, 50000)).astype(np.float32)
    out = torch.zeros(7, device="cuda")
    scratch = torch.zeros(64 * 7, device="cuda")
    rd = dev(rows)
    _lib.call("esgd_rowsum_f32", out.data_ptr(), 0, rd.data_ptr(), 50000, 0, 7, 50000, 1, scratch.data_ptr(),
              stream_ptr())
    assert rel_err(host(out), rows.astype(np.float64).sum(axis=1)) < 1e-5


@pytest.mark.parametrize("m,n,k,c_mcontig", [(300, 70, 96, 1), (1000, 200, 64, 1), (257, 130, 40, 0),
                                              (128, 64, 32, 1)])
def test_tcgen05_gemm_tma_store_epilogue(m, n, k, c_mcontig):
    """TMA-store epilogue for both output orientations (M-contiguous conv /
    dcolT outputs, N-contiguous weight gradients), with bias + relu + edges."""
    rng = np.random.default_rng(m + 3 * n + k)
    kp = (k + 3) // 4 * 4
    A = np.zeros((m, kp), np.float32)
    B = np.zeros((n, kp), np.float32)
    A[:, :k] = rng.standard_normal((m, k))
    B[:, :k] = rng.standard_normal((n, k))
    bias = rng.standard_normal(n).astype(np.float32)
    mp, np_ = (m + 3) // 4 * 4, (n + 3) // 4 * 4
    c_sm, c_sn = (1, mp) if c_mcontig else (np_, 1)
    Cd = torch.full((mp * np_,), -5.0, device="cuda")
    Ad, Bd, bd = dev(A), dev(B), dev(bias)
    d = _lib.TcGemmDesc(m, n, k, 1, Ad.data_ptr(), kp, 0, Bd.data_ptr(), kp, 0, Cd.data_ptr(), c_sm, c_sn, 0,
                        bd.data_ptr(), 0, None, 0, 0, 0, 1, 0, 3, 0, 0, None, 0)
    _lib.check(_lib.load().esgd_tc_gemm_f32(C.byref(d), stream_ptr()))
    out = host(Cd)
    got = np.array([[out[i * c_sm + j * c_sn] for j in range(n)] for i in range(m)])
    ref = np.maximum(_gemm_ref(A[:, :k], B[:, :k].T) + bias, 0)
    assert rel_err(got, ref) < 3e-6
    # padding outside the m x n window untouched
    if c_mcontig and mp > m:
        assert out[m] == -5.0


def _cnhw(x, plane):
    n, c, h, w = x.shape
    out = np.zeros((c, plane), np.float32)
    out[:, :n * h * w] = x.transpose(1, 0, 2, 3).reshape(c, -1)
    return out


def _from_cnhw(a, n, c, h, w):
    return a[:, :n * h * w].reshape(c, n, h, w).transpose(1, 0, 2, 3)


@pytest.mark.parametrize("k,p,h,w", [(3, 1, 13, 13), (5, 2, 27, 27), (3, 1, 8, 7), (5, 2, 9, 12), (11, 2, 35, 35)])
def test_square_kernel_im2col_col2im_cnhw_batched(k, p, h, w):
    """the square-kernel engine paths (stride-1 col2im, any-stride im2col) on
    CNHW planes with two replicas (z strides), bit-exact vs the oracle"""
    rng = np.random.default_rng(k * 100 + h + w)
    n, c, reps = 3, 5, 2
    s = 4 if k == 11 else 1
    oh, ow = (h + 2 * p - k) // s + 1, (w + 2 * p - k) // s + 1
    npix = n * oh * ow
    np4 = (npix + 3) // 4 * 4
    plane = (n * h * w + 3) // 4 * 4
    K = c * k * k
    xs = [rng.standard_normal((n, c, h, w)).astype(np.float32) for _ in range(reps)]
    xd = dev(np.stack([_cnhw(x, plane) for x in xs]))
    colT = torch.zeros((reps, K, np4), device="cuda")
    _lib.call("esgd_im2col_f32", colT.data_ptr(), 1, np4, K * np4, xd.data_ptr(), _lib.cnhw(n, c, h, w, plane),
              c * plane, k, k, s, p, oh, ow, reps, stream_ptr())
    for z in range(reps):
        ref, _, _ = O._im2col(xs[z], k, s, p)
        assert np.array_equal(host(colT[z])[:, :npix].T, ref), z
    if s != 1:
        return
    dcolT = np.zeros((reps, K, np4), np.float32)
    dcolT[:, :, :npix] = rng.standard_normal((reps, K, npix))
    masks = [rng.standard_normal((n, c, h, w)).astype(np.float32) for _ in range(reps)]
    dd, md = dev(dcolT), dev(np.stack([_cnhw(m, plane) for m in masks]))
    dx = torch.zeros((reps, c, plane), device="cuda")
    _lib.call("esgd_col2im_f32", dx.data_ptr(), _lib.cnhw(n, c, h, w, plane), c * plane, dd.data_ptr(), 1, np4,
              K * np4, k, k, s, p, oh, ow, md.data_ptr(), c * plane, reps, stream_ptr())
    for z in range(reps):
        exp = O._col2im(dcolT[z, :, :npix].T.copy(), (n, c, h, w), k, s, p, oh, ow)
        exp = exp * (masks[z] > 0)
        assert np.array_equal(_from_cnhw(host(dx[z]), n, c, h, w), exp), z


@pytest.mark.parametrize("k,h,w", [(3, 55, 55), (3, 13, 13), (3, 14, 9), (2, 24, 24), (2, 7, 8), (3, 27, 28)])
def test_stride2_maxpool_cnhw_batched(k, h, w):
    """the stride-2 max-pool paths (AlexNet 3/2, LeNet 2/2) on CNHW planes,
    two replicas, ties and the relu mask, bit-exact vs the oracle"""
    rng = np.random.default_rng(k * 1000 + h * 10 + w)
    n, c, reps, s = 2, 3, 2, 2
    oh, ow = (h - k) // s + 1, (w - k) // s + 1
    plane, oplane = (n * h * w + 3) // 4 * 4, (n * oh * ow + 3) // 4 * 4
    xs = [rng.standard_normal((n, c, h, w)).astype(np.float32) for _ in range(reps)]
    xs[0][0, 0, :5, :5] = 0.5  # ties: first max in scan order wins
    xd = dev(np.stack([_cnhw(x, plane) for x in xs]))
    y = torch.zeros((reps, c, oplane), device="cuda")
    am = torch.zeros((reps, n, c, oh, ow), dtype=torch.int32, device="cuda")
    _lib.call("esgd_maxpool_fwd_f32", y.data_ptr(), _lib.cnhw(n, c, oh, ow, oplane), c * oplane, am.data_ptr(),
              xd.data_ptr(), _lib.cnhw(n, c, h, w, plane), c * plane, k, s, 0, reps, stream_ptr())
    dys = [rng.standard_normal((n, c, oh, ow)).astype(np.float32) for _ in range(reps)]
    dyd = dev(np.stack([_cnhw(d, oplane) for d in dys]))
    dx = torch.zeros((reps, c, plane), device="cuda")
    _lib.call("esgd_maxpool_bwd_f32", dx.data_ptr(), _lib.cnhw(n, c, h, w, plane), c * plane, dyd.data_ptr(),
              _lib.cnhw(n, c, oh, ow, oplane), c * oplane, am.data_ptr(), xd.data_ptr(), c * plane, k, s, 0,
              reps, stream_ptr())
    for z in range(reps):
        ey, ea = O._maxpool(xs[z], k, s, 0)
        assert np.array_equal(_from_cnhw(host(y[z]), n, c, oh, ow), ey), z
        assert np.array_equal(host(am[z]), ea), z
        exp = O._maxpool_bwd(dys[z], ea, (n, c, h, w)) * (xs[z] > 0)
        assert np.array_equal(_from_cnhw(host(dx[z]), n, c, h, w), exp), z


@pytest.mark.parametrize("nrep,n", [(1, 1031), (2, 4096), (3, 999), (5, 64), (8, 1027)])
def test_sync_update_sum_equals_update_then_tree_sum(nrep, n):
    """esgd_sync_update_sum_f32 == esgd_sync_update_f32 followed by the
    replica tree sum of the updated replicas, bit for bit (S_next aliasing S)"""
    rng = np.random.default_rng(nrep * 100 + n)
    ld = (n + 63) // 64 * 64
    W0 = rng.standard_normal((nrep, ld)).astype(np.float32)
    G0 = rng.standard_normal((nrep, ld)).astype(np.float32)
    C0 = rng.standard_normal(ld).astype(np.float32)
    S0 = rng.standard_normal(ld).astype(np.float32)
    hy = U.HyperParams(eta=0.05, rho=0.25)
    W1, G1, C1, S1 = dev(W0), dev(G0), dev(C0), dev(S0)
    U.sync_update_(W1, G1, C1, S1, n, 7, hy)
    T1 = torch.zeros(ld, device="cuda")
    collectives.replica_sum_(T1, W1, n)
    W2, G2, C2, S2 = dev(W0), dev(G0), dev(C0), dev(S0)
    U.sync_update_sum_(W2, G2, C2, S2, S2, n, 7, hy)
    torch.cuda.synchronize()
    assert torch.equal(W1[:, :n], W2[:, :n])
    assert torch.equal(C1[:n], C2[:n])
    assert torch.equal(T1[:n], S2[:n])


@pytest.mark.parametrize("m,n,k,a_major,b_major,bias", [
    (500, 192, 300, 1, 0, True),     # BN = 192 tile, bias + relu epilogue (conv2 forward shape class)
    (300, 384, 200, 0, 0, False),    # BN = 192, two n tiles
    (192, 1600, 4096, 0, 0, False),  # M = 192 weight gradient: swapped orientation, BN = 192, split-K
    (64, 363, 20000, 0, 0, False),   # M = 64 weight gradient: swapped orientation, split-K
    (1000, 1600, 192, 1, 0, False),  # dgrad shape class, BN = 192 with a padded last tile
    (2048, 256, 512, 1, 0, True),    # conv4/5 forward class: swapped to N = 2048 with the bias per row
    (3000, 64, 364, 1, 0, True),     # conv1 forward class (N = 64): swapped, bias per row, M-padded swap
    (4000, 256, 96, 1, 0, True),     # swapped, split-free short K, bias + relu
])
def test_tcgen05_gemm_wide_tiles_and_orientation(m, n, k, a_major, b_major, bias):
    """the 192-wide N tiles (TMEM A ring of 2) and the padded-work orientation
    choice (C^T = B.A^T) against an fp64 reference"""
    rng = np.random.default_rng(m + n + k)
    A = rng.standard_normal((m, k)).astype(np.float32)
    B = rng.standard_normal((n, k)).astype(np.float32)
    As = np.ascontiguousarray(A.T) if a_major else A
    Bs = np.ascontiguousarray(B.T) if b_major else B
    lda, ldb = (m if a_major else k), (n if b_major else k)
    bvec = rng.standard_normal(n).astype(np.float32)
    Ad, Bd, bd = dev(As), dev(Bs), dev(bvec)
    Cd = torch.zeros((m, n), device="cuda")
    ws = torch.zeros(1 << 24, device="cuda")
    d = _lib.TcGemmDesc(m, n, k, 1, Ad.data_ptr(), lda, 0, Bd.data_ptr(), ldb, 0, Cd.data_ptr(), n, 1, 0,
                        bd.data_ptr() if bias else None, 0, None, 0, 0, 0, 1 if bias else 0, 0, 3,
                        a_major, b_major, ws.data_ptr(), ws.numel())
    _lib.check(_lib.load().esgd_tc_gemm_f32(C.byref(d), stream_ptr()))
    torch.cuda.synchronize()
    ref = _gemm_ref(A, B.T)
    if bias:
        ref = np.maximum(ref + bvec.astype(np.float64), 0.0)
    assert rel_err(host(Cd), ref) < 3e-6, rel_err(host(Cd), ref)


@pytest.mark.parametrize("k,s,p,h,w", [(3, 2, 0, 55, 55), (3, 2, 0, 14, 9), (2, 2, 0, 7, 8), (3, 2, 1, 16, 16),
                                       (3, 2, 1, 15, 17), (3, 1, 1, 9, 10), (2, 1, 0, 6, 5), (4, 3, 1, 20, 19)])
def test_maxpool_bwd_relu_equals_input_mask_bitwise(k, s, p, h, w):
    """esgd_maxpool_bwd_relu_f32 (relu' gated by the pooled output) == the
    input-mask form esgd_maxpool_bwd_f32(mask = x) bit for bit, both stride-2
    and generic paths, two replicas, ties and ReLU zeros in the input"""
    rng = np.random.default_rng(k * 10000 + s * 1000 + p * 100 + h + w)
    n, c, reps = 2, 3, 2
    oh, ow = (h + 2 * p - k) // s + 1, (w + 2 * p - k) // s + 1
    plane, oplane = (n * h * w + 3) // 4 * 4, (n * oh * ow + 3) // 4 * 4
    xs = [np.maximum(rng.standard_normal((n, c, h, w)), 0).astype(np.float32) for _ in range(reps)]
    xs[0][0, 0, :5, :5] = 0.5
    xs[1][1, 2] = 0.0  # an all-zero plane: every window's max is 0
    xd = dev(np.stack([_cnhw(x, plane) for x in xs]))
    y = torch.zeros((reps, c, oplane), device="cuda")
    am = torch.zeros((reps, n, c, oh, ow), dtype=torch.int32, device="cuda")
    yd4, xd4 = _lib.cnhw(n, c, oh, ow, oplane), _lib.cnhw(n, c, h, w, plane)
    _lib.call("esgd_maxpool_fwd_f32", y.data_ptr(), yd4, c * oplane, am.data_ptr(), xd.data_ptr(), xd4, c * plane,
              k, s, p, reps, stream_ptr())
    dyd = dev(np.stack([_cnhw(rng.standard_normal((n, c, oh, ow)).astype(np.float32), oplane) for _ in range(reps)]))
    dx0 = torch.full((reps, c, plane), 7.0, device="cuda")
    dx1 = torch.full((reps, c, plane), 7.0, device="cuda")
    _lib.call("esgd_maxpool_bwd_f32", dx0.data_ptr(), xd4, c * plane, dyd.data_ptr(), yd4, c * oplane, am.data_ptr(),
              xd.data_ptr(), c * plane, k, s, p, reps, stream_ptr())
    _lib.call("esgd_maxpool_bwd_relu_f32", dx1.data_ptr(), xd4, c * plane, dyd.data_ptr(), yd4, c * oplane,
              am.data_ptr(), y.data_ptr(), c * oplane, k, s, p, reps, stream_ptr())
    npix = n * h * w
    assert torch.equal(dx0[:, :, :npix].view(torch.int32), dx1[:, :, :npix].view(torch.int32))


@pytest.mark.parametrize("k,s,p,h,w", [(3, 2, 0, 13, 13), (2, 2, 0, 8, 7), (3, 2, 1, 15, 17), (3, 1, 1, 9, 10)])
@pytest.mark.parametrize("gate", ["none", "mask", "relu"])
def test_maxpool_bwd_strided_layouts(k, s, p, h, w, gate):
    """NHWC planes (not the dense rows the tile kernel stages) take the
    register-gather kernels: bit-exact vs the oracle, each gating form"""
    rng = np.random.default_rng(k * 100 + s * 10 + p + h * w)
    n, c = 2, 3
    oh, ow = (h + 2 * p - k) // s + 1, (w + 2 * p - k) // s + 1
    x = np.maximum(rng.standard_normal((n, c, h, w)), -0.2).astype(np.float32)
    xd4, yd4 = _lib.nhwc(n, c, h, w), _lib.nhwc(n, c, oh, ow)
    xdev = dev(np.ascontiguousarray(x.transpose(0, 2, 3, 1)))
    y = torch.zeros((n, oh, ow, c), device="cuda")
    am = torch.zeros((n, c, oh, ow), dtype=torch.int32, device="cuda")
    _lib.call("esgd_maxpool_fwd_f32", y.data_ptr(), yd4, 0, am.data_ptr(), xdev.data_ptr(), xd4, 0, k, s, p, 1,
              stream_ptr())
    ey, ea = O._maxpool(x, k, s, p)
    assert np.array_equal(host(y).transpose(0, 3, 1, 2), ey) and np.array_equal(host(am), ea)
    dy = rng.standard_normal((n, c, oh, ow)).astype(np.float32)
    dyd = dev(np.ascontiguousarray(dy.transpose(0, 2, 3, 1)))
    dx = torch.full((n, h, w, c), 7.0, device="cuda")
    if gate == "relu":
        _lib.call("esgd_maxpool_bwd_relu_f32", dx.data_ptr(), xd4, 0, dyd.data_ptr(), yd4, 0, am.data_ptr(),
                  y.data_ptr(), 0, k, s, p, 1, stream_ptr())
    else:
        _lib.call("esgd_maxpool_bwd_f32", dx.data_ptr(), xd4, 0, dyd.data_ptr(), yd4, 0, am.data_ptr(),
                  xdev.data_ptr() if gate == "mask" else None, 0, k, s, p, 1, stream_ptr())
    exp = O._maxpool_bwd(dy, ea, (n, c, h, w))
    if gate != "none":
        exp = exp * (x > 0)
    assert np.array_equal(host(dx).transpose(0, 3, 1, 2), exp)


@pytest.mark.parametrize("m,n,k,batch,a_major,b_major", [
    (1000, 1600, 192, 1, 1, 0),    # conv2 data-gradient class
    (2048, 1024, 128, 1, 1, 0),    # FC weight-gradient class: K = batch
    (300, 520, 160, 2, 0, 0),      # ragged M / N, two replicas
    (129, 520, 40, 1, 0, 1),       # ragged K (two k-blocks, the second partial), N-major B
    (197, 640, 96, 3, 1, 1),
    (40000, 640, 192, 1, 1, 0),    # several waves of tiles
])
def test_tcgen05_gemm_short_k_many_n_tiles(m, n, k, batch, a_major, b_major):
    """short-K GEMMs over many N tiles (conv2's data gradient and the FC
    weight gradients are this class; ragged edges, replicas, every operand
    major): within the 3xTF32 tolerance of fp64 and deterministic"""
    rng = np.random.default_rng(m + 7 * n + 13 * k + batch)
    A = rng.standard_normal((batch, m, k)).astype(np.float32)
    B = rng.standard_normal((batch, n, k)).astype(np.float32)
    As = np.ascontiguousarray(A.transpose(0, 2, 1)) if a_major else A
    Bs = np.ascontiguousarray(B.transpose(0, 2, 1)) if b_major else B
    lda = m if a_major else k
    ldb = n if b_major else k
    if lda % 4 or ldb % 4:
        pytest.skip("TMA needs 16-B pitches")
    Ad, Bd = dev(As), dev(Bs)
    Cd = torch.full((batch, m, n), 5.0, device="cuda")
    d = _lib.TcGemmDesc(m, n, k, batch, Ad.data_ptr(), lda, m * k, Bd.data_ptr(), ldb, n * k,
                        Cd.data_ptr(), n, 1, m * n, None, 0, None, 0, 0, 0, 0, 0, 3,
                        a_major, b_major, None, 0)
    _lib.check(_lib.load().esgd_tc_gemm_f32(C.byref(d), stream_ptr()))
    torch.cuda.synchronize()
    for z in range(batch):
        ref = _gemm_ref(A[z], B[z].T)
        assert rel_err(host(Cd[z]), ref) < 3e-6, (z, rel_err(host(Cd[z]), ref))
    C2 = torch.zeros_like(Cd)
    d.c = C2.data_ptr()
    _lib.check(_lib.load().esgd_tc_gemm_f32(C.byref(d), stream_ptr()))
    assert torch.equal(Cd, C2)


@pytest.mark.parametrize("rows,cols,ld,batch", [(7, 50000, 50000, 1), (5, 4099, 4100, 2), (3, 9001, 9001, 1),
                                                (64, 387200, 387200, 1), (2, 3, 4, 3)])
def test_rowsum_vector_and_scalar_paths(rows, cols, ld, batch):
    """esgd_rowsum_f32 (conv bias gradients): the 16-B-load path (ld % 4 ==
    0, with a cols % 4 tail) and the scalar path, vs fp64, deterministic"""
    rng = np.random.default_rng(rows * cols + ld)
    x = np.zeros((batch, rows, ld), np.float32)
    x[:, :, :cols] = rng.standard_normal((batch, rows, cols))
    x[:, :, cols:] = 1e6  # padding beyond cols must not be summed
    xd = dev(x)
    out = torch.zeros((batch, rows), device="cuda")
    scratch = torch.zeros(64 * rows * batch + 64, device="cuda")
    _lib.call("esgd_rowsum_f32", out.data_ptr(), rows, xd.data_ptr(), ld, rows * ld, rows, cols, batch,
              scratch.data_ptr(), stream_ptr())
    ref = x[:, :, :cols].astype(np.float64).sum(axis=2)
    assert rel_err(host(out), ref) < 1e-5
    out2 = torch.zeros_like(out)
    _lib.call("esgd_rowsum_f32", out2.data_ptr(), rows, xd.data_ptr(), ld, rows * ld, rows, cols, batch,
              scratch.data_ptr(), stream_ptr())
    assert torch.equal(out, out2)
