"""Implicit-GEMM convolutions on the tcgen05 3xTF32 kernel
(esgd_tc_conv_f32): the forward, weight-gradient and data-gradient
contractions gathered straight from CNHW activations, against fp64 numpy
built from the oracle's im2col / col2im (oracle/esgd_oracle.py)."""

import ctypes as C

import numpy as np
import pytest
import torch

from oracle import esgd_oracle as O
from paper_1708_02983_b200 import _lib
from paper_1708_02983_b200.device import stream_ptr
from _gpu_util import rel_err

pytestmark = pytest.mark.gpu
TOL = 1e-5


def r4(x):
    return (x + 3) // 4 * 4


def cnhw(x, nrep):
    """(nrep, n, c, h, w) -> device (nrep, c*plane) CNHW with a 4-float plane pitch."""
    _, n, c, h, w = x.shape
    plane = r4(n * h * w)
    out = np.zeros((nrep, c, plane), dtype=np.float32)
    out[:, :, :n * h * w] = x.transpose(0, 2, 1, 3, 4).reshape(nrep, c, n * h * w)
    return torch.from_numpy(out.reshape(nrep, -1)).cuda(), plane


def run_conv(d, g, side):
    need = C.c_int64(0)
    _lib.check(_lib.load().esgd_tc_conv_ws_floats(C.byref(d), C.byref(need)))
    ws = torch.zeros(max(4, need.value), device="cuda")
    d.ws, d.ws_floats = ws.data_ptr(), ws.numel()
    _lib.check(_lib.load().esgd_tc_conv_f32(C.byref(d), C.byref(g), side, stream_ptr()), "tc_conv")
    torch.cuda.synchronize()


GEOMS = [  # (n, cin, h, cout, k, s, p, nrep)
    (4, 1, 28, 20, 5, 1, 0, 2),      # LeNet conv1
    (3, 3, 47, 64, 11, 4, 2, 1),     # AlexNet conv1 shape class (stride 4)
    (3, 16, 13, 48, 5, 1, 2, 2),     # conv2 class
    (2, 32, 13, 40, 3, 1, 1, 1),     # conv3-5 class, odd Cout
    (8, 64, 27, 192, 5, 1, 2, 1),    # AlexNet conv2 at b=8 (BN = 192, 2 M tiles per image row)
]


@pytest.mark.parametrize("n,cin,h,cout,k,s,p,nrep", GEOMS)
def test_conv_forward_wgrad_dgrad_vs_fp64(n, cin, h, cout, k, s, p, nrep):
    rng = np.random.default_rng(n * 1000 + cin * 10 + k)
    oh = (h + 2 * p - k) // s + 1
    K = cin * k * k
    X = rng.standard_normal((nrep, n, cin, h, h)).astype(np.float32)
    Wt = (rng.standard_normal((nrep, cout, K)) / np.sqrt(K)).astype(np.float32)
    bias = rng.standard_normal((nrep, cout)).astype(np.float32)
    D = rng.standard_normal((nrep, n, cout, oh, oh)).astype(np.float32)
    Xd, xplane = cnhw(X, nrep)
    Dd, oplane = cnhw(D, nrep)
    kp = r4(K)
    Wp = np.zeros((nrep, cout, kp), dtype=np.float32)
    Wp[:, :, :K] = Wt
    Wd = torch.from_numpy(Wp.reshape(nrep, -1)).cuda()
    bd = torch.from_numpy(bias).cuda()
    npo, npi = n * oh * oh, n * h * h

    # ---- forward: out[co][pix] = relu(sum_k col[pix][k] W[co][k] + b[co])
    out = torch.zeros((nrep, cout * oplane), device="cuda")
    d = _lib.TcGemmDesc(npo, cout, K, nrep, None, 0, 0, Wd.data_ptr(), kp, Wd.stride(0),
                        out.data_ptr(), 1, oplane, out.stride(0), bd.data_ptr(), bd.stride(0),
                        None, 0, 0, 0, 1, 0, 3, 0, 0, None, 0)
    g = _lib.ConvGather(Xd.data_ptr(), Xd.stride(0), xplane, 0, h, h, oh, oh, s, -p, -p, 1, k, k, npo, cin)
    run_conv(d, g, 1)
    cols = []
    for z in range(nrep):
        col, _, _ = O._im2col(X[z].astype(np.float64), k, s, p)
        cols.append(col)
        ref = np.maximum(col @ Wt[z].astype(np.float64).T + bias[z], 0.0)   # (npix, cout)
        got = out[z].reshape(cout, oplane)[:, :npo].T.cpu().numpy()
        assert rel_err(got, ref) < TOL, ("fwd", z, rel_err(got, ref))

    # ---- weight gradient: dW[co][k] = sum_pix delta[co][pix] col[pix][k]
    dW = torch.zeros((nrep, cout * K), device="cuda")
    d = _lib.TcGemmDesc(cout, K, npo, nrep, Dd.data_ptr(), oplane, Dd.stride(0), None, 0, 0,
                        dW.data_ptr(), K, 1, dW.stride(0), None, 0, None, 0, 0, 0, 0, 0, 3, 0, 0, None, 0)
    g = _lib.ConvGather(Xd.data_ptr(), Xd.stride(0), xplane, 0, h, h, oh, oh, s, -p, -p, 1, k, k, npo, cin)
    run_conv(d, g, 2)
    for z in range(nrep):
        dz = D[z].astype(np.float64).transpose(1, 0, 2, 3).reshape(cout, -1)   # (cout, npix) CNHW order
        ref = dz @ cols[z]
        got = dW[z].reshape(cout, K).cpu().numpy()
        assert rel_err(got, ref) < TOL, ("wgrad", z, rel_err(got, ref))

    if s != 1:
        return
    # ---- data gradient (stride 1): dx[ci][pix_in] = sum_{co,kh,kw} W[co][ci][kh][kw] delta[co][pix_in+p-k]
    kd = cout * k * k
    kdp = r4(kd)
    Wperm = np.zeros((nrep, cin, kdp), dtype=np.float32)
    Wperm[:, :, :kd] = Wt.reshape(nrep, cout, cin, k * k).transpose(0, 2, 1, 3).reshape(nrep, cin, kd)
    Wpd = torch.from_numpy(Wperm.reshape(nrep, -1)).cuda()
    dx = torch.zeros((nrep, cin * xplane), device="cuda")
    d = _lib.TcGemmDesc(npi, cin, kd, nrep, None, 0, 0, Wpd.data_ptr(), kdp, Wpd.stride(0),
                        dx.data_ptr(), 1, xplane, dx.stride(0), None, 0, None, 0, 0, 0, 0, 0, 3, 0, 0, None, 0)
    g = _lib.ConvGather(Dd.data_ptr(), Dd.stride(0), oplane, 0, oh, oh, h, h, 1, p, p, -1, k, k, npi, cout)
    run_conv(d, g, 1)
    for z in range(nrep):
        dz = D[z].astype(np.float64).transpose(0, 2, 3, 1).reshape(-1, cout)   # (npix NHW, cout)
        dcol = dz @ Wt[z].astype(np.float64)
        ref = O._col2im(dcol, (n, cin, h, h), k, 1, p, oh, oh)                 # (n, cin, h, w)
        ref = ref.transpose(1, 0, 2, 3).reshape(cin, -1)
        got = dx[z].reshape(cin, xplane)[:, :npi].cpu().numpy()
        assert rel_err(got, ref) < TOL, ("dgrad", z, rel_err(got, ref))


def test_conv_rejects_bad_geometry():
    d = _lib.TcGemmDesc(10, 4, 9, 1, None, 0, 0, None, 0, 0, None, 1, 12, 0, None, 0, None, 0, 0, 0, 0, 0, 3,
                        0, 0, None, 0)
    g = _lib.ConvGather(None, 0, 16, 0, 4, 4, 4, 4, 1, 0, 0, 1, 3, 3, 16, 1)
    rc = _lib.load().esgd_tc_conv_f32(C.byref(d), C.byref(g), 1, None)
    assert rc != 0


def nhwc(x):
    """(nrep, n, c, h, w) -> device (nrep, n*h*w*c) NHWC (replicas contiguous)."""
    nrep = x.shape[0]
    return torch.from_numpy(np.ascontiguousarray(x.transpose(0, 1, 3, 4, 2)).reshape(nrep, -1)).cuda()


def run_conv_tma(d, g, side):
    need = C.c_int64(0)
    _lib.check(_lib.load().esgd_tc_conv_ws_floats(C.byref(d), C.byref(need)))
    ws = torch.zeros(max(4, need.value), device="cuda")
    d.ws, d.ws_floats = ws.data_ptr(), ws.numel()
    _lib.check(_lib.load().esgd_tc_conv_tma_f32(C.byref(d), C.byref(g), side, stream_ptr()), "tc_conv_tma")
    torch.cuda.synchronize()


TMA_GEOMS = [  # (n, cin, h, cout, k, s, p, nrep); channels of the im2col side multiples of 32
    (3, 32, 13, 64, 3, 1, 1, 2),     # conv3-5 class; the source is < 128 KB (driver workaround path)
    (2, 64, 27, 192, 5, 1, 2, 1),    # AlexNet conv2 class
    (4, 64, 15, 40, 3, 2, 1, 1),     # stride 2 (forward / weight gradient only), odd Cout
    (8, 96, 13, 96, 3, 1, 1, 2),     # replicas, several M tiles
    (2, 32, 9, 32, 5, 1, 0, 1),      # no padding
]


@pytest.mark.parametrize("n,cin,h,cout,k,s,p,nrep", TMA_GEOMS)
def test_conv_tma_im2col_forward_wgrad_dgrad_vs_fp64(n, cin, h, cout, k, s, p, nrep):
    """esgd_tc_conv_tma_f32: the im2col operand loaded by TMA in im2col mode
    from NHWC activations (K ordered (kh, kw, c)); forward with bias + relu,
    weight gradient (split-K over pixels), and the stride-1 data gradient as
    the forward conv of the NHWC output gradient with flipped weights"""
    rng = np.random.default_rng(n * 1000 + cin * 10 + k + s)
    oh = (h + 2 * p - k) // s + 1
    K = cin * k * k
    X = rng.standard_normal((nrep, n, cin, h, h)).astype(np.float32)
    Wt = (rng.standard_normal((nrep, cout, K)) / np.sqrt(K)).astype(np.float32)   # packed (c, kh, kw)
    bias = rng.standard_normal((nrep, cout)).astype(np.float32)
    D = rng.standard_normal((nrep, n, cout, oh, oh)).astype(np.float32)
    Xn = nhwc(X)
    Dd, oplane = cnhw(D, nrep)
    Wf = np.ascontiguousarray(Wt.reshape(nrep, cout, cin, k, k).transpose(0, 1, 3, 4, 2)).reshape(nrep, cout, K)
    Wfd = torch.from_numpy(Wf.reshape(nrep, -1)).cuda()
    bd = torch.from_numpy(bias).cuda()
    npo, npi = n * oh * oh, n * h * h

    out = torch.zeros((nrep, cout * oplane), device="cuda")
    d = _lib.TcGemmDesc(npo, cout, K, nrep, None, 0, 0, Wfd.data_ptr(), K, Wfd.stride(0),
                        out.data_ptr(), 1, oplane, out.stride(0), bd.data_ptr(), bd.stride(0),
                        None, 0, 0, 0, 1, 0, 3, 0, 0, None, 0)
    g = _lib.ConvGather(Xn.data_ptr(), Xn.stride(0), 0, 0, h, h, oh, oh, s, -p, -p, 1, k, k, npo, cin)
    run_conv_tma(d, g, 1)
    cols = []
    for z in range(nrep):
        col, _, _ = O._im2col(X[z].astype(np.float64), k, s, p)
        cols.append(col)
        ref = np.maximum(col @ Wt[z].astype(np.float64).T + bias[z], 0.0)
        got = out[z].reshape(cout, oplane)[:, :npo].T.cpu().numpy()
        assert rel_err(got, ref) < TOL, ("fwd", z, rel_err(got, ref))

    dW = torch.zeros((nrep, cout * K), device="cuda")
    d = _lib.TcGemmDesc(cout, K, npo, nrep, Dd.data_ptr(), oplane, Dd.stride(0), None, 0, 0,
                        dW.data_ptr(), K, 1, dW.stride(0), None, 0, None, 0, 0, 0, 0, 0, 3, 0, 0, None, 0)
    g = _lib.ConvGather(Xn.data_ptr(), Xn.stride(0), 0, 0, h, h, oh, oh, s, -p, -p, 1, k, k, npo, cin)
    run_conv_tma(d, g, 2)
    for z in range(nrep):
        dz = D[z].astype(np.float64).transpose(1, 0, 2, 3).reshape(cout, -1)
        ref = (dz @ cols[z]).reshape(cout, cin, k, k).transpose(0, 2, 3, 1).reshape(cout, K)   # (kh, kw, c)
        got = dW[z].reshape(cout, K).cpu().numpy()
        assert rel_err(got, ref) < TOL, ("wgrad", z, rel_err(got, ref))

    if s != 1 or cout % 32:
        return
    kd = cout * k * k
    Wflip = np.ascontiguousarray(Wt.reshape(nrep, cout, cin, k, k)[:, :, :, ::-1, ::-1].transpose(0, 2, 3, 4, 1))
    Wdd = torch.from_numpy(Wflip.reshape(nrep, -1)).cuda()                   # [ci][(kh', kw', co)]
    Dn = nhwc(D)
    xplane = r4(npi)
    dx = torch.zeros((nrep, cin * xplane), device="cuda")
    d = _lib.TcGemmDesc(npi, cin, kd, nrep, None, 0, 0, Wdd.data_ptr(), kd, Wdd.stride(0),
                        dx.data_ptr(), 1, xplane, dx.stride(0), None, 0, None, 0, 0, 0, 0, 0, 3, 0, 0, None, 0)
    q = k - 1 - p
    g = _lib.ConvGather(Dn.data_ptr(), Dn.stride(0), 0, 0, oh, oh, h, h, 1, -q, -q, 1, k, k, npi, cout)
    run_conv_tma(d, g, 1)
    for z in range(nrep):
        dz = D[z].astype(np.float64).transpose(0, 2, 3, 1).reshape(-1, cout)
        dcol = dz @ Wt[z].astype(np.float64)
        ref = O._col2im(dcol, (n, cin, h, h), k, 1, p, oh, oh).transpose(1, 0, 2, 3).reshape(cin, -1)
        got = dx[z].reshape(cin, xplane)[:, :npi].cpu().numpy()
        assert rel_err(got, ref) < TOL, ("dgrad", z, rel_err(got, ref))


def test_conv_tma_rejects_bad_geometry():
    d = _lib.TcGemmDesc(16, 4, 27, 1, None, 0, 0, None, 0, 0, None, 1, 16, 0, None, 0, None, 0, 0, 0, 0, 0, 3,
                        0, 0, None, 0)
    x = torch.zeros(4 * 4 * 3, device="cuda")
    g = _lib.ConvGather(x.data_ptr(), 0, 0, 0, 4, 4, 4, 4, 1, -1, -1, 1, 3, 3, 16, 3)   # 3 channels
    assert _lib.load().esgd_tc_conv_tma_f32(C.byref(d), C.byref(g), 1, None) != 0
