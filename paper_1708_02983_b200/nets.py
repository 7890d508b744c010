"""Device executor for the per-worker gradient (trainers/problems.py:42-47:
sample -> forward -> softmax-CE -> backward into one packed gradient).

One ``DeviceNet`` serves ``nrep`` local worker replicas at once: every
kernel is batched over replicas (grid.z / batch strides), so P workers on one
GPU cost the same number of launches as one. Layouts in HBM:

* parameters / gradients: rows of a (nrep, ldw) fp32 tensor, the reference's
  packed order (network.view_table);
* sampled batch: (nrep, b, C*H*W) — dataset rows are CHW-flat;
* conv / pool activations: channel-major over the batch ("CNHW"): channel c
  is one plane of b*OH*OW pixels (pitch NP4 = b*OH*OW rounded up to 4), so
  every elementwise / gather kernel walks unit-stride pixels and the GEMMs
  store coalesced;
* im2col is transposed, colT[K][NP4]; then
    forward  out[pix, co]  = colT^T . W^T        (A M-major, B K-major)
    wgrad    dW[co, kk]    = delta . colT^T      (A K-major, B K-major)
    dgrad    dcolT[kk,pix] = (delta^T . W)^T     (A M-major, B N-major)
  and col2im gathers dcolT back to the input planes;
* dense activations: (b, out); the conv->dense flatten is converted to the
  reference's (c, h, w) order by one strided copy.

Contractions go to the tcgen05 3xTF32 GEMM (csrc/gemm_tc.cu) when their
operands are K-major and big enough to fill 128-row tiles; the small ones
(LeNet/MLP sizes, launch-latency bound) run on the FFMA GEMM.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import ACT, ConvGather, GemmDesc, TcGemmDesc, Tensor4, cnhw, nchw
from .device import round_up
from .errors import InputError, ShapeError
from .network import Conv, ConvNetSpec, Dense, ModelSpec, Pool, view_table

import os

# a contraction goes to the tensor cores when M*N*K reaches this and its
# operands suit TMA (a unit-stride dim, 16-B pitches); the rest take the
# CUDA-core FFMA kernel. 2^27 MACs puts CIFAR-quick's convolutions (b = 64:
# 1.6-4.2e8 MACs) and every AlexNet contraction on tcgen05 and keeps LeNet's
# (<= 1.0e8) on FFMA. Measured (B200, bench.py, 1 worker, Sync round):
# all-tcgen05 makes CIFAR-quick 0.409 -> 0.346 ms and LeNet 0.1886 -> 0.1823
# ms, but LeNet's configs[0] trajectory is chaotic (ReLU / max-pool flips):
# with 3xTF32's ~1e-6 GEMM error it leaves the fp32 envelope of the fp64 run
# by round 20-50 (1.6e-5 vs the fp32 oracle's 9e-7, tests/test_gpu_parity.py),
# so LeNet keeps the FFMA kernel's fp32-exact sums. ESGD_TC_MIN_MACS overrides.
TC_MIN_FLOPS = int(os.environ.get("ESGD_TC_MIN_MACS", str(1 << 27)))
# ESGD_IMPLICIT=1: tensor-core conv layers as implicit GEMMs (esgd_tc_conv_f32:
# operands gathered from the activations, no im2col / col2im buffers). Off by
# default: on AlexNet b=128 the gathered-operand GEMMs measured slower than
# TMA-fed explicit GEMMs + im2col/col2im (profiles/r02_implicit_conv.md)
IMPLICIT = os.environ.get("ESGD_IMPLICIT", "0") == "1"


class _FakeRows:
    """Stand-in for the (nrep, ldw) weight / gradient tensors during the
    launch-free workspace-planning pass (only pointers and strides are read)."""

    def __init__(self, ldw: int):
        self.ldw = ldw

    def data_ptr(self) -> int:
        return 1 << 20

    def stride(self, dim: int) -> int:
        return self.ldw


class _NullLib:
    """libesgd stand-in for the planning pass: every launcher is a no-op."""

    def __getattr__(self, name):
        return lambda *args: 0


_NULL_LIB = _NullLib()


@dataclass
class _Layer:
    kind: str                  # conv | pool | dense
    lay: object
    cin: int
    hin: int
    win: int
    cout: int
    hout: int
    wout: int
    act: int
    w_off: int = -1
    b_off: int = -1
    k: int = 0                 # conv reduction dim Cin*k*k
    kp: int = 0                # K rounded up to 4 (padded weight pitch)
    flatten_in: bool = False   # dense whose input is a spatial tensor
    np4: int = 0               # output plane pitch (b*OH*OW rounded up to 4)
    implicit: bool = False     # conv as implicit GEMMs (esgd_tc_conv_f32)


class DeviceNet:
    """Forward/backward executor for one model on one device, nrep replicas,
    fixed batch ``b``."""

    def __init__(self, spec, b: int, nrep: int, device: torch.device, ldw: int | None = None,
                 use_tc: bool = True, precision: int = 3, implicit: bool | None = None):
        if isinstance(spec, ModelSpec):
            spec = spec.as_layers()
        if not isinstance(spec, ConvNetSpec):
            raise InputError(f"unsupported model spec {type(spec).__name__}")
        self.spec = spec
        self.b, self.nrep, self.device = int(b), int(nrep), device
        self.n = spec.parameter_count()
        self.ldw = ldw if ldw is not None else round_up(self.n, 64)
        self.use_tc = use_tc
        self.precision = precision
        self.implicit = (IMPLICIT if implicit is None else implicit) and use_tc and precision == 3
        views = {v.name: v for v in view_table(spec)}
        self.layers: list[_Layer] = []
        prev_spatial = False
        for g in spec.geometry():
            lay = g.layer
            cin, hin, win = g.in_shape
            cout, hout, wout = g.out_shape
            if isinstance(lay, Conv):
                if lay.act not in ("none", "relu"):
                    raise InputError("conv layers support relu or no activation")
                L = _Layer("conv", lay, cin, hin, win, cout, hout, wout, ACT[lay.act],
                           views[f"W{g.param_index}"].offset, views[f"b{g.param_index}"].offset,
                           k=cin * lay.k * lay.k, kp=round_up(cin * lay.k * lay.k, 4))
                prev_spatial = True
            elif isinstance(lay, Pool):
                L = _Layer("pool", lay, cin, hin, win, cout, hout, wout, 0)
                prev_spatial = True
            else:
                L = _Layer("dense", lay, cin, 1, 1, cout, 1, 1, ACT[lay.act],
                           views[f"W{g.param_index}"].offset, views[f"b{g.param_index}"].offset,
                           flatten_in=prev_spatial)
                # geometry reports the flattened fan-in; recover the spatial shape
                if prev_spatial:
                    p = self.layers[-1]
                    L.cin, L.hin, L.win = p.cout, p.hout, p.wout
                prev_spatial = False
            self.layers.append(L)
        self.c0, self.h0, self.w0 = spec.input_shape
        self.d_in = self.c0 * self.h0 * self.w0
        self.classes = spec.num_classes
        self._alloc()

    # ---- workspace ---------------------------------------------------------
    def _t(self, per_rep: int, dtype=torch.float32) -> torch.Tensor:
        return torch.zeros((self.nrep, max(4, round_up(per_rep, 4))), dtype=dtype, device=self.device)

    def _alloc(self):
        b = self.b
        self.x = self._t(b * self.d_in)
        self.y = self._t(b, torch.int32)
        self.row_loss = self._t(b)
        self.outs, self.cols, self.amax, self.flat, self.pre = [], [], [], [], []
        max_act = b * self.d_in
        max_cols = 1
        first_param = next(j for j, L in enumerate(self.layers) if L.kind != "pool")
        for j, L in enumerate(self.layers):
            if L.kind in ("conv", "pool"):
                L.np4 = round_up(b * L.hout * L.wout, 4)
                size = L.cout * L.np4
            else:
                size = b * L.cout
            if L.kind == "conv":
                # implicit only where the tensor cores take the layer, and the data
                # gradient (when needed) is a stride-1 transposed window
                L.implicit = (self.implicit and L.np4 * L.k * L.cout >= TC_MIN_FLOPS and
                              (L.lay.stride == 1 or j <= first_param))
            max_act = max(max_act, size, b * L.cin * L.hin * L.win)
            if L.flatten_in or L.kind != "dense":
                prev = self.layers[self.layers.index(L) - 1] if self.layers.index(L) > 0 else None
                if prev is not None and prev.kind != "dense":
                    max_act = max(max_act, prev.cout * prev.np4)
            self.outs.append(self._t(size))
            self.cols.append(self._t(L.k * L.np4) if (L.kind == "conv" and not L.implicit) else None)
            self.amax.append(self._t(b * L.cout * L.hout * L.wout, torch.int32) if L.kind == "pool" else None)
            self.flat.append(self._t(b * L.cin * L.hin * L.win) if (L.kind == "dense" and L.flatten_in) else None)
            self.pre.append(self._t(size) if (L.kind == "dense" and L.act in (2, 3)) else None)
            if L.kind in ("conv", "dense"):
                max_cols = max(max_cols, L.cout)
        self.d_a = self._t(max_act)
        self.d_b = self._t(max_act)
        self.dcol = self._t(max((L.k * L.np4 for L in self.layers if L.kind == "conv" and not L.implicit),
                                default=4))
        # implicit data gradient: W permuted to [Cin][Cout*k*k] per round (K-major B)
        self.wd = [self._t(L.cin * round_up(L.cout * L.lay.k * L.lay.k, 4)) if (L.kind == "conv" and L.implicit)
                   else None for L in self.layers]
        self.scratch = torch.zeros(256 * max_cols * self.nrep + 64, dtype=torch.float32, device=self.device)
        self.bad_label = torch.zeros(1, dtype=torch.int32, device=self.device)
        # split-K partials of the GEMMs (weight gradients reduce over b*OH*OW),
        # sized below from the plan's own GEMMs (the libraries error out rather
        # than change the split when a workspace is short)
        self.gemm_ws = self.tc_ws = None
        # conv weights whose row (K) is not a multiple of 4 floats get a padded
        # copy each round so the forward GEMM can take them through TMA
        self.wpad = [self._t(L.cout * L.kp) if (L.kind == "conv" and L.k % 4) else None for L in self.layers]
        # re-laid-out operands so no tensor-core GEMM takes two MN-major inputs
        # (measured ~5x slower): W^T [K][Cout4] for conv dgrad, delta^T [out][b4]
        # for dense wgrad; refreshed every round (they depend on W / delta)
        self.wt, self.dT = [], []
        for L in self.layers:
            big = self.use_tc and L.kind == "conv" and L.np4 * L.k * L.cout >= TC_MIN_FLOPS and not L.implicit
            self.wt.append(self._t(L.k * round_up(L.cout, 4)) if big else None)
            fan_in = L.cin * L.hin * L.win
            big = self.use_tc and L.kind == "dense" and b * fan_in * L.cout >= TC_MIN_FLOPS and fan_in >= 128
            self.dT.append(self._t(L.cout * round_up(b, 4)) if big else None)
        self.tc_calls = self.ffma_calls = 0
        self.record = None  # list to capture (kind, descriptor, flops) of each GEMM launch
        self._dry = None
        self._size_workspaces()

    def _size_workspaces(self) -> None:
        """Walk one gradient pass without launching anything and ask each
        GEMM how much split-K workspace it uses (esgd_*gemm_ws_floats)."""
        self._dry = {"tc": 0, "ffma": 0}
        fake = _FakeRows(self.ldw)
        try:
            self.gradient(fake, fake, 0)
        finally:
            need, self._dry = self._dry, None
        self.tc_ws = torch.zeros(max(4, need["tc"]), dtype=torch.float32, device=self.device)
        self.gemm_ws = torch.zeros(max(4, need["ffma"]), dtype=torch.float32, device=self.device)

    def _L(self):
        return _NULL_LIB if self._dry is not None else _lib.load()

    def _out_desc(self, i: int) -> Tensor4:
        L = self.layers[i]
        if L.kind in ("conv", "pool"):
            return cnhw(self.b, L.cout, L.hout, L.wout, L.np4)
        return nchw(self.b, L.cout, 1, 1)

    # ---- GEMM routing ------------------------------------------------------
    def _gemm(self, stream, m, n, k, a, a_sm, a_sk, a_sb, bm, b_sk, b_sn, b_sb, c, c_sm, c_sn, c_sb,
              bias=None, bias_sb=0, mask=None, mask_sm=0, mask_sn=0, mask_sb=0, act=0, pre=None):
        """C = act(A.B + bias) (*mask). Routed to the tcgen05 3xTF32 kernel when
        both operands have a unit-stride dim with 16-B-aligned pitch (either
        K-major or MN-major) and the problem is big enough; else FFMA."""
        nb = self.nrep
        tc = None
        if self.use_tc and pre is None and m * n * k >= TC_MIN_FLOPS and a % 16 == 0 and bm % 16 == 0:
            a_major = 0 if a_sk == 1 else (1 if a_sm == 1 else None)
            b_major = 0 if b_sk == 1 else (1 if b_sn == 1 else None)
            if a_major is not None and b_major is not None:
                lda = a_sm if a_major == 0 else a_sk
                ldb = b_sn if b_major == 0 else b_sk
                if lda % 4 == 0 and ldb % 4 == 0 and (nb == 1 or (a_sb % 4 == 0 and b_sb % 4 == 0)):
                    tc = (a_major, b_major, lda, ldb)
        if tc is not None:
            a_major, b_major, lda, ldb = tc
            ws = self.tc_ws
            d = TcGemmDesc(m, n, k, nb, a, lda, a_sb, bm, ldb, b_sb, c, c_sm, c_sn, c_sb,
                           bias, bias_sb, mask, mask_sm, mask_sn, mask_sb, act, 0, self.precision,
                           a_major, b_major, ws.data_ptr() if ws is not None else None,
                           ws.numel() if ws is not None else 0)
            if self._dry is not None:
                need = C.c_int64(0)
                _lib.check(_lib.load().esgd_tc_gemm_ws_floats(C.byref(d), C.byref(need)), "tc_gemm_ws")
                self._dry["tc"] = max(self._dry["tc"], need.value)
                return
            _lib.check(_lib.load().esgd_tc_gemm_f32(C.byref(d), stream), "tc_gemm")
            self.tc_calls += 1
            if self.record is not None:
                self.record.append(("tc", d, 2.0 * m * n * k * nb))
        else:
            ws = self.gemm_ws
            d = GemmDesc(m, n, k, nb, a, a_sm, a_sk, a_sb, bm, b_sk, b_sn, b_sb, c, c_sm, c_sn, c_sb,
                         bias, bias_sb, mask, mask_sm, mask_sn, mask_sb, pre, act, 0,
                         ws.data_ptr() if ws is not None else None, ws.numel() if ws is not None else 0)
            if self._dry is not None:
                need = C.c_int64(0)
                _lib.check(_lib.load().esgd_gemm_ws_floats(C.byref(d), C.byref(need)), "gemm_ws")
                self._dry["ffma"] = max(self._dry["ffma"], need.value)
                return
            _lib.check(_lib.load().esgd_gemm_f32(C.byref(d), stream), "gemm")
            self.ffma_calls += 1
            if self.record is not None:
                self.record.append(("ffma", d, 2.0 * m * n * k * nb))

    def _conv(self, stream, side, m, n, k, a, lda, a_sb, bm, ldb, b_sb, c, c_sm, c_sn, c_sb, src, src_sb, sd,
              grid_h, grid_w, stride, off, sgn, kwin, chans, bias=None, bias_sb=0, mask=None, mask_sm=0,
              mask_sn=0, mask_sb=0, act=0):
        """Implicit-GEMM convolution (esgd_tc_conv_f32): side 1 gathers A (rows =
        pixels of the grid_h x grid_w grid), side 2 gathers B (rows = (ch, kh,
        kw)) from the activation tensor `src` described by Tensor4 `sd`."""
        ws = self.tc_ws
        d = TcGemmDesc(m, n, k, self.nrep, a, lda, a_sb, bm, ldb, b_sb, c, c_sm, c_sn, c_sb,
                       bias, bias_sb, mask, mask_sm, mask_sn, mask_sb, act, 0, 3, 0, 0,
                       ws.data_ptr() if ws is not None else None, ws.numel() if ws is not None else 0)
        npix = (m if side == 1 else k)
        g = ConvGather(src, src_sb, sd.sc, sd.sn, sd.h, sd.w, grid_h, grid_w, stride, off, off, sgn,
                       kwin, kwin, npix, chans)
        if self._dry is not None:
            need = C.c_int64(0)
            _lib.check(_lib.load().esgd_tc_conv_ws_floats(C.byref(d), C.byref(need)), "tc_conv_ws")
            self._dry["tc"] = max(self._dry["tc"], need.value)
            return
        _lib.check(_lib.load().esgd_tc_conv_f32(C.byref(d), C.byref(g), side, stream), "tc_conv")
        self.tc_calls += 1
        if self.record is not None:
            self.record.append(("tcconv", d, 2.0 * m * n * k * self.nrep, g, side))

    # ---- passes ----------------------------------------------------------------
    def forward(self, W: torch.Tensor, stream: int, x: torch.Tensor | None = None) -> torch.Tensor:
        """Forward of all replicas on self.x (or ``x``, same shape); returns
        the logits tensor (nrep, b*classes pitch)."""
        lib = self._L()
        b, nb = self.b, self.nrep
        wp, ldw = W.data_ptr(), W.stride(0)
        xin = self.x if x is None else x
        cur, cur_sb = xin.data_ptr(), xin.stride(0)
        cur_d = nchw(b, self.c0, self.h0, self.w0)
        for i, L in enumerate(self.layers):
            out = self.outs[i]
            o, o_sb = out.data_ptr(), out.stride(0)
            if L.kind == "conv" and L.implicit:
                lay = L.lay
                w_ptr, w_pitch, w_sb = wp + 4 * L.w_off, L.k, ldw
                if self.wpad[i] is not None:
                    pw = self.wpad[i]
                    _lib.check(lib.esgd_copy4_f32(pw.data_ptr(), Tensor4(1, L.cout, 1, L.k, 0, L.kp, 0, 1),
                                                  pw.stride(0), w_ptr, Tensor4(1, L.cout, 1, L.k, 0, L.k, 0, 1),
                                                  ldw, nb, stream), "pad_weights")
                    w_ptr, w_pitch, w_sb = pw.data_ptr(), L.kp, pw.stride(0)
                # out[co][pix] = act(sum_k col[pix][k] W[co][k] + b[co]), col gathered from the input
                self._conv(stream, 1, b * L.hout * L.wout, L.cout, L.k, None, 0, 0, w_ptr, w_pitch, w_sb,
                           o, 1, L.np4, o_sb, cur, cur_sb, cur_d, L.hout, L.wout, lay.stride, -lay.pad, 1, lay.k,
                           L.cin, bias=wp + 4 * L.b_off, bias_sb=ldw, act=L.act)
            elif L.kind == "conv":
                col = self.cols[i]
                lay = L.lay
                npix = b * L.hout * L.wout
                _lib.check(lib.esgd_im2col_f32(col.data_ptr(), 1, L.np4, col.stride(0), cur, cur_d, cur_sb,
                                               lay.k, lay.k, lay.stride, lay.pad, L.hout, L.wout, nb,
                                               stream), "im2col")
                w_ptr, w_pitch, w_sb = wp + 4 * L.w_off, L.k, ldw
                if self.wpad[i] is not None:
                    pw = self.wpad[i]
                    _lib.check(lib.esgd_copy4_f32(pw.data_ptr(), Tensor4(1, L.cout, 1, L.k, 0, L.kp, 0, 1),
                                                  pw.stride(0), w_ptr, Tensor4(1, L.cout, 1, L.k, 0, L.k, 0, 1),
                                                  ldw, nb, stream), "pad_weights")
                    w_ptr, w_pitch, w_sb = pw.data_ptr(), L.kp, pw.stride(0)
                # out[pix, co] = sum_k colT[k, pix] W[co, k] + b[co]  (CNHW store)
                self._gemm(stream, npix, L.cout, L.k,
                           col.data_ptr(), 1, L.np4, col.stride(0),
                           w_ptr, 1, w_pitch, w_sb,
                           o, 1, L.np4, o_sb, bias=wp + 4 * L.b_off, bias_sb=ldw, act=L.act)
            elif L.kind == "pool":
                lay = L.lay
                _lib.check(lib.esgd_maxpool_fwd_f32(o, self._out_desc(i), o_sb, self.amax[i].data_ptr(), cur,
                                                    cur_d, cur_sb, lay.k, lay.stride, lay.pad, nb, stream),
                           "maxpool")
            else:
                if L.flatten_in:
                    f = self.flat[i]
                    _lib.check(lib.esgd_copy4_f32(f.data_ptr(), nchw(b, L.cin, L.hin, L.win), f.stride(0),
                                                  cur, cur_d, cur_sb, nb, stream), "flatten")
                    cur, cur_sb = f.data_ptr(), f.stride(0)
                fan_in = L.cin * L.hin * L.win
                pre = self.pre[i]
                self._gemm(stream, b, L.cout, fan_in, cur, fan_in, 1, cur_sb,
                           wp + 4 * L.w_off, L.cout, 1, ldw, o, L.cout, 1, o_sb,
                           bias=wp + 4 * L.b_off, bias_sb=ldw, act=L.act,
                           pre=None if pre is None else pre.data_ptr())
            cur, cur_sb = o, o_sb
            cur_d = self._out_desc(i)
        return self.outs[-1]

    def _input_of(self, i: int):
        """(ptr, batch stride, tensor4, producer-act) of layer i's input."""
        b = self.b
        if i == 0:
            return (self.x.data_ptr(), self.x.stride(0), nchw(b, self.c0, self.h0, self.w0), 0)
        P = self.layers[i - 1]
        t = self.outs[i - 1]
        act = P.act if P.kind != "pool" else 0
        return (t.data_ptr(), t.stride(0), self._out_desc(i - 1), act)

    def _other(self, t: torch.Tensor) -> torch.Tensor:
        return self.d_b if t is self.d_a else self.d_a

    def _act_bwd(self, d: torch.Tensor, z_ptr: int, z_sb: int, n_el: int, act: int, stream: int) -> None:
        # d[r] *= act'(z[r]) for each replica (relu'(a) == relu'(z) for a = relu(z))
        lib = self._L()
        for r in range(self.nrep):
            _lib.check(lib.esgd_act_bwd_f32(d.data_ptr() + 4 * r * d.stride(0), z_ptr + 4 * r * z_sb,
                                            n_el, act, stream), "act_bwd")

    def gradient(self, G: torch.Tensor, W: torch.Tensor, stream: int) -> None:
        """G[r] = d(mean CE)/dW[r] on the sampled batch in self.x/self.y."""
        lib = self._L()
        b, nb = self.b, self.nrep
        logits = self.forward(W, stream)
        # dlogits = (softmax - onehot)/rows, in place over the logits (kernels.py:85-106)
        _lib.check(lib.esgd_softmax_xent_f32(logits.data_ptr(), self.row_loss.data_ptr(), logits.data_ptr(),
                                             self.classes, logits.stride(0), self.y.data_ptr(),
                                             self.y.stride(0), b, self.classes, nb,
                                             self.bad_label.data_ptr(), stream), "softmax_xent")
        self.backward(G, W, stream)

    def backward(self, G: torch.Tensor, W: torch.Tensor, stream: int) -> None:
        """G[r] = the packed gradient for the logits' gradient held in the last
        layer's output buffer (self.outs[-1], (nrep, b*classes)), after a
        forward of the same W (network.py:176-200)."""
        lib = self._L()
        b, nb = self.b, self.nrep
        wp, ldw = W.data_ptr(), W.stride(0)
        gp, ldg = G.data_ptr(), G.stride(0)
        dcur = self.outs[-1]
        first_param = next(j for j, L in enumerate(self.layers) if L.kind != "pool")
        for i in range(len(self.layers) - 1, -1, -1):
            L = self.layers[i]
            d_sb = dcur.stride(0)
            xin, x_sb, xd, pact = self._input_of(i)
            need_dx = i > first_param
            if L.kind == "dense":
                fan_in = L.cin * L.hin * L.win
                a_ptr, a_sb = (self.flat[i].data_ptr(), self.flat[i].stride(0)) if L.flatten_in else (xin, x_sb)
                # dW[in, out] = x^T . delta   (network.py:194)
                if self.dT[i] is not None:
                    dT, bp = self.dT[i], round_up(b, 4)
                    _lib.check(lib.esgd_transpose_f32(dT.data_ptr(), bp, dT.stride(0), dcur.data_ptr(), L.cout, d_sb,
                                                      b, L.cout, nb, stream), "transpose")
                    self._gemm(stream, fan_in, L.cout, b, a_ptr, 1, fan_in, a_sb,
                               dT.data_ptr(), 1, bp, dT.stride(0),
                               gp + 4 * L.w_off, L.cout, 1, ldg)
                else:
                    self._gemm(stream, fan_in, L.cout, b, a_ptr, 1, fan_in, a_sb,
                               dcur.data_ptr(), L.cout, 1, d_sb,
                               gp + 4 * L.w_off, L.cout, 1, ldg)
                # db = sum_rows delta   (network.py:195)
                _lib.check(lib.esgd_colsum_f32(gp + 4 * L.b_off, ldg, dcur.data_ptr(), L.cout, d_sb, b, L.cout,
                                               nb, self.scratch.data_ptr(), stream), "colsum")
                if not need_dx:
                    continue
                # delta_prev = (delta . W^T) * act'(z_prev)   (network.py:197-199)
                dnext = self._other(dcur)
                mask = xin if (pact == 1 and not L.flatten_in) else None
                self._gemm(stream, b, fan_in, L.cout, dcur.data_ptr(), L.cout, 1, d_sb,
                           wp + 4 * L.w_off, 1, L.cout, ldw,
                           dnext.data_ptr(), fan_in, 1, dnext.stride(0),
                           mask=mask, mask_sm=fan_in, mask_sn=1, mask_sb=x_sb)
                if pact in (2, 3):
                    self._act_bwd(dnext, self.pre[i - 1].data_ptr(), self.pre[i - 1].stride(0), b * fan_in,
                                  pact, stream)
                if L.flatten_in:
                    # (c,h,w)-flat gradient back to the producer's NHWC layout
                    dback = self._other(dnext)
                    _lib.check(lib.esgd_copy4_f32(dback.data_ptr(), xd, dback.stride(0), dnext.data_ptr(),
                                                  nchw(b, L.cin, L.hin, L.win), dnext.stride(0), nb, stream),
                               "unflatten")
                    if pact == 1:
                        self._act_bwd(dback, xin, x_sb, xd.c * xd.sc, 1, stream)
                    dnext = dback
                dcur = dnext
            elif L.kind == "pool":
                lay = L.lay
                yd = self._out_desc(i)
                dnext = self._other(dcur)
                if pact == 1:  # relu' of the pool input, read off the (4x smaller) pooled output
                    yo = self.outs[i]
                    _lib.check(lib.esgd_maxpool_bwd_relu_f32(dnext.data_ptr(), xd, dnext.stride(0), dcur.data_ptr(),
                                                             yd, d_sb, self.amax[i].data_ptr(), yo.data_ptr(),
                                                             yo.stride(0), lay.k, lay.stride, lay.pad, nb, stream),
                               "maxpool_bwd_relu")
                else:
                    _lib.check(lib.esgd_maxpool_bwd_f32(dnext.data_ptr(), xd, dnext.stride(0), dcur.data_ptr(), yd,
                                                        d_sb, self.amax[i].data_ptr(), None, 0, lay.k, lay.stride,
                                                        lay.pad, nb, stream), "maxpool_bwd")
                dcur = dnext
            elif L.implicit:  # conv as implicit GEMMs; delta is CNHW [Cout][np4]
                lay = L.lay
                npix = b * L.hout * L.wout
                # dW[co][k] = sum_pix delta[co][pix] col[pix][k], col gathered from the input
                self._conv(stream, 2, L.cout, L.k, npix, dcur.data_ptr(), L.np4, d_sb, None, 0, 0,
                           gp + 4 * L.w_off, L.k, 1, ldg, xin, x_sb, xd, L.hout, L.wout, lay.stride, -lay.pad, 1,
                           lay.k, L.cin)
                _lib.check(lib.esgd_rowsum_f32(gp + 4 * L.b_off, ldg, dcur.data_ptr(), L.np4, d_sb, L.cout, npix,
                                               nb, self.scratch.data_ptr(), stream), "rowsum")
                if not need_dx:
                    continue
                # dx[ci][pix] = sum_{co,kh,kw} W[co][ci][kh][kw] delta[co][pix+pad-k] (stride 1), relu
                # mask of the producer in the epilogue; B = W permuted to [ci][co*k*k]
                kk = lay.k * lay.k
                wd, pitch = self.wd[i], round_up(L.cout * kk, 4)
                _lib.check(lib.esgd_copy4_f32(wd.data_ptr(), Tensor4(1, L.cout, L.cin, kk, 0, kk, pitch, 1),
                                              wd.stride(0), wp + 4 * L.w_off,
                                              Tensor4(1, L.cout, L.cin, kk, 0, L.cin * kk, kk, 1), ldw, nb, stream),
                           "permute_weights")
                dnext = self._other(dcur)
                mask = xin if pact == 1 else None
                yd = self._out_desc(i)
                self._conv(stream, 1, b * L.hin * L.win, L.cin, L.cout * kk, None, 0, 0, wd.data_ptr(), pitch,
                           wd.stride(0), dnext.data_ptr(), 1, xd.sc, dnext.stride(0), dcur.data_ptr(), d_sb, yd,
                           L.hin, L.win, 1, lay.pad, -1, lay.k, L.cout,
                           mask=mask, mask_sm=1, mask_sn=xd.sc, mask_sb=x_sb)
                dcur = dnext
            else:  # conv: delta is CNHW [Cout][np4]
                lay = L.lay
                col = self.cols[i]
                npix = b * L.hout * L.wout
                # dW[co, kk] = sum_pix delta[co, pix] colT[kk, pix]
                self._gemm(stream, L.cout, L.k, npix, dcur.data_ptr(), L.np4, 1, d_sb,
                           col.data_ptr(), 1, L.np4, col.stride(0),
                           gp + 4 * L.w_off, L.k, 1, ldg)
                _lib.check(lib.esgd_rowsum_f32(gp + 4 * L.b_off, ldg, dcur.data_ptr(), L.np4, d_sb, L.cout, npix,
                                               nb, self.scratch.data_ptr(), stream), "rowsum")
                if not need_dx:
                    continue
                # dcolT[kk, pix] = sum_co W[co, kk] delta[co, pix]; dx = col2im(dcolT)
                if self.wt[i] is not None:
                    wt, cp = self.wt[i], round_up(L.cout, 4)
                    _lib.check(lib.esgd_transpose_f32(wt.data_ptr(), cp, wt.stride(0), wp + 4 * L.w_off, L.k, ldw,
                                                      L.cout, L.k, nb, stream), "transpose")
                    b_ptr, b_sk, b_sn, b_sb = wt.data_ptr(), 1, cp, wt.stride(0)
                else:
                    b_ptr, b_sk, b_sn, b_sb = wp + 4 * L.w_off, L.k, 1, ldw
                self._gemm(stream, npix, L.k, L.cout, dcur.data_ptr(), 1, L.np4, d_sb,
                           b_ptr, b_sk, b_sn, b_sb,
                           self.dcol.data_ptr(), 1, L.np4, self.dcol.stride(0))
                dnext = self._other(dcur)
                mask = xin if pact == 1 else None
                _lib.check(lib.esgd_col2im_f32(dnext.data_ptr(), xd, dnext.stride(0), self.dcol.data_ptr(), 1,
                                               L.np4, self.dcol.stride(0), lay.k, lay.k, lay.stride, lay.pad,
                                               L.hout, L.wout, mask, x_sb, nb, stream), "col2im")
                dcur = dnext
