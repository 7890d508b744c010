"""Training problems — the plugin boundary the trainers are generic over.

Reference protocol (trainers/problems.py:1-14): ``init_weights()``,
``gradient(weights, rng, batch_size)``, ``train_loss(w)``,
``test_accuracy(w)``, ``batch_nbytes(b)``, ``layer_nbytes()``,
``fingerprint()``, ``n_params``. Every problem here keeps that protocol
(host arrays in, host arrays out, for drop-in use) and adds the device
protocol the engines use:

    plan = problem.bind(device, nrep, batch_size, ldw)
    plan.set_streams(seeds)            # one SplitMix64 stream per replica
    plan.gradient(G, W, stream)        # G[r] = grad at W[r] (rows, pitch ldw)

A plan keeps datasets, RNG state (seed, counter) and workspaces resident in
HBM; its gradient enqueues kernels only (no host sync), so a whole round can
be captured in a CUDA graph. There is no host fallback: without a usable
B200 the problem raises ``CudaError``.
"""

from __future__ import annotations

import numpy as np
import torch

from .. import _lib
from ..datasets import Dataset
from ..device import require_cuda, round_up, stream_ptr
from ..errors import InputError, ShapeError
from ..nets import DeviceNet
from ..network import ConvNetSpec, ModelSpec, init_buffer
from ..rng import CounterRng
from .records import weights_digest


def _as_device_row(weights, device, n: int) -> torch.Tensor:
    if isinstance(weights, torch.Tensor):
        t = weights.detach().reshape(-1)[:n]
        if t.device != device or t.dtype != torch.float32:
            t = t.to(device=device, dtype=torch.float32)
        return t.contiguous()
    arr = np.asarray(weights)
    if arr.size != n:
        raise ShapeError(f"buffer size {arr.size} != layout size {n}")
    return torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float32)).to(device)


class _RngState:
    """Per-replica (seed, counter) pairs resident on the device."""

    def __init__(self, nrep: int, device):
        self.state = torch.zeros((nrep, 2), dtype=torch.int64, device=device)
        self.ticket = torch.zeros(max(1, nrep), dtype=torch.int32, device=device)

    def set(self, seeds, counters=None):
        counters = counters if counters is not None else [0] * len(seeds)
        host = np.array([[s & ((1 << 64) - 1), c] for s, c in zip(seeds, counters)], dtype=np.uint64)
        self.state.copy_(torch.from_numpy(host.view(np.int64)))

    def counters(self) -> list[int]:
        return [int(x) for x in self.state[:, 1].cpu().numpy().view(np.uint64)]


class NetworkPlan:
    """Gradient plan of a NetworkProblem: device sampling + DeviceNet."""

    def __init__(self, problem: "NetworkProblem", device, nrep: int, b: int, ldw: int,
                 use_tc: bool = True):
        self.problem, self.device, self.nrep, self.b = problem, device, nrep, b
        if not 1 <= b <= problem.train.n:
            raise InputError(f"batch size {b} out of range [1, {problem.train.n}]")
        self.X, self.Y = problem.device_train(device)
        self.net = DeviceNet(problem.spec, b, nrep, device, ldw=ldw, use_tc=use_tc)
        self.rng = _RngState(nrep, device)

    def set_streams(self, seeds, counters=None):
        self.rng.set(seeds, counters)

    def sample(self, stream: int) -> None:
        net = self.net
        _lib.check(_lib.load().esgd_sample_batch_f32(
            net.x.data_ptr(), net.x.stride(0), net.y.data_ptr(), None, self.X.data_ptr(),
            self.Y.data_ptr(), self.X.shape[0], self.X.shape[1], self.rng.state.data_ptr(),
            self.rng.ticket.data_ptr(), self.b, self.nrep, stream), "sample_batch")

    def gradient(self, G: torch.Tensor, W: torch.Tensor, stream: int) -> None:
        self.sample(stream)
        self.net.gradient(G, W, stream)

    def staged_gradient(self, G, W, x_dev, y_dev, stream: int) -> None:
        """Gradient on a batch staged by the caller (host->device data path)."""
        self.net.x.copy_(x_dev, non_blocking=True)
        self.net.y.copy_(y_dev, non_blocking=True)
        self.net.gradient(G, W, stream)


class NetworkProblem:
    """Classification on a dataset pair with an MLP (``ModelSpec``) or a CNN
    (``ConvNetSpec``) — reference trainers/problems.py:23-71."""

    def __init__(self, spec, train: Dataset, test: Dataset | None = None,
                 loss_eval_samples: int = 1024, eval_batch: int = 1024):
        if isinstance(spec, ModelSpec):
            in_dim = spec.dims[0]
        elif isinstance(spec, ConvNetSpec):
            in_dim = spec.input_dim
        else:
            raise InputError(f"unsupported spec {type(spec).__name__}")
        if train.dim != in_dim:
            raise InputError(f"samples dim {train.dim} != model input dim {in_dim}")
        self.spec = spec
        self.train = train
        self.test = test
        self.loss_k = min(loss_eval_samples, train.n)
        self.eval_batch = eval_batch
        self.n_params = spec.parameter_count()
        self._dev: dict = {}
        self._eval_nets: dict = {}

    # -- reference protocol ---------------------------------------------------
    def init_weights(self) -> np.ndarray:
        return init_buffer(self.spec)

    def gradient(self, weights, rng: CounterRng, batch_size: int) -> np.ndarray:
        """Host-in/host-out gradient at ``weights`` on a batch drawn from
        ``rng`` (advanced by batch_size), computed on the device."""
        dev = require_cuda()
        n = self.n_params
        plan = self.bind(dev, 1, batch_size, round_up(n, 64))
        plan.set_streams([rng.seed], [rng.counter])
        W = torch.zeros((1, plan.net.ldw), dtype=torch.float32, device=dev)
        W[0, :n] = _as_device_row(weights, dev, n)
        G = torch.zeros_like(W)
        plan.gradient(G, W, stream_ptr())
        rng.counter += batch_size
        return G[0, :n].cpu().numpy().astype(self.spec.dtype, copy=False)

    def train_loss(self, weights) -> float:
        losses, _ = self._eval(weights, self.train, self.loss_k)
        return float(losses.mean())

    def test_accuracy(self, weights) -> float:
        if self.test is None:
            return float("nan")
        _, correct = self._eval(weights, self.test, self.test.n)
        return float(correct.mean())

    def batch_nbytes(self, batch_size: int) -> int:
        return batch_size * self.train.dim * 8  # the reference prices 8 B/elem (problems.py:62-63)

    def layer_nbytes(self) -> list[int]:
        from ..network import view_table
        vt = view_table(self.spec)
        return [(vt[i].size + vt[i + 1].size) * 8 for i in range(0, len(vt), 2)]

    def fingerprint(self) -> str:
        head = weights_digest(self.train.samples[: min(16, self.train.n)])[:12]
        name = getattr(self.spec, "name", None) or f"net{self.spec.dims}"
        if isinstance(self.spec, ModelSpec):
            name = f"net{self.spec.dims}"
        return f"{name}-n{self.train.n}-{head}"

    # -- device protocol ------------------------------------------------------------
    def device_train(self, device):
        key = ("train", device)
        if key not in self._dev:
            self._dev[key] = (
                torch.from_numpy(np.ascontiguousarray(self.train.samples, dtype=np.float32)).to(device),
                torch.from_numpy(self.train.labels.astype(np.int32)).to(device))
        return self._dev[key]

    def device_set(self, which: str, device):
        if which == "train":
            return self.device_train(device)
        key = ("test", device)
        if key not in self._dev:
            self._dev[key] = (
                torch.from_numpy(np.ascontiguousarray(self.test.samples, dtype=np.float32)).to(device),
                torch.from_numpy(self.test.labels.astype(np.int32)).to(device))
        return self._dev[key]

    def bind(self, device, nrep: int, batch_size: int, ldw: int, use_tc: bool = True) -> NetworkPlan:
        return NetworkPlan(self, device, nrep, batch_size, ldw, use_tc=use_tc)

    def _eval_net(self, device, rows: int) -> DeviceNet:
        key = (device, rows)
        if key not in self._eval_nets:
            self._eval_nets[key] = DeviceNet(self.spec, rows, 1, device)
        return self._eval_nets[key]

    def _eval(self, weights, data: Dataset, count: int):
        """Per-row losses and correctness of the first ``count`` rows (off the clock)."""
        dev = require_cuda()
        n = self.n_params
        which = "train" if data is self.train else "test"
        X, Y = self.device_set(which, dev)
        w = _as_device_row(weights, dev, n)
        lib = _lib.load()
        losses, correct = [], []
        s = stream_ptr()
        for lo in range(0, count, self.eval_batch):
            rows = min(self.eval_batch, count - lo)
            net = self._eval_net(dev, rows)
            W = torch.zeros((1, net.ldw), dtype=torch.float32, device=dev)
            W[0, :n] = w
            net.x[0, :rows * net.d_in].copy_(X[lo:lo + rows].reshape(-1))
            net.y[0, :rows].copy_(Y[lo:lo + rows])
            logits = net.forward(W, s)
            pred = torch.empty(rows, dtype=torch.int32, device=dev)
            _lib.check(lib.esgd_argmax_rows_f32(pred.data_ptr(), logits.data_ptr(), net.classes, rows,
                                                net.classes, s), "argmax")
            rl = torch.empty(rows, dtype=torch.float32, device=dev)
            scratch = torch.empty_like(logits)
            _lib.check(lib.esgd_softmax_xent_f32(scratch.data_ptr(), rl.data_ptr(), logits.data_ptr(),
                                                 net.classes, logits.stride(0), net.y.data_ptr(),
                                                 net.y.stride(0), rows, net.classes, 1, None, s), "xent")
            losses.append(rl.double().cpu().numpy())
            correct.append((pred.cpu().numpy() == data.labels[lo:lo + rows]))
        return np.concatenate(losses), np.concatenate(correct)


class QuadraticPlan:
    def __init__(self, problem, device, nrep: int, b: int, ldw: int):
        self.nrep, self.b = nrep, b
        n = problem.n_params
        self.target = torch.zeros(ldw, dtype=torch.float32, device=device)
        self.curv = torch.zeros(ldw, dtype=torch.float32, device=device)
        self.target[:n] = torch.from_numpy(problem.target.astype(np.float32))
        self.curv[:n] = torch.from_numpy(problem.curvature.astype(np.float32))
        self.n = n
        self.zero = getattr(problem, "_zero_grad", False)

    def set_streams(self, seeds, counters=None):
        pass  # deterministic gradient: no sampling

    def gradient(self, G: torch.Tensor, W: torch.Tensor, stream: int) -> None:
        if self.zero:
            G.zero_()
            return
        _lib.check(_lib.load().esgd_quadratic_grad_f32(
            G.data_ptr(), G.stride(0), W.data_ptr(), W.stride(0), W.shape[0], self.target.data_ptr(),
            self.curv.data_ptr(), self.n, stream), "quadratic_grad")


class QuadraticProblem:
    """0.5 (w - target)' D (w - target) with a deterministic gradient
    (reference trainers/problems.py:74-117)."""

    def __init__(self, target, curvature=None):
        self.target = np.asarray(target, dtype=np.float64)
        self.curvature = (np.ones_like(self.target) if curvature is None
                          else np.asarray(curvature, dtype=np.float64))
        self.n_params = self.target.size

    @classmethod
    def random(cls, dim: int, seed: int) -> "QuadraticProblem":
        rng = CounterRng(seed)
        target = rng.normal_block(dim)
        curvature = 0.5 + rng.uniform_block(dim)
        return cls(target, curvature)

    def init_weights(self) -> np.ndarray:
        return np.zeros_like(self.target)

    def gradient(self, weights, rng: CounterRng, batch_size: int) -> np.ndarray:
        dev = require_cuda()
        plan = self.bind(dev, 1, batch_size, round_up(self.n_params, 64))
        W = torch.zeros((1, plan.target.numel()), dtype=torch.float32, device=dev)
        W[0, :self.n_params] = _as_device_row(weights, dev, self.n_params)
        G = torch.zeros_like(W)
        plan.gradient(G, W, stream_ptr())
        return G[0, :self.n_params].cpu().numpy()

    def train_loss(self, weights) -> float:
        w = _host(weights)
        d = w - self.target
        return float(0.5 * np.dot(d, self.curvature * d))

    def distance_to_optimum(self, weights) -> float:
        return float(np.linalg.norm(_host(weights) - self.target))

    def test_accuracy(self, weights) -> float:
        return float("nan")

    def batch_nbytes(self, batch_size: int) -> int:
        return 0

    def layer_nbytes(self) -> list[int]:
        return [self.n_params * 8]

    def fingerprint(self) -> str:
        return f"quadratic-{self.n_params}-{weights_digest(self.target)[:12]}"

    def bind(self, device, nrep: int, batch_size: int, ldw: int, use_tc: bool = True) -> QuadraticPlan:
        return QuadraticPlan(self, device, nrep, batch_size, ldw)


class ZeroGradientProblem(QuadraticProblem):
    """Gradients identically zero; isolates the elastic exchange terms."""

    _zero_grad = True

    def __init__(self, dim: int, init=None, seed: int = 0):
        super().__init__(np.zeros(dim))
        self._init = (CounterRng(seed).normal_block(dim) if init is None
                      else np.asarray(init, dtype=np.float64))

    def init_weights(self) -> np.ndarray:
        return self._init.copy()

    def gradient(self, weights, rng, batch_size):
        return np.zeros(self.n_params)

    def fingerprint(self) -> str:
        return f"zerograd-{self.n_params}"


def _host(weights) -> np.ndarray:
    if isinstance(weights, torch.Tensor):
        return weights.detach().cpu().numpy().astype(np.float64)
    return np.asarray(weights, dtype=np.float64)
