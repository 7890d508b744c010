"""Model descriptions and the packed single-buffer parameter layout.

``ModelSpec`` is the reference's MLP description (network.py:24-61) with the
same packed layout ``W1 (d0 x d1), b1, W2, b2, ...`` (network.py:116-125)
and Xavier-uniform init from ``CounterRng(mix64(seed ^ 0xE1A57F17))``
(network.py:128-140).

``ConvNetSpec`` adds the north star's CNNs (LeNet, CIFAR-quick, AlexNet),
which the reference does not have. They follow the same
conventions so that one flat buffer carries the whole model:
  * packed order per parameter layer l: W{l} then b{l};
  * conv W shape (out, in, k, k), row-major; dense W shape (in, out);
  * Xavier bound sqrt(6/(fan_in+fan_out)) with conv fan_in = in*k*k and
    fan_out = out*k*k, drawn sequentially across layers in fp64, biases 0;
  * activations are NCHW, the conv->dense flatten is (c, h, w) order;
  * max pooling, argmax = first maximum in (ky, kx) scan order;
  * the last layer is linear (logits feed softmax cross-entropy).
The CPU restatement of these conventions is oracle/esgd_oracle.py.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .errors import InputError, ShapeError, StaleCacheError
from .rng import CounterRng, mix64

ACT_IDS = {"none": 0, "relu": 1, "tanh": 2, "sigmoid": 3}
_INIT_SALT = 0xE1A57F17


# --- MLP (reference ModelSpec) ---------------------------------------------

@dataclass(frozen=True)
class ModelSpec:
    """Layer dims (input, hidden..., output), hidden activation, init seed.

    ``dtype`` is the host dtype of init/returned buffers; the device computes
    in fp32 regardless (libesgd is an fp32 engine).
    """

    dims: tuple[int, ...]
    activation: str | tuple[str, ...] = "relu"
    seed: int = 0
    dtype: np.dtype = np.float64

    def __post_init__(self):
        if len(self.dims) < 2:
            raise InputError("a model needs at least an input and an output dim")
        if any(d < 1 for d in self.dims):
            raise InputError(f"all dims must be >= 1, got {self.dims}")
        for kind in self.hidden_activations():
            if kind not in ("relu", "tanh", "sigmoid"):
                raise InputError(f"unknown activation {kind!r}")

    def hidden_activations(self) -> tuple[str, ...]:
        n_hidden = len(self.dims) - 2
        if isinstance(self.activation, str):
            return (self.activation,) * n_hidden
        if len(self.activation) != n_hidden:
            raise InputError(f"need {n_hidden} activation kinds, got {len(self.activation)}")
        return tuple(self.activation)

    @property
    def num_layers(self) -> int:
        return len(self.dims) - 1

    def parameter_count(self) -> int:
        return sum(fi * fo + fo for fi, fo in zip(self.dims[:-1], self.dims[1:]))

    # uniform description used by the device executor
    def as_layers(self) -> "ConvNetSpec":
        acts = self.hidden_activations() + ("none",)
        layers = tuple(Dense(d, a) for d, a in zip(self.dims[1:], acts))
        return ConvNetSpec((self.dims[0], 1, 1), layers, seed=self.seed, dtype=self.dtype,
                           name=f"mlp{self.dims}")


# --- CNN layers -------------------------------------------------------------

@dataclass(frozen=True)
class Conv:
    out: int
    k: int
    stride: int = 1
    pad: int = 0
    act: str = "none"


@dataclass(frozen=True)
class Pool:
    """Max pooling (k x k window, stride, zero-free padding)."""

    k: int
    stride: int
    pad: int = 0


@dataclass(frozen=True)
class Dense:
    out: int
    act: str = "none"


@dataclass(frozen=True)
class LayerGeom:
    layer: object
    in_shape: tuple[int, int, int]   # (C, H, W)
    out_shape: tuple[int, int, int]
    param_index: int | None          # l of W{l}/b{l}, None for pools


@dataclass(frozen=True)
class ConvNetSpec:
    input_shape: tuple[int, int, int]
    layers: tuple
    seed: int = 0
    dtype: np.dtype = np.float32
    name: str = "convnet"

    def __post_init__(self):
        if not self.layers or not isinstance(self.layers[-1], Dense):
            raise InputError("the last layer must be Dense (logits)")
        if self.layers[-1].act != "none":
            raise InputError("the last layer is linear (logits feed softmax cross-entropy)")
        for lay in self.layers:
            act = getattr(lay, "act", "none")
            if act not in ACT_IDS:
                raise InputError(f"unknown activation {act!r}")
        self.geometry()  # validates shapes

    def geometry(self) -> list[LayerGeom]:
        c, h, w = self.input_shape
        out: list[LayerGeom] = []
        pidx = 0
        flat = False
        for lay in self.layers:
            if isinstance(lay, Conv):
                if flat:
                    raise InputError("Conv after Dense is not supported")
                oh = (h + 2 * lay.pad - lay.k) // lay.stride + 1
                ow = (w + 2 * lay.pad - lay.k) // lay.stride + 1
                if oh < 1 or ow < 1:
                    raise ShapeError(f"conv {lay} produces empty output from {(c, h, w)}")
                pidx += 1
                out.append(LayerGeom(lay, (c, h, w), (lay.out, oh, ow), pidx))
                c, h, w = lay.out, oh, ow
            elif isinstance(lay, Pool):
                if flat:
                    raise InputError("Pool after Dense is not supported")
                if lay.pad >= lay.k:
                    raise InputError("pool padding must be smaller than the window")
                oh = (h + 2 * lay.pad - lay.k) // lay.stride + 1
                ow = (w + 2 * lay.pad - lay.k) // lay.stride + 1
                if oh < 1 or ow < 1:
                    raise ShapeError(f"pool {lay} produces empty output from {(c, h, w)}")
                out.append(LayerGeom(lay, (c, h, w), (c, oh, ow), None))
                h, w = oh, ow
            elif isinstance(lay, Dense):
                fan_in = c * h * w
                pidx += 1
                out.append(LayerGeom(lay, (fan_in, 1, 1), (lay.out, 1, 1), pidx))
                c, h, w = lay.out, 1, 1
                flat = True
            else:
                raise InputError(f"unknown layer {lay!r}")
        return out

    @property
    def input_dim(self) -> int:
        c, h, w = self.input_shape
        return c * h * w

    @property
    def num_classes(self) -> int:
        return self.layers[-1].out

    def parameter_count(self) -> int:
        return sum(v.size for v in view_table(self))

    def flops_per_sample(self) -> int:
        """Forward+backward multiply-adds x2 of the contractions (3x forward)."""
        f = 0
        for g in self.geometry():
            if isinstance(g.layer, Conv):
                _, oh, ow = g.out_shape
                f += 2 * oh * ow * g.layer.out * g.in_shape[0] * g.layer.k ** 2
            elif isinstance(g.layer, Dense):
                f += 2 * g.in_shape[0] * g.layer.out
        return 3 * f


@dataclass
class View:
    name: str
    offset: int
    shape: tuple[int, ...]

    @property
    def size(self) -> int:
        return int(np.prod(self.shape))


def view_table(spec) -> list[View]:
    """Packed layout: alternating W{l}, b{l} views (network.py:116-125)."""
    if isinstance(spec, ModelSpec):
        spec = spec.as_layers()
    views: list[View] = []
    off = 0
    for g in spec.geometry():
        lay = g.layer
        if g.param_index is None:
            continue
        if isinstance(lay, Conv):
            shape = (lay.out, g.in_shape[0], lay.k, lay.k)
        else:
            shape = (g.in_shape[0], lay.out)
        views.append(View(f"W{g.param_index}", off, shape))
        off += int(np.prod(shape))
        views.append(View(f"b{g.param_index}", off, (lay.out,)))
        off += lay.out
    return views


def _fans(spec, v: View) -> tuple[int, int]:
    if len(v.shape) == 4:
        o, i, kh, kw = v.shape
        return i * kh * kw, o * kh * kw
    return v.shape[0], v.shape[1]


class PackedWeights:
    """Contiguous parameter buffer plus the per-layer view table (reference
    network.py:80-113): views are disjoint, contiguous and cover the buffer
    exactly; a tensor from :meth:`view` writes through to its slice. The
    buffer may be a host ndarray or a device tensor of the same layout."""

    def __init__(self, buffer, views: list[View]):
        covered = 0
        for v in views:
            if v.offset != covered:
                raise ShapeError(f"view {v.name} at offset {v.offset}, expected {covered}")
            covered += v.size
        size = buffer.numel() if hasattr(buffer, "numel") else buffer.size
        if covered != size:
            raise ShapeError(f"views cover {covered} elements, buffer has {size}")
        self.buffer = buffer
        self.views = views

    def view(self, name: str):
        for v in self.views:
            if v.name == name:
                return self.buffer[v.offset:v.offset + v.size].reshape(v.shape)
        raise KeyError(name)

    def clone(self) -> "PackedWeights":
        return PackedWeights(self.buffer.clone() if hasattr(self.buffer, "clone") else self.buffer.copy(),
                             self.views)

    @property
    def size(self) -> int:
        return int(self.buffer.numel() if hasattr(self.buffer, "numel") else self.buffer.size)

    @property
    def nbytes(self) -> int:
        return int(self.size * (self.buffer.element_size() if hasattr(self.buffer, "element_size")
                                else self.buffer.itemsize))


def packed_weights_for(spec, buffer) -> PackedWeights:
    """Wrap an existing flat buffer in the view table of ``spec`` (network.py:236-242)."""
    expected = spec.parameter_count()
    size = buffer.numel() if hasattr(buffer, "numel") else np.asarray(buffer).size
    if size != expected:
        raise ShapeError(f"buffer size {size} != layout size {expected}")
    if not hasattr(buffer, "numel"):
        buffer = np.ascontiguousarray(buffer, dtype=spec.dtype)
    return PackedWeights(buffer, view_table(spec))


def build_model(spec) -> PackedWeights:
    """Xavier-uniform weights, zero biases, deterministic in ``spec.seed``
    (network.py:128-140; sequential draws across layers), as PackedWeights
    over a host buffer; ``init_buffer`` returns the flat buffer alone."""
    return PackedWeights(init_buffer(spec), view_table(spec))


@dataclass
class ForwardCache:
    """What backward needs from a forward pass (network.py:144-150): here the
    device executor that ran it, holding the activations in HBM."""

    net: object
    weights_token: int
    spec: object
    W: object


def _device_batch(spec, weights: PackedWeights, batch):
    import torch

    from .device import require_cuda
    from .nets import DeviceNet

    dev = require_cuda()
    batch = np.asarray(batch, dtype=np.float32)
    d_in = spec.input_dim if isinstance(spec, ConvNetSpec) else spec.dims[0]
    if batch.ndim != 2 or batch.shape[1] != d_in:
        raise InputError(f"batch shape {batch.shape} does not match input dim {d_in}")
    n = spec.parameter_count()
    net = DeviceNet(spec, batch.shape[0], 1, dev)
    W = torch.zeros((1, net.ldw), dtype=torch.float32, device=dev)
    buf = weights.buffer
    W[0, :n] = (buf.to(dev, torch.float32) if hasattr(buf, "numel")
                else torch.from_numpy(np.ascontiguousarray(buf, dtype=np.float32)).to(dev))
    net.x[0, :batch.size] = torch.from_numpy(batch.reshape(-1)).to(dev)
    return net, W


def forward(spec, weights: PackedWeights, batch) -> tuple[ForwardCache, np.ndarray]:
    """Run the network on a (b, input_dim) batch on the device; returns
    (cache, logits) like the reference (network.py:153-173)."""
    import torch

    from .device import stream_ptr

    net, W = _device_batch(spec, weights, batch)
    logits = net.forward(W, stream_ptr())
    out = logits[0, :net.b * net.classes].reshape(net.b, net.classes).cpu().numpy()
    torch.cuda.synchronize()
    return ForwardCache(net, id(weights), spec, W), out.astype(spec.dtype)


def backward(spec, weights: PackedWeights, cache: ForwardCache, dlogits) -> np.ndarray:
    """Gradient of the loss w.r.t. every packed parameter for the logits'
    gradient ``dlogits`` (network.py:176-200): one buffer of the packed layout."""
    import torch

    from .device import stream_ptr

    if cache.weights_token != id(weights) or cache.spec is not spec:
        raise StaleCacheError("cache was produced by a different forward pass")
    net = cache.net
    dl = np.asarray(dlogits, dtype=np.float32)
    if dl.shape != (net.b, net.classes):
        raise ShapeError(f"dlogits shape {dl.shape} != logits shape {(net.b, net.classes)}")
    net.outs[-1][0, :dl.size] = torch.from_numpy(dl.reshape(-1)).to(net.device)
    G = torch.zeros_like(cache.W)
    net.backward(G, cache.W, stream_ptr())
    return G[0, :spec.parameter_count()].cpu().numpy().astype(spec.dtype)


def init_buffer(spec) -> np.ndarray:
    """Flat host buffer: Xavier-uniform weights, zero biases, deterministic in
    ``spec.seed`` (network.py:128-140; sequential draws across layers)."""
    views = view_table(spec)
    total = sum(v.size for v in views)
    dtype = spec.dtype
    buf = np.zeros(total, dtype=dtype)
    rng = CounterRng(mix64(spec.seed ^ _INIT_SALT))
    for v in views:
        if not v.name.startswith("W"):
            continue
        fan_in, fan_out = _fans(spec, v)
        bound = np.sqrt(6.0 / (fan_in + fan_out))
        w = (rng.uniform_block(v.size) * 2.0 - 1.0) * bound
        buf[v.offset:v.offset + v.size] = w.astype(dtype)
    return buf


def view(spec, buffer: np.ndarray, name: str) -> np.ndarray:
    for v in view_table(spec):
        if v.name == name:
            return buffer[v.offset:v.offset + v.size].reshape(v.shape)
    raise KeyError(name)


# --- the north star's models ----------------------------------------------------

def lenet(seed: int = 0, dtype=np.float32) -> ConvNetSpec:
    """Caffe LeNet: conv20-5, pool2, conv50-5, pool2, fc500+relu, fc10
    (431,080 parameters)."""
    return ConvNetSpec((1, 28, 28), (
        Conv(20, 5), Pool(2, 2), Conv(50, 5), Pool(2, 2), Dense(500, "relu"), Dense(10),
    ), seed=seed, dtype=dtype, name="lenet")


def cifar_quick(seed: int = 0, dtype=np.float32) -> ConvNetSpec:
    """CIFAR-quick: three conv5x5(pad 2)+relu+maxpool3/2(pad 1) stages
    (32, 32, 64 maps), fc64, fc10 (145,578 parameters)."""
    return ConvNetSpec((3, 32, 32), (
        Conv(32, 5, pad=2, act="relu"), Pool(3, 2, 1),
        Conv(32, 5, pad=2, act="relu"), Pool(3, 2, 1),
        Conv(64, 5, pad=2, act="relu"), Pool(3, 2, 1),
        Dense(64, "relu"), Dense(10),
    ), seed=seed, dtype=dtype, name="cifar-quick")


def alexnet(seed: int = 0, dtype=np.float32, num_classes: int = 1000) -> ConvNetSpec:
    """AlexNet at 224x224 (torchvision shapes, no dropout; 61,100,840
    parameters for 1000 classes)."""
    return ConvNetSpec((3, 224, 224), (
        Conv(64, 11, stride=4, pad=2, act="relu"), Pool(3, 2),
        Conv(192, 5, pad=2, act="relu"), Pool(3, 2),
        Conv(384, 3, pad=1, act="relu"),
        Conv(256, 3, pad=1, act="relu"),
        Conv(256, 3, pad=1, act="relu"), Pool(3, 2),
        Dense(4096, "relu"), Dense(4096, "relu"), Dense(num_classes),
    ), seed=seed, dtype=dtype, name="alexnet")


MODELS = {"lenet": lenet, "cifar-quick": cifar_quick, "alexnet": alexnet}


# EFW1 checkpoints (reference network.py:203-233), implemented in formats.py
from .formats import load_weights, save_weights  # noqa: E402,F401
