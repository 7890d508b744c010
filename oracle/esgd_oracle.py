"""CPU ORACLE — test infrastructure only, never the product path.

A plain-numpy restatement of the reference package ``elasticsgd``
(/root/reference/pkg/src/elasticsgd, cited below as ``file:line``) for the
north-star path: counter RNG, synthetic data + sampling, the dense network,
softmax cross-entropy, the update rules, the fixed-order tree sum and the
Sync-EASGD round loop. Plus the CNN layers (conv / max-pool) the reference
does not have, restated under the conventions documented in
paper_1708_02983_b200/network.py.

Pinning: tests/test_oracle_golden.py checks every function here against
golden vectors produced by running the real reference in this container
(oracle/make_golden.py -> tests/golden/*.npz). The CNN functions have no
reference counterpart: parity for them is "unpinned" beyond the shared
dense/loss/update pieces and the adjoint / finite-difference identities
tested in tests/test_oracle_cnn.py.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module.
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
from numpy.lib.stride_tricks import sliding_window_view

# ---------------------------------------------------------------------------
# rng.py:30-105
GOLDEN = 0x9E3779B97F4A7C15
MASK64 = (1 << 64) - 1


def mix64(x: int) -> int:
    """rng.py:37-42"""
    z = x & MASK64
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9 & MASK64
    z = (z ^ (z >> 27)) * 0x94D049BB133111EB & MASK64
    return z ^ (z >> 31)


def mix64_vec(z: np.ndarray) -> np.ndarray:
    """rng.py:44-49"""
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def stream_seed(seed: int, worker_id: int) -> int:
    """rng.py:52-54"""
    return mix64(mix64(seed) ^ (worker_id + 1))


class CounterRng:
    """rng.py:57-100"""

    def __init__(self, seed: int, counter: int = 0):
        self.seed = seed & MASK64
        self.counter = counter

    def raw(self, n: int) -> np.ndarray:
        with np.errstate(over="ignore"):
            idx = np.arange(self.counter + 1, self.counter + n + 1, dtype=np.uint64)
            self.counter += n
            return mix64_vec(np.uint64(self.seed) + idx * np.uint64(GOLDEN))

    def uniform_block(self, n: int) -> np.ndarray:
        return (self.raw(n) >> np.uint64(11)).astype(np.float64) * 2.0**-53

    def randint_block(self, n: int, upper: int) -> np.ndarray:
        return (self.raw(n) % np.uint64(upper)).astype(np.int64)

    def randint(self, upper: int) -> int:
        return int(self.randint_block(1, upper)[0])

    def normal_block(self, n: int) -> np.ndarray:
        u1 = ((self.raw(n) >> np.uint64(11)).astype(np.float64) + 1.0) * 2.0**-53
        u2 = self.uniform_block(n)
        return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)


def worker_rng(seed: int, w: int) -> CounterRng:
    """rng.py:103-105"""
    return CounterRng(stream_seed(seed, w))


# ---------------------------------------------------------------------------
# datasets.py:129-171

def gen_synthetic(classes, dim, per_class, seed, separation=6.0):
    """datasets.py:129-147 -> (samples float64 (n, dim), labels int64)"""
    rng = CounterRng(seed)
    n = classes * per_class
    noise = rng.normal_block(n * dim).reshape(n, dim)
    labels = np.repeat(np.arange(classes, dtype=np.int64), per_class)
    means = np.zeros((classes, dim))
    means[np.arange(classes), np.arange(classes)] = separation
    return means[labels] + noise, labels


def normalize(samples):
    """datasets.py:150-163"""
    mean = samples.mean(axis=0)
    std = samples.std(axis=0)
    scale = np.where(std > 0.0, std, 1.0)
    out = (samples - mean) / scale
    out[:, std == 0.0] = 0.0
    return out


def sample_batch(samples, labels, b, rng):
    """datasets.py:166-171"""
    idx = rng.randint_block(b, samples.shape[0])
    return samples[idx], labels[idx]


# ---------------------------------------------------------------------------
# kernels.py:30-106

def relu(z):
    return np.maximum(z, 0.0)


def relu_grad(z):
    return (z > 0).astype(z.dtype)


def tanh_grad(z):
    t = np.tanh(z)
    return 1.0 - t * t


def sigmoid(z):
    out = np.empty_like(z)
    pos = z >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-z[pos]))
    ez = np.exp(z[~pos])
    out[~pos] = ez / (1.0 + ez)
    return out


def sigmoid_grad(z):
    s = sigmoid(z)
    return s * (1.0 - s)


ACT = {"relu": (relu, relu_grad), "tanh": (np.tanh, tanh_grad), "sigmoid": (sigmoid, sigmoid_grad),
       "none": (lambda z: z, lambda z: np.ones_like(z))}


def softmax_cross_entropy(logits, labels):
    """kernels.py:85-106 -> (mean loss, dlogits)"""
    rows = logits.shape[0]
    shifted = logits - logits.max(axis=1, keepdims=True)
    e = np.exp(shifted)
    probs = e / e.sum(axis=1, keepdims=True)
    picked = probs[np.arange(rows), labels]
    loss = float(-np.log(picked).mean())
    d = probs.copy()
    d[np.arange(rows), labels] -= 1.0
    d /= rows
    return loss, d


def row_losses(logits, labels):
    shifted = logits - logits.max(axis=1, keepdims=True)
    e = np.exp(shifted)
    probs = e / e.sum(axis=1, keepdims=True)
    return -np.log(probs[np.arange(logits.shape[0]), labels])


# ---------------------------------------------------------------------------
# Layer description shared by the MLP and the CNNs:
#   ("conv", out, k, stride, pad, act) | ("pool", k, stride, pad) | ("dense", out, act)

def mlp_layers(dims, activation="relu"):
    acts = [activation] * (len(dims) - 2) if isinstance(activation, str) else list(activation)
    acts = acts + ["none"]
    return (dims[0], 1, 1), [("dense", d, a) for d, a in zip(dims[1:], acts)]


LENET = ((1, 28, 28), [("conv", 20, 5, 1, 0, "none"), ("pool", 2, 2, 0),
                       ("conv", 50, 5, 1, 0, "none"), ("pool", 2, 2, 0),
                       ("dense", 500, "relu"), ("dense", 10, "none")])
CIFAR_QUICK = ((3, 32, 32), [("conv", 32, 5, 1, 2, "relu"), ("pool", 3, 2, 1),
                             ("conv", 32, 5, 1, 2, "relu"), ("pool", 3, 2, 1),
                             ("conv", 64, 5, 1, 2, "relu"), ("pool", 3, 2, 1),
                             ("dense", 64, "relu"), ("dense", 10, "none")])


def alexnet_layers(classes=1000):
    return ((3, 224, 224), [("conv", 64, 11, 4, 2, "relu"), ("pool", 3, 2, 0),
                            ("conv", 192, 5, 1, 2, "relu"), ("pool", 3, 2, 0),
                            ("conv", 384, 3, 1, 1, "relu"), ("conv", 256, 3, 1, 1, "relu"),
                            ("conv", 256, 3, 1, 1, "relu"), ("pool", 3, 2, 0),
                            ("dense", 4096, "relu"), ("dense", 4096, "relu"),
                            ("dense", classes, "none")])


def param_views(input_shape, layers):
    """Packed layout W{l}, b{l} per parameter layer (network.py:116-125
    generalised: conv W (out, in, k, k), dense W (in, out))."""
    c, h, w = input_shape
    views, off = [], 0
    for L in layers:
        if L[0] == "conv":
            _, o, k, s, p, _a = L
            views.append(((o, c, k, k), off)); off += o * c * k * k
            views.append(((o,), off)); off += o
            c, h, w = o, (h + 2 * p - k) // s + 1, (w + 2 * p - k) // s + 1
        elif L[0] == "pool":
            _, k, s, p = L
            h, w = (h + 2 * p - k) // s + 1, (w + 2 * p - k) // s + 1
        else:
            _, o, _a = L
            fan = c * h * w
            views.append(((fan, o), off)); off += fan * o
            views.append(((o,), off)); off += o
            c, h, w = o, 1, 1
    return views, off


def build_model(input_shape, layers, seed, dtype):
    """network.py:128-140: Xavier-uniform from CounterRng(mix64(seed ^ 0xE1A57F17)),
    sequential draws across layers in fp64, cast, zero biases."""
    views, total = param_views(input_shape, layers)
    buf = np.zeros(total, dtype=dtype)
    rng = CounterRng(mix64(seed ^ 0xE1A57F17))
    for shape, off in views[0::2]:
        if len(shape) == 4:
            o, i, kh, kw = shape
            fi, fo = i * kh * kw, o * kh * kw
        else:
            fi, fo = shape
        size = int(np.prod(shape))
        bound = np.sqrt(6.0 / (fi + fo))
        buf[off:off + size] = ((rng.uniform_block(size) * 2.0 - 1.0) * bound).astype(dtype)
    return buf


# Data-movement helpers of the CNN restatement. They are pure copies / fixed-
# order accumulations, written with strided views and split over the batch
# across host threads (ESGD_ORACLE_THREADS, default all cores): per element the
# values and the accumulation order are those of the plain per-tap loops
# (tests/test_oracle_cnn.py pins them against those loops), only faster, so the
# CPU baseline is not dominated by slow numpy indexing.
_POOL = None


def _nthreads():
    return max(1, int(os.environ.get("ESGD_ORACLE_THREADS", os.cpu_count() or 1)))


def _par(fn, n, size):
    """fn(a, b) over batch chunks [a, b) on the thread pool (one chunk when small)."""
    global _POOL
    t = min(_nthreads(), n) if size >= (1 << 20) else 1
    bounds = np.linspace(0, n, t + 1).astype(int)
    chunks = [(int(bounds[i]), int(bounds[i + 1])) for i in range(t) if bounds[i + 1] > bounds[i]]
    if len(chunks) == 1:
        fn(*chunks[0])
        return
    if _POOL is None:
        _POOL = ThreadPoolExecutor(_nthreads())
    list(_POOL.map(lambda c: fn(*c), chunks))


def _im2col(x, k, s, p):
    """x (n, c, h, w) -> col (n*oh*ow, c*k*k) with column order (ci, ky, kx)."""
    n, c, h, w = x.shape
    oh, ow = (h + 2 * p - k) // s + 1, (w + 2 * p - k) // s + 1
    col = np.empty((n, oh, ow, c, k, k), dtype=x.dtype)

    def part(a, b):
        xp = np.zeros((b - a, c, h + 2 * p, w + 2 * p), dtype=x.dtype)
        xp[:, :, p:p + h, p:p + w] = x[a:b]
        v = sliding_window_view(xp, (k, k), axis=(2, 3))[:, :, ::s, ::s][:, :, :oh, :ow]
        col[a:b] = v.transpose(0, 2, 3, 1, 4, 5)

    _par(part, n, col.size)
    return col.reshape(n * oh * ow, c * k * k), oh, ow


def _col2im(dcol, shape, k, s, p, oh, ow):
    """Adjoint of _im2col; accumulation order per input element is (ky, kx)."""
    n, c, h, w = shape
    d = dcol.reshape(n, oh, ow, c, k, k)
    dx = np.empty((n, c, h, w), dtype=dcol.dtype)

    def part(a, b):
        dT = np.ascontiguousarray(d[a:b].transpose(0, 3, 4, 5, 1, 2))  # (m, c, k, k, oh, ow)
        dxp = np.zeros((b - a, c, h + 2 * p, w + 2 * p), dtype=dcol.dtype)
        for ky in range(k):
            for kx in range(k):
                dxp[:, :, ky:ky + s * oh:s, kx:kx + s * ow:s] += dT[:, :, ky, kx]
        dx[a:b] = dxp[:, :, p:p + h, p:p + w]

    _par(part, n, dcol.size)
    return dx


def _maxpool(x, k, s, p):
    """max over k x k windows (padding excluded); argmax = first max in
    (ky, kx) scan order, as flat h*W+w of the input plane."""
    n, c, h, w = x.shape
    oh, ow = (h + 2 * p - k) // s + 1, (w + 2 * p - k) // s + 1
    best = np.empty((n, c, oh, ow), dtype=x.dtype)
    arg = np.empty((n, c, oh, ow), dtype=np.int64)

    def part(a, b):
        m = b - a
        hp, wp = max(h + 2 * p, (oh - 1) * s + k), max(w + 2 * p, (ow - 1) * s + k)
        xp = np.full((m, c, hp, wp), -np.inf, dtype=x.dtype)
        xp[:, :, p:p + h, p:p + w] = x[a:b]
        bst = np.full((m, c, oh, ow), -np.inf, dtype=x.dtype)
        ag = np.full((m, c, oh, ow), -1, dtype=np.int64)
        for ky in range(k):
            for kx in range(k):
                iy = np.arange(oh) * s - p + ky
                ix = np.arange(ow) * s - p + kx
                valid = ((iy >= 0) & (iy < h))[:, None] & ((ix >= 0) & (ix < w))[None, :]
                cand = xp[:, :, ky:ky + s * (oh - 1) + 1:s, kx:kx + s * (ow - 1) + 1:s]
                cand = np.where(valid, cand, -np.inf).astype(x.dtype, copy=False)
                upd = (cand > bst) | ((ag < 0) & valid)
                np.copyto(bst, cand, where=upd)
                np.copyto(ag, np.broadcast_to(iy[:, None] * w + ix[None, :], ag.shape), where=upd)
        best[a:b], arg[a:b] = bst, ag

    _par(part, n, x.size)
    return best, arg


def _maxpool_bwd(dy, arg, shape):
    """dx[argmax] += dy, outputs visited in (oy, ox) order (the device's
    gather order)."""
    n, c, h, w = shape
    oh, ow = dy.shape[2:]
    dx = np.zeros((n, c, h * w), dtype=dy.dtype)

    def part(a, b):
        sub = dx[a:b]
        nn, cc = np.meshgrid(np.arange(b - a), np.arange(c), indexing="ij")
        for oy in range(oh):
            for ox in range(ow):
                # one target per (n, c) plane per output: no duplicate indices
                sub[nn, cc, arg[a:b, :, oy, ox]] += dy[a:b, :, oy, ox]

    _par(part, n, dx.size)
    return dx.reshape(n, c, h, w)


def forward(input_shape, layers, buf, x):
    """x (b, C*H*W) CHW-flat -> (cache, logits). NCHW activations, the
    conv->dense flatten in (c, h, w) order."""
    views, _ = param_views(input_shape, layers)
    b = x.shape[0]
    a = x.reshape(b, *input_shape)
    cache = []
    vi = 0
    for L in layers:
        if L[0] == "conv":
            _, o, k, s, p, act = L
            (ws, wo), (bs, bo) = views[vi], views[vi + 1]; vi += 2
            W = buf[wo:wo + int(np.prod(ws))].reshape(o, -1)
            bias = buf[bo:bo + o]
            col, oh, ow = _im2col(a, k, s, p)
            z = col @ W.T + bias                      # (b*oh*ow, o)
            z = z.reshape(b, oh, ow, o).transpose(0, 3, 1, 2)
            out = ACT[act][0](z)
            cache.append(("conv", a, col, z, L))
        elif L[0] == "pool":
            _, k, s, p = L
            out, arg = _maxpool(a, k, s, p)
            cache.append(("pool", a, arg, None, L))
        else:
            _, o, act = L
            (ws, wo), (bs, bo) = views[vi], views[vi + 1]; vi += 2
            W = buf[wo:wo + ws[0] * ws[1]].reshape(ws)
            bias = buf[bo:bo + o]
            xin = a.reshape(b, -1)
            z = xin @ W + bias                        # network.py:166
            out = ACT[act][0](z)
            cache.append(("dense", xin, None, z, L))
        a = out
    return cache, a


def backward(input_shape, layers, buf, cache, dlogits):
    """network.py:176-200 generalised to conv/pool; one packed gradient."""
    views, total = param_views(input_shape, layers)
    grad = np.zeros(total, dtype=buf.dtype)
    vidx = [i for i, L in enumerate(layers) if L[0] != "pool"]
    first = vidx[0]
    delta = dlogits
    for li in range(len(layers) - 1, -1, -1):
        kind, xin, aux, z, L = cache[li]
        if kind == "dense":
            vi = 2 * vidx.index(li)
            (ws, wo), (bs, bo) = views[vi], views[vi + 1]
            W = buf[wo:wo + ws[0] * ws[1]].reshape(ws)
            grad[wo:wo + ws[0] * ws[1]] = (xin.T @ delta).reshape(-1)
            grad[bo:bo + L[1]] = delta.sum(axis=0)
            if li > first:
                d_in = delta @ W.T
                prev_z, prev_act = _producer(cache, layers, li)
                if prev_act is not None:
                    d_in = d_in.reshape(prev_z.shape) * ACT[prev_act][1](prev_z)
                delta = d_in  # consumers (pool / conv / dense) reshape as they need
        elif kind == "pool":
            _, k, s, p = L
            delta = delta.reshape(_out_shape(cache, li))
            d_in = _maxpool_bwd(delta, aux, xin.shape)
            prev_z, prev_act = _producer(cache, layers, li)
            if prev_act is not None:
                d_in = d_in * ACT[prev_act][1](prev_z)
            delta = d_in
        else:
            _, o, k, s, p, act = L
            vi = 2 * vidx.index(li)
            (ws, wo), (bs, bo) = views[vi], views[vi + 1]
            W = buf[wo:wo + int(np.prod(ws))].reshape(o, -1)
            b, _, oh, ow = z.shape
            dz = delta.reshape(b, o, oh, ow).transpose(0, 2, 3, 1).reshape(-1, o)
            grad[wo:wo + W.size] = (dz.T @ aux).reshape(-1)
            grad[bo:bo + o] = dz.sum(axis=0)
            if li > first:
                dcol = dz @ W
                d_in = _col2im(dcol, xin.shape, k, s, p, oh, ow)
                prev_z, prev_act = _producer(cache, layers, li)
                if prev_act is not None:
                    d_in = d_in * ACT[prev_act][1](prev_z)
                delta = d_in
    return grad


def _producer(cache, layers, li):
    """(pre-activation, activation) of the layer that produced layer li's
    input, or (None, None) when no activation derivative applies."""
    if li == 0:
        return None, None
    kind, _, _, z, L = cache[li - 1]
    if kind == "pool":
        return None, None
    act = L[-1]
    if act == "none":
        return None, None
    return z, act


def _out_shape(cache, li):
    kind, xin, aux, z, L = cache[li]
    if kind == "pool":
        return aux.shape
    return z.shape


def gradient(input_shape, layers, buf, samples, labels, b, rng):
    """NetworkProblem.gradient (trainers/problems.py:42-47)"""
    xb, yb = sample_batch(samples, labels, b, rng)
    xb = np.asarray(xb, dtype=buf.dtype)
    cache, logits = forward(input_shape, layers, buf, xb)
    _, dl = softmax_cross_entropy(logits, yb)
    return backward(input_shape, layers, buf, cache, dl)


# ---------------------------------------------------------------------------
# updates.py:71-154 (pure; scalars are weak Python floats -> cast at use)

def sgd_step(w, g, eta):
    return w - eta * g


def msgd_step(w, v, g, eta, mu):
    v_new = mu * v - eta * g
    return w + v_new, v_new


def easgd_worker_step(w, g, c, eta, rho):
    """updates.py:85-93"""
    return (w - eta * g) - (eta * rho) * (w - c)


def easgd_center_step_from_sum(c, s, p, eta, rho):
    """updates.py:113-119"""
    return c + (eta * rho) * (s - p * c)


def easgd_center_step(c, snaps, eta, rho):
    """updates.py:96-110"""
    total = np.zeros_like(c)
    for s in snaps:
        total += s - c
    return c + (eta * rho) * total


def easgd_center_incremental(c, w, eta, rho):
    """updates.py:122-131"""
    return c + (eta * rho) * (w - c)


def measgd_worker_step(w, v, g, c, eta, mu, rho):
    """updates.py:134-140"""
    v_new = mu * v - eta * g
    return (w + v_new) - (eta * rho) * (w - c), v_new


def tree_sum(buffers):
    """fabric/collectives.py:18-32"""
    partial = [b.copy() for b in buffers]
    d = 1
    while d < len(buffers):
        for pos in range(0, len(buffers), 2 * d):
            if pos + d < len(buffers):
                partial[pos] = partial[pos] + partial[pos + d]
        d *= 2
    return partial[0]


def grouped_tree_sum(buffers, groups):
    """trainers/synchronous.py:50-54"""
    size = len(buffers) // groups
    return tree_sum([tree_sum(buffers[g * size:(g + 1) * size]) for g in range(groups)])


# ---------------------------------------------------------------------------
# problems restated for the trainer loop

class NetProblem:
    def __init__(self, input_shape, layers, samples, labels, seed=0, dtype=np.float32):
        self.input_shape, self.layers = input_shape, layers
        self.samples = np.asarray(samples, dtype=dtype)
        self.labels = np.asarray(labels, dtype=np.int64)
        self.seed, self.dtype = seed, dtype

    def init_weights(self):
        return build_model(self.input_shape, self.layers, self.seed, self.dtype)

    def gradient(self, w, rng, b):
        return gradient(self.input_shape, self.layers, w, self.samples, self.labels, b, rng)

    def loss(self, w, k=1024):
        _, logits = forward(self.input_shape, self.layers, w, self.samples[:k])
        return softmax_cross_entropy(logits, self.labels[:k])[0]


class QuadProblem:
    """trainers/problems.py:74-117 in a chosen dtype"""

    def __init__(self, target, curvature, dtype=np.float64):
        self.target = np.asarray(target, dtype=dtype)
        self.curvature = np.asarray(curvature, dtype=dtype)

    @classmethod
    def random(cls, dim, seed, dtype=np.float64):
        rng = CounterRng(seed)
        t = rng.normal_block(dim)
        c = 0.5 + rng.uniform_block(dim)
        return cls(t, c, dtype)

    def init_weights(self):
        return np.zeros_like(self.target)

    def gradient(self, w, rng, b):
        return self.curvature * (w - self.target)


# ---------------------------------------------------------------------------
# trainers/synchronous.py:57-64, 75-153 (arithmetic only; no pricing)

def run_sync(problem, workers, iterations, batch_size, eta, rho, seed, groups=1, on_round=None,
             state=None):
    """state = (C, W, t0) starts from a given round-t0 state (the workers'
    RNG counters at t0*batch_size); on_round(t, C, W) sees every state."""
    if state is None:
        init = problem.init_weights()
        W = [init.copy() for _ in range(workers)]
        C, t0 = init.copy(), 0
    else:
        C, W, t0 = state[0].copy(), [w.copy() for w in state[1]], state[2]
    rngs = [CounterRng(stream_seed(seed, w), t0 * batch_size) for w in range(workers)]
    for t in range(t0, t0 + iterations):
        grads = [problem.gradient(W[i], rngs[i], batch_size) for i in range(workers)]
        s = grouped_tree_sum(W, groups)
        W = [easgd_worker_step(w, g, C, eta, rho) for w, g in zip(W, grads)]
        C = easgd_center_step_from_sum(C, s, workers, eta, rho)
        if on_round is not None:
            on_round(t + 1, C, W)
    return C, W


# ---------------------------------------------------------------------------
# fabric/engine.py:156-189

def hogwild_apply(center, delta):
    center += delta


def interleaved_apply(center, delta_fns, rng, num_blocks=8):
    fns = list(delta_fns)
    if not fns:
        return
    bounds = np.linspace(0, center.size, min(num_blocks, center.size) + 1).astype(int)
    for blk in range(len(bounds) - 1):
        sl = slice(int(bounds[blk]), int(bounds[blk + 1]))
        order = list(range(len(fns)))
        for i in range(len(order) - 1, 0, -1):
            j = rng.randint(i + 1)
            order[i], order[j] = order[j], order[i]
        for i in order:
            center[sl] += fns[i](center[sl], sl)


# ---------------------------------------------------------------------------
# trainers/synchronous.py:156-219 (the reference's threaded engine: one OS
# thread per worker, three barriers per round, thread 0 sums in tree order and
# steps the center; the worker step uses the pre-update center snapshot)

def run_sync_threaded(problem, workers, iterations, batch_size, eta, rho, seed, groups=1):
    import threading

    rngs = [worker_rng(seed, w) for w in range(workers)]
    init = problem.init_weights()
    W = [init.copy() for _ in range(workers)]
    grads = [None] * workers
    shared = {"center": init.copy(), "snap": None, "failure": None}
    barrier = threading.Barrier(workers)

    def body(w):
        try:
            for _ in range(iterations):
                grads[w] = problem.gradient(W[w], rngs[w], batch_size)
                barrier.wait()
                if w == 0:
                    s = grouped_tree_sum(W, groups)
                    shared["snap"] = shared["center"]
                    shared["center"] = easgd_center_step_from_sum(shared["center"], s, workers, eta, rho)
                barrier.wait()
                W[w] = easgd_worker_step(W[w], grads[w], shared["snap"], eta, rho)
                barrier.wait()
        except Exception as exc:  # surfaced to the caller (synchronous.py:209-210)
            shared["failure"] = exc
            barrier.abort()

    threads = [threading.Thread(target=body, args=(w,)) for w in range(workers)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    if shared["failure"] is not None:
        raise shared["failure"]
    return shared["center"], W
