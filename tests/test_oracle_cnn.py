"""The CNN half of the oracle has no reference counterpart, so
it is pinned by identities instead: finite differences of the mean CE loss
(float64, every coordinate of a small net) and im2col/col2im adjointness."""

import numpy as np

from oracle import esgd_oracle as O

TINY = ((2, 7, 6), [("conv", 3, 3, 2, 1, "relu"), ("pool", 2, 1, 0), ("conv", 4, 2, 1, 0, "relu"),
                    ("dense", 5, "tanh"), ("dense", 3, "none")])


def _loss(buf, x, y):
    _, logits = O.forward(*TINY, buf, x)
    return O.softmax_cross_entropy(logits, y)[0]


def test_cnn_gradient_finite_differences():
    rng = np.random.default_rng(0)
    buf = O.build_model(*TINY, seed=3, dtype=np.float64) + 0.05 * rng.standard_normal(
        O.param_views(*TINY)[1])
    x = rng.standard_normal((4, 2 * 7 * 6))
    y = rng.integers(0, 3, 4)
    cache, logits = O.forward(*TINY, buf, x)
    _, dl = O.softmax_cross_entropy(logits, y)
    g = O.backward(*TINY, buf, cache, dl)
    eps = 1e-6
    num = np.empty_like(buf)
    for i in range(buf.size):
        e = np.zeros_like(buf)
        e[i] = eps
        num[i] = (_loss(buf + e, x, y) - _loss(buf - e, x, y)) / (2 * eps)
    assert np.abs(num - g).max() <= 1e-5 * max(1.0, np.abs(num).max())


def test_im2col_col2im_adjoint():
    rng = np.random.default_rng(1)
    x = rng.standard_normal((2, 3, 9, 8))
    col, oh, ow = O._im2col(x, 3, 2, 1)
    y = rng.standard_normal(col.shape)
    lhs = np.sum(col * y)
    rhs = np.sum(x * O._col2im(y, x.shape, 3, 2, 1, oh, ow))
    assert abs(lhs - rhs) < 1e-10 * max(1, abs(lhs))


def test_maxpool_backward_is_routing():
    rng = np.random.default_rng(2)
    x = rng.standard_normal((1, 2, 6, 6))
    y, arg = O._maxpool(x, 3, 2, 1)
    dy = np.ones_like(y)
    dx = O._maxpool_bwd(dy, arg, x.shape)
    assert dx.sum() == y.size
    assert np.all(x.reshape(1, 2, -1)[0, 0, arg[0, 0].ravel()] == y[0, 0].ravel())


def test_reference_param_counts():
    assert O.param_views(*O.LENET)[1] == 431_080
    assert O.param_views(*O.CIFAR_QUICK)[1] == 145_578
    assert O.param_views(*O.alexnet_layers())[1] == 61_100_840


# ---- the oracle's vectorised / threaded data movement == plain per-tap loops

def _im2col_loops(x, k, s, p):
    n, c, h, w = x.shape
    oh, ow = (h + 2 * p - k) // s + 1, (w + 2 * p - k) // s + 1
    xp = np.zeros((n, c, h + 2 * p, w + 2 * p), dtype=x.dtype)
    xp[:, :, p:p + h, p:p + w] = x
    col = np.empty((n, oh, ow, c, k, k), dtype=x.dtype)
    for ky in range(k):
        for kx in range(k):
            col[:, :, :, :, ky, kx] = xp[:, :, ky:ky + s * oh:s, kx:kx + s * ow:s].transpose(0, 2, 3, 1)
    return col.reshape(n * oh * ow, c * k * k), oh, ow


def _col2im_loops(dcol, shape, k, s, p, oh, ow):
    n, c, h, w = shape
    d = dcol.reshape(n, oh, ow, c, k, k)
    dxp = np.zeros((n, c, h + 2 * p, w + 2 * p), dtype=dcol.dtype)
    for ky in range(k):
        for kx in range(k):
            dxp[:, :, ky:ky + s * oh:s, kx:kx + s * ow:s] += d[:, :, :, :, ky, kx].transpose(0, 3, 1, 2)
    return dxp[:, :, p:p + h, p:p + w]


def _maxpool_loops(x, k, s, p):
    n, c, h, w = x.shape
    oh, ow = (h + 2 * p - k) // s + 1, (w + 2 * p - k) // s + 1
    best = np.full((n, c, oh, ow), -np.inf, dtype=x.dtype)
    arg = np.full((n, c, oh, ow), -1, dtype=np.int64)
    for b in range(n):
        for ch in range(c):
            for oy in range(oh):
                for ox in range(ow):
                    for ky in range(k):
                        for kx in range(k):
                            iy, ix = oy * s - p + ky, ox * s - p + kx
                            if 0 <= iy < h and 0 <= ix < w and (arg[b, ch, oy, ox] < 0 or
                                                                 x[b, ch, iy, ix] > best[b, ch, oy, ox]):
                                best[b, ch, oy, ox], arg[b, ch, oy, ox] = x[b, ch, iy, ix], iy * w + ix
    return best, arg


def _maxpool_bwd_loops(dy, arg, shape):
    n, c, h, w = shape
    dx = np.zeros((n, c, h * w), dtype=dy.dtype)
    for oy in range(dy.shape[2]):
        for ox in range(dy.shape[3]):
            for b in range(n):
                for ch in range(c):
                    dx[b, ch, arg[b, ch, oy, ox]] += dy[b, ch, oy, ox]
    return dx.reshape(shape)


import pytest  # noqa: E402


@pytest.mark.parametrize("n,c,h,k,s,p", [(5, 3, 23, 11, 4, 2), (9, 6, 13, 5, 1, 2), (3, 4, 9, 3, 2, 1),
                                         (17, 8, 16, 3, 1, 1), (2, 3, 7, 2, 2, 0)])
def test_fast_data_movement_matches_loops(n, c, h, k, s, p, monkeypatch):
    """bit-identical to the per-tap loops, with the batch split over threads
    (threshold forced to 0 so even these small cases take the threaded path)."""
    monkeypatch.setenv("ESGD_ORACLE_THREADS", "4")
    rng = np.random.default_rng(n * 100 + h)
    x = rng.standard_normal((n, c, h, h)).astype(np.float32)
    x[0, 0, 0, :3] = x[0, 0, 0, 0]  # ties: first max in scan order wins
    orig = O._par
    monkeypatch.setattr(O, "_par", lambda fn, n_, size: orig(fn, n_, 1 << 30))
    col, oh, ow = O._im2col(x, k, s, p)
    ref, _, _ = _im2col_loops(x, k, s, p)
    assert np.array_equal(col, ref)
    d = rng.standard_normal(col.shape).astype(np.float32)
    assert np.array_equal(O._col2im(d, x.shape, k, s, p, oh, ow), _col2im_loops(d, x.shape, k, s, p, oh, ow))
    kp = min(k, 3)
    y, arg = O._maxpool(x, kp, 2, min(p, kp // 2))
    y0, arg0 = _maxpool_loops(x, kp, 2, min(p, kp // 2))
    assert np.array_equal(y, y0) and np.array_equal(arg, arg0)
    dy = rng.standard_normal(y.shape).astype(np.float32)
    assert np.array_equal(O._maxpool_bwd(dy, arg, x.shape), _maxpool_bwd_loops(dy, arg, x.shape))


def test_threaded_engine_equals_simulated():
    """trainers/synchronous.py:156-219 restated: bit-identical to run_sync
    (the reference's tests/test_threaded.py:31-38 property)."""
    rng = np.random.default_rng(4)
    X = rng.standard_normal((60, 2 * 7 * 6))
    Y = rng.integers(0, 3, 60)
    prob = O.NetProblem(*TINY, X, Y, seed=2, dtype=np.float32)
    C0, W0 = O.run_sync(prob, 3, 4, 5, 0.05, 0.25, seed=1)
    C1, W1 = O.run_sync_threaded(prob, 3, 4, 5, 0.05, 0.25, seed=1)
    assert np.array_equal(C0, C1) and all(np.array_equal(a, b) for a, b in zip(W0, W1))
