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
