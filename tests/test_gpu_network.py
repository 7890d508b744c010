"""Per-worker gradient on the B200 vs the reference (MLP, golden fixtures)
and vs the pinned oracle (CNNs). fp32 device math; tolerance 1e-5 relative
(BASELINE.json north_star)."""

import numpy as np
import pytest
import torch

from oracle import esgd_oracle as O
from paper_1708_02983_b200 import ModelSpec, network
from paper_1708_02983_b200.datasets import Dataset
from paper_1708_02983_b200.rng import CounterRng, worker_rng
from paper_1708_02983_b200.trainers import NetworkProblem
from _gpu_util import rel_err

pytestmark = pytest.mark.gpu
TOL = 1e-5


@pytest.mark.parametrize("act", ["relu", "tanh", "sigmoid"])
def test_mlp_gradient_vs_reference(golden, act):
    g = golden("net")
    spec = ModelSpec((32, 24, 16, 10), activation=act, seed=1, dtype=np.float32)
    prob = NetworkProblem(spec, Dataset(g["train_x"], g["train_y"], 10), Dataset(g["test_x"], g["test_y"], 10))
    w = prob.init_weights()
    assert np.array_equal(w, g[f"float32_{act}_init"])
    rng = worker_rng(3, 0)
    g1 = prob.gradient(w, rng, 16)
    g2 = prob.gradient(w, rng, 16)
    assert rng.counter == 32
    assert rel_err(g1, g[f"float32_{act}_grad"]) < TOL
    assert rel_err(g2, g[f"float32_{act}_grad2"]) < TOL
    assert abs(prob.train_loss(w) - g[f"float32_{act}_loss"][0]) < 1e-5 * max(1, abs(g[f"float32_{act}_loss"][0]))


def _cnn_case(spec, layers, n, b, seed=0):
    rng = np.random.default_rng(seed)
    d = spec.input_dim
    X = rng.standard_normal((n, d)).astype(np.float64)
    Y = rng.integers(0, spec.num_classes, n).astype(np.int64)
    prob = NetworkProblem(spec, Dataset(X, Y, spec.num_classes))
    w = prob.init_weights()
    shape, lay = layers
    ow = O.build_model(shape, lay, spec.seed, np.float32)
    assert np.array_equal(w, ow), "init layout/draw order differs from the oracle"
    # perturb biases so every path is exercised with nonzero values
    w = w + np.float32(0.01) * rng.standard_normal(w.size).astype(np.float32)
    g_dev = prob.gradient(w, CounterRng(77), b)
    oprob = O.NetProblem(shape, lay, X, Y, seed=spec.seed, dtype=np.float32)
    g_ref = oprob.gradient(w, O.CounterRng(77), b)
    return g_dev, g_ref


@pytest.fixture(params=["tcgen05", "default", "ffma", "implicit"])
def gemm_routing(request, monkeypatch):
    """'tcgen05' sends every contraction above 4M MACs to the tensor-core
    kernel (so small test batches exercise it); 'default' is the engine's
    production routing; 'ffma' forces the CUDA-core FFMA kernel; 'implicit'
    additionally runs the tensor-core conv layers as implicit GEMMs
    (esgd_tc_conv_f32, no im2col / col2im)."""
    from paper_1708_02983_b200 import nets
    if request.param in ("tcgen05", "implicit"):
        monkeypatch.setattr(nets, "TC_MIN_FLOPS", 1 << 22)
    if request.param == "ffma":
        monkeypatch.setattr(nets, "TC_MIN_FLOPS", 1 << 62)
    if request.param == "implicit":
        monkeypatch.setattr(nets, "IMPLICIT", True)
    return request.param


def test_lenet_gradient_vs_oracle(gemm_routing):
    g_dev, g_ref = _cnn_case(network.lenet(), O.LENET, 300, 16)
    assert rel_err(g_dev, g_ref) < TOL


def test_cifar_quick_gradient_vs_oracle(gemm_routing):
    g_dev, g_ref = _cnn_case(network.cifar_quick(), O.CIFAR_QUICK, 200, 8)
    assert rel_err(g_dev, g_ref) < TOL


def test_alexnet_gradient_vs_oracle(gemm_routing):
    """full AlexNet geometry (61.1M params) at a small batch: with the
    tcgen05 routing every conv / fc contraction runs on the 3xTF32 kernel."""
    spec = network.alexnet(num_classes=1000)
    g_dev, g_ref = _cnn_case(spec, O.alexnet_layers(1000), 6, 2)
    assert rel_err(g_dev, g_ref) < TOL
