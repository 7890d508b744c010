"""The rest of the reference's public surface on the device: the snapshot
center step (updates.py:96-110), PackedWeights / build_model /
packed_weights_for / forward / backward (network.py:80-242) and evaluate /
eval_loss (trainers/records.py:92-108) — against the reference's golden
outputs (tests/golden, made by oracle/make_golden.py from the reference)."""

import numpy as np
import pytest

from paper_1708_02983_b200 import ModelSpec, network, updates
from paper_1708_02983_b200.errors import ShapeError, StaleCacheError
from paper_1708_02983_b200.network import PackedWeights, backward, build_model, forward, packed_weights_for
from paper_1708_02983_b200.rng import worker_rng
from paper_1708_02983_b200.trainers import eval_loss, evaluate
from _gpu_util import dev, host, rel_err

pytestmark = pytest.mark.gpu


def test_snapshot_center_step_bitwise_vs_reference(golden):
    """a8: easgd_center_step (fixed-order sum of W_i - C) bitwise."""
    g = golden("updates")
    w, v, gr, c, s = g["float32_in"]
    eta, rho = float(g["scalars"][0]), float(g["scalars"][1])
    out = updates.easgd_center_step(dev(c), [dev(x) for x in g["float32_snaps"]], eta, rho)
    assert np.array_equal(host(out), g["float32_center_snap"])


def _mlp(golden, act):
    net = golden("net")
    spec = ModelSpec((32, 24, 16, 10), activation=act, seed=1, dtype=np.float32)
    return spec, net


@pytest.mark.parametrize("act", ["relu", "tanh", "sigmoid"])
def test_forward_backward_vs_reference(golden, act):
    """forward + host softmax-CE + backward == the reference gradient of the
    first sampled batch (float32 golden) within 1e-5; build_model ==
    the reference init bitwise."""
    from oracle import esgd_oracle as O

    spec, net = _mlp(golden, act)
    pw = build_model(spec)
    assert isinstance(pw, PackedWeights)
    assert np.array_equal(pw.buffer, net[f"float32_{act}_init"])
    assert pw.view("W1").shape == (32, 24) and pw.view("b3").shape == (10,)
    rng = worker_rng(3, 0)
    idx = rng.randint_block(16, net["train_x"].shape[0])
    xb, yb = net["train_x"][idx], net["train_y"][idx]
    cache, logits = forward(spec, pw, xb)
    assert logits.shape == (16, 10)
    _, dl = O.softmax_cross_entropy(logits.astype(np.float32), yb)
    grad = backward(spec, pw, cache, dl.astype(np.float32))
    assert rel_err(grad, net[f"float32_{act}_grad"]) < 1e-5
    with pytest.raises(StaleCacheError):
        backward(spec, pw.clone(), cache, dl)
    with pytest.raises(ShapeError):
        packed_weights_for(spec, np.zeros(7, dtype=np.float32))


def test_evaluate_and_eval_loss_vs_reference(golden):
    spec, net = _mlp(golden, "relu")
    w = net["float32_relu_init"]
    k = min(1024, net["train_x"].shape[0])
    loss = eval_loss(spec, w, net["train_x"][:k], net["train_y"][:k])
    assert abs(loss - float(net["float32_relu_loss"][0])) < 1e-5 * max(1.0, abs(loss))
    acc = evaluate(spec, packed_weights_for(spec, w), net["test_x"], net["test_y"])
    from oracle import esgd_oracle as O

    _, ref_logits = O.forward(*O.mlp_layers((32, 24, 16, 10), "relu"), w.astype(np.float64), net["test_x"])
    assert acc == float((ref_logits.argmax(axis=1) == net["test_y"]).mean())
