"""End-to-end Sync EASGD through run_trainer on the B200 vs the reference's
own runs (golden) and the pinned oracle."""

import numpy as np
import pytest

from oracle import esgd_oracle as O
from paper_1708_02983_b200 import HyperParams, ModelSpec, make_config, run_trainer
from paper_1708_02983_b200.datasets import Dataset
from paper_1708_02983_b200.trainers import NetworkProblem, QuadraticProblem, ZeroGradientProblem
from _gpu_util import rel_err

pytestmark = pytest.mark.gpu
HY = HyperParams(eta=0.05, rho=0.25, mu=0.9)


def _mlp_problem(golden):
    g = golden("net")
    spec = ModelSpec((32, 24, 16, 10), activation="relu", seed=1, dtype=np.float32)
    return NetworkProblem(spec, Dataset(g["train_x"], g["train_y"], 10), Dataset(g["test_x"], g["test_y"], 10))


@pytest.mark.parametrize("P,T", [(1, 5), (2, 10), (4, 10)])
def test_sync_mlp_matches_reference_run(golden, P, T):
    """center + every worker + losses within 1e-5 relative of the reference's
    float32 sync-easgd2 run (same seeds, same data)."""
    g = golden("trainers")
    rec = run_trainer(make_config("sync-easgd2", workers=P, iterations=T, batch_size=16, hyper=HY,
                                  eval_every=5, seed=3), _mlp_problem(golden))
    assert rel_err(rec.final_weights, g[f"float32_mlp_P{P}_T{T}_center"]) < 1e-5
    assert rel_err(np.stack(rec.final_worker_weights), g[f"float32_mlp_P{P}_T{T}_workers"]) < 1e-5
    assert rel_err(rec.train_loss, g[f"float32_mlp_P{P}_T{T}_loss"]) < 1e-5
    assert rec.test_accuracy == list(g[f"float32_mlp_P{P}_T{T}_acc"])


@pytest.mark.parametrize("method,groups", [("sync-easgd2", 1), ("group-easgd", 2)])
def test_sync_quadratic_bitwise_vs_oracle_fp32(method, groups):
    """elementwise path end to end: bitwise equal to the (reference-pinned)
    oracle evaluated in float32."""
    prob = QuadraticProblem.random(300, seed=2)
    hq = HyperParams(eta=0.1, rho=0.5)
    rec = run_trainer(make_config(method, workers=4, iterations=20, hyper=hq, groups=groups, seed=5), prob)
    oq = O.QuadProblem.random(300, 2, dtype=np.float32)
    C, W = O.run_sync(oq, 4, 20, 1, 0.1, 0.5, seed=5, groups=groups)
    assert np.array_equal(rec.final_weights, C)
    assert np.array_equal(np.stack(rec.final_worker_weights), np.stack(W))


def test_sync_quadratic_close_to_reference_fp64(golden):
    g = golden("trainers")
    prob = QuadraticProblem(g["quad_target"], g["quad_curv"])
    rec = run_trainer(make_config("sync-easgd2", workers=4, iterations=20, hyper=HyperParams(0.1, 0.5),
                                  seed=5), prob)
    assert rel_err(rec.final_weights, g["quad_sync-easgd2_center"]) < 1e-6


def test_sync_family_bit_identical(golden):
    digests = set()
    for m in ("sync-easgd1", "sync-easgd2", "sync-easgd3"):
        rec = run_trainer(make_config(m, workers=4, iterations=12, batch_size=16, hyper=HY, seed=1),
                          _mlp_problem(golden))
        digests.add(rec.weights_digest)
    assert len(digests) == 1


def test_deterministic(golden):
    cfg = make_config("sync-easgd3", workers=3, iterations=15, batch_size=16, hyper=HY, eval_every=5, seed=7)
    a = run_trainer(cfg, _mlp_problem(golden))
    b = run_trainer(cfg, _mlp_problem(golden))
    assert a.same_series(b)


def test_conservation_zero_gradient():
    prob = ZeroGradientProblem(257, seed=3)
    for P in (2, 4, 8):
        rec = run_trainer(make_config("sync-easgd2", workers=P, iterations=30, hyper=HyperParams(0.05, 0.3),
                                      seed=1), prob)
        total0 = (P + 1) * prob.init_weights()
        total = rec.final_weights.astype(np.float64) + np.sum(np.stack(rec.final_worker_weights), axis=0)
        assert np.abs(total - total0).max() < 1e-4 * P


def test_quadratic_converges():
    prob = QuadraticProblem.random(50, seed=9)
    rec = run_trainer(make_config("sync-easgd3", workers=4, iterations=600, hyper=HyperParams(0.1, 0.2),
                                  seed=2), prob)
    assert prob.distance_to_optimum(rec.final_weights) < 1e-3
    assert rec.total_seconds > 0 and set(rec.breakdown) >= {"peer_param", "forward_backward"}


@pytest.mark.parametrize("model", ["lenet", "cifar-quick"])
@pytest.mark.parametrize("tc", [True, False])
def test_sync_cnn_multi_replica_vs_oracle(model, tc, monkeypatch):
    """P workers as batched replicas of one DeviceNet (every CNN kernel runs
    with batch = P) against the oracle's sequential workers, three rounds, at
    the north-star 1e-5 (measured on the B200: center 3e-9 / 7e-9, workers
    2e-8 / 3e-8 for LeNet / CIFAR-quick; the fp32 oracle is 4e-8 from fp64)."""
    from paper_1708_02983_b200 import network, nets

    # tc: contractions above 4M MACs on tcgen05; else all on the FFMA kernel
    monkeypatch.setattr(nets, "TC_MIN_FLOPS", (1 << 22) if tc else (1 << 62))
    spec = network.MODELS[model](seed=1)
    layers = {"lenet": O.LENET, "cifar-quick": O.CIFAR_QUICK}[model]
    rng = np.random.default_rng(7)
    X = rng.standard_normal((400, spec.input_dim))
    Y = rng.integers(0, 10, 400)
    prob = NetworkProblem(spec, Dataset(X, Y, 10))
    rec = run_trainer(make_config("sync-easgd3", workers=3, iterations=3, batch_size=8, hyper=HY, seed=2), prob)
    oprob = O.NetProblem(*layers, X, Y, seed=1, dtype=np.float32)
    C, W = O.run_sync(oprob, 3, 3, 8, 0.05, 0.25, seed=2)
    assert rel_err(rec.final_weights, C) < 1e-5
    for w_dev, w_ref in zip(rec.final_worker_weights, W):
        assert rel_err(w_dev, w_ref) < 1e-5


@pytest.mark.parametrize("model", ["mlp", "lenet"])
def test_resume_from_state_is_bitwise(model, golden, tmp_path):
    """ESR1 save / load (formats.py): 3 rounds, checkpoint,
    a fresh engine restored from it, 3 more rounds == 6 rounds straight."""
    import torch

    from paper_1708_02983_b200 import formats, network
    from paper_1708_02983_b200.trainers.synchronous import SyncEngine

    if model == "mlp":
        prob = _mlp_problem(golden)
    else:
        rng = np.random.default_rng(3)
        prob = NetworkProblem(network.lenet(seed=0), Dataset(rng.standard_normal((300, 784)),
                                                             rng.integers(0, 10, 300), 10))
    cfg = make_config("sync-easgd3", workers=3, iterations=6, batch_size=8, hyper=HY, seed=4)

    def rounds(eng, k):
        for _ in range(k):
            eng.step()
        torch.cuda.synchronize()

    a = SyncEngine(cfg, prob)
    rounds(a, 6)
    b = SyncEngine(cfg, prob)
    rounds(b, 3)
    formats.save_state(tmp_path / "s.esr1", b, 3)
    c = SyncEngine(cfg, prob)
    assert formats.load_state(tmp_path / "s.esr1", c) == 3
    rounds(c, 3)
    assert np.array_equal(a.center_host(), c.center_host())
    for wa, wc in zip(a.workers_host(), c.workers_host()):
        assert np.array_equal(wa, wc)
