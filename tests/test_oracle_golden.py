"""Pin the CPU oracle (oracle/esgd_oracle.py) against golden vectors that the
real reference produced (oracle/make_golden.py). Bitwise where the reference
is deterministic numpy; the oracle is the checker for every GPU parity test."""

import numpy as np
import pytest

from oracle import esgd_oracle as O


def test_rng_streams(golden):
    g = golden("rng")
    seeds = [O.stream_seed(s, w) for s in (0, 3, 7) for w in range(8)]
    assert np.array_equal(np.array(seeds, dtype=np.uint64), g["stream_seeds"])
    assert np.array_equal(O.CounterRng(12345).raw(16), g["raw"])
    r = O.worker_rng(3, 2)
    assert np.array_equal(r.randint_block(256, 60000), g["randint_60000"])
    assert r.counter == int(g["randint_after_counter"][0])
    assert np.array_equal(O.CounterRng(99).uniform_block(64), g["uniform"])
    assert np.array_equal(O.CounterRng(7).normal_block(64), g["normal"])


def test_synthetic_and_normalize(golden):
    g = golden("data")
    x, y = O.gen_synthetic(10, 32, 20, seed=5, separation=5.0)
    assert np.array_equal(x, g["samples"]) and np.array_equal(y, g["labels"])
    assert np.array_equal(O.normalize(x), g["normalized"])


@pytest.mark.parametrize("dt", ["float32", "float64"])
def test_update_rules_bitwise(golden, dt):
    g = golden("updates")
    eta, rho, mu, P = (float(x) for x in g["scalars"])
    P = int(P)
    w, v, gr, c, s = g[f"{dt}_in"]
    assert np.array_equal(O.easgd_worker_step(w, gr, c, eta, rho), g[f"{dt}_worker"])
    assert np.array_equal(O.easgd_center_step_from_sum(c, s, P, eta, rho), g[f"{dt}_center_from_sum"])
    assert np.array_equal(O.easgd_center_incremental(c, w, eta, rho), g[f"{dt}_center_incr"])
    mw, mv = O.measgd_worker_step(w, v, gr, c, eta, mu, rho)
    assert np.array_equal(mw, g[f"{dt}_measgd_w"]) and np.array_equal(mv, g[f"{dt}_measgd_v"])
    assert np.array_equal(O.sgd_step(w, gr, eta), g[f"{dt}_sgd"])
    a, b = O.msgd_step(w, v, gr, eta, mu)
    assert np.array_equal(a, g[f"{dt}_msgd_w"]) and np.array_equal(b, g[f"{dt}_msgd_v"])
    assert np.array_equal(O.easgd_center_step(c, list(g[f"{dt}_snaps"]), eta, rho), g[f"{dt}_center_snap"])
    for p in (1, 2, 3, 5, 8, 13):
        assert np.array_equal(O.tree_sum(list(g[f"{dt}_tree_in_{p}"])), g[f"{dt}_tree_out_{p}"])


@pytest.mark.parametrize("dt", ["float32", "float64"])
@pytest.mark.parametrize("act", ["relu", "tanh", "sigmoid"])
def test_mlp_init_gradient_loss(golden, dt, act):
    g = golden("net")
    shape, layers = O.mlp_layers((32, 24, 16, 10), act)
    w = O.build_model(shape, layers, 1, np.dtype(dt).type)
    assert np.array_equal(w, g[f"{dt}_{act}_init"])
    prob = O.NetProblem(shape, layers, g["train_x"], g["train_y"], seed=1, dtype=np.dtype(dt).type)
    rng = O.worker_rng(3, 0)
    assert np.array_equal(prob.gradient(w, rng, 16), g[f"{dt}_{act}_grad"])
    assert np.array_equal(prob.gradient(w, rng, 16), g[f"{dt}_{act}_grad2"])
    assert prob.loss(w) == g[f"{dt}_{act}_loss"][0]


def test_big_init_and_xent(golden):
    g = golden("net")
    shape, layers = O.mlp_layers((784, 100, 10))
    w = O.build_model(shape, layers, 0, np.float64)
    assert np.array_equal(w[:4096], g["big_init_head"])
    loss, dl = O.softmax_cross_entropy(g["xent_logits"], g["xent_labels"])
    assert loss == g["xent_loss"][0]
    assert np.array_equal(dl, g["xent_dlogits"])


@pytest.mark.parametrize("dt", ["float32", "float64"])
@pytest.mark.parametrize("P,T", [(1, 5), (2, 10), (4, 10)])
def test_sync_trainer_bitwise(golden, dt, P, T):
    g, net = golden("trainers"), golden("net")
    shape, layers = O.mlp_layers((32, 24, 16, 10), "relu")
    prob = O.NetProblem(shape, layers, net["train_x"], net["train_y"], seed=1, dtype=np.dtype(dt).type)
    C, W = O.run_sync(prob, P, T, 16, 0.05, 0.25, seed=3)
    assert np.array_equal(C, g[f"{dt}_mlp_P{P}_T{T}_center"])
    assert np.array_equal(np.stack(W), g[f"{dt}_mlp_P{P}_T{T}_workers"])


@pytest.mark.parametrize("method,groups", [("sync-easgd2", 1), ("group-easgd", 2)])
def test_sync_quadratic_bitwise(golden, method, groups):
    g = golden("trainers")
    prob = O.QuadProblem(g["quad_target"], g["quad_curv"])
    assert np.array_equal(prob.target, O.QuadProblem.random(300, 2).target)
    C, W = O.run_sync(prob, 4, 20, 1, 0.1, 0.5, seed=5, groups=groups)
    assert np.array_equal(C, g[f"quad_{method}_center"])
    assert np.array_equal(np.stack(W), g[f"quad_{method}_workers"])
