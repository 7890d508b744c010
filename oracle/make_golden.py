"""Generate tests/golden/*.npz by running the REAL reference package.

Run in the build container (the reference is read-only at /root/reference and
does not exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python oracle/make_golden.py

The fixtures pin the oracle restatement (tests/test_oracle_golden.py) and are
the reference side of the GPU parity tests (tests/test_gpu_*.py). Small
sizes only: the whole set is a few hundred KB.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True
if "/root/reference/pkg/src" not in sys.path:
    sys.path.insert(0, "/root/reference/pkg/src")

from elasticsgd import CostModel, HyperParams, ModelSpec  # noqa: E402
from elasticsgd import rng as R  # noqa: E402
from elasticsgd.datasets import gen_synthetic, normalize  # noqa: E402
from elasticsgd.fabric.collectives import tree_sum  # noqa: E402
from elasticsgd.kernels import softmax_cross_entropy  # noqa: E402
from elasticsgd.network import build_model  # noqa: E402
from elasticsgd.trainers import NetworkProblem, QuadraticProblem, make_config, run_trainer  # noqa: E402
from elasticsgd import updates as U  # noqa: E402

OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"


def rng_fixture():
    d = {}
    d["stream_seeds"] = np.array([R.stream_seed(s, w) for s in (0, 3, 7) for w in range(8)], dtype=np.uint64)
    g = R.CounterRng(12345)
    d["raw"] = np.array([g.u64() for _ in range(16)], dtype=np.uint64)
    g = R.worker_rng(3, 2)
    d["randint_60000"] = g.randint_block(256, 60000)
    d["randint_after_counter"] = np.array([g.counter], dtype=np.int64)
    d["uniform"] = R.CounterRng(99).uniform_block(64)
    d["normal"] = R.CounterRng(7).normal_block(64)
    return d


def data_fixture():
    ds = gen_synthetic(10, 32, 20, seed=5, separation=5.0)
    nd = normalize(ds)
    return {"samples": ds.samples, "labels": ds.labels, "normalized": nd.samples}


def update_fixture():
    d = {}
    rng = R.CounterRng(2024)
    n = 1031  # odd size: vector tails
    for dt in (np.float32, np.float64):
        tag = np.dtype(dt).name
        w, v, g, c, s = (rng.normal_block(n).astype(dt) for _ in range(5))
        eta, rho, mu, P = 0.05, 0.25, 0.9, 8
        d[f"{tag}_in"] = np.stack([w, v, g, c, s])
        d[f"{tag}_worker"] = U.easgd_worker_step(w, g, c, eta, rho)
        d[f"{tag}_center_from_sum"] = U.easgd_center_step_from_sum(c, s, P, eta, rho)
        d[f"{tag}_center_incr"] = U.easgd_center_incremental(c, w, eta, rho)
        mw, mv = U.measgd_worker_step(w, v, g, c, eta, mu, rho)
        d[f"{tag}_measgd_w"], d[f"{tag}_measgd_v"] = mw, mv
        d[f"{tag}_sgd"] = U.sgd_step(w, g, eta)
        a, b = U.msgd_step(w, v, g, eta, mu)
        d[f"{tag}_msgd_w"], d[f"{tag}_msgd_v"] = a, b
        snaps = [rng.normal_block(n).astype(dt) for _ in range(5)]
        d[f"{tag}_snaps"] = np.stack(snaps)
        d[f"{tag}_center_snap"] = U.easgd_center_step(c, snaps, eta, rho)
        for p in (1, 2, 3, 5, 8, 13):
            bufs = [rng.normal_block(n).astype(dt) for _ in range(p)]
            d[f"{tag}_tree_in_{p}"] = np.stack(bufs)
            d[f"{tag}_tree_out_{p}"] = tree_sum(bufs)
    d["scalars"] = np.array([0.05, 0.25, 0.9, 8.0])
    return d


def net_fixture():
    d = {}
    train = normalize(gen_synthetic(10, 32, 40, seed=5, separation=5.0))
    test = normalize(gen_synthetic(10, 32, 10, seed=6, separation=5.0))
    d["train_x"], d["train_y"] = train.samples, train.labels
    d["test_x"], d["test_y"] = test.samples, test.labels
    for dt in (np.float32, np.float64):
        tag = np.dtype(dt).name
        for act in ("relu", "tanh", "sigmoid"):
            spec = ModelSpec((32, 24, 16, 10), activation=act, seed=1, dtype=dt)
            prob = NetworkProblem(spec, train, test)
            w = prob.init_weights()
            d[f"{tag}_{act}_init"] = w
            rng = R.worker_rng(3, 0)
            d[f"{tag}_{act}_grad"] = prob.gradient(w, rng, 16)
            d[f"{tag}_{act}_grad2"] = prob.gradient(w, rng, 16)  # second draw, same weights
            d[f"{tag}_{act}_loss"] = np.array([prob.train_loss(w)])
    spec = ModelSpec((784, 100, 10), seed=0)
    d["big_init_head"] = build_model(spec).buffer[:4096]
    logits = R.CounterRng(4).normal_block(12 * 7).reshape(12, 7) * 3
    labels = R.CounterRng(5).randint_block(12, 7)
    loss, dl = softmax_cross_entropy(logits, labels)
    d["xent_logits"], d["xent_labels"], d["xent_loss"], d["xent_dlogits"] = logits, labels, np.array([loss]), dl
    return d


def trainer_fixture():
    d = {}
    train = normalize(gen_synthetic(10, 32, 40, seed=5, separation=5.0))
    test = normalize(gen_synthetic(10, 32, 10, seed=6, separation=5.0))
    hy = HyperParams(eta=0.05, rho=0.25, mu=0.9)
    cm = CostModel(alpha=0.0, beta=0.0)
    for dt in (np.float32, np.float64):
        tag = np.dtype(dt).name
        spec = ModelSpec((32, 24, 16, 10), activation="relu", seed=1, dtype=dt)
        prob = NetworkProblem(spec, train, test)
        for P, T in ((1, 5), (2, 10), (4, 10)):
            rec = run_trainer(make_config("sync-easgd2", workers=P, iterations=T, batch_size=16,
                                          hyper=hy, eval_every=5, seed=3), prob, cm)
            d[f"{tag}_mlp_P{P}_T{T}_center"] = rec.final_weights
            d[f"{tag}_mlp_P{P}_T{T}_workers"] = np.stack(rec.final_worker_weights)
            d[f"{tag}_mlp_P{P}_T{T}_loss"] = np.array(rec.train_loss)
            d[f"{tag}_mlp_P{P}_T{T}_acc"] = np.array(rec.test_accuracy)
    quad = QuadraticProblem.random(300, seed=2)
    hq = HyperParams(eta=0.1, rho=0.5, mu=0.9)
    for method, groups in (("sync-easgd2", 1), ("group-easgd", 2)):
        rec = run_trainer(make_config(method, workers=4, iterations=20, hyper=hq, groups=groups, seed=5),
                          quad, cm)
        d[f"quad_{method}_center"] = rec.final_weights
        d[f"quad_{method}_workers"] = np.stack(rec.final_worker_weights)
    d["quad_target"], d["quad_curv"] = quad.target, quad.curvature
    for method in ("async-measgd", "async-easgd", "hogwild-easgd"):
        rec = run_trainer(make_config(method, workers=4, iterations=400, hyper=hq, seed=5), quad,
                          CostModel.preset("fdr"))
        d[f"quad_{method}_center"] = rec.final_weights
        d[f"quad_{method}_dist"] = np.array([quad.distance_to_optimum(rec.final_weights)])
    return d


def async_fixture():
    """Loss curves of the reference's async / Hogwild schedules on the MLP
    problem (simulated engine, FCFS by virtual time) for statistical parity."""
    d = {}
    train = normalize(gen_synthetic(10, 32, 40, seed=5, separation=5.0))
    test = normalize(gen_synthetic(10, 32, 10, seed=6, separation=5.0))
    spec = ModelSpec((32, 24, 16, 10), activation="relu", seed=1, dtype=np.float32)
    prob = NetworkProblem(spec, train, test)
    cm = CostModel.preset("fdr")
    for method, hy in (("async-measgd", HyperParams(eta=0.02, rho=0.25, mu=0.9)),
                       ("async-easgd", HyperParams(eta=0.05, rho=0.25)),
                       ("hogwild-easgd", HyperParams(eta=0.05, rho=0.25))):
        rec = run_trainer(make_config(method, workers=4, iterations=800, batch_size=16, hyper=hy,
                                      eval_every=200, seed=3), prob, cm)
        d[f"{method}_loss"] = np.array(rec.train_loss)
        d[f"{method}_acc"] = np.array(rec.test_accuracy)
    d["init_loss"] = np.array([prob.train_loss(prob.init_weights())])
    return d


def formats_fixture():
    """Bytes written by the reference's IDX writer and EFW1 checkpointer
    (datasets.py:111-126, network.py:203-211), and what its loaders read
    back, for the format round-trip tests."""
    import os
    import tempfile

    from elasticsgd.datasets import load_idx, write_idx
    from elasticsgd.network import PackedWeights, build_model, load_weights, save_weights  # noqa: F401

    d = {}
    ds = normalize(gen_synthetic(3, 12, 4, seed=9, separation=5.0))
    samples01 = (ds.samples - ds.samples.min()) / (ds.samples.max() - ds.samples.min())
    with tempfile.TemporaryDirectory() as tmp:
        ip, lp = os.path.join(tmp, "img.idx"), os.path.join(tmp, "lab.idx")
        write_idx(ip, lp, samples01, ds.labels, rows=3, cols=4)
        d["idx_images"] = np.frombuffer(open(ip, "rb").read(), dtype=np.uint8)
        d["idx_labels"] = np.frombuffer(open(lp, "rb").read(), dtype=np.uint8)
        back = load_idx(ip, lp)
        d["idx_samples"], d["idx_labels_loaded"] = back.samples, back.labels
        d["idx_input"] = samples01
        d["idx_input_labels"] = ds.labels
        spec = ModelSpec((5, 4, 3), seed=2)
        model = build_model(spec)
        cp = os.path.join(tmp, "w.efw1")
        save_weights(cp, spec, model)
        d["efw1_bytes"] = np.frombuffer(open(cp, "rb").read(), dtype=np.uint8)
        dims, buf = load_weights(cp)
        d["efw1_dims"], d["efw1_buf"] = np.array(dims), buf
    return d


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    only = sys.argv[1:]
    for name, fn in (("rng", rng_fixture), ("data", data_fixture), ("updates", update_fixture),
                     ("net", net_fixture), ("trainers", trainer_fixture), ("async", async_fixture),
                     ("formats", formats_fixture)):
        if only and name not in only:
            continue
        path = OUT / f"{name}.npz"
        np.savez_compressed(path, **fn())
        print(path, path.stat().st_size)


if __name__ == "__main__":
    main()
