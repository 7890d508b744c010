"""Host-side logic of the drop-in package (no GPU): model layouts and init,
datasets, RNG, configs/validation, records."""

import numpy as np
import pytest

from oracle import esgd_oracle as O
from paper_1708_02983_b200 import ClusterSpec, HyperParams, ModelSpec, make_config, network
from paper_1708_02983_b200.datasets import gen_synthetic, normalize
from paper_1708_02983_b200.errors import ElasticSGDError, InputError, ShapeError
from paper_1708_02983_b200.rng import CounterRng, stream_seed, worker_rng
from paper_1708_02983_b200.trainers import METHODS, RunRecord


def test_parameter_counts_match_survey():
    assert network.lenet().parameter_count() == 431_080
    assert network.cifar_quick().parameter_count() == 145_578
    assert network.alexnet().parameter_count() == 61_100_840
    assert ModelSpec((784, 300, 100, 10)).parameter_count() == 266_610


def test_mlp_view_offsets():
    vt = network.view_table(ModelSpec((784, 100, 10)))
    assert {v.name: v.offset for v in vt} == {"W1": 0, "b1": 78400, "W2": 78500, "b2": 79500}


@pytest.mark.parametrize("factory,layers", [(network.lenet, O.LENET), (network.cifar_quick, O.CIFAR_QUICK)])
def test_cnn_layout_and_init_equal_oracle(factory, layers):
    spec = factory(seed=4)
    views, total = O.param_views(*layers)
    assert total == spec.parameter_count()
    assert [(v.shape, v.offset) for v in network.view_table(spec)] == [(tuple(s), o) for s, o in views]
    assert np.array_equal(network.build_model(spec).buffer, O.build_model(*layers, 4, np.float32))


def test_mlp_init_equals_reference(golden):
    g = golden("net")
    for dt in ("float32", "float64"):
        for act in ("relu", "tanh", "sigmoid"):
            spec = ModelSpec((32, 24, 16, 10), activation=act, seed=1, dtype=np.dtype(dt).type)
            assert np.array_equal(network.build_model(spec).buffer, g[f"{dt}_{act}_init"])
    assert np.array_equal(network.build_model(ModelSpec((784, 100, 10), seed=0)).buffer[:4096], g["big_init_head"])


def test_rng_equals_reference(golden):
    g = golden("rng")
    assert [stream_seed(s, w) for s in (0, 3, 7) for w in range(8)] == [int(x) for x in g["stream_seeds"]]
    r = worker_rng(3, 2)
    assert np.array_equal(r.randint_block(256, 60000), g["randint_60000"])
    assert np.array_equal(CounterRng(7).normal_block(64), g["normal"])


def test_synthetic_data_equals_reference(golden):
    g = golden("data")
    ds = gen_synthetic(10, 32, 20, seed=5, separation=5.0)
    assert np.array_equal(ds.samples, g["samples"]) and np.array_equal(ds.labels, g["labels"])
    assert np.array_equal(normalize(ds).samples, g["normalized"])


def test_synthetic_chunking_is_invisible():
    # > one 16M-draw chunk: must equal one normal_block over all draws
    a = gen_synthetic(3, 5_600_000 // 3 + 1, 1, seed=9)
    x, _ = O.gen_synthetic(3, 5_600_000 // 3 + 1, 1, seed=9)
    assert np.array_equal(a.samples, x)


def test_config_validation():
    assert len(METHODS) == 11
    cfg = make_config("sync-easgd3", workers=4, iterations=3, batch_size=8)
    assert cfg.cluster.engine == "cuda" and cfg.cluster.scheduler == "bulk-synchronous"
    with pytest.raises(InputError):
        make_config("nope", workers=1, iterations=1)
    with pytest.raises(InputError):
        make_config("sync-easgd2", workers=4, iterations=1, groups=2)
    with pytest.raises(InputError):
        make_config("group-easgd", workers=4, iterations=1, groups=3)
    with pytest.raises(InputError):
        make_config("sync-easgd2", workers=4, iterations=0)


@pytest.mark.parametrize("engine", ["simulated", "threaded", "bogus"])
def test_cpu_engines_rejected(engine):
    with pytest.raises(InputError):
        ClusterSpec(4, engine=engine)


def test_hyperparams():
    with pytest.raises(InputError):
        HyperParams(eta=0.0)
    with pytest.raises(InputError):
        HyperParams(rho=-1)
    with pytest.raises(InputError):
        HyperParams(mu=1.0)
    h = HyperParams(eta=0.05, rho=0.25)
    assert h.etarho32 == float(np.float32(0.05 * 0.25))


def test_error_taxonomy():
    assert issubclass(ShapeError, ValueError) and issubclass(InputError, ElasticSGDError)


def test_run_record_helpers():
    r = RunRecord("sync-easgd3", "w", times=[1.0, 2.0], iterations=[1, 2], test_accuracy=[0.5, 0.9],
                  breakdown={"peer_param": 1.0, "data_stage": 0.0, "master_param": 0.0,
                             "forward_backward": 3.0, "worker_update": 0.0, "master_update": 0.0},
                  total_seconds=4.0)
    assert r.comm_ratio == 0.25
    assert r.time_to_accuracy(0.7) == pytest.approx(1.5)
    assert r.time_to_accuracy(0.95) is None


def test_model_specs_validate():
    with pytest.raises(InputError):
        network.ConvNetSpec((1, 8, 8), (network.Conv(4, 3),))
    with pytest.raises(Exception):
        network.ConvNetSpec((1, 4, 4), (network.Conv(4, 7), network.Dense(2)))


def test_costmodel_recalibration_helpers():
    """alpha-beta fit, the B200 preset, and the sync-round
    predictor (overlap: no exposed comm while compute covers it)."""
    from paper_1708_02983_b200.fabric import costmodel as cmod

    a, b = cmod.fit_alpha_beta([1e3, 1e6, 1e8], [2e-6 + 1e3 * 3e-12, 2e-6 + 1e6 * 3e-12, 2e-6 + 1e8 * 3e-12])
    assert abs(a - 2e-6) < 1e-9 and abs(b - 3e-12) < 1e-15
    cm = cmod.CostModel.preset("b200-nvlink")
    assert cm.alpha > 0 and cm.beta > 0
    one = cmod.predict_sync_round(cm, 4e-3, 61_100_840, 1)
    assert one["comm_seconds"] == 0 and one["weak_scaling_efficiency"] == 1.0
    eight = cmod.predict_sync_round(cm, 4e-3, 61_100_840, 8, interference=0.0)
    assert eight["exposed_comm_seconds"] == 0.0 and eight["weak_scaling_efficiency"] == 1.0
    tiny = cmod.predict_sync_round(cm, 1e-6, 61_100_840, 8)
    assert tiny["exposed_comm_seconds"] > 0 and tiny["weak_scaling_efficiency"] < 0.1
    pc = cmod.packed_vs_perlayer_cost([100, 200, 300], cm)
    assert abs(pc.per_layer - pc.packed - 2 * cm.alpha) < 1e-15
