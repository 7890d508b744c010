"""The trainer catalog behind one entry point (reference
trainers/__init__.py:15-29): ``run_trainer(cfg, problem, cost_model)``."""

from __future__ import annotations

from ..errors import InputError
from ..fabric.costmodel import CostModel
from .config import METHOD_SCHEDULERS, METHODS, TrainerConfig, make_config
from .problems import NetworkProblem, QuadraticProblem, ZeroGradientProblem
from .records import RunRecord, eval_loss, evaluate, weights_digest
from .synchronous import SYNC_METHODS, SyncEngine, run_synchronous
from .hostfeed import HostFedRun

ASYNC_METHODS = ("async-sgd", "async-easgd", "async-msgd", "async-measgd")
HOGWILD_METHODS = ("hogwild-sgd", "hogwild-easgd")


def run_trainer(cfg: TrainerConfig, problem, cost_model: CostModel | None = None) -> RunRecord:
    """Run one configured trainer on a problem on the device.

    ``cost_model`` is accepted for signature compatibility; the device engine
    measures real time (CUDA events) instead of pricing events.
    """
    if cfg.cluster.engine != "cuda":
        raise InputError(f"engine {cfg.cluster.engine!r} is not available; use 'cuda'")
    if cfg.method in SYNC_METHODS:
        return run_synchronous(cfg, problem, cost_model)
    if cfg.method in ASYNC_METHODS:
        from .asynchronous import run_asynchronous
        return run_asynchronous(cfg, problem, cost_model)
    if cfg.method in HOGWILD_METHODS:
        from .hogwild import run_hogwild
        return run_hogwild(cfg, problem, cost_model)
    if cfg.method == "original-easgd":
        from .roundrobin import run_original_easgd
        return run_original_easgd(cfg, problem, cost_model)
    raise InputError(f"unknown method {cfg.method!r}")


__all__ = [
    "HostFedRun",
    "ASYNC_METHODS",
    "HOGWILD_METHODS",
    "METHODS",
    "METHOD_SCHEDULERS",
    "NetworkProblem",
    "QuadraticProblem",
    "RunRecord",
    "SYNC_METHODS",
    "SyncEngine",
    "TrainerConfig",
    "ZeroGradientProblem",
    "eval_loss",
    "evaluate",
    "make_config",
    "run_trainer",
    "weights_digest",
]
