"""alpha-beta cost model (reference fabric/costmodel.py:27-132), kept so that
``run_trainer(cfg, problem, cost_model)`` accepts the same arguments and so
``predict``-style extrapolation can use measured NVLink constants. The
device engine measures real time and does not consult it.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable

from ..errors import InputError

ComputeFn = Callable[[int, int, int], float]


def constant_compute(seconds: float) -> ComputeFn:
    def model(worker: int, batch_size: int, n_weights: int) -> float:
        return seconds
    return model


@dataclass(frozen=True)
class CostModel:
    alpha: float
    beta: float
    compute: ComputeFn = field(default_factory=lambda: constant_compute(0.0))
    worker_update: Callable[[int], float] = lambda n_weights: 0.0
    master_update: Callable[[int], float] = lambda n_weights: 0.0
    group_speedup: Callable[[int], float] = lambda groups: 1.0

    def __post_init__(self):
        if self.alpha < 0 or self.beta < 0:
            raise InputError("alpha and beta must be >= 0")

    @classmethod
    def preset(cls, name: str, **overrides) -> "CostModel":
        try:
            alpha, beta = _PRESETS[name]
        except KeyError:
            raise InputError(f"unknown cost preset {name!r}; have {sorted(_PRESETS)}")
        return cls(alpha=alpha, beta=beta, **overrides)

    def message_seconds(self, nbytes: int) -> float:
        return message_cost(nbytes, self)


_PRESETS = {
    "fdr": (0.7e-6, 0.2e-9),
    "qdr": (1.2e-6, 0.3e-9),
    "10gbe": (7.2e-6, 0.9e-9),
}
PRESET_NAMES = tuple(sorted(_PRESETS))


def message_cost(nbytes: int, cm: CostModel) -> float:
    if nbytes < 0:
        raise InputError(f"message size must be >= 0, got {nbytes}")
    return cm.alpha + cm.beta * nbytes


def tree_depth(participants: int) -> int:
    if participants < 1:
        raise InputError("participants must be >= 1")
    return math.ceil(math.log2(participants)) if participants > 1 else 0
