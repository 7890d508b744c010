from .cluster import ClusterSpec
from .collectives import allreduce_sum_, replica_sum_, tree_sum, world
from .costmodel import CostModel, constant_compute, message_cost, tree_depth
from .engine import CATEGORIES, COMM_CATEGORIES, hogwild_apply, hogwild_elastic_apply

__all__ = [
    "CATEGORIES",
    "COMM_CATEGORIES",
    "ClusterSpec",
    "CostModel",
    "allreduce_sum_",
    "constant_compute",
    "hogwild_apply",
    "hogwild_elastic_apply",
    "message_cost",
    "replica_sum_",
    "tree_depth",
    "tree_sum",
    "world",
]
