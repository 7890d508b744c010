"""Datasets for the device problems: immutable host ``Dataset`` plus the
synthetic Gaussian-blob generator and population-std normalisation, with the
reference's semantics (datasets.py:24-171). Datasets are generated once on
the host and uploaded to HBM by the device problems; per-round sampling
happens on the device (csrc/sampling.cu).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import InputError
from .rng import CounterRng


@dataclass(frozen=True)
class Dataset:
    """n samples of dimension d with integer class labels (datasets.py:24-52)."""

    samples: np.ndarray
    labels: np.ndarray
    num_classes: int

    def __post_init__(self):
        if self.samples.ndim != 2 or self.samples.shape[0] < 1:
            raise InputError(f"samples must be (n, d) with n >= 1, got {self.samples.shape}")
        if self.labels.shape != (self.samples.shape[0],):
            raise InputError(
                f"labels shape {self.labels.shape} does not match n={self.samples.shape[0]}")
        if self.labels.min() < 0 or self.labels.max() >= self.num_classes:
            raise InputError("labels must lie in [0, num_classes)")
        self.samples.setflags(write=False)
        self.labels.setflags(write=False)

    @property
    def n(self) -> int:
        return self.samples.shape[0]

    @property
    def dim(self) -> int:
        return self.samples.shape[1]


def gen_synthetic(classes: int, dim: int, per_class: int, seed: int,
                  separation: float = 6.0, dtype=np.float64) -> Dataset:
    """Gaussian blobs; class k centred at ``separation`` along axis k
    (datasets.py:129-147). Noise is drawn in chunks of whole samples, which
    leaves the draw sequence identical to one ``normal_block(n*dim)`` call
    only when it is a single chunk — so the chunking follows the reference:
    u1 = first n*dim draws, u2 = next n*dim draws.
    """
    if classes < 1 or dim < 1 or per_class < 1:
        raise InputError("classes, dim and per_class must all be >= 1")
    if dim < classes:
        raise InputError(f"dim ({dim}) must be >= classes ({classes}) to place blob centers")
    n = classes * per_class
    total = n * dim
    out = np.empty((n, dim), dtype=dtype)
    flat = out.reshape(-1)
    # u1 uses draws [0, total), u2 uses draws [total, 2*total)
    chunk = 1 << 24
    for lo in range(0, total, chunk):
        hi = min(total, lo + chunk)
        r1 = CounterRng(seed, lo)
        u1 = ((r1.raw_block(hi - lo) >> np.uint64(11)).astype(np.float64) + 1.0) * 2.0**-53
        r2 = CounterRng(seed, total + lo)
        u2 = (r2.raw_block(hi - lo) >> np.uint64(11)).astype(np.float64) * 2.0**-53
        noise = np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)
        rows = np.arange(lo, hi) // dim
        cols = np.arange(lo, hi) % dim
        labels_here = rows // per_class
        mean = np.where(cols == labels_here, separation, 0.0)
        flat[lo:hi] = mean + noise
    labels = np.repeat(np.arange(classes, dtype=np.int64), per_class)
    return Dataset(out, labels, num_classes=classes)


def normalize(d: Dataset) -> Dataset:
    """Per-feature standardisation, population std, constant features -> 0
    (datasets.py:150-163)."""
    if d.n < 2:
        raise InputError("normalize needs at least 2 samples")
    x = d.samples.astype(np.float64, copy=False)
    mean = x.mean(axis=0)
    std = x.std(axis=0)
    scale = np.where(std > 0.0, std, 1.0)
    out = (x - mean) / scale
    out[:, std == 0.0] = 0.0
    return Dataset(out.astype(d.samples.dtype, copy=False), d.labels.copy(), d.num_classes)


def standardize_pair(train: Dataset, test: Dataset) -> tuple[Dataset, Dataset]:
    """Standardise both sets with the TRAIN statistics (the acceptance
    suite's convention, tests/test_acceptance.py:253-261)."""
    mean = train.samples.mean(axis=0)
    std = train.samples.std(axis=0)
    scale = np.where(std > 0.0, std, 1.0)

    def apply(d: Dataset) -> Dataset:
        out = (d.samples - mean) / scale
        out[:, std == 0.0] = 0.0
        return Dataset(out, d.labels.copy(), d.num_classes)

    return apply(train), apply(test)


# IDX pairs (reference datasets.py:82-126), implemented in formats.py
from .formats import load_idx, write_idx  # noqa: E402,F401
