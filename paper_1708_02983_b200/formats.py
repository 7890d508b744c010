"""Data and checkpoint formats on either side of the round:

* IDX image/label pairs (MNIST's format) — reference ``datasets.py:82-126``:
  big-endian headers (magic 0x00000803 / 0x00000801, counts, rows, cols),
  uint8 payloads, ``.gz`` read transparently, pixels scaled to [0, 1] on
  load and rounded back to bytes on write (load(write(load(x))) is exact).
* EFW1 weight checkpoints — reference ``network.py:203-233``: b"EFW1",
  uint32 dim count, uint32 dims, then the packed buffer as little-endian
  float64. Device buffers (fp32 CUDA tensors) are accepted and widened.
* ESR1 run state (new — the reference cannot resume): the Sync-EASGD
  engine's worker replicas, center and per-worker RNG (seed, counter), so a
  run continues bit-identically after a restart.
"""

from __future__ import annotations

import gzip
import io
import json
import struct

import numpy as np

from .errors import DataFormatError, InputError

IMAGE_MAGIC = 0x00000803
LABEL_MAGIC = 0x00000801
CHECKPOINT_MAGIC = b"EFW1"
STATE_MAGIC = b"ESR1"


def _open(path):
    return gzip.open(path, "rb") if str(path).endswith(".gz") else open(path, "rb")


def _take(fh, count: int, offset: int, what: str) -> bytes:
    data = fh.read(count)
    if len(data) != count:
        raise DataFormatError(f"truncated file while reading {what}", offset=offset)
    return data


def load_idx(image_path, label_path):
    """IDX image/label pair -> Dataset (float64 pixels in [0, 1], int64 labels)."""
    from .datasets import Dataset

    with _open(image_path) as fh:
        magic, n, rows, cols = struct.unpack(">IIII", _take(fh, 16, 0, "image header"))
        if magic != IMAGE_MAGIC:
            raise DataFormatError(f"bad image magic 0x{magic:08x}, expected 0x{IMAGE_MAGIC:08x}", offset=0)
        pixels = np.frombuffer(_take(fh, n * rows * cols, 16, "pixel data"), dtype=np.uint8)
    with _open(label_path) as fh:
        magic, n_labels = struct.unpack(">II", _take(fh, 8, 0, "label header"))
        if magic != LABEL_MAGIC:
            raise DataFormatError(f"bad label magic 0x{magic:08x}, expected 0x{LABEL_MAGIC:08x}", offset=0)
        labels = np.frombuffer(_take(fh, n_labels, 8, "label data"), dtype=np.uint8)
    if n_labels != n:
        raise DataFormatError(f"image count {n} != label count {n_labels}", offset=4)
    samples = pixels.reshape(n, rows * cols).astype(np.float64) / 255.0
    return Dataset(samples, labels.astype(np.int64), num_classes=int(labels.max()) + 1 if n else 0)


def write_idx(image_path, label_path, samples, labels, rows: int | None = None, cols: int | None = None) -> None:
    """Dataset arrays -> IDX pair; float samples in [0, 1] are rounded to bytes."""
    samples = np.asarray(samples)
    if samples.dtype != np.uint8:
        samples = np.rint(samples * 255.0).astype(np.uint8)
    n, d = samples.shape
    if rows is None:
        rows, cols = 1, d
    if rows * cols != d:
        raise InputError(f"rows*cols = {rows * cols} != sample dim {d}")
    with open(image_path, "wb") as fh:
        fh.write(struct.pack(">IIII", IMAGE_MAGIC, n, rows, cols))
        fh.write(np.ascontiguousarray(samples).tobytes())
    with open(label_path, "wb") as fh:
        fh.write(struct.pack(">II", LABEL_MAGIC, n))
        fh.write(np.asarray(labels, dtype=np.uint8).tobytes())


def _host_f64(buffer) -> np.ndarray:
    if hasattr(buffer, "detach"):  # torch tensor (device or host)
        buffer = buffer.detach().float().cpu().numpy()
    return np.asarray(buffer, dtype=np.float64).reshape(-1)


def save_weights(path, spec, weights) -> None:
    """EFW1 checkpoint of an MLP ``ModelSpec``'s packed buffer (numpy or a
    device tensor of the packed layout, possibly padded: the first
    ``parameter_count()`` values are written)."""
    dims = getattr(spec, "dims", None)
    if dims is None:
        raise InputError("EFW1 stores MLP dims only (reference network.py:203-211); use save_state for CNNs")
    buf = _host_f64(getattr(weights, "buffer", weights))
    count = spec.parameter_count()
    if buf.size < count:
        raise DataFormatError(f"buffer holds {buf.size} values, spec needs {count}")
    with open(path, "wb") as fh:
        fh.write(CHECKPOINT_MAGIC)
        fh.write(struct.pack("<I", len(dims)))
        fh.write(struct.pack(f"<{len(dims)}I", *dims))
        fh.write(buf[:count].astype("<f8").tobytes())


def load_weights(path) -> tuple[tuple[int, ...], np.ndarray]:
    """EFW1 checkpoint -> (dims, float64 packed buffer)."""
    from .network import ModelSpec

    with open(path, "rb") as fh:
        magic = fh.read(4)
        if magic != CHECKPOINT_MAGIC:
            raise DataFormatError(f"bad checkpoint magic {magic!r}", offset=0)
        (ndims,) = struct.unpack("<I", _take(fh, 4, 4, "dim count"))
        dims = struct.unpack(f"<{ndims}I", _take(fh, 4 * ndims, 8, "dims"))
        buf = np.frombuffer(fh.read(), dtype="<f8").astype(np.float64)
    expected = ModelSpec(dims).parameter_count()
    if buf.size != expected:
        raise DataFormatError(f"buffer holds {buf.size} values, dims {dims} need {expected}",
                              offset=8 + 4 * ndims)
    return tuple(int(d) for d in dims), buf


# ---- run state (resume) ------------------------------------------------------

def write_state(path, method: str, center, workers, rng_rows, rounds_done: int, fingerprint: str = "") -> None:
    """ESR1 from host arrays: json header (method, P, n, rounds_done,
    fingerprint, rng_rows) + the center (n), the worker replicas (P x n) and
    the workers' RNG (seed, counter) rows, raw little-endian. The format
    save_state writes; also how a state computed elsewhere (e.g. a CPU run of
    the reference algorithm) is handed to a device engine (load_state)."""
    C = np.ascontiguousarray(center, dtype="<f4").reshape(-1)
    W = np.ascontiguousarray(workers, dtype="<f4").reshape(-1, C.size)
    rng = np.ascontiguousarray(rng_rows, dtype="<u8").reshape(-1, 2)
    head = {"method": method, "workers": int(W.shape[0]), "n": int(C.size), "rounds_done": int(rounds_done),
            "fingerprint": fingerprint, "rng_rows": int(rng.shape[0])}
    hb = json.dumps(head).encode()
    with open(path, "wb") as fh:
        fh.write(STATE_MAGIC)
        fh.write(struct.pack("<I", len(hb)))
        fh.write(hb)
        fh.write(C.tobytes())
        fh.write(W.tobytes())
        fh.write(rng.tobytes())


def save_state(path, engine, rounds_done: int) -> None:
    """ESR1 of a single-process engine: its center, every local worker
    replica and the workers' RNG (seed, counter) pairs (write_state)."""
    import torch

    if getattr(engine, "world", 1) != 1:
        raise InputError("save_state: single-process engines only (gather the replicas first)")
    n = engine.n
    rng = engine.plan.rng.state.detach().cpu().numpy().view("<u8") if hasattr(engine.plan, "rng") else \
        np.zeros((engine.nrep, 2), dtype="<u8")
    torch.cuda.synchronize()
    write_state(path, engine.cfg.method, engine.C[:n].detach().cpu().numpy(),
                engine.W[:, :n].detach().cpu().numpy(), rng, rounds_done,
                getattr(engine.problem, "fingerprint", lambda: "")())


def load_state(path, engine) -> int:
    """Restore an ESR1 state into a freshly built engine of the same config
    and problem; returns rounds_done."""
    import torch

    with open(path, "rb") as fh:
        raw = fh.read()
    buf = io.BytesIO(raw)
    if buf.read(4) != STATE_MAGIC:
        raise DataFormatError("bad state magic", offset=0)
    if len(raw) < 8:
        raise DataFormatError("truncated state header", offset=len(raw))
    (hl,) = struct.unpack("<I", buf.read(4))
    if 8 + hl > len(raw):
        raise DataFormatError(f"state header of {hl} bytes runs past the end of the file", offset=8)
    try:
        head = json.loads(buf.read(hl))
    except ValueError as exc:
        raise DataFormatError(f"unreadable state header: {exc}", offset=8) from exc
    n, P = engine.n, engine.P
    if head["n"] != n or head["workers"] != P or head["method"] != engine.cfg.method:
        raise InputError(f"state {head['method']} P={head['workers']} n={head['n']} does not match the engine")
    fp = getattr(engine.problem, "fingerprint", lambda: "")()
    if head.get("fingerprint") and fp and head["fingerprint"] != fp:
        raise InputError("state was written for a different problem (fingerprint mismatch)")
    # check every payload length before anything is copied into the engine
    expect = 8 + hl + 4 * n + 4 * n * engine.nrep + 16 * int(head.get("rng_rows", 0))
    if len(raw) != expect:
        raise DataFormatError(f"state payload is {len(raw)} bytes, expected {expect} "
                              f"(header + center + {engine.nrep} workers + RNG rows)",
                              offset=min(len(raw), expect))
    C = np.frombuffer(buf.read(4 * n), dtype="<f4")
    W = np.frombuffer(buf.read(4 * n * engine.nrep), dtype="<f4").reshape(engine.nrep, n)
    rng = np.frombuffer(buf.read(16 * head["rng_rows"]), dtype="<u8").reshape(-1, 2)
    dev = engine.W.device
    engine.C[:n].copy_(torch.from_numpy(C.copy()).to(dev))
    engine.W[:, :n].copy_(torch.from_numpy(W.copy()).to(dev))
    if hasattr(engine.plan, "rng") and rng.size:
        engine.plan.rng.state.copy_(torch.from_numpy(rng.copy().view(np.int64)).to(dev))
    engine.after_external_write()
    return int(head["rounds_done"])
