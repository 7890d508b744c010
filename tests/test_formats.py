"""Data / checkpoint formats against bytes the reference
wrote (tests/golden/formats.npz, oracle/make_golden.py): IDX pairs
(datasets.py:82-126) and EFW1 checkpoints (network.py:203-233)."""

import gzip

import numpy as np
import pytest

from paper_1708_02983_b200 import formats
from paper_1708_02983_b200.errors import DataFormatError, InputError
from paper_1708_02983_b200.network import ModelSpec, build_model


@pytest.fixture(scope="module")
def g(golden):
    return golden("formats")


def test_idx_writer_bytes_equal_reference(tmp_path, g):
    ip, lp = tmp_path / "i.idx", tmp_path / "l.idx"
    formats.write_idx(ip, lp, g["idx_input"], g["idx_input_labels"], rows=3, cols=4)
    assert np.array_equal(np.frombuffer(ip.read_bytes(), dtype=np.uint8), g["idx_images"])
    assert np.array_equal(np.frombuffer(lp.read_bytes(), dtype=np.uint8), g["idx_labels"])


def test_idx_loader_reads_reference_files(tmp_path, g):
    ip, lp = tmp_path / "i.idx", tmp_path / "l.idx"
    ip.write_bytes(g["idx_images"].tobytes())
    lp.write_bytes(g["idx_labels"].tobytes())
    ds = formats.load_idx(ip, lp)
    assert np.array_equal(ds.samples, g["idx_samples"]) and np.array_equal(ds.labels, g["idx_labels_loaded"])
    # gz transparently, and load(write(load(x))) is exact
    gi, gl = tmp_path / "i.idx.gz", tmp_path / "l.idx.gz"
    gi.write_bytes(gzip.compress(g["idx_images"].tobytes()))
    gl.write_bytes(gzip.compress(g["idx_labels"].tobytes()))
    ds2 = formats.load_idx(gi, gl)
    formats.write_idx(tmp_path / "r.idx", tmp_path / "rl.idx", ds2.samples, ds2.labels, rows=3, cols=4)
    assert (tmp_path / "r.idx").read_bytes() == g["idx_images"].tobytes()


def test_idx_errors(tmp_path, g):
    ip, lp = tmp_path / "i.idx", tmp_path / "l.idx"
    bad = bytearray(g["idx_images"].tobytes())
    bad[3] = 0x01
    ip.write_bytes(bytes(bad))
    lp.write_bytes(g["idx_labels"].tobytes())
    with pytest.raises(DataFormatError, match="magic"):
        formats.load_idx(ip, lp)
    ip.write_bytes(g["idx_images"].tobytes()[:-3])
    with pytest.raises(DataFormatError, match="truncated"):
        formats.load_idx(ip, lp)
    with pytest.raises(InputError):
        formats.write_idx(ip, lp, np.zeros((2, 5)), [0, 1], rows=2, cols=2)


def test_efw1_bytes_and_load_equal_reference(tmp_path, g):
    spec = ModelSpec((5, 4, 3), seed=2, dtype=np.float64)
    p = tmp_path / "w.efw1"
    formats.save_weights(p, spec, build_model(spec))
    assert np.array_equal(np.frombuffer(p.read_bytes(), dtype=np.uint8), g["efw1_bytes"])
    ref = tmp_path / "ref.efw1"
    ref.write_bytes(g["efw1_bytes"].tobytes())
    dims, buf = formats.load_weights(ref)
    assert dims == tuple(g["efw1_dims"]) and np.array_equal(buf, g["efw1_buf"])


def test_efw1_errors(tmp_path, g):
    p = tmp_path / "w.efw1"
    p.write_bytes(b"XXXX" + g["efw1_bytes"].tobytes()[4:])
    with pytest.raises(DataFormatError, match="magic"):
        formats.load_weights(p)
    p.write_bytes(g["efw1_bytes"].tobytes()[:-8])
    with pytest.raises(DataFormatError, match="need"):
        formats.load_weights(p)
    from paper_1708_02983_b200 import network

    with pytest.raises(InputError):
        formats.save_weights(p, network.lenet(), np.zeros(10))


def test_load_state_rejects_truncated_payload(tmp_path):
    """ESR1 payload lengths are checked before anything is copied into the
    engine (truncated / mismatched files -> DataFormatError with an offset)."""
    import json
    import struct
    from types import SimpleNamespace

    import torch

    from paper_1708_02983_b200 import formats
    from paper_1708_02983_b200.errors import DataFormatError

    n, nrep = 10, 2
    head = json.dumps({"method": "sync-easgd3", "workers": nrep, "n": n, "rounds_done": 3,
                       "fingerprint": "", "rng_rows": nrep}).encode()
    body = formats.STATE_MAGIC + struct.pack("<I", len(head)) + head
    payload = np.zeros(4 * n + 4 * n * nrep + 16 * nrep, dtype=np.uint8).tobytes()
    C0 = torch.full((n,), 7.0)
    eng = SimpleNamespace(n=n, P=nrep, nrep=nrep, cfg=SimpleNamespace(method="sync-easgd3"),
                          problem=SimpleNamespace(), C=C0, W=torch.zeros(nrep, n))
    for cut in (1, 17, len(payload) // 2):
        p = tmp_path / f"s{cut}.esr1"
        p.write_bytes(body + payload[:-cut])
        with pytest.raises(DataFormatError):
            formats.load_state(p, eng)
    p = tmp_path / "long.esr1"
    p.write_bytes(body + payload + b"\0")
    with pytest.raises(DataFormatError):
        formats.load_state(p, eng)
    p = tmp_path / "head.esr1"
    p.write_bytes(formats.STATE_MAGIC + struct.pack("<I", 1000) + head)
    with pytest.raises(DataFormatError):
        formats.load_state(p, eng)
    assert torch.all(C0 == 7.0)  # nothing was copied
