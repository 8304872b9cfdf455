"""BPQI/BPQT read + write in the reference layout (storage.py:253-360).
The written bytes must hash-match the reference's own serialisation of the
same index (tests/golden/storage_sha256.json, from make_golden.py)."""

import hashlib
import json
import struct
from pathlib import Path

import numpy as np
import pytest

from paper_1404_1831_b200 import storage

GOLD = Path(__file__).resolve().parent / "golden"


def test_writer_matches_reference_bytes(c0, hbpq_rig):
    sha = json.loads((GOLD / "storage_sha256.json").read_text())
    b = storage.index_bytes(c0["c1"], c0["c2"], c0["offsets"], c0["ids"], c0["codes"], books=c0["books"])
    assert hashlib.sha256(b).hexdigest() == sha["c0_bpqi_sha256"]
    t = storage.tables_bytes(c0["cn1"], c0["cn2"], c0["fine_norms"], c0["cross1"], c0["cross2"])
    assert hashlib.sha256(t).hexdigest() == sha["c0_bpqt_sha256"]
    g = hbpq_rig
    hb = storage.index_bytes(g["c1"], g["c2"], g["offsets"], g["ids"], g["hcodes"], bank1=g["bank1"], bank2=g["bank2"])
    assert hashlib.sha256(hb).hexdigest() == sha["hbpq_bpqi_sha256"]


def test_round_trip(tmp_path, c0):
    p = tmp_path / "x.bpqi"
    storage.save_index_arrays(p, c1=c0["c1"], c2=c0["c2"], offsets=c0["offsets"], ids=c0["ids"], codes=c0["codes"],
                              books=c0["books"])
    rec = storage.load_index_arrays(p)
    for k in ("c1", "c2", "offsets", "ids", "codes", "books"):
        np.testing.assert_array_equal(rec[k], c0[k])
    q = tmp_path / "x.bpqt"
    storage.save_tables_arrays(q, c0["cn1"], c0["cn2"], c0["fine_norms"], c0["cross1"], c0["cross2"])
    for a, k in zip(storage.load_tables_arrays(q), ("cn1", "cn2", "fine_norms", "cross1", "cross2")):
        np.testing.assert_array_equal(a, c0[k])


def test_strict_reader_rejects_corruption(tmp_path, c0):
    p = tmp_path / "x.bpqi"
    storage.save_index_arrays(p, c1=c0["c1"], c2=c0["c2"], offsets=c0["offsets"], ids=c0["ids"], codes=c0["codes"],
                              books=c0["books"])
    raw = p.read_bytes()
    for bad, msg in ((b"XXXX" + raw[4:], "magic"), (raw[:4] + struct.pack("<I", 9) + raw[8:], "version"),
                     (raw[:-3], "truncated"), (raw + b"\0", "trailing")):
        q = tmp_path / "bad.bpqi"
        q.write_bytes(bad)
        with pytest.raises(storage.StorageError, match=msg):
            storage.load_index_arrays(q)
