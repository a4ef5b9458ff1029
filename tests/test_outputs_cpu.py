"""Native output path (cli.py:386-390, hsio.py:85-101, manifest.py:22-27) on CPU:
Python float repr, sha256, and the merge-log JSONL pinned to the sha256 of the
reference's own JSONL recorded in the golden fixtures."""

import hashlib
import json
import math
import struct

import numpy as np
import pytest

from golden_io import load
from paper_2106_12942_b200 import outputs
from paper_2106_12942_b200.graph import LabelMap
from paper_2106_12942_b200.recursive import RecordList, RhsegResult
from paper_2106_12942_b200.sections import SectionId


def test_format_float_matches_python_repr():
    rng = np.random.default_rng(5)
    vals = [0.0, -0.0, 1.0, 2.0, 0.5, 0.1, 1e-4, 1e-5, 9.999e-5, 1e15, 1e16, 1e17, 123456789012345678.0,
            1.5e300, 5e-324, 2.2250738585072014e-308, 1.7976931308623157e308, math.pi, math.sqrt(2),
            float("inf"), -float("inf")]
    vals += [2.0 ** e for e in range(-1074, 1024)]
    vals += [struct.unpack("<d", rng.bytes(8))[0] for _ in range(50000)]
    vals += list(rng.normal(0, 100, 20000)) + list(np.sqrt(rng.uniform(0, 1e6, 20000)))
    vals += [float(v) for v in rng.integers(0, 10 ** 6, 2000)]
    for v in vals:
        if math.isnan(v):
            continue
        assert outputs.format_float(v) == json.dumps(v), (v, outputs.format_float(v), json.dumps(v))


def test_sha256_matches_hashlib():
    rng = np.random.default_rng(1)
    for n in (0, 1, 55, 56, 63, 64, 65, 1000, 123457):
        data = rng.bytes(n)
        assert outputs.sha256_hex(data) == hashlib.sha256(data).hexdigest()


def _result_from_fixture(z):
    lev, row, col = z["log_level"], z["log_row"], z["log_col"]
    logs, start = [], 0
    n = len(lev)
    for k in range(1, n + 1):
        if k == n or (lev[k], row[k], col[k]) != (lev[start], row[start], col[start]):
            sl = slice(start, k)
            logs.append((SectionId(int(lev[start]), int(row[start]), int(col[start])),
                         RecordList(z["log_survivor"][sl].astype(np.int32), z["log_absorbed"][sl].astype(np.int32),
                                    z["log_dissim"][sl].astype(np.float64), z["log_kind"][sl].astype(np.uint8))))
            start = k
    labels = z["labels"]
    return RhsegResult(section_logs=logs, root_initial=None, root_hierarchy=None, graph=None,
                       labels=LabelMap(labels.shape[1], labels.shape[0], labels))


@pytest.mark.parametrize("name", ["c1_64x64x32.npz", "rhseg_32x32x224_L2.npz", "crit2_64x64x16_L3.npz",
                                  "c2_144x144x220_L3.npz"])
def test_native_jsonl_equals_reference_bytes(name, tmp_path):
    z = load(name)
    res = _result_from_fixture(z)
    out = outputs.write_outputs(res, tmp_path / "x.pgm", tmp_path / "x.merges.jsonl")
    jsonl = (tmp_path / "x.merges.jsonl").read_bytes()
    assert hashlib.sha256(jsonl).hexdigest() == str(z["jsonl_sha256"])
    # the same bytes json.dumps produces over flat_log (cli.py:387-390)
    py = "".join(json.dumps(r) + "\n" for r in res.flat_log()).encode()
    assert jsonl == py
    labels = np.asarray(z["labels"], np.int64)
    pgm = f"P5\n{labels.shape[1]} {labels.shape[0]}\n65535\n".encode() + labels.astype(">u2").tobytes()
    assert (tmp_path / "x.pgm").read_bytes() == pgm
    assert out["content_hash"] == hashlib.sha256(pgm + jsonl).hexdigest()


def _tiny_result(labels):
    recs = RecordList(np.array([0], np.int32), np.array([1], np.int32), np.array([1.5]), np.array([0], np.uint8))
    lab = np.asarray(labels)
    return RhsegResult([(SectionId(1, 0, 0), recs)], None, None, None, LabelMap(lab.shape[1], lab.shape[0], lab))


def test_write_outputs_errors_map_to_reference_types(tmp_path):
    """A label above 65535 raises TooManyLabels (hsio.py:88-92) with a message and
    writes nothing; an unopenable path raises OSError and leaves no partial file set."""
    from paper_2106_12942_b200 import TooManyLabels

    big = _tiny_result([[0, 70000], [1, 2]])
    with pytest.raises(TooManyLabels, match="70000"):
        outputs.write_outputs(big, tmp_path / "a.pgm", tmp_path / "a.merges.jsonl")
    assert not (tmp_path / "a.pgm").exists() and not (tmp_path / "a.merges.jsonl").exists()
    ok = _tiny_result([[0, 1], [1, 2]])
    with pytest.raises(OSError, match="cannot open"):
        outputs.write_outputs(ok, tmp_path / "b.pgm", tmp_path / "missing_dir" / "b.merges.jsonl")
    assert not (tmp_path / "b.pgm").exists()
    out = outputs.write_outputs(ok, tmp_path / "c.pgm", tmp_path / "c.merges.jsonl")
    assert len(out["content_hash"]) == 64
