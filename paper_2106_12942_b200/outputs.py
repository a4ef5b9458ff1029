"""The reference CLI's output files at scale (cli.py:386-390, hsio.py:85-101,
manifest.py:22-27), written natively: the labels PGM, the merge-log JSONL (one
`json.dumps(record)` line per merge of `RhsegResult.flat_log()`, Python float
repr) and the manifest content hash sha256(pgm || jsonl). Byte-identical to the
reference's files, without building millions of Python dicts.
"""

from __future__ import annotations

import ctypes
from pathlib import Path

import numpy as np

from . import _lib
from .recursive import RecordList


def format_float(x: float) -> str:
    """Python repr(x) (json.dumps spelling for inf/nan), computed natively."""
    buf = ctypes.create_string_buffer(48)
    _lib.check(_lib.load().rhseg_format_float(float(x), buf, 48), "rhseg_format_float")
    return buf.value.decode()


def sha256_hex(data: bytes) -> str:
    out = ctypes.create_string_buffer(65)
    arr = np.frombuffer(data, dtype=np.uint8) if data else np.zeros(1, np.uint8)
    _lib.check(_lib.load().rhseg_sha256_hex(arr.ctypes.data_as(ctypes.c_void_p), len(data), out), "sha256")
    return out.value.decode()


def _log_arrays(result):
    a, b, d, k, lev, row, col, cnt = [], [], [], [], [], [], [], []
    for sid, recs in result.section_logs:
        if isinstance(recs, RecordList):
            ra, rb, rd, rk = recs.arrays()
        else:
            ra = [r.survivor_id for r in recs]
            rb = [r.absorbed_id for r in recs]
            rd = [r.dissimilarity for r in recs]
            rk = [int(r.kind) for r in recs]
        a.append(np.asarray(ra, np.int32)); b.append(np.asarray(rb, np.int32))
        d.append(np.asarray(rd, np.float64)); k.append(np.asarray(rk, np.uint8))
        lev.append(sid.level); row.append(sid.row); col.append(sid.col); cnt.append(len(ra))
    cat = (lambda xs, dt: np.ascontiguousarray(np.concatenate(xs), dt) if xs else np.zeros(1, dt))
    return (cat(a, np.int32), cat(b, np.int32), cat(d, np.float64), cat(k, np.uint8),
            np.asarray(lev, np.int32), np.asarray(row, np.int32), np.asarray(col, np.int32),
            np.asarray(cnt, np.int64))


def write_outputs(result, pgm_path, jsonl_path) -> dict:
    """Write `<stem>.pgm` and `<stem>.merges.jsonl` like `rhseg segment` does and
    return {"content_hash", "jsonl_bytes", "pgm", "jsonl"} (the manifest's
    content_hash covers exactly these two files, in this order)."""
    labels = np.ascontiguousarray(result.labels.labels, dtype=np.int32)
    h, w = labels.shape
    a, b, d, k, lev, row, col, cnt = _log_arrays(result)
    out = ctypes.create_string_buffer(65)
    nbytes = ctypes.c_int64(0)
    p = _lib.ptr
    _lib.check(_lib.load().rhseg_write_outputs_host(
        str(pgm_path).encode(), str(jsonl_path).encode(), w, h, p(labels), len(lev), p(lev), p(row), p(col),
        p(cnt), p(a), p(b), p(d), p(k), out, ctypes.byref(nbytes)), "rhseg_write_outputs_host")
    return {"content_hash": out.value.decode(), "jsonl_bytes": nbytes.value, "pgm": Path(pgm_path),
            "jsonl": Path(jsonl_path)}
