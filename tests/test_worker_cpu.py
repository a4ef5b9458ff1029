"""Wire protocol of the B200 worker on CPU: frames and ASSIGN payloads made by
the unmodified reference (tests/golden/wire_frames.npz, oracle/gen_golden.py
wire) decode to the expected fields; malformed frames raise the reference's
ProtocolError subclasses; RESULT encoding of the reference's own reply data
round-trips to the reference's bytes."""

import struct

import numpy as np
import pytest

from golden_io import load
from paper_2106_12942_b200 import worker
from paper_2106_12942_b200.errors import BadMagic, BadVersion, Truncated, UnknownType


def _frames():
    z = load("wire_frames.npz")
    for k in range(int(z["n"])):
        yield z[f"assign_{k}"].tobytes(), z[f"result_{k}"].tobytes()


def test_assign_frames_decode():
    for frame, reply in _frames():
        t, payload = worker.decode_message(frame)
        assert t == worker.ASSIGN
        sid, samples, w, target = worker.decode_assign(payload)
        assert samples.dtype == np.float32 and samples.shape[1] == samples.shape[2]
        assert 0.0 <= w <= 1.0 and target >= 1 and sid[0] >= 1
        rt, _ = worker.decode_message(reply)
        assert rt == worker.RESULT


def _parse_result(body, edge, bands):
    """Reference RESULT payload -> arrays (for re-encoding)."""
    off = 5
    (n,) = struct.unpack_from("<I", body, off); off += 4
    rec = np.frombuffer(body, dtype=np.dtype([("s", "<u4"), ("a", "<u4"), ("d", "<f8"), ("k", "u1")]), count=n,
                        offset=off)
    off += rec.nbytes
    (nr,) = struct.unpack_from("<I", body, off); off += 4
    R = edge * edge
    counts = np.zeros(R, np.int64); sums = np.zeros((R, bands)); bits = np.zeros((R, (R + 31) // 32), np.uint32)
    for _ in range(nr):
        rid, cnt = struct.unpack_from("<II", body, off); off += 8
        sums[rid] = np.frombuffer(body, "<f8", bands, off); off += 8 * bands
        (na,) = struct.unpack_from("<H", body, off); off += 2
        for a in np.frombuffer(body, "<u4", na, off):
            bits[rid, a // 32] |= np.uint32(1 << (int(a) % 32))
        off += 4 * na
        counts[rid] = cnt
    assign = np.frombuffer(body, "<u4", R, off)
    return struct.unpack_from("<BHH", body), rec, counts, sums, bits, assign


def test_result_encoding_reproduces_reference_bytes():
    for frame, reply in _frames():
        _, payload = worker.decode_message(frame)
        sid, samples, _, _ = worker.decode_assign(payload)
        bands, edge, _ = samples.shape
        _, body = worker.decode_message(reply)
        sid2, rec, counts, sums, bits, assign = _parse_result(body, edge, bands)
        assert sid2 == sid
        again = worker.encode_result(sid, rec["s"], rec["a"], rec["d"], rec["k"], counts, sums, bits, assign)
        assert again == body


def test_malformed_frames_raise_protocol_errors():
    good = worker.encode_message(worker.HELLO)
    with pytest.raises(BadMagic):
        worker.decode_message(b"XXXX" + good[4:])
    with pytest.raises(BadVersion):
        worker.decode_message(good[:4] + bytes([2]) + good[5:])
    with pytest.raises(UnknownType):
        worker.decode_message(good[:5] + bytes([9]) + good[6:])
    with pytest.raises(Truncated):
        worker.decode_message(good[:5])
    frame, _ = next(_frames())
    _, payload = worker.decode_message(frame)
    with pytest.raises(Truncated):
        worker.decode_assign(payload[:-3])
    with pytest.raises(Truncated):
        worker.decode_assign(payload + b"\0")
