"""The B200 worker answers the reference master's ASSIGN frames with RESULT
frames byte-identical to the unmodified reference worker's replies
(tests/golden/wire_frames.npz), directly and over a loopback TCP connection."""

import socket

import pytest

from golden_io import load
from paper_2106_12942_b200 import worker

pytestmark = pytest.mark.gpu


def _frames():
    z = load("wire_frames.npz")
    for k in range(int(z["n"])):
        yield z[f"assign_{k}"].tobytes(), z[f"result_{k}"].tobytes()


def test_run_assign_matches_reference_result():
    for frame, reply in _frames():
        _, payload = worker.decode_message(frame)
        assert worker.run_assign(payload) == reply


def test_tcp_worker_session():
    server = worker.GpuWorkerServer("127.0.0.1", 0).start()
    try:
        with socket.create_connection(server.endpoint, timeout=60) as s:
            rd = s.makefile("rb")
            s.sendall(worker.encode_message(worker.HELLO))
            assert worker.read_message(rd)[0] == worker.HELLO
            for frame, reply in _frames():
                s.sendall(frame)
                t, body = worker.read_message(rd)
                assert t == worker.RESULT and worker.encode_message(t, body) == reply
            # a bad assignment is reported, not fatal
            _, payload = worker.decode_message(next(_frames())[0])
            bad = bytearray(payload)
            bad[5 + 16:5 + 20] = (0).to_bytes(4, "little")  # section_target 0 -> ValueError
            s.sendall(worker.encode_message(worker.ASSIGN, bytes(bad)))
            t, body = worker.read_message(rd)
            assert t == worker.ERROR and b"ValueError" in body
            s.sendall(worker.encode_message(worker.SHUTDOWN))
    finally:
        server.stop()
