"""A B200 worker for the reference's cluster protocol.

The reference scales out with a TCP master/worker pair (cluster.py:53-338) that
speaks a framed binary protocol (wire.py): the master sends ASSIGN (a section's
f32 sub-cube + merge parameters), the worker runs the section's HSEG and replies
RESULT (merge log, region graph, pixel assignment, f64 everything bit-exact).
This module restates that protocol and serves it from the GPU: a reference
`ClusterExecutor` pointed at this worker gets byte-identical RESULT frames
(pinned against the reference worker's own replies in tests/golden/wire_frames.npz).

Frame (wire.py:23-44): b"RHSG" | u8 version 1 | u8 type | u32 payload length (LE).
ASSIGN payload (wire.py:112-123): <BHH section (level,row,col), <IIdIBH (edge, bands,
weight, section_target, strategy code, tile_k), f32 samples [bands][edge][edge].
RESULT payload (wire.py:151-169): <BHH section, <I n_records, n x <IIdB (survivor,
absorbed, dissim, kind), <I n_regions, per live region ascending: <II (id, count),
f64 sums[bands], <H n_adj, u32 adjacency ascending; u32 pixel assignment [edge*edge].
"""

from __future__ import annotations

import argparse
import logging
import socket
import struct
import threading

import numpy as np

from .errors import BadMagic, BadVersion, ProtocolError, Truncated, UnknownType

MAGIC = b"RHSG"
VERSION = 1
HELLO, ASSIGN, RESULT, ERROR, SHUTDOWN = 1, 2, 3, 4, 5
_TYPES = {HELLO, ASSIGN, RESULT, ERROR, SHUTDOWN}
_HEADER = struct.Struct("<4sBBI")
HEADER_SIZE = _HEADER.size
STRATEGY_CODES = {"seq": 0, "per-region": 1, "per-pair": 2}
_SECTION = struct.Struct("<BHH")
_ASSIGN_FIXED = struct.Struct("<IIdIBH")

log = logging.getLogger("paper_2106_12942_b200.worker")


def encode_message(msg_type: int, payload: bytes = b"") -> bytes:
    if msg_type not in _TYPES:
        raise UnknownType(f"unknown message type {msg_type}")
    return _HEADER.pack(MAGIC, VERSION, msg_type, len(payload)) + payload


def encode_error(reason: str) -> bytes:
    return encode_message(ERROR, reason.encode("utf-8", errors="replace"))


def _check_header(magic, version, msg_type):
    if magic != MAGIC:
        raise BadMagic(f"bad magic {magic!r}")
    if version != VERSION:
        raise BadVersion(f"unsupported version {version}")
    if msg_type not in _TYPES:
        raise UnknownType(f"unknown message type {msg_type}")


def decode_message(data: bytes) -> tuple[int, bytes]:
    if len(data) < HEADER_SIZE:
        raise Truncated(f"frame header needs {HEADER_SIZE} bytes, got {len(data)}")
    magic, version, msg_type, length = _HEADER.unpack_from(data)
    _check_header(magic, version, msg_type)
    if len(data) < HEADER_SIZE + length:
        raise Truncated(f"payload declares {length} bytes, frame holds {len(data) - HEADER_SIZE}")
    return msg_type, data[HEADER_SIZE:HEADER_SIZE + length]


def read_message(stream) -> tuple[int, bytes]:
    header = stream.read(HEADER_SIZE)
    if len(header) < HEADER_SIZE:
        raise Truncated("connection closed mid-header")
    magic, version, msg_type, length = _HEADER.unpack(header)
    _check_header(magic, version, msg_type)
    payload = stream.read(length)
    if len(payload) < length:
        raise Truncated("connection closed mid-payload")
    return msg_type, payload


def decode_assign(payload: bytes):
    """-> (section (level,row,col), samples f32 [bands][edge][edge], weight, target)."""
    fixed = _SECTION.size + _ASSIGN_FIXED.size
    if len(payload) < fixed:
        raise Truncated(f"payload ends {fixed - len(payload)} bytes short")
    sid = _SECTION.unpack_from(payload)
    edge, bands, weight, target, code, _tile = _ASSIGN_FIXED.unpack_from(payload, _SECTION.size)
    if code not in STRATEGY_CODES.values():
        raise UnknownType(f"unknown strategy code {code}")
    need = fixed + edge * edge * bands * 4
    if len(payload) < need:
        raise Truncated(f"payload ends {need - len(payload)} bytes short")
    if len(payload) > need:
        raise Truncated(f"{len(payload) - need} trailing bytes in payload")
    samples = np.frombuffer(payload, dtype="<f4", count=edge * edge * bands, offset=fixed)
    return sid, samples.reshape(bands, edge, edge).astype(np.float32), weight, target


def encode_result(sid, survivor, absorbed, dissim, kind, counts, sums, adj_bits, assignment) -> bytes:
    """RESULT payload from device result arrays (wire.py:151-169 layout).
    counts[R] (0 = dead), sums[R][bands] f64, adj_bits[R][ceil(R/32)] u32, assignment[npx]."""
    n = len(survivor)
    rec = np.zeros(n, dtype=np.dtype([("s", "<u4"), ("a", "<u4"), ("d", "<f8"), ("k", "u1")]))
    rec["s"], rec["a"], rec["d"], rec["k"] = survivor, absorbed, dissim, kind
    parts = [_SECTION.pack(*sid), struct.pack("<I", n), rec.tobytes()]
    live = np.nonzero(counts > 0)[0]
    parts.append(struct.pack("<I", len(live)))
    R = len(counts)
    bits = np.unpackbits(adj_bits.view(np.uint8), axis=1, bitorder="little")[:, :R]
    for rid in live:
        nbr = np.nonzero(bits[rid])[0].astype("<u4")
        parts.append(struct.pack("<II", int(rid), int(counts[rid])))
        parts.append(np.ascontiguousarray(sums[rid], dtype="<f8").tobytes())
        parts.append(struct.pack("<H", len(nbr)))
        parts.append(nbr.tobytes())
    parts.append(np.ascontiguousarray(assignment, dtype="<u4").tobytes())
    return b"".join(parts)


def run_assign(payload: bytes, device: int | None = None) -> bytes:
    """One ASSIGN -> RESULT frame, computed on the B200 (cluster.py:309-327
    semantics: init_region_graph(image, 8) + hseg_run to section_target)."""
    import ctypes

    from . import _lib
    from .recursive import B200Executor, RhsegParams
    from .engine import HsegParams

    try:
        sid, samples, weight, target = decode_assign(payload)
        bands, edge, _ = samples.shape
        ex = B200Executor(connectivity=8, device=device)
        params = RhsegParams(HsegParams(weight, target), 1, target)
        cp = ex.c_params(params)
        ctx = _lib.context(device)
        L = _lib.load()
        with ctx.lock:
            info = _lib.ResultInfoC()
            _lib.check(L.rhseg_run_host(ctx.handle, _lib.ptr(np.ascontiguousarray(samples)), edge, bands,
                                        ctypes.byref(cp), None, None, None, None, None, None, ctypes.byref(info)),
                       "rhseg_run_host")
            n = int(info.n_records)
            sa, sb = np.zeros(max(n, 1), np.int32), np.zeros(max(n, 1), np.int32)
            sd, sk = np.zeros(max(n, 1), np.float64), np.zeros(max(n, 1), np.uint8)
            _lib.check(L.rhseg_result_log(ctx.handle, _lib.ptr(sa), _lib.ptr(sb), _lib.ptr(sd), _lib.ptr(sk)),
                       "rhseg_result_log")
            R = int(info.root_idspace)
            counts = np.zeros(R, np.int64)
            sums = np.zeros((R, bands), np.float64)
            wo = max((R + 31) // 32, 1)
            bits = np.zeros((R, wo), np.uint32)
            assign = np.zeros(edge * edge, np.int32)
            _lib.check(L.rhseg_result_root(ctx.handle, 1, _lib.ptr(counts), _lib.ptr(sums), _lib.ptr(bits),
                                           _lib.ptr(assign)), "rhseg_result_root")
        body = encode_result(sid, sa[:n], sb[:n], sd[:n], sk[:n], counts, sums, bits, assign)
        return encode_message(RESULT, body)
    except Exception as exc:  # noqa: BLE001 - reported to the master like the reference worker
        return encode_error(f"{type(exc).__name__}: {exc}")


class GpuWorkerServer:
    """Serves the reference master (cluster.py:220-327 WorkerServer interface):
    HELLO -> HELLO, ASSIGN -> RESULT/ERROR, SHUTDOWN stops the server."""

    def __init__(self, host: str = "127.0.0.1", port: int = 0, device: int | None = None):
        self.device = device
        self._stop = threading.Event()
        self._sock = socket.socket(socket.AF_INET, socket.SOCK_STREAM)
        self._sock.setsockopt(socket.SOL_SOCKET, socket.SO_REUSEADDR, 1)
        self._sock.bind((host, port))
        self._sock.listen(8)
        self._sock.settimeout(0.2)
        self.address = self._sock.getsockname()
        self._threads: list[threading.Thread] = []
        self._accept_thread: threading.Thread | None = None

    @property
    def endpoint(self) -> tuple[str, int]:
        return self.address[0], self.address[1]

    def start(self) -> "GpuWorkerServer":
        self._accept_thread = threading.Thread(target=self._accept_loop, daemon=True)
        self._accept_thread.start()
        return self

    def serve_forever(self):
        self._accept_loop()

    def stop(self):
        self._stop.set()
        if self._accept_thread is not None:
            self._accept_thread.join(timeout=5)
        for t in self._threads:
            t.join(timeout=5)
        self._sock.close()

    def _accept_loop(self):
        while not self._stop.is_set():
            try:
                conn, _ = self._sock.accept()
            except socket.timeout:
                continue
            except OSError:
                break
            t = threading.Thread(target=self._handle, args=(conn,), daemon=True)
            t.start()
            self._threads.append(t)

    def _handle(self, conn: socket.socket):
        try:
            rd, wr = conn.makefile("rb"), conn.makefile("wb")
            while not self._stop.is_set():
                try:
                    msg_type, payload = read_message(rd)
                except ProtocolError:
                    return
                if msg_type == HELLO:
                    wr.write(encode_message(HELLO))
                elif msg_type == SHUTDOWN:
                    self._stop.set()
                    return
                elif msg_type == ASSIGN:
                    wr.write(run_assign(payload, self.device))
                else:
                    wr.write(encode_error(f"unexpected message {msg_type}"))
                wr.flush()
        finally:
            conn.close()


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description="B200 worker for the rhseg cluster protocol")
    ap.add_argument("--listen", default="127.0.0.1:0", help="host:port")
    ap.add_argument("--device", type=int, default=0)
    a = ap.parse_args(argv)
    host, port = a.listen.rsplit(":", 1)
    server = GpuWorkerServer(host, int(port), a.device)
    print(f"rhseg-b200 worker listening on {server.endpoint[0]}:{server.endpoint[1]}", flush=True)
    try:
        server.serve_forever()
    finally:
        server._sock.close()
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
