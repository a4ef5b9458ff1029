"""ctypes wrapper around the C oracle (oracle/rhseg_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py, always as the checker or the
timed CPU reference -- never by the product package.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "librhseg_oracle.so")

_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(
        os.path.join(HERE, "rhseg_oracle.c")
    ):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        i64, i32, f64, vp = ctypes.c_int64, ctypes.c_int32, ctypes.c_double, ctypes.c_void_p
        L.oracle_scan_adjacent.argtypes = [i64, i64, i64, i64, vp, vp, vp, vp, vp, vp]
        L.oracle_scan_adjacent.restype = None
        L.oracle_scan_nonadjacent.argtypes = [i64, i64, i64, i64, i64, vp, vp, vp, vp, vp, vp]
        L.oracle_scan_nonadjacent.restype = None
        L.oracle_hseg_graph.argtypes = [i64, i64, vp, vp, vp, vp, i64, f64, i64, i64, vp, vp, vp, vp, vp]
        L.oracle_hseg_graph.restype = i64
        L.oracle_rhseg_run.argtypes = [vp, i64, i64, i32, f64, i64, i64, i32, i64] + [vp] * 11
        L.oracle_rhseg_run.restype = i64
        L.oracle_rhseg_replay_leaves.argtypes = [vp, i64, i64, i32, f64, i64, i64, i32, i64] + [vp] * 16
        L.oracle_rhseg_replay_leaves.restype = i64
        L.oracle_run_leaf.argtypes = [vp, i64, i64, i64, i64, i64, f64, i64, i32, i64]
        L.oracle_run_leaf.restype = i64
        L.oracle_run_leaves.argtypes = [vp, i64, i64, i64, vp, vp, i64, f64, i64, i32, vp]
        L.oracle_run_leaves.restype = None
        L.oracle_set_threads.argtypes = [ctypes.c_int]
        L.oracle_set_threads.restype = None
        L.oracle_set_incremental.argtypes = [ctypes.c_int]
        L.oracle_set_incremental.restype = None
        L.oracle_set_measure.argtypes = [ctypes.c_int]
        L.oracle_set_measure.restype = None
        L.oracle_acos.argtypes = [ctypes.c_double]
        L.oracle_acos.restype = ctypes.c_double
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def set_threads(n: int) -> None:
    lib().oracle_set_threads(int(n))


def set_incremental(on: bool) -> None:
    """Process-wide HSEG mode of every following call: False (default) = the literal
    restatement (both per-row tables rebuilt every step, engine.py:309-342); True = the
    exact incremental checker (cached D and per-row bests, sections of a level in
    parallel) -- the same records bit for bit, affordable at the full BASELINE sizes."""
    lib().oracle_set_incremental(1 if on else 0)


MEASURE_CODES = {"sqrt-bsmse": 0, "euclidean": 1, "sam": 2}


def set_measure(name: str) -> None:
    """Dissimilarity for every following call (process-wide): "sqrt-bsmse"
    (the reference's), or the extensions "euclidean" / "sam"."""
    lib().oracle_set_measure(MEASURE_CODES[name])


def acos(x: float) -> float:
    return lib().oracle_acos(float(x))


def scan_adjacent(row_start, row_stop, counts, sums, indptr, indices, out_d, out_j):
    """Restatement of rhseg._kernels.scan_adjacent (_kernels.py:31-59)."""
    counts = np.ascontiguousarray(counts, dtype=np.float64)
    sums = np.ascontiguousarray(sums, dtype=np.float64)
    indptr = np.ascontiguousarray(indptr, dtype=np.int64)
    indices = np.ascontiguousarray(indices, dtype=np.int64)
    n, nb = sums.shape
    lib().oracle_scan_adjacent(row_start, row_stop, n, nb, _p(counts), _p(sums), _p(indptr),
                               _p(indices), _p(out_d), _p(out_j))


def scan_nonadjacent(row_start, row_stop, col_tile, counts, sums, indptr, indices, out_d, out_j):
    """Restatement of rhseg._kernels.scan_nonadjacent (_kernels.py:62-115)."""
    counts = np.ascontiguousarray(counts, dtype=np.float64)
    sums = np.ascontiguousarray(sums, dtype=np.float64)
    indptr = np.ascontiguousarray(indptr, dtype=np.int64)
    indices = np.ascontiguousarray(indices, dtype=np.int64)
    n, nb = sums.shape
    lib().oracle_scan_nonadjacent(row_start, row_stop, col_tile, n, nb, _p(counts), _p(sums),
                                  _p(indptr), _p(indices), _p(out_d), _p(out_j))


def hseg_graph(counts, sums, adj, weight, target, assign=None):
    """hseg_run (engine.py:345-371) on a dense-index graph. Mutates copies;
    returns dict(records=(surv, abs, d, kind), counts, sums, adj, assign, converged)."""
    counts = np.array(counts, dtype=np.int64)
    sums = np.array(sums, dtype=np.float64, order="C")
    adj = np.array(adj, dtype=np.uint8, order="C")
    R0, nb = sums.shape
    cap = max(R0, 1)
    surv = np.zeros(cap, np.int32)
    absd = np.zeros(cap, np.int32)
    d = np.zeros(cap, np.float64)
    kind = np.zeros(cap, np.uint8)
    conv = np.zeros(1, np.int32)
    if assign is not None:
        assign = np.array(assign, dtype=np.int32)
        npx = assign.size
        ap = _p(assign)
    else:
        npx, ap = 0, None
    n = lib().oracle_hseg_graph(R0, nb, _p(counts), _p(sums), _p(adj), ap, npx, float(weight),
                                int(target), cap, _p(surv), _p(absd), _p(d), _p(kind), _p(conv))
    return dict(records=(surv[:n], absd[:n], d[:n], kind[:n]), counts=counts, sums=sums, adj=adj,
                assign=assign, converged=bool(conv[0]))


def rhseg_run(samples, levels, weight, target, section_target=None, connectivity=8):
    """SequentialExecutor.execute (recursive.py:173-209) restated. samples:
    float32 BSQ (bands, edge, edge). Returns dict of flat-log arrays + labels."""
    samples = np.ascontiguousarray(samples, dtype=np.float32)
    nb, edge, _ = samples.shape
    if section_target is None:
        section_target = target
    cap = edge * edge * 2 + 16
    out = {
        "log_level": np.zeros(cap, np.int16),
        "log_row": np.zeros(cap, np.int32),
        "log_col": np.zeros(cap, np.int32),
        "log_survivor": np.zeros(cap, np.int32),
        "log_absorbed": np.zeros(cap, np.int32),
        "log_dissim": np.zeros(cap, np.float64),
        "log_kind": np.zeros(cap, np.uint8),
    }
    labels = np.zeros(edge * edge, np.int32)
    assignment = np.zeros(edge * edge, np.int32)
    rootinit = np.zeros(1, np.int64)
    conv = np.zeros(1, np.int32)
    n = lib().oracle_rhseg_run(
        _p(samples), edge, nb, int(levels), float(weight), int(target), int(section_target),
        int(connectivity), cap, _p(out["log_level"]), _p(out["log_row"]), _p(out["log_col"]),
        _p(out["log_survivor"]), _p(out["log_absorbed"]), _p(out["log_dissim"]),
        _p(out["log_kind"]), _p(labels), _p(assignment), _p(rootinit), _p(conv))
    if n < 0:
        raise ValueError(f"edge {edge} not divisible by {2 ** (levels - 1)} (levels={levels})")
    res = {k: v[:n] for k, v in out.items()}
    res["labels"] = labels.reshape(edge, edge)
    res["assignment"] = assignment.reshape(edge, edge)
    res["root_initial_count"] = int(rootinit[0])
    res["converged_early"] = bool(conv[0])
    return res


def rhseg_replay_leaves(samples, levels, weight, target, section_target, leaf_logs, connectivity=8):
    """rhseg_run with the leaf level REPLAYED from `leaf_logs` = (counts per leaf
    row-major, survivor, absorbed, dissim, kind) and every upper level computed
    from scratch (recursive.py:145-170): checks all upper levels of a run too big
    for the from-scratch oracle. Returns the same dict as rhseg_run."""
    samples = np.ascontiguousarray(samples, dtype=np.float32)
    nb, edge, _ = samples.shape
    counts, sv, ab, dd, kk = leaf_logs
    counts = np.ascontiguousarray(counts, np.int64)
    sv = np.ascontiguousarray(sv, np.int32)
    ab = np.ascontiguousarray(ab, np.int32)
    dd = np.ascontiguousarray(dd, np.float64)
    kk = np.ascontiguousarray(kk, np.uint8)
    cap = int(counts.sum()) + edge * edge + 16
    out = {
        "log_level": np.zeros(cap, np.int16),
        "log_row": np.zeros(cap, np.int32),
        "log_col": np.zeros(cap, np.int32),
        "log_survivor": np.zeros(cap, np.int32),
        "log_absorbed": np.zeros(cap, np.int32),
        "log_dissim": np.zeros(cap, np.float64),
        "log_kind": np.zeros(cap, np.uint8),
    }
    labels = np.zeros(edge * edge, np.int32)
    assignment = np.zeros(edge * edge, np.int32)
    rootinit = np.zeros(1, np.int64)
    conv = np.zeros(1, np.int32)
    n = lib().oracle_rhseg_replay_leaves(
        _p(samples), edge, nb, int(levels), float(weight), int(target), int(section_target),
        int(connectivity), cap, _p(out["log_level"]), _p(out["log_row"]), _p(out["log_col"]),
        _p(out["log_survivor"]), _p(out["log_absorbed"]), _p(out["log_dissim"]),
        _p(out["log_kind"]), _p(labels), _p(assignment), _p(rootinit), _p(conv),
        _p(counts), _p(sv), _p(ab), _p(dd), _p(kk))
    if n < 0:
        raise ValueError(f"edge {edge} not divisible by {2 ** (levels - 1)} (levels={levels})")
    res = {k: v[:n] for k, v in out.items()}
    res["labels"] = labels.reshape(edge, edge)
    res["assignment"] = assignment.reshape(edge, edge)
    res["root_initial_count"] = int(rootinit[0])
    res["converged_early"] = bool(conv[0])
    return res


def run_leaf(samples, orow, ocol, sec_edge, weight, target, connectivity=8, max_steps=-1):
    """run_leaf (recursive.py:130-142) restated; returns merges performed."""
    samples = np.ascontiguousarray(samples, dtype=np.float32)
    nb, edge, _ = samples.shape
    return lib().oracle_run_leaf(_p(samples), edge, nb, orow, ocol, sec_edge, float(weight),
                                 int(target), int(connectivity), int(max_steps))


def run_leaves(samples, origins, sec_edge, weight, target, connectivity=8):
    """Section-parallel CPU baseline: whole leaves (run_leaf, recursive.py:130-142),
    one leaf per host thread (the process-per-section strategy of cluster.py), each
    leaf's scans single-threaded. origins: [(row, col), ...]. Returns merges per leaf."""
    samples = np.ascontiguousarray(samples, dtype=np.float32)
    nb, edge, _ = samples.shape
    o = np.ascontiguousarray(np.asarray(origins, dtype=np.int64).reshape(-1, 2))
    orow = np.ascontiguousarray(o[:, 0])
    ocol = np.ascontiguousarray(o[:, 1])
    merges = np.zeros(len(o), np.int64)
    lib().oracle_run_leaves(_p(samples), edge, nb, len(o), _p(orow), _p(ocol), int(sec_edge), float(weight),
                            int(target), int(connectivity), _p(merges))
    return merges
