"""HSEG engine drop-in (API of rhseg/engine.py:29-371), executed on the B200.

* `hseg_run` (engine.py:345-371) runs the whole merge loop of one region graph
  on the device (persistent cluster kernel, csrc/hseg_kernels.cu) and then
  applies the returned merge log to the caller's graph with the reference's
  merge semantics, so the graph is mutated in place exactly as the reference
  would mutate it.
* `scan_adjacent` / `scan_nonadjacent` have the signatures of the reference's
  numba kernels (_kernels.py:31-115) and fill the same per-row tables on the
  device; `search_table`/`reduce_best`/`hseg_step` are built on them.
* Search strategies (Sequential / PerRegion / PerPair) are accepted for API
  compatibility; results never depend on them (engine.py:8-11), and the device
  path ignores them.
"""

from __future__ import annotations

import ctypes
import sys
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .dissim import MEASURE_CODES, resolve_measure
from .graph import MergeHierarchy, MergeKind, MergeRecord, RegionGraph, merge_regions


@dataclass
class HsegParams:
    """engine.py:29-42: spectral weight w in [0, 1], stopping count, measure."""

    spectral_weight: float = 0.21
    target_regions: int = 1
    measure: str = "sqrt-bsmse"

    def __post_init__(self):
        if not 0.0 <= self.spectral_weight <= 1.0:
            raise ValueError(f"spectral_weight must be in [0, 1], got {self.spectral_weight}")
        if self.target_regions < 1:
            raise ValueError(f"target_regions must be >= 1, got {self.target_regions}")
        resolve_measure(self.measure)


@dataclass(frozen=True)
class Sequential:
    pass


@dataclass(frozen=True)
class PerRegion:
    workers: int = 1

    def __post_init__(self):
        if self.workers < 1:
            raise ValueError("workers must be >= 1")


@dataclass(frozen=True)
class PerPair:
    tile_k: int = 16
    workers: int = 1

    def __post_init__(self):
        if self.tile_k < 1:
            raise ValueError("tile_k must be >= 1")
        if self.workers < 1:
            raise ValueError("workers must be >= 1")


SearchStrategy = Sequential | PerRegion | PerPair
STRATEGY_NAMES = {"seq": Sequential, "per-region": PerRegion, "per-pair": PerPair}


def make_strategy(name: str, tile_k: int = 16, workers: int = 1):
    if name == "seq":
        return Sequential()
    if name == "per-region":
        return PerRegion(workers=workers)
    if name == "per-pair":
        return PerPair(tile_k=tile_k, workers=workers)
    raise ValueError(f"unknown strategy {name!r}; choose from {sorted(STRATEGY_NAMES)}")


@dataclass
class ProfileStats:
    """engine.py:120-132. dissim_ns = device time of the dissimilarity kernels
    (all-pairs init + merge loop), total_ns = wall time of the call."""

    dissim_ns: int = 0
    total_ns: int = 0
    steps: int = 0

    @property
    def dissim_fraction(self) -> float:
        return 0.0 if self.total_ns == 0 else self.dissim_ns / self.total_ns


@dataclass
class BestPairTable:
    stage: MergeKind
    ids: np.ndarray
    partner_ids: np.ndarray
    dissims: np.ndarray

    def __len__(self) -> int:
        return len(self.ids)


@dataclass
class GraphSnapshot:
    """Dense ascending-id view (engine.py:155-191)."""

    ids: np.ndarray
    counts: np.ndarray
    sums: np.ndarray
    indptr: np.ndarray
    indices: np.ndarray


def snapshot(graph) -> GraphSnapshot:
    order = sorted(graph.regions)
    n = len(order)
    ids = np.asarray(order, dtype=np.int64)
    counts = np.fromiter((graph.regions[r].pixel_count for r in order), dtype=np.float64, count=n)
    sums = np.empty((n, graph.bands))
    for k, r in enumerate(order):
        sums[k] = graph.regions[r].band_sums
    degrees = np.fromiter((len(graph.regions[r].adjacency) for r in order), dtype=np.int64, count=n)
    nbr = np.fromiter(
        (x for r in order for x in graph.regions[r].adjacency), dtype=np.int64, count=int(degrees.sum())
    )
    cols = np.searchsorted(ids, nbr)
    rows = np.repeat(np.arange(n, dtype=np.int64), degrees)
    perm = np.lexsort((cols, rows))
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(degrees, out=indptr[1:])
    return GraphSnapshot(ids, counts, sums, indptr, np.ascontiguousarray(cols[perm]))


# ---------------------------------------------------------------------------
# B3: kernel seam (_kernels.py:31-115)
# ---------------------------------------------------------------------------
def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _scan_out(out, dtype):
    if out.dtype != dtype or not out.flags.c_contiguous:
        raise TypeError(f"output buffer must be C-contiguous {dtype}")
    return out


def scan_adjacent(row_start, row_stop, counts, sums, indptr, indices, out_d, out_j):
    """Device version of rhseg._kernels.scan_adjacent: best adjacent partner per
    row in [row_start, row_stop); writes only those rows of out_d / out_j."""
    counts, sums, indptr, indices = _f64(counts), _f64(sums), _i64(indptr), _i64(indices)
    n, nb = sums.shape
    _lib.check(
        _lib.load().rhseg_scan_adjacent(
            int(row_start), int(row_stop), n, nb, _lib.ptr(counts), _lib.ptr(sums), _lib.ptr(indptr),
            _lib.ptr(indices), _lib.ptr(_scan_out(out_d, np.float64)), _lib.ptr(_scan_out(out_j, np.int64)),
        ),
        "rhseg_scan_adjacent",
    )


def scan_nonadjacent(row_start, row_stop, col_tile, counts, sums, indptr, indices, out_d, out_j):
    """Device version of rhseg._kernels.scan_nonadjacent (col_tile accepted,
    result-invariant as in the reference)."""
    counts, sums, indptr, indices = _f64(counts), _f64(sums), _i64(indptr), _i64(indices)
    n, nb = sums.shape
    _lib.check(
        _lib.load().rhseg_scan_nonadjacent(
            int(row_start), int(row_stop), int(col_tile), n, nb, _lib.ptr(counts), _lib.ptr(sums),
            _lib.ptr(indptr), _lib.ptr(indices), _lib.ptr(_scan_out(out_d, np.float64)),
            _lib.ptr(_scan_out(out_j, np.int64)),
        ),
        "rhseg_scan_nonadjacent",
    )


def search_table(graph_or_snapshot, stage, strategy=Sequential(), profile: ProfileStats | None = None):
    snap = graph_or_snapshot if isinstance(graph_or_snapshot, GraphSnapshot) else snapshot(graph_or_snapshot)
    n = len(snap.ids)
    out_d = np.empty(n)
    out_j = np.empty(n, dtype=np.int64)
    t0 = time.perf_counter_ns()
    if n:
        if int(stage) == int(MergeKind.ADJACENT):
            scan_adjacent(0, n, snap.counts, snap.sums, snap.indptr, snap.indices, out_d, out_j)
        else:
            scan_nonadjacent(0, n, max(n, 1), snap.counts, snap.sums, snap.indptr, snap.indices, out_d, out_j)
    if profile is not None:
        profile.dissim_ns += time.perf_counter_ns() - t0
    partner = np.where(out_j >= 0, snap.ids[np.maximum(out_j, 0)], np.int64(-1))
    return BestPairTable(stage=MergeKind(int(stage)), ids=snap.ids, partner_ids=partner, dissims=out_d)


def reduce_best(table: BestPairTable):
    """engine.py:281-296: first row holding the minimum; None if not finite."""
    if len(table) == 0:
        return None
    k = int(np.argmin(table.dissims))
    d = float(table.dissims[k])
    if not np.isfinite(d):
        return None
    a, b = int(table.ids[k]), int(table.partner_ids[k])
    return ((a, b) if a < b else (b, a)), d


def best_adjacent_pair(graph, strategy=Sequential()):
    return reduce_best(search_table(graph, MergeKind.ADJACENT, strategy))


def best_nonadjacent_pair(graph, strategy=Sequential()):
    return reduce_best(search_table(graph, MergeKind.NON_ADJACENT, strategy))


def parallel_search_per_region(graph, stage, workers: int):
    return search_table(graph, stage, PerRegion(workers=workers))


def parallel_search_per_pair(graph, stage, tile_k: int, workers: int):
    return search_table(graph, stage, PerPair(tile_k=tile_k, workers=workers))


def _graph_api(graph):
    """(MergeHierarchy, MergeKind, merge_regions) of the module that defines
    `graph`'s class, so reference RegionGraph objects get reference records."""
    mod = sys.modules.get(type(graph).__module__)
    if mod is not None and all(hasattr(mod, n) for n in ("MergeHierarchy", "MergeKind", "merge_regions")):
        return mod.MergeHierarchy, mod.MergeKind, mod.merge_regions
    return MergeHierarchy, MergeKind, merge_regions


def hseg_step(graph, params, strategy=Sequential(), profile: ProfileStats | None = None):
    """One merge (engine.py:309-342) from device-built per-row tables. The B3
    table kernels are sqrt-bsmse only (as _kernels.py is); the extension
    measures take one step of the device loop instead (same rule, same pick)."""
    resolve_measure(params.measure)
    if params.measure != "sqrt-bsmse":
        if graph.live_count <= 1:
            return None
        h = hseg_run(graph, HsegParams(params.spectral_weight, graph.live_count - 1, params.measure), strategy,
                     profile)
        return h.records[0] if h.records else None
    _, Kind, merge = _graph_api(graph)
    snap = snapshot(graph)
    adjacent = reduce_best(search_table(snap, MergeKind.ADJACENT, strategy, profile))
    chosen, kind = None, None
    if params.spectral_weight > 0.0:
        spectral = reduce_best(search_table(snap, MergeKind.NON_ADJACENT, strategy, profile))
        if spectral is not None:
            d_a = adjacent[1] if adjacent is not None else np.inf
            if spectral[1] < params.spectral_weight * d_a:
                chosen, kind = spectral, Kind.NON_ADJACENT
    if chosen is None and adjacent is not None:
        chosen, kind = adjacent, Kind.ADJACENT
    if chosen is None:
        return None
    if profile is not None:
        profile.steps += 1
    (a, b), d = chosen
    return merge(graph, a, b, d, kind)


def hseg_run(graph, params, strategy=Sequential(), profile: ProfileStats | None = None, stop_check=None,
             device: int | None = None, cluster: int = 0):
    """Merge until target_regions remain (engine.py:345-371), on the device.

    The whole loop runs in one persistent kernel (no per-step host round trip).
    `stop_check` keeps the reference's contract exactly (engine.py:351-363): it is
    called before every step, with the caller's graph at that step boundary, and a
    True ends the run with `interrupted` set. That is possible without stopping the
    device because the merge sequence does not depend on when a run stops -- the
    reference's interrupted run is a prefix of the full one -- so the device computes
    the whole log and the host applies it one merge per stop_check."""
    t0 = time.perf_counter_ns()
    Hier, Kind, merge = _graph_api(graph)
    resolve_measure(params.measure)
    hierarchy = Hier(initial_region_count=graph.live_count)
    target = int(params.target_regions)
    if graph.live_count > target:
        if stop_check is not None and stop_check():
            hierarchy.interrupted = True
        else:
            snap = snapshot(graph)
            n, nb = snap.sums.shape
            cap = max(n, 1)
            sa = np.empty(cap, np.int32)
            sb = np.empty(cap, np.int32)
            sd = np.empty(cap, np.float64)
            sk = np.empty(cap, np.uint8)
            nrec = ctypes.c_int64(0)
            conv = ctypes.c_int32(0)
            ctx = _lib.context(device)
            with ctx.lock:
                _lib.check(
                    _lib.load().rhseg_hseg_graph(
                        ctx.handle, n, nb, _lib.ptr(snap.counts), _lib.ptr(np.ascontiguousarray(snap.sums)),
                        _lib.ptr(snap.indptr), _lib.ptr(snap.indices), float(params.spectral_weight),
                        min(target, 2**62), int(cluster), MEASURE_CODES[params.measure], _lib.ptr(sa),
                        _lib.ptr(sb), _lib.ptr(sd), _lib.ptr(sk), ctypes.byref(nrec), ctypes.byref(conv),
                    ),
                    "rhseg_hseg_graph",
                )
                dev_ms = _phase_ms(ctx)
            ids = snap.ids
            applied = 0
            for k in range(nrec.value):
                # the first step's check already ran above
                if k > 0 and stop_check is not None and stop_check():
                    hierarchy.interrupted = True
                    break
                hierarchy.records.append(
                    merge(graph, int(ids[sa[k]]), int(ids[sb[k]]), float(sd[k]), Kind(int(sk[k])))
                )
                applied += 1
            if not hierarchy.interrupted and conv.value:
                # the reference checks once more before the step that finds no pair
                if applied > 0 and stop_check is not None and stop_check():
                    hierarchy.interrupted = True
                else:
                    hierarchy.converged_early = True
            if profile is not None:
                profile.steps += applied
                profile.dissim_ns += int((dev_ms[1] + dev_ms[2]) * 1e6)
    if profile is not None:
        profile.total_ns += time.perf_counter_ns() - t0
    return hierarchy


def _phase_ms(ctx) -> np.ndarray:
    ms = np.zeros(4, np.float32)
    st = _lib.load().rhseg_result_phase_ms(ctx.handle, _lib.ptr(ms))
    return ms if st == 0 else np.zeros(4, np.float32)


def measure_code(name: str) -> int:
    resolve_measure(name)
    return MEASURE_CODES[name]
