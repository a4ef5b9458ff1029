"""RHSEG recursion drop-in (API of rhseg/recursive.py:30-223) on the B200.

`B200Executor.execute(image, params, strategy, profile) -> RhsegResult` is the
executor seam of the reference (recursive.py:179-185): the whole quadtree --
leaf HSEG, stitching, every upper level, root labels -- runs on the device
through one C-ABI call (rhseg_run_host / rhseg_run_device), and the result is
assembled with the reference's field names and canonical log order.
"""

from __future__ import annotations

import ctypes
import time
from collections.abc import Sequence
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .dissim import MEASURE_CODES
from .engine import HsegParams, ProfileStats, Sequential, _phase_ms, hseg_run
from .graph import (LabelMap, MergeHierarchy, MergeKind, MergeRecord, RegionGraph, extract_labels,
                    label_map_from_graph)
from .sections import SectionId, check_divisible, log_order, section_side, stitch


@dataclass
class RhsegParams:
    """recursive.py:30-59: recursion depth + merge-loop parameters."""

    hseg: HsegParams = field(default_factory=HsegParams)
    levels: int = 1
    section_target_regions: int | None = None

    def __post_init__(self):
        if self.levels < 1:
            raise ValueError(f"levels must be >= 1, got {self.levels}")
        if self.section_target_regions is None:
            self.section_target_regions = self.hseg.target_regions
        if self.section_target_regions < 1:
            raise ValueError("section_target_regions must be >= 1")

    def target_for(self, section_id: SectionId) -> int:
        return self.hseg.target_regions if section_id.level == 1 else self.section_target_regions

    def section_params(self, section_id: SectionId) -> HsegParams:
        return HsegParams(self.hseg.spectral_weight, self.target_for(section_id), self.hseg.measure)


class RecordList(Sequence):
    """Lazy sequence of MergeRecord over device-returned arrays (a C4 run has
    4.2 M records; materialising them eagerly would dominate the host side)."""

    __slots__ = ("_a", "_b", "_d", "_k")

    def __init__(self, a, b, d, k):
        self._a, self._b, self._d, self._k = a, b, d, k

    def __len__(self):
        return len(self._a)

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[j] for j in range(*i.indices(len(self)))]
        if i < 0:
            i += len(self)
        if not 0 <= i < len(self):
            raise IndexError(i)
        return MergeRecord(i, int(self._a[i]), int(self._b[i]), float(self._d[i]), MergeKind(int(self._k[i])))

    def __eq__(self, other):
        """Field by field, so a list of the reference's own MergeRecord objects (another
        class with the same fields, graph.py:41-47) compares equal to the same records."""
        try:
            if len(self) != len(other):
                return False
            return all(
                (x.step, x.survivor_id, x.absorbed_id, x.dissimilarity, int(x.kind))
                == (y.step, y.survivor_id, y.absorbed_id, y.dissimilarity, int(y.kind))
                for x, y in zip(self, other)
            )
        except (TypeError, AttributeError):
            return NotImplemented

    def arrays(self):
        return self._a, self._b, self._d, self._k


@dataclass
class RhsegResult:
    """recursive.py:62-92."""

    section_logs: list
    root_initial: RegionGraph
    root_hierarchy: MergeHierarchy
    graph: RegionGraph
    labels: LabelMap
    converged_early: bool = False
    spectral_pairs: int = 0
    device_ms: float = 0.0

    def labels_at(self, region_count: int) -> LabelMap:
        return extract_labels(self.root_hierarchy, self.root_initial, region_count)

    def flat_log(self):
        step = 0
        for sid, records in self.section_logs:
            a, b, d, k = records.arrays() if isinstance(records, RecordList) else _rec_arrays(records)
            for i in range(len(a)):
                yield {
                    "step": step,
                    "level": sid.level,
                    "section": [sid.row, sid.col],
                    "survivor": int(a[i]),
                    "absorbed": int(b[i]),
                    "dissim": float(d[i]),
                    "kind": "adjacent" if int(k[i]) == 0 else "non_adjacent",
                }
                step += 1


def _rec_arrays(records):
    return (
        [r.survivor_id for r in records],
        [r.absorbed_id for r in records],
        [r.dissimilarity for r in records],
        [int(r.kind) for r in records],
    )


def _hseg_fields(params):
    h = params.hseg
    measure = getattr(h, "measure", "sqrt-bsmse")
    if measure not in MEASURE_CODES:
        raise ValueError(f"unknown measure {measure!r}; available: {sorted(MEASURE_CODES)}")
    return float(h.spectral_weight), int(h.target_regions), MEASURE_CODES[measure]


class B200Executor:
    """Executor seam (recursive.py:173-209) running every section on one B200.

    cluster: CTAs per section (0 = auto: leaves of few-section levels get up
    to 16 SMs each, many-section levels one CTA per section)."""

    def __init__(self, connectivity: int = 8, device: int | None = None, cluster: int = 0):
        if connectivity not in (4, 8):
            raise ValueError(f"connectivity must be 4 or 8, got {connectivity}")
        self.connectivity = connectivity
        self.device = device
        self.cluster = cluster
        self.last_phase_ms = np.zeros(4, np.float32)

    def c_params(self, params):
        w, t, m = _hseg_fields(params)
        return _lib.make_params(w, t, params.section_target_regions or t, params.levels, self.connectivity, m,
                                self.cluster)

    def execute(self, image, params, strategy=Sequential(), profile: ProfileStats | None = None) -> RhsegResult:
        t0 = time.perf_counter_ns()
        check_divisible(image.width, params.levels)
        samples = np.ascontiguousarray(image.samples, dtype=np.float32)
        cp = self.c_params(params)
        ctx = _lib.context(self.device)
        info = _lib.ResultInfoC()
        with ctx.lock:
            _lib.check(
                _lib.load().rhseg_run_host(ctx.handle, _lib.ptr(samples), image.width, image.bands,
                                           ctypes.byref(cp), None, None, None, None, None, None,
                                           ctypes.byref(info)),
                "rhseg_run_host",
            )
            result = collect_result(ctx, info, image.width, image.bands, params.levels)
            self.last_phase_ms = _phase_ms(ctx)
        if profile is not None:
            ms = self.last_phase_ms
            profile.dissim_ns += int((ms[1] + ms[2]) * 1e6)
            profile.steps += int(info.n_records)
            profile.total_ns += time.perf_counter_ns() - t0
        return result

    def execute_device(self, samples_dev_ptr: int, edge: int, bands: int, params, stream: int = 0):
        """Run on a cube already resident in HBM (e.g. a torch CUDA tensor's
        data_ptr()); results stay on the device until collect_result()."""
        cp = self.c_params(params)
        ctx = _lib.context(self.device)
        with ctx.lock:
            _lib.check(
                _lib.load().rhseg_run_device(ctx.handle, ctypes.c_void_p(samples_dev_ptr), edge, bands,
                                             ctypes.byref(cp), ctypes.c_void_p(stream) if stream else None),
                "rhseg_run_device",
            )
        return ctx


def result_info(ctx) -> _lib.ResultInfoC:
    info = _lib.ResultInfoC()
    _lib.check(_lib.load().rhseg_result_info_get(ctx.handle, ctypes.byref(info)), "rhseg_result_info_get")
    return info


def collect_result(ctx, info, edge: int, bands: int, levels: int) -> RhsegResult:
    """Copy a finished device run into an RhsegResult (host objects)."""
    L = _lib.load()
    n = int(info.n_records)
    ns = int(info.n_sections)
    lev = np.empty(ns, np.int32)
    row = np.empty(ns, np.int32)
    col = np.empty(ns, np.int32)
    off = np.empty(ns, np.int64)
    cnt = np.empty(ns, np.int64)
    _lib.check(L.rhseg_result_sections(ctx.handle, _lib.ptr(lev), _lib.ptr(row), _lib.ptr(col), _lib.ptr(off),
                                       _lib.ptr(cnt)), "rhseg_result_sections")
    sa = np.empty(n, np.int32)
    sb = np.empty(n, np.int32)
    sd = np.empty(n, np.float64)
    sk = np.empty(n, np.uint8)
    _lib.check(L.rhseg_result_log(ctx.handle, _lib.ptr(sa), _lib.ptr(sb), _lib.ptr(sd), _lib.ptr(sk)),
               "rhseg_result_log")
    section_logs = []
    for s in range(ns):
        o, c = int(off[s]), int(cnt[s])
        section_logs.append(
            (SectionId(int(lev[s]), int(row[s]), int(col[s])), RecordList(sa[o:o + c], sb[o:o + c], sd[o:o + c],
                                                                          sk[o:o + c]))
        )
    npx = edge * edge
    labels = np.empty(npx, np.int32)
    _lib.check(L.rhseg_result_labels(ctx.handle, _lib.ptr(labels), None), "rhseg_result_labels")
    R = int(info.root_idspace)
    wo = (R + 31) // 32
    graphs = []
    for which in (0, 1):
        counts = np.empty(R, np.int64)
        sums = np.empty((R, bands), np.float64)
        bits = np.empty((R, max(wo, 1)), np.uint32)
        assign = np.empty(npx, np.int32)
        _lib.check(L.rhseg_result_root(ctx.handle, which, _lib.ptr(counts), _lib.ptr(sums), _lib.ptr(bits),
                                       _lib.ptr(assign)), "rhseg_result_root")
        graphs.append(RegionGraph.from_arrays(edge, edge, counts, sums, bits[:, :wo], assign))
    root_initial, root = graphs
    root_records = section_logs[-1][1]
    root.merges_done = len(root_records)
    hierarchy = MergeHierarchy(initial_region_count=root_initial.live_count, records=root_records,
                               converged_early=bool(info.converged_early))
    return RhsegResult(
        section_logs=section_logs,
        root_initial=root_initial,
        root_hierarchy=hierarchy,
        graph=root,
        labels=LabelMap(edge, edge, labels.reshape(edge, edge)),
        converged_early=bool(info.converged_early),
        spectral_pairs=int(info.spectral_pairs),
        device_ms=float(info.device_ms),
    )


def run_leaf(task, params: RhsegParams, strategy=Sequential(), connectivity: int = 8,
             profile: ProfileStats | None = None):
    """recursive.py:130-142: one leaf section (its HSEG on the device through the B2
    seam); returns (graph, records, converged_early, pre-merge copy if the leaf is the
    root)."""
    from .graph import init_region_graph

    graph = init_region_graph(task.image, connectivity)
    root_initial = graph.copy() if task.section_id.level == 1 else None
    hier = hseg_run(graph, params.section_params(task.section_id), strategy, profile)
    return graph, hier.records, hier.converged_early, root_initial


def run_upper_levels(params: RhsegParams, strategy, connectivity: int, graphs: dict, logs: dict,
                     profile: ProfileStats | None = None):
    """recursive.py:145-170: stitch and HSEG every level above the leaves (each section
    on the device), mutating `graphs` and `logs`; returns (root_initial, converged_early)."""
    converged_early, root_initial = False, None
    for level in range(params.levels - 1, 0, -1):
        side = section_side(level)
        for r in range(side):
            for c in range(side):
                sid = SectionId(level, r, c)
                graph = stitch([graphs[k] for k in sid.children()], connectivity)
                if level == 1:
                    root_initial = graph.copy()
                hier = hseg_run(graph, params.section_params(sid), strategy, profile)
                converged_early |= hier.converged_early
                graphs[sid] = graph
                logs[sid] = hier.records
    return root_initial, converged_early


def assemble_result(params: RhsegParams, logs: dict, root_initial, root_graph, converged_early: bool) -> RhsegResult:
    """recursive.py:107-127: logs in log_order, the root's hierarchy and dense labels."""
    ordered = [(sid, logs[sid]) for sid in log_order(params.levels)]
    hierarchy = MergeHierarchy(initial_region_count=root_initial.live_count,
                               records=list(logs[SectionId(1, 0, 0)]), converged_early=converged_early)
    return RhsegResult(section_logs=ordered, root_initial=root_initial, root_hierarchy=hierarchy, graph=root_graph,
                       labels=label_map_from_graph(root_graph), converged_early=converged_early)


def rhseg_run(image, params: RhsegParams, strategy=Sequential(), executor=None,
              profile: ProfileStats | None = None) -> RhsegResult:
    """recursive.py:212-223; the default executor is the B200 one."""
    if executor is None:
        executor = B200Executor()
    return executor.execute(image, params, strategy, profile=profile)


__all__ = [
    "RhsegParams", "RhsegResult", "RecordList", "B200Executor", "rhseg_run", "log_order", "section_side",
    "collect_result", "result_info", "run_leaf", "run_upper_levels", "assemble_result",
]
