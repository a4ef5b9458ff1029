"""ctypes binding of librhseg_b200.so (include/rhseg_b200.h).

There is no CPU fallback anywhere in the product path: if the in-tree
extension is missing or no sm_100a device is visible, every compute call
raises ExtensionMissing / DeviceError.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from .errors import DeviceError, ExtensionMissing, IndivisibleImage, TooManyLabels

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RHSEG_LIB_PATH") or os.path.join(PKG, "_lib", "librhseg_b200.so")

RHSEG_OK = 0
RHSEG_E_INVALID = 1
RHSEG_E_INDIVISIBLE = 2
RHSEG_E_CUDA = 3
RHSEG_E_TOO_LARGE = 4
RHSEG_E_STATE = 5
RHSEG_E_TOO_MANY_LABELS = 6
RHSEG_E_IO = 7

i32, i64, f64, vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p


class RhsegParamsC(ctypes.Structure):
    _fields_ = [
        ("spectral_weight", f64),
        ("target_regions", i32),
        ("section_target_regions", i32),
        ("levels", i32),
        ("connectivity", i32),
        ("measure", i32),
        ("cluster", i32),
    ]


class ResultInfoC(ctypes.Structure):
    _fields_ = [
        ("n_records", i64),
        ("spectral_pairs", i64),
        ("n_sections", i32),
        ("levels", i32),
        ("edge", i32),
        ("bands", i32),
        ("root_idspace", i32),
        ("root_initial_regions", i32),
        ("root_regions", i32),
        ("converged_early", i32),
        ("device_ms", ctypes.c_float),
        ("pad_", ctypes.c_float),
    ]


# name -> (argtypes); every entry point returns int status except the two noted
_SIGS = {
    "rhseg_abi_version": [],
    "rhseg_last_error": [],
    "rhseg_ctx_create": [ctypes.c_int, ctypes.POINTER(vp)],
    "rhseg_ctx_destroy": [vp],
    "rhseg_run_device": [vp, vp, i32, i32, ctypes.POINTER(RhsegParamsC), vp],
    "rhseg_run_host": [vp, vp, i32, i32, ctypes.POINTER(RhsegParamsC), vp, vp, vp, vp, vp, vp,
                       ctypes.POINTER(ResultInfoC)],
    "rhseg_run_subtrees": [vp, vp, i32, i32, ctypes.POINTER(RhsegParamsC), i32, i32, i32, i32, i32, vp],
    "rhseg_top_info": [vp, vp, vp, vp, vp, vp],
    "rhseg_pack_bytes": [i32, i32, i32, vp],
    "rhseg_export_top": [vp, i32, vp, vp],
    "rhseg_run_upper": [vp, vp, i32, i32, vp, vp, i32, i32, ctypes.POINTER(RhsegParamsC), vp],
    "rhseg_result_log_device": [vp, vp, vp, vp, vp, vp],
    "rhseg_result_info_get": [vp, ctypes.POINTER(ResultInfoC)],
    "rhseg_result_sections": [vp, vp, vp, vp, vp, vp],
    "rhseg_result_log": [vp, vp, vp, vp, vp],
    "rhseg_result_labels": [vp, vp, vp],
    "rhseg_result_root": [vp, i32, vp, vp, vp, vp],
    "rhseg_hseg_graph": [vp, i64, i64, vp, vp, vp, vp, f64, i64, i32, i32, vp, vp, vp, vp, vp, vp],
    "rhseg_scan_adjacent": [i64, i64, i64, i64, vp, vp, vp, vp, vp, vp],
    "rhseg_scan_nonadjacent": [i64, i64, i64, i64, i64, vp, vp, vp, vp, vp, vp],
    "rhseg_result_phase_ms": [vp, vp],
    "rhseg_result_launches": [vp, vp],
    "rhseg_result_rescans": [vp, ctypes.c_int32, vp],
    "rhseg_result_level_info": [vp, i32, vp, vp, vp, vp, vp],
    "rhseg_format_float": [f64, vp, i32],
    "rhseg_sha256_hex": [vp, i64, vp],
    "rhseg_write_outputs_host": [ctypes.c_char_p, ctypes.c_char_p, i32, i32, vp, i32, vp, vp, vp, vp, vp, vp, vp, vp,
                                 vp, vp],
    "rhseg_fp64_peak": [vp, vp],
    "rhseg_fp64_fma_peak": [vp, vp],
}
EXPORTS = tuple(_SIGS)

_lib = None
_lock = threading.RLock()  # context() -> Context() -> load() re-enters


def load():
    """Load the in-tree extension (raises ExtensionMissing if absent)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ExtensionMissing(
                f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        try:
            L = ctypes.CDLL(LIB_PATH)
        except OSError as exc:  # pragma: no cover - depends on the host
            raise ExtensionMissing(f"cannot load {LIB_PATH}: {exc}") from exc
        for name, args in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = ctypes.c_int
        L.rhseg_last_error.restype = ctypes.c_char_p
        _lib = L
        return L


def last_error() -> str:
    return load().rhseg_last_error().decode(errors="replace")


def check(status: int, what: str = "") -> None:
    if status == RHSEG_OK:
        return
    msg = last_error()
    if status == RHSEG_E_INVALID:
        raise ValueError(msg)
    if status == RHSEG_E_INDIVISIBLE:
        raise IndivisibleImage(msg)
    if status == RHSEG_E_TOO_MANY_LABELS:
        raise TooManyLabels(msg)
    if status == RHSEG_E_IO:
        raise OSError(msg)
    raise DeviceError(f"{what}: {msg} (status {status})")


def ptr(a: np.ndarray | None):
    if a is None:
        return None
    return a.ctypes.data_as(vp)


class Context:
    """One librhseg context (device stream, memory pool, last result)."""

    def __init__(self, device: int = 0):
        self.device = device
        self.lock = threading.Lock()
        h = vp()
        check(load().rhseg_ctx_create(device, ctypes.byref(h)), "rhseg_ctx_create")
        self.handle = h

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            if getattr(self, "handle", None) and _lib is not None:
                _lib.rhseg_ctx_destroy(self.handle)
        except Exception:
            pass


_contexts: dict[int, Context] = {}


def context(device: int | None = None) -> Context:
    if device is None:
        device = _current_device()
    with _lock:
        ctx = _contexts.get(device)
        if ctx is None:
            ctx = Context(device)
            _contexts[device] = ctx
        return ctx


def _current_device() -> int:
    try:
        import torch

        if torch.cuda.is_available():
            return torch.cuda.current_device()
    except Exception:  # pragma: no cover
        pass
    return int(os.environ.get("LOCAL_RANK", "0")) if os.environ.get("RHSEG_USE_LOCAL_RANK") else 0


def make_params(weight, target, section_target, levels, connectivity=8, measure=0, cluster=0):
    p = RhsegParamsC()
    p.spectral_weight = float(weight)
    # the C struct holds int32 targets: a larger target means "no merge" exactly as
    # INT32_MAX does (no section has that many regions), so clamp instead of wrapping
    p.target_regions = min(int(target), 2**31 - 1)
    p.section_target_regions = min(int(section_target or 0), 2**31 - 1)
    p.levels = int(levels)
    p.connectivity = int(connectivity)
    p.measure = int(measure)
    p.cluster = int(cluster)
    return p


LOOP_NAMES = {0: "adjacent (w=0)", 1: "mean stream", 2: "APO", 3: "APO re-cut", 4: "grid"}


def level_info(handle, level: int) -> dict:
    """Which merge loop ran on one level of the context's last run, its sections,
    capacity, CTAs per section, merges and D-row rescans (rhseg_result_level_info /
    rhseg_result_rescans)."""
    L = load()
    ns, rp, cl, var = (ctypes.c_int32(0) for _ in range(4))
    mg, rs = ctypes.c_int64(0), ctypes.c_int64(0)
    check(L.rhseg_result_level_info(handle, level, ctypes.byref(ns), ctypes.byref(rp), ctypes.byref(cl),
                                    ctypes.byref(var), ctypes.byref(mg)), "rhseg_result_level_info")
    check(L.rhseg_result_rescans(handle, level, ctypes.byref(rs)), "rhseg_result_rescans")
    return {"nsec": ns.value, "rp": rp.value, "cluster": cl.value, "variant": var.value,
            "loop": LOOP_NAMES.get(var.value, str(var.value)), "merges": mg.value, "rescans": rs.value}


def phase_ms(handle):
    """Per-kernel device ms of the context's last run: [init, all-pairs D, loops, stitch+labels]."""
    import numpy as np

    ms = np.zeros(4, np.float32)
    check(load().rhseg_result_phase_ms(handle, ms.ctypes.data_as(ctypes.c_void_p)), "rhseg_result_phase_ms")
    return ms.astype(np.float64)

