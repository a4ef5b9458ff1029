"""Bind the B200 path into an imported reference `rhseg` package.

The reference looks its seams up in three ways, and each needs its own patch:

* B2 `hseg_run` (engine.py:345-371) is imported BY NAME at import time into
  recursive.py:16 (run_leaf, run_upper_levels), cluster.py:17 (the worker) and
  hybrid.py:19, and re-exported by the package __init__; patching only
  `rhseg.engine.hseg_run` would leave every caller on the CPU path.
* B3 `scan_adjacent` / `scan_nonadjacent` are looked up as attributes of
  `rhseg._kernels` at call time (engine.py:213-218): one module patch suffices.
* B1 is the `executor=` argument of `rhseg_run` (recursive.py:212-223); with
  `default_executor=True` a call without one gets `B200Executor`.

`install()` returns a handle whose `uninstall()` restores the originals.
"""

from __future__ import annotations

import importlib
import sys

_HSEG_RUN_HOLDERS = ("engine", "recursive", "cluster", "hybrid")


class Binding:
    def __init__(self):
        self._saved = []

    def _set(self, obj, name, value):
        if hasattr(obj, name):
            self._saved.append((obj, name, getattr(obj, name)))
            setattr(obj, name, value)

    def uninstall(self):
        for obj, name, value in reversed(self._saved):
            setattr(obj, name, value)
        self._saved.clear()


def install(rhseg=None, kernels: bool = True, default_executor: bool = False, device: int | None = None) -> Binding:
    """Route the reference package's hot path to librhseg_b200.so."""
    from . import engine as b200_engine
    from .recursive import B200Executor

    if rhseg is None:
        rhseg = sys.modules.get("rhseg") or importlib.import_module("rhseg")
    bind = Binding()

    def hseg_run(graph, params, strategy=None, profile=None, stop_check=None):
        kw = {} if strategy is None else {"strategy": strategy}
        return b200_engine.hseg_run(graph, params, profile=profile, stop_check=stop_check, device=device, **kw)

    hseg_run.__doc__ = b200_engine.hseg_run.__doc__
    hseg_run.__wrapped__ = b200_engine.hseg_run
    for name in _HSEG_RUN_HOLDERS:
        mod = sys.modules.get(f"{rhseg.__name__}.{name}")
        if mod is not None:
            bind._set(mod, "hseg_run", hseg_run)
    bind._set(rhseg, "hseg_run", hseg_run)
    if kernels:
        k = sys.modules.get(f"{rhseg.__name__}._kernels")
        if k is not None:
            bind._set(k, "scan_adjacent", b200_engine.scan_adjacent)
            bind._set(k, "scan_nonadjacent", b200_engine.scan_nonadjacent)
    if default_executor:
        rec = sys.modules.get(f"{rhseg.__name__}.recursive")
        orig = rec.rhseg_run

        def rhseg_run(image, params, strategy=None, executor=None, profile=None):
            kw = {} if strategy is None else {"strategy": strategy}
            return orig(image, params, executor=executor or B200Executor(device=device), profile=profile, **kw)

        bind._set(rec, "rhseg_run", rhseg_run)
        bind._set(rhseg, "rhseg_run", rhseg_run)
    return bind
