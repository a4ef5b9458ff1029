"""BASELINE.md §4 CPU-baseline plan, run once on the GPU box's host (not part of the
default bench, which samples ~20 s): the C restatement of the reference algorithm
(oracle/, test infrastructure) timed two ways per workload, the faster reported --

  within:   one leaf at a time, the per-step row scans spread over every host thread
            (the reference's PerPair/PerRegion strategies, engine.py:50-76);
  sections: one whole leaf per host thread, each leaf's scans single-threaded (the
            process-per-section strategy of cluster.py:68-131, `Sequential` inside).

Both time the same fixed random sample of >= 2 x ncores leaves (C3/C4/C5w1, then
extrapolated to the whole leaf level; upper levels < 0.01% of the pairs at t=16), or
every leaf (C2, C5 w=0). C1 (one 4096-region section, HSEG to 2 regions) is timed on
all threads and, as the paper's speedup denominator, on ONE core over
the first K steps, extrapolated with the per-step cost model sum_steps R_live^2
(the scans are O(R^2 B) per step).

    python tools/cpu_baseline.py [c4 c3b c5w1 c5w0 c2 c1 ...] > profiles/r02_cpu_baseline.jsonl
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bench  # noqa: E402
from oracle import oracle  # noqa: E402


def leaves_of(name, nsample):
    spec, crop, levels, w, t, st = bench.WORKLOADS[name]
    bands, edge, _ = bench.cube_shape(name)
    side = 1 << (levels - 1)
    se = edge // side
    nleaf = side * side
    rng = np.random.default_rng(1234)
    order = rng.permutation(nleaf)[: min(nsample, nleaf)]
    origins = [((int(k) // side) * se, (int(k) % side) * se) for k in order]
    return origins, se, nleaf, bands, edge, w, (t if levels == 1 else st)


def time_within(samples, origins, se, w, tgt, threads):
    oracle.set_threads(threads)
    t0 = time.perf_counter()
    m = [oracle.run_leaf(samples, r, c, se, w, tgt) for r, c in origins]
    return time.perf_counter() - t0, int(sum(m))


def time_sections(samples, origins, se, w, tgt, threads):
    oracle.set_threads(threads)
    t0 = time.perf_counter()
    m = oracle.run_leaves(samples, origins, se, w, tgt)
    return time.perf_counter() - t0, int(m.sum())


def leaf_workload(name, ncores, nsample):
    samples = bench.make_cube(name)
    oracle.set_measure(bench.MEASURE_OF.get(name, "sqrt-bsmse"))
    origins, se, nleaf, bands, edge, w, tgt = leaves_of(name, nsample)
    out = {"workload": name, "descr": bench.DESCR[name], "cores": ncores, "leaves_sampled": len(origins),
           "leaves_total": nleaf, "leaf": f"{se}x{se}x{bands}"}
    pxb = len(origins) * se * se * bands
    for strat, fn in (("within", time_within), ("sections", time_sections)):
        dt, merges = fn(samples, origins, se, w, tgt, ncores)
        out[strat] = {"seconds": dt, "merges": merges, "pixel_bands_per_s": pxb / dt,
                      "whole_cube_seconds_extrapolated": dt * nleaf / len(origins)}
        print(f"# {name} {strat}: {dt:.1f}s for {len(origins)} leaves", file=sys.stderr, flush=True)
    best = max(("within", "sections"), key=lambda s: out[s]["pixel_bands_per_s"])
    out["best"] = best
    out["value"] = out[best]["pixel_bands_per_s"]
    out["extrapolated"] = len(origins) < nleaf
    return out


def c1(ncores, single_steps):
    """C1: HSEG over the whole 64x64x32 cube to 2 regions (L=1): all threads in full,
    and one core over the first `single_steps` steps, extrapolated by sum R^2."""
    name = "c1"
    samples = bench.make_cube(name)
    oracle.set_measure("sqrt-bsmse")
    spec, crop, levels, w, t, st = bench.WORKLOADS[name]
    bands, edge, _ = bench.cube_shape(name)
    R0 = edge * edge
    out = {"workload": name, "descr": bench.DESCR[name], "cores": ncores}
    oracle.set_threads(ncores)
    t0 = time.perf_counter()
    m = oracle.run_leaf(samples, 0, 0, edge, w, t)
    dt = time.perf_counter() - t0
    out["within"] = {"seconds": dt, "merges": int(m), "pixel_bands_per_s": R0 * bands / dt}
    oracle.set_threads(1)
    t0 = time.perf_counter()
    m1 = oracle.run_leaf(samples, 0, 0, edge, w, t, max_steps=single_steps)
    d1 = time.perf_counter() - t0
    full = sum(float(R) ** 2 for R in range(t + 1, R0 + 1))
    part = sum(float(R) ** 2 for R in range(R0 - int(m1) + 1, R0 + 1))
    est = d1 * full / part
    out["single_core"] = {"seconds_first_steps": d1, "steps": int(m1), "seconds_extrapolated": est,
                          "pixel_bands_per_s": R0 * bands / est,
                          "model": "per-step cost proportional to R_live^2 (from-scratch O(R^2 B) scans)"}
    out["value"] = out["within"]["pixel_bands_per_s"]
    return out


def main():
    names = [a for a in sys.argv[1:] if not a.startswith("-")] or ["c4", "c3b", "c5w1", "c5w0", "c2", "c1"]
    ncores = os.cpu_count() or 1
    oracle.build()
    print(json.dumps({"host_cores": ncores, "cpu": open("/proc/cpuinfo").read().split("model name")[1]
                      .split("\n")[0].strip(": ") if os.path.exists("/proc/cpuinfo") else None}), flush=True)
    for name in names:
        if name == "c1":
            res = c1(ncores, single_steps=50)
        elif name in ("c2", "c5w0"):
            res = leaf_workload(name, ncores, 1 << 30)  # every leaf
        else:
            res = leaf_workload(name, ncores, 2 * ncores)
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
