"""RHSEG throughput bench (driver contract: one JSON line from rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c4|c2|c1|c3b|c5w0|c5w1]

A "step" is one full RHSEG run (every quadtree level, stitching, root labels)
over one synthetic cube (BASELINE.json configs; SURVEY §8(d) pins the open
parameters). Metric: pixel-bands/s = edge^2 * bands / step time; spectral
pairs/s (reference-equivalent, sum over steps of R(R-1)/2 - E) rides along.

ours:      `value` is device time (CUDA events on the run stream) with the cube
           already resident in HBM; `e2e` is the same metric through the C-ABI
           host call rhseg_run_host (pinned cube H2D, run, merge log + labels
           D2H), wall-clocked.
reference: the CPU restatement of the reference algorithm (oracle/, a C port of
           rhseg's from-scratch per-step scans, OpenMP over all host threads)
           timed on a bounded sample of the same workload's leaves; only this
           leg and `cpu_baseline` touch oracle/.

Multi-GPU (--gpus N under torchrun): the quadtree's leaf level is sharded by
contiguous subtrees; see paper_2106_12942_b200/distributed.py.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

# name -> (gen_synthetic args, crop edge or None, levels, weight, target, section_target)
# measure: MEASURE_OF (default sqrt-bsmse, the reference's only measure)
WORKLOADS = {
    "c1": ((64, 32, 4, 6, 3.0, 2), None, 1, 0.5, 2, 2),
    "c3": ((512, 224, 16, 25, 3.0, 512), None, 5, 0.21, 16, 16),
    "c2": ((145, 220, 16, 25, 3.0, 145), 144, 3, 0.5, 16, 16),
    "c3b": ((512, 224, 16, 25, 3.0, 512), None, 5, 0.21, 16, 16),
    "c4": ((2048, 224, 16, 25, 3.0, 2048), None, 7, 0.21, 16, 16),
    "c5w0": ((1024, 64, 4, 6, 3.0, 1024), None, 6, 0.0, 16, 16),
    "c5w1": ((1024, 64, 4, 6, 3.0, 1024), None, 6, 1.0, 16, 16),
}
MEASURE_OF = {"c3": "sam"}
DESCR = {
    "c3": "C3 gen_synthetic(512,224,16,25,3.0,512) RHSEG L=5 SAM w=0.21 t=16 (extension measure)",
    "c1": "C1 gen_synthetic(64,32,4,6,3.0,2) HSEG L=1 w=0.5 t=2",
    "c2": "C2 gen_synthetic(145,220,16,25,3.0,145).crop(144) RHSEG L=3 w=0.5 t=16",
    "c3b": "C3 gen_synthetic(512,224,16,25,3.0,512) RHSEG L=5 w=0.21 t=16 (BSMSE twin)",
    "c4": "C4 gen_synthetic(2048,224,16,25,3.0,2048) RHSEG L=7 w=0.21 t=16",
    "c5w0": "C5 gen_synthetic(1024,64,4,6,3.0,1024) RHSEG L=6 w=0.0 t=16",
    "c5w1": "C5 gen_synthetic(1024,64,4,6,3.0,1024) RHSEG L=6 w=1.0 t=16",
}
METRIC = "RHSEG pixel-bands/sec"
UNIT = "pixel-bands/s"
L2_BYTES = 126 * 1024 * 1024


def config_of(name):
    """The workload's config dict -- identical in both arms (the driver compares them);
    arm-specific execution details go to the line's top-level "execution" key."""
    spec, crop, levels, w, t, st = WORKLOADS[name]
    bands, edge, _ = cube_shape(name)
    return {"workload": DESCR[name], "edge": edge, "bands": bands, "levels": levels, "spectral_weight": w,
            "target_regions": t, "section_target_regions": st, "connectivity": 8,
            "measure": MEASURE_OF.get(name, "sqrt-bsmse"),
            "l2": "flushed between timed steps (2x126 MB write); CPU arm: n/a"}


def make_cube(name, out=None):
    from paper_2106_12942_b200.synth import gen_synthetic

    spec, crop, *_ = WORKLOADS[name]
    edge = spec[0]
    if crop is None:
        img, _ = gen_synthetic(*spec, out=out)
        return img.samples
    full, _ = gen_synthetic(*spec)
    s = np.ascontiguousarray(full.samples[:, :crop, :crop])
    if out is not None:
        out[...] = s
        return out
    return s


def cube_shape(name):
    spec, crop, *_ = WORKLOADS[name]
    e = crop or spec[0]
    return spec[1], e, e


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the
    timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.rows = []
        if self.proc is None:
            return
        time.sleep(0.25)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
            out, _ = self.proc.communicate()
        for line in out.splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 9:
                self.rows.append(f)

    def summary(self):
        rows = getattr(self, "rows", [])
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------------------
# CPU legs (oracle = the reference algorithm restated in C; test infra only)
# ---------------------------------------------------------------------------
def cpu_sample(name, samples, seconds_hint=20.0, threads=None, max_leaves=None, max_steps=-1):
    """Time whole leaves of the workload (the reference's per-step from-scratch
    scans; run_leaf, recursive.py:130-142) until ~seconds_hint of CPU work.
    Upper levels carry <0.01% of the pairs at t=16 and are not
    sampled; the leaf rate is extrapolated to the whole cube."""
    from oracle import oracle

    oracle.build()
    threads = threads or os.cpu_count() or 1
    oracle.set_threads(threads)
    oracle.set_measure(MEASURE_OF.get(name, "sqrt-bsmse"))
    spec, crop, levels, w, t, st = WORKLOADS[name]
    bands, edge, _ = samples.shape
    side = 1 << (levels - 1)
    se = edge // side
    nleaves = side * side
    leaf_t = t if levels == 1 else st
    rng = np.random.default_rng(1234)
    order = rng.permutation(nleaves)
    done, t0 = 0, time.perf_counter()
    limit = max_leaves or nleaves
    while done < limit:
        k = int(order[done])
        oracle.run_leaf(samples, (k // side) * se, (k % side) * se, se, w, leaf_t, max_steps=max_steps)
        done += 1
        if time.perf_counter() - t0 > seconds_hint:
            break
    dt = time.perf_counter() - t0
    pxb = done * se * se * bands
    return {
        "value": pxb / dt,
        "unit": UNIT,
        "cores": threads,
        "kind": "port",
        "sample": f"{done}/{nleaves} random leaves ({se}x{se}x{bands}, {dt:.1f}s) through the C restatement of "
                  f"rhseg run_leaf/hseg_run (from-scratch scans every step, OpenMP {threads} threads); "
                  f"pixel-bands/s extrapolated from leaves (upper levels <0.01% of pairs)",
        "seconds": dt,
        "leaves": done,
    }


def full_cpu_plan(name):
    """The BASELINE.md §4 plan measured once on the box's host (tools/cpu_baseline.py:
    >= 2 x ncores leaves, within-leaf OpenMP vs one leaf per core, the faster kept),
    committed as profiles/r02_cpu_baseline.jsonl; None if this workload was not run."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_cpu_baseline.jsonl")) as f:
            rows = [json.loads(x) for x in f if x.strip()]
    except OSError:
        return None
    for r in rows:
        if r.get("workload") == name:
            out = {"source": "profiles/r02_cpu_baseline.jsonl", "cores": r["cores"], "value": r["value"],
                   "unit": UNIT}
            if "best" in r:
                out.update(best=r["best"], leaves=f"{r['leaves_sampled']}/{r['leaves_total']}",
                           within=r["within"]["pixel_bands_per_s"], sections=r["sections"]["pixel_bands_per_s"],
                           extrapolated=r["extrapolated"])
            if "single_core" in r:
                out["single_core"] = r["single_core"]["pixel_bands_per_s"]
            return out
    return None


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    name = args.workload
    samples = make_cube(name)
    for _ in range(args.warmup):
        cpu_sample(name, samples, seconds_hint=0.0, max_leaves=1, max_steps=4)
    vals = []
    last = None
    for _ in range(args.steps):
        last = cpu_sample(name, samples, seconds_hint=args.ref_seconds)
        vals.append(last["value"])
    value = float(np.median(vals))
    bands, edge, _ = samples.shape
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": last["seconds"] * 1e3,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (gen_synthetic, bit-identical to the reference generator)",
        "config": config_of(name),
        "execution": f"CPU (no GPU): the reference algorithm restated in C (oracle/), OpenMP over "
                     f"{last['cores']} host threads, bounded random leaf sample",
        "cpu_baseline": {k: last[k] for k in ("value", "unit", "cores", "kind", "sample")} | {"value": value},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args):
    import ctypes

    import torch

    import paper_2106_12942_b200 as rh
    from paper_2106_12942_b200 import _lib
    from paper_2106_12942_b200.recursive import result_info

    rank, world, local = dist_env()
    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device (the product path has no CPU fallback)")
    if world > 1:
        from paper_2106_12942_b200 import distributed as rdist

        return rdist.bench_sharded(args, sys.modules[__name__])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    name = args.workload
    spec, crop, levels, w, t, st = WORKLOADS[name]
    bands, edge, _ = cube_shape(name)
    host = torch.empty((bands, edge, edge), dtype=torch.float32, pin_memory=True)
    make_cube(name, out=host.numpy())
    cube = host.to(dev, non_blocking=False)
    params = rh.RhsegParams(rh.HsegParams(w, t, MEASURE_OF.get(name, "sqrt-bsmse")), levels, st)
    ex = rh.B200Executor(device=local)
    stream = torch.cuda.Stream(device=dev)  # the run and its events share one non-default stream
    sptr = stream.cuda_stream
    flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.int32, device=dev)
    lib = _lib.load()

    def step():
        ctx = ex.execute_device(cube.data_ptr(), edge, bands, params, stream=sptr)
        return ctx

    with torch.cuda.stream(stream):
        for _ in range(max(args.warmup, 0)):
            ctx = step()
    torch.cuda.synchronize()
    info = result_info(ctx)
    pairs = int(info.spectral_pairs)
    launches = ctypes.c_int64(0)
    times, walls, phases, launch_total = [], [], np.zeros(4), 0
    with ClockSampler(local) as clk, torch.cuda.stream(stream):
        for _ in range(args.steps):
            flush.zero_()  # L2 flush between timed steps (on the run stream)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            e0.record(stream)
            ctx = step()
            e1.record(stream)
            torch.cuda.synchronize()
            walls.append(time.perf_counter() - t0)
            times.append(e0.elapsed_time(e1))
            phases += _phase_ms_of(ctx)
            lib.rhseg_result_launches(ctx.handle, ctypes.byref(launches))
            launch_total += int(launches.value)
    ms = float(np.sum(times)) / args.steps
    phases /= args.steps
    npxb = edge * edge * bands
    value = npxb / (ms * 1e-3)

    # ---- e2e through the C-ABI host call (pinned cube in, log + labels out) ----
    n_rec = int(info.n_records)
    oa = torch.empty(max(n_rec, 1), dtype=torch.int32, pin_memory=True)
    ob = torch.empty(max(n_rec, 1), dtype=torch.int32, pin_memory=True)
    od = torch.empty(max(n_rec, 1), dtype=torch.float64, pin_memory=True)
    ok = torch.empty(max(n_rec, 1), dtype=torch.uint8, pin_memory=True)
    olab = torch.empty(edge * edge, dtype=torch.int32, pin_memory=True)
    cp = ex.c_params(params)
    inf2 = _lib.ResultInfoC()
    hctx = _lib.context(local)
    e2e_t = []
    for it in range(2 + args.steps):
        t0 = time.perf_counter()
        with hctx.lock:
            _lib.check(lib.rhseg_run_host(hctx.handle, ctypes.c_void_p(host.data_ptr()), edge, bands,
                                          ctypes.byref(cp), None, ctypes.c_void_p(oa.data_ptr()),
                                          ctypes.c_void_p(ob.data_ptr()), ctypes.c_void_p(od.data_ptr()),
                                          ctypes.c_void_p(ok.data_ptr()), ctypes.c_void_p(olab.data_ptr()),
                                          ctypes.byref(inf2)), "rhseg_run_host")
        if it >= 2:
            e2e_t.append(time.perf_counter() - t0)
    e2e_s = float(np.median(e2e_t))
    h2d = edge * edge * bands * 4
    d2h = n_rec * (4 + 4 + 8 + 1) + edge * edge * 4

    # ---- roofline of the dominant kernel ----
    roof, roof2 = roofline(name, edge, bands, levels, w, phases, ctx.handle)

    line = {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": 1,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (gen_synthetic, bit-identical to the reference generator)",
        "config": config_of(name),
        "execution": "1 GPU, every section of a quadtree level in one persistent launch",
        "spectral_pairs_per_s": pairs / (ms * 1e-3),
        "merges": n_rec,
        "host_wall_ms_per_step": float(np.mean(walls)) * 1e3,
        "phase_ms": {"init_stitch": phases[0], "dinit_allpairs": phases[1], "merge_loop": phases[2],
                     "resolve_labels": phases[3]},
        "gpu_launches": launch_total,
        "e2e": {"value": npxb / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": e2e_s * 1e3},
        "roofline": roof,
        "roofline_secondary": roof2,
        "clocks": clk.summary(),
    }
    if not args.no_cpu_baseline:
        cb = cpu_sample(name, host.numpy(), seconds_hint=args.ref_seconds)
        line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
        fp = full_cpu_plan(name)
        if fp:
            line["cpu_baseline"]["full_plan"] = fp
    print(json.dumps(line), flush=True)
    return 0


def _phase_ms_of(ctx):
    import ctypes

    from paper_2106_12942_b200 import _lib

    ms = np.zeros(4, np.float32)
    _lib.check(_lib.load().rhseg_result_phase_ms(ctx.handle, ms.ctypes.data_as(ctypes.c_void_p)), "phase_ms")
    return ms.astype(np.float64)


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


def ncu_traffic(name, kernel):
    """DRAM bytes (read + write) of one leaf-level launch from the committed ncu
    capture (profiles/traffic.json), or None when this workload was not captured."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f).get(name, {}).get(kernel)
    except (OSError, ValueError):
        return None
    return None if not t else t["dram_read_bytes"] + t["dram_write_bytes"]


def roofline(name, edge, bands, levels, w, phases, handle, leaf=None):
    """Roofline entries of the two heavy kernels; the longer one is the line's
    `roofline` (DESIGN.md §4 states the per-unit algorithmic work):
      merge loop (HBM): the leaf level's loop -- the variant that ACTUALLY ran
        (rhseg_result_level_info), >99% of the merges at t=16:
          APO:    per step D rows a and b read, row and column a' written (4 R 8 bytes),
                  a's and b's band sums + a's new mean (4 B 8), every rescanned row's
                  live D entries (rescans counted by the kernel x mean R x 8);
          stream: the live regions' mean columns once per step, sum_steps R (8B + 16);
          w = 0:  ~10 band-sum rows of 8B bytes per step;
      all-pairs D init (FP64): sum over leaves of R0(R0+1)/2 pairs x (3B + 5) flops,
        against the measured DFMA flop rate (rhseg_fp64_fma_peak)."""
    import ctypes

    from paper_2106_12942_b200 import _lib

    lib = _lib.load()
    peaks = measured_peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    side = 1 << (levels - 1)
    se = edge // side
    nleaf = side * side
    R0 = se * se
    t = WORKLOADS[name][4] if levels == 1 else WORKLOADS[name][5]
    loop_ms, dinit_ms = float(phases[2]), float(phases[1])
    leaf = leaf or _lib.level_info(handle, levels)
    var = leaf["variant"]
    resc_per_sec = leaf["rescans"] / max(1, leaf["nsec"])  # (multi-GPU: from this rank's leaves)
    steps = range(t + 1, R0 + 1)
    if var in (2, 3):
        rbar = sum(steps) / max(1, len(steps))
        per_sec = sum(4 * R * 8 + 4 * bands * 8 for R in steps) + resc_per_sec * rbar * 8
        note = ("APO loop: sum_steps (4R*8 + 4B*8) + rescans*mean(R)*8 bytes; %.0f rescans per leaf "
                "(latency-bound step chain, not a stream)" % resc_per_sec)
    elif var in (1, 4):
        per_sec = sum(R * (8 * bands + 16) for R in steps)
        note = ("mean-stream loop" if var == 1 else "grid loop (one section on a group of CTAs)") + \
            ": the live regions' fp64 means once per step, sum_steps R_live*(8B+16)"
    else:
        per_sec = (R0 - t) * 10 * 8 * bands
        note = "w=0 loop: ~10 band-sum rows of 8B bytes per step (latency-bound, not a stream)"
    algo = nleaf * per_sec
    achieved = algo / (loop_ms * 1e-3) / 1e9 if loop_ms > 0 else 0.0
    kname = "hseg_grid_kernel" if var == 4 else \
        {3: "hseg_apo_kernel", 0: "hseg_adj_kernel"}.get(var, "hseg_loop_kernel") if leaf["cluster"] == 1 \
        else "hseg_loop_kernel"
    loop = {"kernel": kname + " (persistent per-section merge loop)",
            "loop_variant": leaf["loop"], "ctas_per_section": leaf["cluster"],
            "bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
            "traffic": ncu_traffic(name, kname),
            "algorithmic_bytes": algo, "algorithmic_model": note, "kernel_ms": loop_ms,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650 GB/s"}
    fma = ctypes.c_double(0.0)
    _lib.check(lib.rhseg_fp64_fma_peak(handle, ctypes.byref(fma)), "fp64_fma_peak")
    flops = nleaf * (R0 * (R0 + 1) // 2) * (3 * bands + 5) if w > 0 else 0
    ach = flops / (dinit_ms * 1e-3) / 1e12 if dinit_ms > 0 else 0.0
    peak = fma.value / 1e12
    dname = "dinit_sparse_kernel" if w <= 0 else ("dinit_iv84_kernel" if var in (2, 3) else "dinit_dense_kernel")
    dinit = {"kernel": dname + " (all-pairs fp64 dissimilarity)",
             "bound": "fp64", "achieved": ach, "peak": peak, "unit": "TFLOP/s",
             "frac": ach / peak if peak else None, "traffic": ncu_traffic(name, dname),
             "kernel_ms": dinit_ms, "algorithmic_flops": flops,
             "algorithmic_model": "leaf pairs R0(R0+1)/2 x (3B+5) flops (sub, mul, add per band + finish)",
             "peak_source": "measured live: rhseg_fp64_fma_peak (DFMA loop, 2 flops/instr)"}
    if loop_ms >= dinit_ms:
        return loop, dinit
    return dinit, loop


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c4")
    ap.add_argument("--ref-seconds", type=float, default=15.0, help="CPU sample budget per reference step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        print("bench.py: warmup < 3 violates the timing rules; using 3", file=sys.stderr)
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
