"""Golden-vector generator: runs the UNMODIFIED reference package in place.

Test infrastructure only (never imported by the product path). Run in the
build container, where /root/reference exists:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
    PYTHONDONTWRITEBYTECODE=1 python oracle/gen_golden.py [small|c1|c2|crit2|all]

Outputs go to tests/golden/*.npz / *.json and are committed, so the GPU box
(which has no /root/reference) can check parity against the reference's own
results. Each fixture records the reference call that produced it.

Reference entry points used (all read-only):
  rhseg.synth.gen_synthetic            synth.py:77-109
  rhseg.graph.init_region_graph        graph.py:161-183
  rhseg.engine.hseg_run / search_table engine.py:253-268, 345-371
  rhseg.recursive.rhseg_run            recursive.py:212-223
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(os.path.dirname(HERE), "tests", "golden")

from rhseg.engine import HsegParams, PerPair, Sequential, hseg_run, search_table, snapshot  # noqa: E402
from rhseg.graph import MergeKind, init_region_graph, label_map_from_graph  # noqa: E402
from rhseg.image import HyperImage  # noqa: E402
from rhseg.recursive import RhsegParams, rhseg_run  # noqa: E402
from rhseg.synth import gen_synthetic  # noqa: E402


def _log_arrays(result):
    rows = list(result.flat_log())
    n = len(rows)
    out = {
        "log_level": np.array([r["level"] for r in rows], dtype=np.int16).reshape(n),
        "log_row": np.array([r["section"][0] for r in rows], dtype=np.int32).reshape(n),
        "log_col": np.array([r["section"][1] for r in rows], dtype=np.int32).reshape(n),
        "log_survivor": np.array([r["survivor"] for r in rows], dtype=np.int32).reshape(n),
        "log_absorbed": np.array([r["absorbed"] for r in rows], dtype=np.int32).reshape(n),
        "log_dissim": np.array([r["dissim"] for r in rows], dtype=np.float64).reshape(n),
        "log_kind": np.array(
            [0 if r["kind"] == "adjacent" else 1 for r in rows], dtype=np.uint8
        ).reshape(n),
    }
    return out


def _jsonl_sha(result):
    h = hashlib.sha256()
    for rec in result.flat_log():
        h.update((json.dumps(rec) + "\n").encode())
    return h.hexdigest()


def gen_synth_hashes():
    cases = [
        (64, 32, 4, 6, 3.0, 2),
        (145, 220, 16, 25, 3.0, 145),
        (12, 4, 3, 3, 0.0, 0),
        (16, 8, 4, 6, 3.0, 16),
        (64, 16, 4, 6, 3.0, 64),
        (128, 8, 4, 6, 3.0, 128),
        (32, 224, 16, 25, 3.0, 32),
        (512, 224, 16, 25, 3.0, 512),
    ]
    out = []
    for c in cases:
        img, gt = gen_synthetic(*c)
        out.append(
            {
                "args": list(c),
                "samples_sha256": hashlib.sha256(img.samples.tobytes()).hexdigest(),
                "labels_sha256": hashlib.sha256(gt.labels.astype(np.int64).tobytes()).hexdigest(),
            }
        )
        print("synth", c, out[-1]["samples_sha256"][:12], flush=True)
    with open(os.path.join(GOLDEN, "synth_hashes.json"), "w") as fh:
        json.dump({"source": "rhseg.synth.gen_synthetic (synth.py:77-109)", "cases": out}, fh, indent=1)


def gen_hseg_corpus(n_cases=300, seed=1405):
    """Criterion-1-style random corpus (test_acceptance.py:56-87), reference hseg_run."""
    rng = np.random.default_rng(seed)
    samples, meta, merges, assigns = [], [], [], []
    for case in range(n_cases):
        edge = int(rng.integers(2, 7))
        bands = int(rng.integers(1, 5))
        conn = int(rng.choice([4, 8]))
        weight = float(rng.choice([0.0, 0.21, 1.0, round(float(rng.uniform()), 3)]))
        # half the cases are integer-valued (tie-heavy)
        if case % 2:
            s = rng.integers(0, 4, size=(bands, edge, edge)).astype(np.float32)
        else:
            s = rng.normal(0.0, 40.0, size=(bands, edge, edge)).astype(np.float32)
        pixels = edge * edge
        target = int(rng.choice([1, int(rng.integers(1, pixels + 1)), pixels]))
        img = HyperImage(edge, edge, bands, s)
        g = init_region_graph(img, conn)
        h = hseg_run(g, HsegParams(weight, target), Sequential())
        samples.append(s.ravel())
        meta.append((edge, bands, conn, weight, target, int(h.converged_early), len(h.records)))
        merges.extend(
            (r.survivor_id, r.absorbed_id, r.dissimilarity, int(r.kind)) for r in h.records
        )
        assigns.append(g.pixel_assignment.astype(np.int32))
    meta_a = np.array(meta, dtype=np.float64)
    np.savez_compressed(
        os.path.join(GOLDEN, "hseg_corpus.npz"),
        source="rhseg.engine.hseg_run (engine.py:345-371), Sequential strategy",
        meta=meta_a,  # edge, bands, conn, weight, target, converged_early, n_records
        samples=np.concatenate(samples).astype(np.float32),
        merge_surv=np.array([m[0] for m in merges], dtype=np.int32),
        merge_abs=np.array([m[1] for m in merges], dtype=np.int32),
        merge_d=np.array([m[2] for m in merges], dtype=np.float64),
        merge_kind=np.array([m[3] for m in merges], dtype=np.uint8),
        assign=np.concatenate(assigns),
    )
    print("corpus", n_cases, "cases", len(merges), "merges", flush=True)


def gen_scan_tables(seed=7):
    """Per-row tables of scan_adjacent / scan_nonadjacent (_kernels.py:31-115)
    at several merge stages, to pin the B3 kernel ABI bitwise."""
    rng = np.random.default_rng(seed)
    recs = {k: [] for k in ("ncase", "counts", "sums", "indptr", "indices", "adj_d", "adj_j", "non_d", "non_j", "meta")}
    for case in range(24):
        edge = int(rng.integers(3, 13))
        bands = int(rng.integers(1, 40))
        if case % 3 == 0:
            s = rng.integers(0, 3, size=(bands, edge, edge)).astype(np.float32)
        else:
            s = rng.normal(0.0, 50.0, size=(bands, edge, edge)).astype(np.float32)
        img = HyperImage(edge, edge, bands, s)
        g = init_region_graph(img, 8)
        target = int(rng.integers(1, edge * edge + 1))
        hseg_run(g, HsegParams(0.21, target))
        snap = snapshot(g)
        ta = search_table(snap, MergeKind.ADJACENT, Sequential())
        tn = search_table(snap, MergeKind.NON_ADJACENT, PerPair(tile_k=3, workers=2))
        # out_j index space: dense row index; recover from partner ids
        idx = {int(v): k for k, v in enumerate(snap.ids)}
        aj = np.array([idx[int(p)] if p >= 0 else -1 for p in ta.partner_ids], dtype=np.int64)
        nj = np.array([idx[int(p)] if p >= 0 else -1 for p in tn.partner_ids], dtype=np.int64)
        recs["meta"].append((len(snap.ids), bands, len(snap.indices)))
        recs["counts"].append(snap.counts)
        recs["sums"].append(snap.sums.ravel())
        recs["indptr"].append(snap.indptr)
        recs["indices"].append(snap.indices)
        recs["adj_d"].append(ta.dissims)
        recs["adj_j"].append(aj)
        recs["non_d"].append(tn.dissims)
        recs["non_j"].append(nj)
    np.savez_compressed(
        os.path.join(GOLDEN, "scan_tables.npz"),
        source="rhseg._kernels.scan_adjacent/scan_nonadjacent via engine.search_table",
        meta=np.array(recs["meta"], dtype=np.int64),
        **{k: np.concatenate(v) for k, v in recs.items() if k not in ("meta", "ncase")},
    )
    print("scan tables", len(recs["meta"]), flush=True)


def gen_rhseg(name, image, params, strategy, note):
    t0 = time.perf_counter()
    res = rhseg_run(image, params, strategy)
    wall = time.perf_counter() - t0
    arrs = _log_arrays(res)
    np.savez_compressed(
        os.path.join(GOLDEN, f"{name}.npz"),
        source="rhseg.recursive.rhseg_run (recursive.py:212-223) with SequentialExecutor",
        note=note,
        labels=res.labels.labels.astype(np.int32),
        final_ids=np.array(sorted(res.graph.regions), dtype=np.int32),
        final_counts=np.array([res.graph.regions[k].pixel_count for k in sorted(res.graph.regions)], dtype=np.int64),
        final_sums=np.array([res.graph.regions[k].band_sums for k in sorted(res.graph.regions)], dtype=np.float64),
        assignment=res.graph.pixel_assignment.astype(np.int32),
        root_initial_count=np.int64(res.root_initial.live_count),
        converged_early=np.int8(res.converged_early),
        jsonl_sha256=_jsonl_sha(res),
        ref_wall_s=np.float64(wall),
        **arrs,
    )
    print(name, "records", len(arrs["log_dissim"]), f"{wall:.1f}s", flush=True)


def gen_small_rhseg():
    cases = []
    rng = np.random.default_rng(2106)
    for k in range(10):
        edge = int(rng.choice([4, 8, 16]))
        levels = int(rng.integers(1, 4))
        while edge % (2 ** (levels - 1)):
            levels -= 1
        bands = int(rng.integers(1, 6))
        w = float(rng.choice([0.0, 0.21, 0.5, 1.0]))
        tgt = int(rng.integers(1, 8))
        st = int(rng.integers(tgt, tgt + 6))
        if k % 2:
            s = rng.integers(0, 3, size=(bands, edge, edge)).astype(np.float32)
        else:
            s = rng.normal(0.0, 30.0, size=(bands, edge, edge)).astype(np.float32)
        img = HyperImage(edge, edge, bands, s)
        params = RhsegParams(HsegParams(w, tgt), levels=levels, section_target_regions=st)
        res = rhseg_run(img, params)
        arrs = _log_arrays(res)
        cases.append(dict(edge=edge, bands=bands, levels=levels, w=w, tgt=tgt, st=st,
                          samples=s.ravel(), labels=res.labels.labels.ravel().astype(np.int32),
                          conv=int(res.converged_early), **arrs))
    flat = {}
    flat["meta"] = np.array([[c["edge"], c["bands"], c["levels"], c["w"], c["tgt"], c["st"], c["conv"], len(c["log_dissim"])] for c in cases], dtype=np.float64)
    for key in ("samples", "labels", "log_level", "log_row", "log_col", "log_survivor", "log_absorbed", "log_dissim", "log_kind"):
        flat[key] = np.concatenate([c[key] for c in cases])
    np.savez_compressed(os.path.join(GOLDEN, "rhseg_small.npz"),
                        source="rhseg.recursive.rhseg_run, SequentialExecutor, random cubes", **flat)
    print("rhseg_small", len(cases), flush=True)


def gen_wire_frames():
    """ASSIGN frames and the unmodified reference worker's RESULT replies
    (wire.py:103-200, cluster.py:309-327) for a GPU worker speaking the same
    protocol. Stored as raw bytes; the worker must reproduce RESULT exactly."""
    from rhseg import wire
    from rhseg.cluster import WorkerServer
    from rhseg.sections import SectionId

    cases = []
    specs = [((16, 8, 4, 6, 3.0, 16), SectionId(3, 1, 2), 0.21, 6),
             ((32, 12, 4, 6, 3.0, 7), SectionId(2, 0, 1), 0.5, 9),
             ((12, 3, 2, 3, 1.0, 3), SectionId(1, 0, 0), 0.0, 4)]
    server = WorkerServer("127.0.0.1", 0)
    try:
        for gen, sid, w, tgt in specs:
            img, _ = gen_synthetic(*gen)
            payload = wire.AssignPayload(sid, img, w, tgt, "seq", 16).encode()
            frame = wire.encode_message(wire.ASSIGN, payload)
            reply = server._run_assign(payload)
            cases.append((frame, reply))
    finally:
        server.stop()
    arrays = {}
    for k, (frame, reply) in enumerate(cases):
        arrays[f"assign_{k}"] = np.frombuffer(frame, np.uint8)
        arrays[f"result_{k}"] = np.frombuffer(reply, np.uint8)
    np.savez_compressed(os.path.join(GOLDEN, "wire_frames.npz"), n=len(cases), **arrays)
    print("wire_frames", [len(r) for _, r in cases])


def main(which):
    os.makedirs(GOLDEN, exist_ok=True)
    workers = int(os.environ.get("GOLDEN_WORKERS", "6"))
    fast = PerPair(tile_k=16, workers=workers)
    if which in ("small", "all"):
        gen_synth_hashes()
        gen_hseg_corpus()
        gen_scan_tables()
        gen_small_rhseg()
        img, _ = gen_synthetic(16, 8, 4, 6, 3.0, 16)
        gen_rhseg("rhseg_16x16x8_L3", img, RhsegParams(HsegParams(0.21, 6), levels=3, section_target_regions=10), fast,
                  "gen_synthetic(16,8,4,6,3.0,16); L=3, w=0.21, target 6, section_target 10")
        img, _ = gen_synthetic(32, 224, 16, 25, 3.0, 32)
        gen_rhseg("rhseg_32x32x224_L2", img, RhsegParams(HsegParams(0.21, 16), levels=2), fast,
                  "gen_synthetic(32,224,16,25,3.0,32); L=2, w=0.21, target 16 (C3/C4 leaf shape)")
    if which in ("wire", "all"):
        gen_wire_frames()
    if which in ("crit2", "all"):
        img, _ = gen_synthetic(64, 16, 4, 6, 3.0, 64)
        gen_rhseg("crit2_64x64x16_L3", img, RhsegParams(HsegParams(0.21, 50), levels=3, section_target_regions=60), fast,
                  "criterion 2 (test_acceptance.py:133-166) 64x64x16 L=3")
    if which in ("c1", "all"):
        img, _ = gen_synthetic(64, 32, 4, 6, 3.0, 2)
        gen_rhseg("c1_64x64x32", img, RhsegParams(HsegParams(0.5, 2), levels=1), fast,
                  "BASELINE config 1: gen_synthetic(64,32,4,6,3.0,2); HSEG L=1, w=0.5, target 2")
    if which in ("c2", "all"):
        img, _ = gen_synthetic(145, 220, 16, 25, 3.0, 145)
        img = img.crop(0, 0, 144, 144)
        gen_rhseg("c2_144x144x220_L3", img, RhsegParams(HsegParams(0.5, 16), levels=3), fast,
                  "BASELINE config 2: gen_synthetic(145,220,16,25,3.0,145).crop(0,0,144,144); L=3, w=0.5, target 16")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "small")
