"""Parity of the sm_100a path against the reference's golden outputs and the
CPU oracle. Every call goes through the C ABI (librhseg_b200.so)."""

import os

import numpy as np
import pytest

import paper_2106_12942_b200 as rh
from golden_io import LOG_KEYS, corpus_cases, load, scan_table_cases, small_rhseg_cases

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _flat(res):
    rows = list(res.flat_log())
    return {
        "log_level": np.array([r["level"] for r in rows], np.int64),
        "log_row": np.array([r["section"][0] for r in rows], np.int64),
        "log_col": np.array([r["section"][1] for r in rows], np.int64),
        "log_survivor": np.array([r["survivor"] for r in rows], np.int64),
        "log_absorbed": np.array([r["absorbed"] for r in rows], np.int64),
        "log_dissim": np.array([r["dissim"] for r in rows], np.float64),
        "log_kind": np.array([0 if r["kind"] == "adjacent" else 1 for r in rows], np.int64),
    }


def assert_log_equal(got, exp, where=""):
    for k in LOG_KEYS:
        g, e = np.asarray(got[k]), np.asarray(exp[k])
        assert g.shape == e.shape, (where, k, g.shape, e.shape)
        if k == "log_dissim":
            bad = np.nonzero(g.view(np.uint64) != e.astype(np.float64).view(np.uint64))[0]
        else:
            bad = np.nonzero(g.astype(np.int64) != e.astype(np.int64))[0]
        assert bad.size == 0, f"{where} {k} differs first at record {bad[:1]}: {g[bad[:3]]} vs {e[bad[:3]]}"


def test_scan_tables_bitwise():
    for c in scan_table_cases():
        n = c["n"]
        d = np.full(n, -7.0)
        j = np.full(n, -7, np.int64)
        rh.scan_adjacent(0, n, c["counts"], c["sums"], c["indptr"], c["indices"], d, j)
        assert np.array_equal(d.view(np.uint64), c["adj_d"].view(np.uint64))
        assert np.array_equal(j, c["adj_j"])
        rh.scan_nonadjacent(0, n, 16, c["counts"], c["sums"], c["indptr"], c["indices"], d, j)
        assert np.array_equal(d.view(np.uint64), c["non_d"].view(np.uint64))
        assert np.array_equal(j, c["non_j"])


def test_scan_partial_rows_untouched():
    c = next(iter(scan_table_cases()))
    n = c["n"]
    lo, hi = n // 3, 2 * n // 3
    d = np.full(n, -7.0)
    j = np.full(n, -7, np.int64)
    rh.scan_nonadjacent(lo, hi, 4, c["counts"], c["sums"], c["indptr"], c["indices"], d, j)
    assert np.all(d[:lo] == -7.0) and np.all(d[hi:] == -7.0)
    assert np.array_equal(d[lo:hi].view(np.uint64), c["non_d"][lo:hi].view(np.uint64))


@pytest.mark.parametrize("cluster", [0, 2])
def test_hseg_run_corpus(cluster):
    """The 300-case criterion-1 corpus (test_acceptance.py:56-87) through the
    device hseg_run: merge tuples, bitwise dissims, converged flag, assignment."""
    n = 0
    for c in corpus_cases():
        img = rh.HyperImage(c["edge"], c["edge"], c["bands"], c["samples"])
        g = rh.init_region_graph(img, c["conn"])
        h = rh.hseg_run(g, rh.HsegParams(c["weight"], c["target"]), cluster=cluster)
        surv, absd, d, kind = c["records"]
        assert [r.survivor_id for r in h.records] == surv.tolist(), n
        assert [r.absorbed_id for r in h.records] == absd.tolist(), n
        got_d = np.array([r.dissimilarity for r in h.records], np.float64)
        assert np.array_equal(got_d.view(np.uint64), d.view(np.uint64)), n
        assert [int(r.kind) for r in h.records] == kind.tolist(), n
        assert h.converged_early == c["converged"], n
        assert np.array_equal(g.pixel_assignment, c["assign"]), n
        n += 1
    assert n == 300


@pytest.mark.parametrize("cluster", [0, 1, 2, 4])
def test_small_rhseg_golden(cluster):
    for c in small_rhseg_cases():
        img = rh.HyperImage(c["edge"], c["edge"], c["bands"], c["samples"])
        params = rh.RhsegParams(rh.HsegParams(c["weight"], c["target"]), c["levels"], c["section_target"])
        res = rh.rhseg_run(img, params, executor=rh.B200Executor(cluster=cluster))
        assert_log_equal(_flat(res), c["log"], f"case edge={c['edge']} L={c['levels']}")
        assert np.array_equal(res.labels.labels, c["labels"])
        assert res.converged_early == c["converged"]


SYNTH = {
    "rhseg_16x16x8_L3": ((16, 8, 4, 6, 3.0, 16), 3, 0.21, 6, 10),
    "rhseg_32x32x224_L2": ((32, 224, 16, 25, 3.0, 32), 2, 0.21, 16, 16),
    "crit2_64x64x16_L3": ((64, 16, 4, 6, 3.0, 64), 3, 0.21, 50, 60),
    "c1_64x64x32": ((64, 32, 4, 6, 3.0, 2), 1, 0.5, 2, 2),
    "c2_144x144x220_L3": ((145, 220, 16, 25, 3.0, 145), 3, 0.5, 16, 16),
}


def synth_image(spec):
    img, _ = rh.gen_synthetic(*spec)
    if img.width == 145:
        img = img.crop(0, 0, 144, 144)
    return img


@pytest.mark.parametrize("name", list(SYNTH))
def test_synthetic_golden(name):
    """Reference rhseg_run outputs on gen_synthetic cubes, incl. BASELINE
    config 1 (HSEG 64x64x32 -> 2 regions) and config 2 (144x144x220, L=3)."""
    if not os.path.exists(os.path.join(GOLDEN, name + ".npz")):
        pytest.skip("fixture not generated")
    z = load(name + ".npz")
    spec, levels, w, t, st = SYNTH[name]
    res = rh.rhseg_run(synth_image(spec), rh.RhsegParams(rh.HsegParams(w, t), levels, st))
    assert_log_equal(_flat(res), z, name)
    assert np.array_equal(res.labels.labels, z["labels"])
    assert np.array_equal(res.graph.pixel_assignment, z["assignment"].astype(np.int64))
    ids = np.array(sorted(res.graph.regions))
    assert np.array_equal(ids, z["final_ids"])
    sums = np.array([res.graph.regions[k].band_sums for k in ids])
    assert np.array_equal(sums.view(np.uint64), z["final_sums"].view(np.uint64))


_ORACLE_CACHE = {}


@pytest.mark.parametrize("cluster", [1, 2, 4, 8, 16])
def test_cluster_sizes_match_oracle(cluster, oracle):
    """Every CTAs-per-section choice gives the oracle's bits (30x30 = 900 regions
    per leaf, so 16 CTAs own >= 56 rows each; the tiny root leaves most of the
    16 CTAs with no rows at all)."""
    img, _ = rh.gen_synthetic(60, 12, 4, 6, 3.0, 60)
    for w, L in ((0.0, 2), (0.21, 2), (1.0, 1)):
        im = img if L == 2 else img.crop(0, 0, 30, 30)
        key = (w, L)
        if key not in _ORACLE_CACHE:
            oracle.set_threads(os.cpu_count() or 1)
            _ORACLE_CACHE[key] = oracle.rhseg_run(im.samples, L, w, 5, 9)
        ref = _ORACLE_CACHE[key]
        res = rh.rhseg_run(im, rh.RhsegParams(rh.HsegParams(w, 5), L, 9),
                           executor=rh.B200Executor(cluster=cluster))
        assert_log_equal(_flat(res), ref, f"w={w} L={L} C={cluster}")
        assert np.array_equal(res.labels.labels, ref["labels"])


def test_random_cases_vs_oracle(oracle):
    rng = np.random.default_rng(99)
    for case in range(12):
        edge = int(rng.choice([8, 12, 16, 24]))
        levels = int(rng.integers(1, 4))
        while edge % (1 << (levels - 1)):
            levels -= 1
        bands = int(rng.integers(1, 20))
        w = float(rng.choice([0.0, 0.21, 0.5, 1.0]))
        conn = int(rng.choice([4, 8]))
        if case % 3 == 0:
            s = rng.integers(0, 3, size=(bands, edge, edge)).astype(np.float32)
        else:
            s = rng.normal(0, 25, size=(bands, edge, edge)).astype(np.float32)
        t = int(rng.integers(1, 10))
        st = int(rng.integers(t, t + 12))
        img = rh.HyperImage(edge, edge, bands, s)
        res = rh.rhseg_run(img, rh.RhsegParams(rh.HsegParams(w, t), levels, st),
                           executor=rh.B200Executor(connectivity=conn))
        ref = oracle.rhseg_run(s, levels, w, t, st, connectivity=conn)
        assert_log_equal(_flat(res), ref, f"case {case}")
        assert np.array_equal(res.labels.labels, ref["labels"])
        assert res.converged_early == ref["converged_early"]


def test_edge_cases():
    # single pixel: nothing to merge
    img = rh.HyperImage(1, 1, 2, np.zeros((2, 1, 1), np.float32))
    res = rh.rhseg_run(img, rh.RhsegParams(rh.HsegParams(0.21, 1)))
    assert list(res.flat_log()) == [] and res.labels.labels.tolist() == [[0]]
    # target == initial -> empty hierarchy
    img2, _ = rh.gen_synthetic(4, 2, 2, 2, 1.0, 3)
    g = rh.init_region_graph(img2, 8)
    assert rh.hseg_run(g, rh.HsegParams(0.21, 16)).records == []
    # indivisible image raises the reference's error type
    with pytest.raises(rh.IndivisibleImage):
        rh.rhseg_run(rh.HyperImage(6, 6, 1, np.zeros((1, 6, 6), np.float32)),
                     rh.RhsegParams(rh.HsegParams(0.21, 1), levels=3))
    # tie-break: [[0,0],[9,9]] -> (0,1,0.0), (2,3,0.0) (test_engine.py:251-258)
    img3 = rh.HyperImage(2, 2, 1, np.array([[0, 0], [9, 9]], np.float32))
    h = rh.hseg_run(rh.init_region_graph(img3, 8), rh.HsegParams(0.21, 2))
    assert [(r.survivor_id, r.absorbed_id, r.dissimilarity) for r in h.records] == [(0, 1, 0.0), (2, 3, 0.0)]
    # converged early on a disconnected graph with w = 0 (test_engine.py:276-301)
    g4 = rh.init_region_graph(rh.HyperImage(2, 2, 1, np.array([[0, 0], [9, 9]], np.float32)), 4)
    for rid in list(g4.regions):
        g4.regions[rid].adjacency.clear()
    h4 = rh.hseg_run(g4, rh.HsegParams(0.0, 1))
    assert h4.converged_early and g4.live_count == 4


def test_profile_steps_and_replay():
    """profile.steps == 34 on 8x8x2 seed 5 target 30 (test_engine.py:318-325);
    recorded dissims equal the scalar formula on a replay (304-315)."""
    rng = np.random.default_rng(5)
    img = rh.HyperImage(8, 8, 2, rng.normal(size=(2, 8, 8)).astype(np.float32))
    g = rh.init_region_graph(img, 8)
    prof = rh.ProfileStats()
    h = rh.hseg_run(g, rh.HsegParams(0.21, 30), profile=prof)
    assert prof.steps == 34 and len(h.records) == 34
    replay = rh.init_region_graph(img, 8)
    for rec in h.records:
        assert rec.dissimilarity == rh.sqrt_bsmse(replay.region(rec.survivor_id), replay.region(rec.absorbed_id))
        rh.merge_regions(replay, rec.survivor_id, rec.absorbed_id, rec.dissimilarity, rec.kind)
    g.check_invariants()


def test_result_graphs_and_labels_at():
    img, _ = rh.gen_synthetic(32, 4, 4, 6, 3.0, 7)
    res = rh.rhseg_run(img, rh.RhsegParams(rh.HsegParams(0.21, 5), 3, 12))
    res.graph.check_invariants(img.samples.astype(np.float64).sum(axis=(1, 2)))
    res.root_initial.check_invariants(img.samples.astype(np.float64).sum(axis=(1, 2)))
    assert res.root_initial.live_count == res.root_hierarchy.initial_region_count
    top = res.labels_at(res.root_hierarchy.initial_region_count - len(res.root_hierarchy.records))
    assert np.array_equal(top.labels, res.labels.labels)
    assert res.labels_at(res.root_initial.live_count).label_count() == res.root_initial.live_count


@pytest.mark.parametrize("measure", ["euclidean", "sam"])
@pytest.mark.parametrize("cluster", [0, 2, 8])
def test_extension_measures_vs_oracle(measure, cluster, oracle):
    """euclidean / sam (north-star extensions, no reference implementation):
    bit-exact against the oracle's restatement, incl. the fdlibm acos on device."""
    rng = np.random.default_rng(17)
    cases = []
    for case in range(8):
        edge = int(rng.choice([8, 12, 16]))
        levels = int(rng.integers(1, 4))
        while edge % (1 << (levels - 1)):
            levels -= 1
        bands = int(rng.integers(1, 12))
        w = float(rng.choice([0.0, 0.21, 1.0]))
        conn = int(rng.choice([4, 8]))
        if case % 3 == 0:
            s = rng.integers(0, 3, size=(bands, edge, edge)).astype(np.float32)
        else:
            s = rng.normal(40, 25, size=(bands, edge, edge)).astype(np.float32)
        t = int(rng.integers(1, 8))
        cases.append((s, levels, w, t, int(rng.integers(t, t + 10)), conn))
    img, _ = rh.gen_synthetic(32, 12, 4, 6, 3.0, 32)
    cases.append((img.samples, 2, 0.21, 4, 9, 8))
    oracle.set_measure(measure)
    try:
        for k, (s, levels, w, t, st, conn) in enumerate(cases):
            bands, edge, _ = s.shape
            img = rh.HyperImage(edge, edge, bands, s)
            res = rh.rhseg_run(img, rh.RhsegParams(rh.HsegParams(w, t, measure), levels, st),
                               executor=rh.B200Executor(connectivity=conn, cluster=cluster))
            ref = oracle.rhseg_run(s, levels, w, t, st, connectivity=conn)
            assert_log_equal(_flat(res), ref, f"{measure} case {k}")
            assert np.array_equal(res.labels.labels, ref["labels"])
            assert res.converged_early == ref["converged_early"]
    finally:
        oracle.set_measure("sqrt-bsmse")


@pytest.mark.parametrize("measure", ["euclidean", "sam"])
def test_extension_measures_hseg_run_and_step(measure, oracle):
    img, _ = rh.gen_synthetic(16, 6, 4, 6, 3.0, 5)
    g = rh.init_region_graph(img, 8)
    h = rh.hseg_run(g, rh.HsegParams(0.5, 3, measure))
    fn = rh.MEASURES[measure]
    replay = rh.init_region_graph(img, 8)
    for rec in h.records:
        assert rec.dissimilarity == fn(replay.region(rec.survivor_id), replay.region(rec.absorbed_id))
        rh.merge_regions(replay, rec.survivor_id, rec.absorbed_id, rec.dissimilarity, rec.kind)
    g2 = rh.init_region_graph(img, 8)
    first = rh.hseg_step(g2, rh.HsegParams(0.5, 3, measure))
    assert (first.survivor_id, first.absorbed_id, first.dissimilarity) == (
        h.records[0].survivor_id, h.records[0].absorbed_id, h.records[0].dissimilarity)


@pytest.mark.parametrize("name", ["c1_64x64x32", "crit2_64x64x16_L3", "c2_144x144x220_L3"])
def test_native_outputs_hash_equals_reference(name, tmp_path):
    """End to end: the device run's merge-log JSONL written natively has the sha256
    of the reference CLI's JSONL for the same cube (cli.py:387-390)."""
    import hashlib

    from paper_2106_12942_b200 import outputs

    z = load(name + ".npz")
    spec, levels, w, t, st = SYNTH[name]
    res = rh.rhseg_run(synth_image(spec), rh.RhsegParams(rh.HsegParams(w, t), levels, st))
    out = outputs.write_outputs(res, tmp_path / "o.pgm", tmp_path / "o.merges.jsonl")
    assert hashlib.sha256((tmp_path / "o.merges.jsonl").read_bytes()).hexdigest() == str(z["jsonl_sha256"])
    assert len(out["content_hash"]) == 64


def test_largest_section_first_merges_vs_oracle(oracle):
    """The largest supported section (128x128 = 16384 regions: 16-CTA cluster,
    1024 rows per CTA, 2 GB D): the first merges against the oracle."""
    img, _ = rh.gen_synthetic(128, 6, 4, 6, 3.0, 11)
    R0 = 128 * 128
    for w in (0.21, 0.0):
        g = rh.init_region_graph(img, 8)
        h = rh.hseg_run(g, rh.HsegParams(w, R0 - 4))
        oracle.set_threads(os.cpu_count() or 1)
        ref = oracle.rhseg_run(img.samples, 1, w, R0 - 4)
        assert [(r.survivor_id, r.absorbed_id) for r in h.records] == list(
            zip(ref["log_survivor"].tolist(), ref["log_absorbed"].tolist()))
        got = np.array([r.dissimilarity for r in h.records])
        assert np.array_equal(got.view(np.uint64), ref["log_dissim"].view(np.uint64))


@pytest.mark.parametrize("bands,conn", [(1, 4), (300, 8), (37, 4)])
def test_band_counts_and_connectivity_vs_oracle(bands, conn, oracle):
    rng = np.random.default_rng(bands)
    s = rng.normal(50, 20, size=(bands, 24, 24)).astype(np.float32)
    img = rh.HyperImage(24, 24, bands, s)
    for w in (0.0, 0.5):
        res = rh.rhseg_run(img, rh.RhsegParams(rh.HsegParams(w, 5), 2, 11),
                           executor=rh.B200Executor(connectivity=conn))
        ref = oracle.rhseg_run(s, 2, w, 5, 11, connectivity=conn)
        assert_log_equal(_flat(res), ref, f"B={bands} conn={conn} w={w}")
        assert np.array_equal(res.labels.labels, ref["labels"])


def test_stress_determinism_and_leaf_parity(oracle):
    """Races show up as run-to-run differences at scale: 64 leaves of 32x32x64
    (two CTAs per SM, every phase of the loop exercised thousands of times),
    repeated runs must agree bit for bit, and sampled leaves must equal an
    independent HSEG of that leaf on the oracle (leaves are independent
    sections, recursive.py:130-142)."""
    img, _ = rh.gen_synthetic(256, 64, 16, 25, 3.0, 256)
    params = rh.RhsegParams(rh.HsegParams(0.21, 16), 4, 16)
    runs = [_flat(rh.rhseg_run(img, params)) for _ in range(3)]
    for k in LOG_KEYS:
        for r in runs[1:]:
            assert np.array_equal(np.asarray(r[k]).view(np.uint8), np.asarray(runs[0][k]).view(np.uint8)), k
    f = runs[0]
    oracle.set_threads(os.cpu_count() or 1)
    for (lr, lc) in ((0, 0), (3, 5), (7, 7), (5, 2)):
        m = (f["log_level"] == 4) & (f["log_row"] == lr) & (f["log_col"] == lc)
        sub = np.ascontiguousarray(img.samples[:, 32 * lr:32 * lr + 32, 32 * lc:32 * lc + 32])
        ref = oracle.rhseg_run(sub, 1, 0.21, 16)
        assert np.array_equal(f["log_survivor"][m], ref["log_survivor"])
        assert np.array_equal(f["log_absorbed"][m], ref["log_absorbed"])
        assert np.array_equal(f["log_dissim"][m].view(np.uint64), ref["log_dissim"].view(np.uint64))


def test_device_resident_path_equals_host_path():
    """rhseg_run_device (cube already in HBM, the bench's `value` leg) and the
    pipelined rhseg_run_host (chunked upload, the e2e leg / executor) agree bit
    for bit (leaf chunks of the host path run on their own streams)."""
    import torch

    from paper_2106_12942_b200.recursive import collect_result, result_info

    img, _ = rh.gen_synthetic(128, 16, 4, 6, 3.0, 12)
    params = rh.RhsegParams(rh.HsegParams(0.21, 8), 4, 12)
    host = _flat(rh.rhseg_run(img, params))
    ex = rh.B200Executor()
    cube = torch.from_numpy(np.ascontiguousarray(img.samples)).cuda()
    ctx = ex.execute_device(cube.data_ptr(), 128, 16, params)
    torch.cuda.synchronize()
    dev = _flat(collect_result(ctx, result_info(ctx), 128, 16, 4))
    for k in LOG_KEYS:
        assert np.array_equal(np.asarray(host[k]).view(np.uint8), np.asarray(dev[k]).view(np.uint8)), k


def test_hseg_step_sequence_equals_hseg_run():
    """hseg_step through the B3 per-row table kernels (engine.py:309-342) merge by
    merge reproduces the device loop's hseg_run (engine.py:345-371)."""
    img, _ = rh.gen_synthetic(12, 5, 4, 6, 3.0, 4)
    g1 = rh.init_region_graph(img, 8)
    h = rh.hseg_run(g1, rh.HsegParams(0.21, 20))
    g2 = rh.init_region_graph(img, 8)
    steps = []
    while g2.live_count > 20:
        rec = rh.hseg_step(g2, rh.HsegParams(0.21, 20))
        if rec is None:
            break
        steps.append((rec.survivor_id, rec.absorbed_id, rec.dissimilarity, int(rec.kind)))
    assert steps == [(r.survivor_id, r.absorbed_id, r.dissimilarity, int(r.kind)) for r in h.records]
    assert np.array_equal(g1.pixel_assignment, g2.pixel_assignment)


@pytest.mark.parametrize("measure", ["sam", "sqrt-bsmse"])
def test_config3_sampled_leaves_vs_oracle(measure, oracle):
    """BASELINE config 3 at full size (512x512x224, L=5, w=0.21, t=16; SAM and its
    BSMSE twin): the device run's logs for sampled leaves equal an independent
    oracle HSEG of those leaves (leaves are independent sections)."""
    img, _ = rh.gen_synthetic(512, 224, 16, 25, 3.0, 512)
    res = rh.rhseg_run(img, rh.RhsegParams(rh.HsegParams(0.21, 16, measure), 5, 16))
    logs = {(s.level, s.row, s.col): r for s, r in res.section_logs}
    oracle.set_threads(os.cpu_count() or 1)
    oracle.set_measure(measure)
    try:
        for (lr, lc) in ((0, 0), (9, 14)):
            sub = np.ascontiguousarray(img.samples[:, 32 * lr:32 * lr + 32, 32 * lc:32 * lc + 32])
            ref = oracle.rhseg_run(sub, 1, 0.21, 16)
            a, b, d, k = logs[(5, lr, lc)].arrays()
            assert np.array_equal(np.asarray(a), ref["log_survivor"])
            assert np.array_equal(np.asarray(b), ref["log_absorbed"])
            assert np.array_equal(np.asarray(d).view(np.uint64), ref["log_dissim"].view(np.uint64))
            assert np.array_equal(np.asarray(k), ref["log_kind"])
        _upper_levels_vs_replay(oracle, img, res, 5, 0.21, 16, 16)
    finally:
        oracle.set_measure("sqrt-bsmse")


def _upper_levels_vs_replay(oracle, img, res, levels, w, t, st):
    """Every level above the leaves: the oracle replays the device's leaf logs and
    computes the upper levels from scratch; logs and labels must match."""
    side = 1 << (levels - 1)
    logs = {(s.level, s.row, s.col): r for s, r in res.section_logs}
    cnt, parts = [], [[], [], [], []]
    for r in range(side):
        for c in range(side):
            arr = logs[(levels, r, c)].arrays()
            cnt.append(len(arr[0]))
            for q in range(4):
                parts[q].append(np.asarray(arr[q]))
    leaf = (cnt, *[np.concatenate(p) for p in parts])
    ref = oracle.rhseg_replay_leaves(img.samples, levels, w, t, st, leaf)
    got = _flat(res)
    for k in LOG_KEYS:
        g, e = np.asarray(got[k]), np.asarray(ref[k])
        if k == "log_dissim":
            assert np.array_equal(g.view(np.uint64), e.view(np.uint64)), k
        else:
            assert np.array_equal(g.astype(np.int64), e.astype(np.int64)), k
    assert np.array_equal(res.labels.labels, ref["labels"])


def test_config4_upper_levels_vs_oracle(oracle):
    """BASELINE config 4: all 1365 sections above the leaves (levels 1-6) and the
    final labels, against the oracle replaying the device's 4096 leaf logs."""
    img, _ = rh.gen_synthetic(2048, 224, 16, 25, 3.0, 2048)
    res = rh.rhseg_run(img, rh.RhsegParams(rh.HsegParams(0.21, 16), 7, 16))
    oracle.set_threads(os.cpu_count() or 1)
    _upper_levels_vs_replay(oracle, img, res, 7, 0.21, 16, 16)


def test_config4_sampled_leaves_vs_oracle(oracle):
    """BASELINE config 4 at full size (2048x2048x224, L=7, 4096 leaves, 4.19 M
    merges) through the executor: sampled leaves equal the oracle bit for bit,
    the merge count is the analytic one, labels are dense and the root holds 16
    regions."""
    img, _ = rh.gen_synthetic(2048, 224, 16, 25, 3.0, 2048)
    res = rh.rhseg_run(img, rh.RhsegParams(rh.HsegParams(0.21, 16), 7, 16))
    assert sum(len(r) for _, r in res.section_logs) == 4194288
    assert res.labels.label_count() == 16 and res.graph.live_count == 16
    logs = {(s.level, s.row, s.col): r for s, r in res.section_logs}
    oracle.set_threads(os.cpu_count() or 1)
    for (lr, lc) in ((0, 0), (37, 50)):
        sub = np.ascontiguousarray(img.samples[:, 32 * lr:32 * lr + 32, 32 * lc:32 * lc + 32])
        ref = oracle.rhseg_run(sub, 1, 0.21, 16)
        a, b, d, k = logs[(7, lr, lc)].arrays()
        assert np.array_equal(np.asarray(a), ref["log_survivor"])
        assert np.array_equal(np.asarray(b), ref["log_absorbed"])
        assert np.array_equal(np.asarray(d).view(np.uint64), ref["log_dissim"].view(np.uint64))


@pytest.mark.parametrize("apo", ["0", "1"])
def test_loop_variants_vs_oracle(apo, oracle, monkeypatch):
    """Both merge-loop formulations of w > 0 single-CTA sections -- APO (row a' bounded
    from D rows a and b, interval D/caches) and the mean stream (RHSEG_APO=0) -- equal the
    oracle, on noisy, tie-heavy integer and large-magnitude cubes (wide intervals,
    exact fallbacks) and both measures they cover."""
    monkeypatch.setenv("RHSEG_APO", apo)
    rng = np.random.default_rng(7 + int(apo))
    cubes = [
        rng.normal(0, 25, size=(12, 32, 32)).astype(np.float32),
        rng.integers(0, 3, size=(7, 32, 32)).astype(np.float32),       # ties everywhere
        (rng.normal(0, 1, size=(20, 16, 16)) * 1e6 + 3e7).astype(np.float32),  # |m| >> d
        rng.integers(0, 2, size=(1, 16, 16)).astype(np.float32),        # one band
    ]
    try:
        for k, s in enumerate(cubes):
            for measure in ("sqrt-bsmse", "euclidean"):
                oracle.set_measure(measure)
                b, e = s.shape[0], s.shape[1]
                img = rh.HyperImage(e, e, b, s)
                res = rh.rhseg_run(img, rh.RhsegParams(rh.HsegParams(0.37, 4, measure), 2, 6))
                ref = oracle.rhseg_run(s, 2, 0.37, 4, 6)
                assert_log_equal(_flat(res), ref, f"cube {k} {measure} APO={apo}")
                assert np.array_equal(res.labels.labels, ref["labels"])
    finally:
        oracle.set_measure("sqrt-bsmse")
