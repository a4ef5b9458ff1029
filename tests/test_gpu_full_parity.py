"""Full-size parity: EVERY section of BASELINE configs 3, 4 and 5 -- all leaves and all
upper levels -- against the oracle's exact incremental HSEG (oracle_set_incremental,
pinned to the from-scratch restatement and the reference's golden fixtures by
tests/test_oracle_incremental.py), plus the two merge-loop formulations against each
other at full size and adversarial cubes for the APO interval bounds.

Every device call goes through the C ABI (librhseg_b200.so)."""

import os

import numpy as np
import pytest

import paper_2106_12942_b200 as rh

pytestmark = pytest.mark.gpu

KEYS = ("log_level", "log_row", "log_col", "log_survivor", "log_absorbed", "log_dissim", "log_kind")

# name -> (gen_synthetic args, levels, weight, target, section_target, measure)
CONFIGS = {
    "c3_sam": ((512, 224, 16, 25, 3.0, 512), 5, 0.21, 16, 16, "sam"),
    "c3_bsmse": ((512, 224, 16, 25, 3.0, 512), 5, 0.21, 16, 16, "sqrt-bsmse"),
    "c4": ((2048, 224, 16, 25, 3.0, 2048), 7, 0.21, 16, 16, "sqrt-bsmse"),
    "c5_w0": ((1024, 64, 4, 6, 3.0, 1024), 6, 0.0, 16, 16, "sqrt-bsmse"),
    "c5_w1": ((1024, 64, 4, 6, 3.0, 1024), 6, 1.0, 16, 16, "sqrt-bsmse"),
}


def device_flat(res):
    """Flat log arrays (log order) straight from the device-returned section arrays."""
    parts = {k: [] for k in KEYS}
    for sid, recs in res.section_logs:
        a, b, d, k = (np.asarray(x) for x in recs.arrays())
        n = len(a)
        parts["log_level"].append(np.full(n, sid.level, np.int64))
        parts["log_row"].append(np.full(n, sid.row, np.int64))
        parts["log_col"].append(np.full(n, sid.col, np.int64))
        parts["log_survivor"].append(a.astype(np.int64))
        parts["log_absorbed"].append(b.astype(np.int64))
        parts["log_dissim"].append(d.astype(np.float64))
        parts["log_kind"].append(k.astype(np.int64))
    return {k: np.concatenate(v) if v else np.zeros(0) for k, v in parts.items()}


def assert_flat_equal(got, ref, where):
    for k in KEYS:
        g, e = np.asarray(got[k]), np.asarray(ref[k])
        assert g.shape == e.shape, (where, k, g.shape, e.shape)
        if k == "log_dissim":
            bad = np.nonzero(g.view(np.uint64) != e.astype(np.float64).view(np.uint64))[0]
        else:
            bad = np.nonzero(g.astype(np.int64) != e.astype(np.int64))[0]
        if bad.size:
            i = int(bad[0])
            sec = (int(ref["log_level"][i]), int(ref["log_row"][i]), int(ref["log_col"][i]))
            pytest.fail(f"{where}: {k} differs at {bad.size} records, first #{i} in section {sec}: "
                        f"{g[bad[:3]]} vs {e[bad[:3]]}")


def oracle_full(oracle, samples, levels, w, t, st, measure):
    oracle.set_threads(os.cpu_count() or 1)
    oracle.set_measure(measure)
    oracle.set_incremental(True)
    try:
        return oracle.rhseg_run(samples, levels, w, t, st)
    finally:
        oracle.set_incremental(False)
        oracle.set_measure("sqrt-bsmse")


@pytest.mark.parametrize("name", list(CONFIGS))
def test_full_config_every_section_vs_oracle(name, oracle):
    """Every record of every section (C4: 4096 leaves + 1365 upper sections, 4,194,288
    merges; C5 w = 0 runs the adjacency-only loop) equals the oracle bit for bit:
    survivor, absorbed, dissimilarity bits, kind, section; then labels and the root
    assignment."""
    spec, levels, w, t, st, measure = CONFIGS[name]
    img, _ = rh.gen_synthetic(*spec)
    res = rh.rhseg_run(img, rh.RhsegParams(rh.HsegParams(w, t, measure), levels, st))
    got = device_flat(res)
    ref = oracle_full(oracle, img.samples, levels, w, t, st, measure)
    side = 1 << (levels - 1)
    nleaf = int(np.unique(ref["log_row"][ref["log_level"] == levels] * side
                          + ref["log_col"][ref["log_level"] == levels]).size)
    assert nleaf == side * side  # every leaf is in the comparison
    assert_flat_equal(got, ref, name)
    assert np.array_equal(res.labels.labels, ref["labels"])
    assert np.array_equal(res.graph.pixel_assignment.reshape(ref["assignment"].shape), ref["assignment"])
    assert res.converged_early == ref["converged_early"]


@pytest.mark.parametrize("name", ["c3_bsmse", "c4", "c5_w1"])
def test_apo_and_stream_loops_identical_at_full_size(name, monkeypatch):
    """the APO loop (interval D entries, hand-derived error bounds) and the
    exact mean-stream loop (RHSEG_APO=0) produce the same bits on every section of the
    full-size configs."""
    spec, levels, w, t, st, measure = CONFIGS[name]
    img, _ = rh.gen_synthetic(*spec)
    params = rh.RhsegParams(rh.HsegParams(w, t, measure), levels, st)
    out = {}
    for apo in ("1", "0"):
        monkeypatch.setenv("RHSEG_APO", apo)
        res = rh.rhseg_run(img, params)
        out[apo] = (device_flat(res), res.labels.labels.copy())
    assert_flat_equal(out["1"][0], out["0"][0], f"{name} APO vs stream")
    assert np.array_equal(out["1"][1], out["0"][1])


def _adversarial_cubes(seed):
    """32x32-leaf cubes that stress the APO interval decisions."""
    rng = np.random.default_rng(seed)
    e, B = 64, int(rng.choice([3, 16, 40]))
    kind = seed % 4
    if kind == 0:
        # near-tie clusters: a few levels, each pixel nudged by 0/1 float32 ulp, so many
        # pair dissimilarities agree to the last bits
        base = rng.integers(0, 3, size=(B, e, e)).astype(np.float32) * np.float32(64.0) + np.float32(1024.0)
        ulp = np.spacing(base)
        s = base + ulp * rng.integers(0, 2, size=base.shape).astype(np.float32)
    elif kind == 1:
        # huge |m| with tiny d: values near 3e7 (ulp 2) differing by a few ulp
        s = (3.0e7 + 2.0 * rng.integers(0, 4, size=(B, e, e))).astype(np.float32)
    elif kind == 2:
        # large blocks (regions grow to hundreds of pixels next to single pixels: tiny
        # count ratios in the merge coefficient) with sparse outliers
        blk = rng.integers(0, 4, size=(B, e // 16, e // 16)).repeat(16, 1).repeat(16, 2)
        s = (blk * 100.0 + rng.normal(0, 0.01, size=(B, e, e))).astype(np.float32)
        out = rng.random((e, e)) < 0.01
        s[:, out] += np.float32(37.0)
    else:
        # mixed magnitudes across bands + exact duplicates
        s = (rng.normal(0, 1, size=(B, e, e)) * np.logspace(-3, 6, B)[:, None, None]).astype(np.float32)
        s[:, 1::2, ::4] = s[:, 0::2, ::4]
    return np.ascontiguousarray(s)


@pytest.mark.parametrize("measure", ["sqrt-bsmse", "euclidean"])
def test_apo_adversarial_cubes_vs_oracle(measure, oracle):
    """Near-tie clusters differing in the last ulp, |m| >> d, tiny count ratios and mixed
    band magnitudes, at the real 32x32 leaf size (APO loop) over many seeds and both
    APO measures, against the oracle."""
    oracle.set_threads(os.cpu_count() or 1)
    oracle.set_incremental(True)
    oracle.set_measure(measure)
    try:
        for seed in range(24):
            s = _adversarial_cubes(seed)
            B, e, _ = s.shape
            w = (0.21, 1.0, 0.5)[seed % 3]
            img = rh.HyperImage(e, e, B, s)
            res = rh.rhseg_run(img, rh.RhsegParams(rh.HsegParams(w, 4, measure), 2, 12))
            ref = oracle.rhseg_run(s, 2, w, 4, 12)
            assert_flat_equal(device_flat(res), ref, f"{measure} seed {seed}")
            assert np.array_equal(res.labels.labels, ref["labels"])
    finally:
        oracle.set_incremental(False)
        oracle.set_measure("sqrt-bsmse")


def test_apo_hseg_graph_extreme_counts_vs_oracle(oracle):
    """B2 hseg_run on graphs whose regions carry counts from 1 to 1e6 (count ratios down
    to 1e-6 in the BSMSE coefficient and the APO mean weights): device == oracle."""
    rng = np.random.default_rng(3)
    for case in range(12):
        n = 700
        nb = int(rng.choice([4, 32]))
        counts = np.where(rng.random(n) < 0.1, rng.integers(10**4, 10**6, n), rng.integers(1, 4, n)).astype(np.int64)
        means = rng.integers(0, 5, size=(n, nb)).astype(np.float64) * 3.0 + rng.normal(0, 1e-3, size=(n, nb))
        sums = means * counts[:, None]
        a = np.zeros((n, n), np.uint8)
        for i in range(n):  # a ring plus random chords
            a[i, (i + 1) % n] = a[(i + 1) % n, i] = 1
        ch = rng.integers(0, n, size=(n, 2))
        a[ch[:, 0], ch[:, 1]] = 1
        a[ch[:, 1], ch[:, 0]] = 1
        np.fill_diagonal(a, 0)
        w, t = float(rng.choice([0.21, 1.0])), 8
        g = rh.RegionGraph(n, 1, nb)
        for i in range(n):
            g.regions[i] = rh.Region(i, int(counts[i]), sums[i].copy(), set(np.nonzero(a[i])[0].tolist()), [i])
            g.pixel_assignment[i] = i
        h = rh.hseg_run(g, rh.HsegParams(w, t))
        oracle.set_incremental(True)
        try:
            ref = oracle.hseg_graph(counts, sums, a, w, t)
        finally:
            oracle.set_incremental(False)
        sv, ab, dd, kk = ref["records"]
        assert [r.survivor_id for r in h.records] == sv.tolist(), case
        assert [r.absorbed_id for r in h.records] == ab.tolist(), case
        got_d = np.array([r.dissimilarity for r in h.records], np.float64)
        assert np.array_equal(got_d.view(np.uint64), dd.view(np.uint64)), case
        assert [int(r.kind) for r in h.records] == kk.tolist(), case
