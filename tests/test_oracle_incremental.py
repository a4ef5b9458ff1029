"""Pin the oracle's exact incremental HSEG mode (oracle_set_incremental, the checker
the full-size GPU parity tests use) against the literal from-scratch restatement and
against every reference golden fixture. CPU only."""

import os

import numpy as np
import pytest

from golden_io import LOG_KEYS, corpus_cases, load, small_rhseg_cases


@pytest.fixture
def inc(oracle):
    oracle.set_incremental(True)
    oracle.set_threads(os.cpu_count() or 1)
    try:
        yield oracle
    finally:
        oracle.set_incremental(False)
        oracle.set_measure("sqrt-bsmse")


def _same(a, b, where=""):
    for k in LOG_KEYS:
        x, y = np.asarray(a[k]), np.asarray(b[k])
        assert x.shape == y.shape, (where, k)
        if k == "log_dissim":
            assert np.array_equal(x.view(np.uint64), y.astype(np.float64).view(np.uint64)), (where, k)
        else:
            assert np.array_equal(x.astype(np.int64), y.astype(np.int64)), (where, k)


def test_incremental_corpus_golden(inc):
    """The 300-case criterion-1 corpus (test_acceptance.py:56-87) made by the reference."""
    n = 0
    for c in corpus_cases():
        res = inc.rhseg_run(c["samples"], 1, c["weight"], c["target"], connectivity=c["conn"])
        surv, absd, d, kind = c["records"]
        assert np.array_equal(res["log_survivor"], surv), n
        assert np.array_equal(res["log_absorbed"], absd), n
        assert np.array_equal(res["log_dissim"].view(np.uint64), d.view(np.uint64)), n
        assert np.array_equal(res["log_kind"], kind), n
        assert res["converged_early"] == c["converged"], n
        assert np.array_equal(res["assignment"].ravel(), c["assign"]), n
        n += 1
    assert n == 300


def test_incremental_small_rhseg_golden(inc):
    for c in small_rhseg_cases():
        res = inc.rhseg_run(c["samples"], c["levels"], c["weight"], c["target"], c["section_target"])
        _same(res, c["log"])
        assert np.array_equal(res["labels"], c["labels"])
        assert res["converged_early"] == c["converged"]


SYNTH = {
    "rhseg_16x16x8_L3": ((16, 8, 4, 6, 3.0, 16), None, 3, 0.21, 6, 10),
    "rhseg_32x32x224_L2": ((32, 224, 16, 25, 3.0, 32), None, 2, 0.21, 16, 16),
    "crit2_64x64x16_L3": ((64, 16, 4, 6, 3.0, 64), None, 3, 0.21, 50, 60),
    "c1_64x64x32": ((64, 32, 4, 6, 3.0, 2), None, 1, 0.5, 2, 2),
    "c2_144x144x220_L3": ((145, 220, 16, 25, 3.0, 145), 144, 3, 0.5, 16, 16),
}


@pytest.mark.parametrize("name", list(SYNTH))
def test_incremental_synthetic_golden(inc, name):
    """The reference's own rhseg_run on gen_synthetic cubes, incl. BASELINE configs 1
    and 2 (the whole runs: every section, every level, labels, assignment)."""
    from paper_2106_12942_b200.synth import gen_synthetic

    spec, crop, levels, w, t, st = SYNTH[name]
    z = load(name + ".npz")
    img, _ = gen_synthetic(*spec)
    s = img.samples if crop is None else np.ascontiguousarray(img.samples[:, :crop, :crop])
    res = inc.rhseg_run(s, levels, w, t, st)
    _same(res, z, name)
    assert np.array_equal(res["labels"], z["labels"])
    assert np.array_equal(res["assignment"].ravel(), z["assignment"])


def _cases(seed, n):
    rng = np.random.default_rng(seed)
    for case in range(n):
        edge = int(rng.choice([6, 8, 12, 16]))
        levels = int(rng.integers(1, 4))
        while edge % (1 << (levels - 1)):
            levels -= 1
        bands = int(rng.integers(1, 24))
        w = float(rng.choice([0.0, 0.21, 0.5, 1.0, 0.05]))
        conn = int(rng.choice([4, 8]))
        kind = case % 4
        if kind == 0:  # ties everywhere
            s = rng.integers(0, 3, size=(bands, edge, edge)).astype(np.float32)
        elif kind == 1:
            s = rng.normal(0, 25, size=(bands, edge, edge)).astype(np.float32)
        elif kind == 2:  # large magnitude, small differences
            s = (rng.normal(0, 1, size=(bands, edge, edge)) * 1e3 + 3e6).astype(np.float32)
        else:  # piecewise-constant blocks + small noise (near ties)
            base = rng.integers(0, 4, size=(bands, 1 + edge // 4, 1 + edge // 4)).repeat(4, 1).repeat(4, 2)
            s = (base[:, :edge, :edge] * 10 + rng.integers(0, 2, size=(bands, edge, edge))).astype(np.float32)
        t = int(rng.integers(1, 10))
        st = int(rng.integers(t, t + 12))
        yield s, levels, w, t, st, conn


@pytest.mark.parametrize("measure", ["sqrt-bsmse", "euclidean", "sam"])
def test_incremental_equals_from_scratch_random(oracle, measure):
    """Random cubes (tie-heavy, noisy, large-magnitude, blocky), every measure,
    w in {0, .05, .21, .5, 1}, 4/8-connectivity, 1-3 levels: the incremental records,
    labels and assignment equal the from-scratch restatement's bit for bit."""
    oracle.set_threads(2)
    try:
        for k, (s, levels, w, t, st, conn) in enumerate(_cases(11 + len(measure), 60)):
            oracle.set_measure(measure)
            oracle.set_incremental(False)
            ref = oracle.rhseg_run(s, levels, w, t, st, connectivity=conn)
            oracle.set_incremental(True)
            got = oracle.rhseg_run(s, levels, w, t, st, connectivity=conn)
            _same(got, ref, f"{measure} case {k}")
            assert np.array_equal(got["labels"], ref["labels"]), k
            assert np.array_equal(got["assignment"], ref["assignment"]), k
            assert got["converged_early"] == ref["converged_early"], k
            assert got["root_initial_count"] == ref["root_initial_count"], k
    finally:
        oracle.set_incremental(False)
        oracle.set_measure("sqrt-bsmse")


def test_incremental_hseg_graph_arbitrary_adjacency(oracle):
    """hseg_graph on random graphs (arbitrary symmetric adjacency, counts > 1, some
    isolated regions -> early convergence at w = 0): incremental == from scratch."""
    rng = np.random.default_rng(5)
    try:
        for case in range(40):
            n = int(rng.integers(2, 40))
            nb = int(rng.integers(1, 9))
            counts = rng.integers(1, 6, size=n)
            sums = rng.integers(0, 4, size=(n, nb)).astype(np.float64) * counts[:, None]
            if case % 2:
                sums += rng.normal(0, 3, size=(n, nb))
            a = (rng.random((n, n)) < rng.choice([0.05, 0.2, 0.6])).astype(np.uint8)
            a = np.triu(a, 1)
            a = a + a.T
            w = float(rng.choice([0.0, 0.3, 1.0]))
            t = int(rng.integers(1, n))
            oracle.set_incremental(False)
            ref = oracle.hseg_graph(counts, sums, a, w, t)
            oracle.set_incremental(True)
            got = oracle.hseg_graph(counts, sums, a, w, t)
            for x, y in zip(got["records"], ref["records"]):
                assert np.array_equal(np.asarray(x).view(np.uint8), np.asarray(y).view(np.uint8)), case
            assert got["converged"] == ref["converged"], case
            assert np.array_equal(got["sums"].view(np.uint64), ref["sums"].view(np.uint64)), case
    finally:
        oracle.set_incremental(False)


def test_incremental_full_leaf_sizes(oracle):
    """Whole 32x32 leaves at the BASELINE band counts (224 and 64; w = 0.21, 1 and 0):
    the full-size leaf shape of C3-C5, incremental == from scratch."""
    from paper_2106_12942_b200.synth import gen_synthetic

    img, _ = gen_synthetic(64, 64, 4, 6, 3.0, 1024)
    sub = np.ascontiguousarray(img.samples[:, :32, :32])
    img2, _ = gen_synthetic(32, 224, 16, 25, 3.0, 512)
    oracle.set_threads(os.cpu_count() or 1)
    try:
        for s, w in ((sub, 0.0), (sub, 1.0), (img2.samples, 0.21)):
            oracle.set_incremental(False)
            ref = oracle.rhseg_run(s, 1, w, 16)
            oracle.set_incremental(True)
            got = oracle.rhseg_run(s, 1, w, 16)
            _same(got, ref, f"w={w} B={s.shape[0]}")
    finally:
        oracle.set_incremental(False)
