"""Pin the CPU oracle (oracle/rhseg_oracle.c) against the reference's own
outputs committed under tests/golden/ (made by oracle/gen_golden.py from the
unmodified reference). CPU only."""

import os

import numpy as np
import pytest

from golden_io import LOG_KEYS, corpus_cases, load, scan_table_cases, small_rhseg_cases


def test_oracle_scan_tables_bitwise(oracle):
    """_kernels.scan_adjacent/scan_nonadjacent per-row tables, bit for bit
    (the reference's test_engine.py:104-129 contract)."""
    ncases = 0
    for c in scan_table_cases():
        n = c["n"]
        d = np.empty(n)
        j = np.empty(n, np.int64)
        oracle.scan_adjacent(0, n, c["counts"], c["sums"], c["indptr"], c["indices"], d, j)
        assert np.array_equal(d.view(np.uint64), c["adj_d"].view(np.uint64))
        assert np.array_equal(j, c["adj_j"])
        oracle.scan_nonadjacent(0, n, 5, c["counts"], c["sums"], c["indptr"], c["indices"], d, j)
        assert np.array_equal(d.view(np.uint64), c["non_d"].view(np.uint64))
        assert np.array_equal(j, c["non_j"])
        ncases += 1
    assert ncases == 24


def test_oracle_hseg_corpus():
    """300 criterion-1-style cases (test_acceptance.py:56-87): merge tuples,
    dissimilarities (bitwise), converged flag and pixel assignment."""
    from oracle import oracle

    n = 0
    for c in corpus_cases():
        res = oracle.rhseg_run(c["samples"], 1, c["weight"], c["target"], connectivity=c["conn"])
        surv, absd, d, kind = c["records"]
        assert np.array_equal(res["log_survivor"], surv), n
        assert np.array_equal(res["log_absorbed"], absd), n
        assert np.array_equal(res["log_dissim"].view(np.uint64), d.view(np.uint64)), n
        assert np.array_equal(res["log_kind"], kind), n
        assert res["converged_early"] == c["converged"], n
        assert np.array_equal(res["assignment"].ravel(), c["assign"]), n
        n += 1
    assert n == 300


def _check_log(res, z_or_dict):
    for k in LOG_KEYS:
        got, exp = res[k], z_or_dict[k]
        if k == "log_dissim":
            assert np.array_equal(got.view(np.uint64), exp.view(np.uint64)), k
        else:
            assert np.array_equal(got.astype(np.int64), exp.astype(np.int64)), k


def test_oracle_small_rhseg():
    from oracle import oracle

    for c in small_rhseg_cases():
        res = oracle.rhseg_run(c["samples"], c["levels"], c["weight"], c["target"], c["section_target"])
        _check_log(res, c["log"])
        assert np.array_equal(res["labels"], c["labels"])
        assert res["converged_early"] == c["converged"]


@pytest.mark.parametrize("name", ["rhseg_16x16x8_L3", "rhseg_32x32x224_L2", "crit2_64x64x16_L3"])
def test_oracle_synthetic_rhseg(name):
    from oracle import oracle
    from paper_2106_12942_b200.synth import gen_synthetic

    path = os.path.join(os.path.dirname(__file__), "golden", name + ".npz")
    if not os.path.exists(path):
        pytest.skip(f"{name} fixture not generated")
    z = load(name + ".npz")
    spec = {
        "rhseg_16x16x8_L3": ((16, 8, 4, 6, 3.0, 16), 3, 0.21, 6, 10),
        "rhseg_32x32x224_L2": ((32, 224, 16, 25, 3.0, 32), 2, 0.21, 16, 16),
        "crit2_64x64x16_L3": ((64, 16, 4, 6, 3.0, 64), 3, 0.21, 50, 60),
    }[name]
    img, _ = gen_synthetic(*spec[0])
    oracle.set_threads(os.cpu_count() or 1)
    res = oracle.rhseg_run(img.samples, spec[1], spec[2], spec[3], spec[4])
    _check_log(res, z)
    assert np.array_equal(res["labels"], z["labels"])
    assert np.array_equal(res["assignment"].ravel(), z["assignment"])


def test_extension_measures_known_answers(oracle):
    """euclidean / sam (north-star extensions; no reference oracle): hand-checked
    values through the oracle's hseg on tiny graphs, and the fdlibm acos
    restatement agreeing with libm to 1 ulp and with the Python scalar bitwise."""
    import math

    from paper_2106_12942_b200.dissim import acos_fdlibm, euclidean_scalar, sam_scalar

    assert euclidean_scalar(1, 1, [0.0, 0.0], [3.0, 4.0]) == 5.0
    assert sam_scalar(1, 1, [1.0, 0.0], [0.0, 2.0]) == acos_fdlibm(0.0)
    assert abs(sam_scalar(1, 1, [1.0, 0.0], [0.0, 2.0]) - math.pi / 2) < 1e-15
    assert sam_scalar(2, 3, [2.0, 4.0], [3.0, 6.0]) == 0.0
    assert sam_scalar(1, 1, [0.0, 0.0], [0.0, 0.0]) == 0.0
    rng = np.random.default_rng(3)
    for x in np.concatenate([rng.uniform(-1, 1, 20000), [1.0, -1.0, 0.0, 0.5, -0.5, 1 - 2 ** -53]]):
        a = oracle.acos(float(x))
        assert a == acos_fdlibm(float(x))
        assert abs(a - math.acos(x)) <= math.ulp(math.acos(x))
    # two regions, one merge: the recorded dissimilarity is the scalar formula
    for name, fn in (("euclidean", euclidean_scalar), ("sam", sam_scalar), ("sqrt-bsmse", None)):
        oracle.set_measure(name)
        try:
            r = oracle.hseg_graph([1, 1], [[1.0, 2.0], [4.0, 6.0]], [[0, 1], [1, 0]], 0.21, 1)
        finally:
            oracle.set_measure("sqrt-bsmse")
        d = r["records"][2][0]
        if fn is not None:
            assert d == fn(1, 1, [1.0, 2.0], [4.0, 6.0]), name
        else:
            assert d == math.sqrt(0.5 * 25.0)


def test_oracle_replay_leaves_equals_full_run(oracle):
    """The upper-level checker (leaves replayed from a log, levels above computed
    from scratch) reproduces the full oracle run."""
    from paper_2106_12942_b200 import gen_synthetic

    img, _ = gen_synthetic(32, 6, 4, 6, 3.0, 5)
    full = oracle.rhseg_run(img.samples, 3, 0.21, 4, 9)
    m = full["log_level"] == 3
    cnt = [int((m & (full["log_row"] == r) & (full["log_col"] == c)).sum()) for r in range(4) for c in range(4)]
    rep = oracle.rhseg_replay_leaves(img.samples, 3, 0.21, 4, 9, (cnt, full["log_survivor"][m],
                                     full["log_absorbed"][m], full["log_dissim"][m], full["log_kind"][m]))
    for k, v in full.items():
        if isinstance(v, np.ndarray):
            assert np.array_equal(v, rep[k]), k
