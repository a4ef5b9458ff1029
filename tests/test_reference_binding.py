"""The drop-in boundary against the real reference package (CPU; skipped where
/root/reference is absent, e.g. on the GPU box):

* bind.install() reaches every caller of the B2 seam -- the names recursive.py:16,
  cluster.py:17 and hybrid.py:19 bound at import time, not just rhseg.engine -- and
  the B3 kernel attributes; on a GPU-less host the calls end in the library's
  DeviceError, i.e. they left the reference's CPU path;
* the host helpers the reference exports (stitch, init_from_presegmentation,
  assemble_result) produce the reference's objects bit for bit."""

import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference package not present")


@pytest.fixture(scope="module")
def ref():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.dont_write_bytecode = True
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import rhseg

    return rhseg


def test_install_patches_every_hseg_run_caller(ref):
    import paper_2106_12942_b200 as b200
    from paper_2106_12942_b200 import bind, engine

    orig = {m: getattr(sys.modules[f"rhseg.{m}"], "hseg_run") for m in ("engine", "recursive", "cluster", "hybrid")}
    orig_scan = sys.modules["rhseg._kernels"].scan_adjacent
    h = bind.install(ref, default_executor=True)
    try:
        for m in orig:
            fn = getattr(sys.modules[f"rhseg.{m}"], "hseg_run")
            assert getattr(fn, "__wrapped__", None) is engine.hseg_run, m
        assert ref.hseg_run.__wrapped__ is engine.hseg_run
        assert sys.modules["rhseg._kernels"].scan_adjacent is b200.scan_adjacent
        assert sys.modules["rhseg._kernels"].scan_nonadjacent is b200.scan_nonadjacent
        img = ref.HyperImage(4, 4, 2, np.arange(32, dtype=np.float32).reshape(2, 4, 4))
        params = ref.RhsegParams(ref.HsegParams(0.21, 2), levels=2)
        task = ref.partition(img, 2)[0]
        try:
            import torch

            has_gpu = torch.cuda.is_available()
        except Exception:
            has_gpu = False
        if not has_gpu:
            # run_leaf (recursive.py:130-142) now calls the library, which has no device here
            with pytest.raises((b200.DeviceError, b200.ExtensionMissing)):
                sys.modules["rhseg.recursive"].run_leaf(task, params, ref.Sequential(), 8)
            with pytest.raises((b200.DeviceError, b200.ExtensionMissing)):
                ref.rhseg_run(img, params)  # default executor -> B200Executor
    finally:
        h.uninstall()
    for m, fn in orig.items():
        assert getattr(sys.modules[f"rhseg.{m}"], "hseg_run") is fn
    assert sys.modules["rhseg._kernels"].scan_adjacent is orig_scan


def _as_ref_graph(ref, g):
    out = ref.RegionGraph(g.width, g.height, g.bands)
    out.pixel_assignment = np.asarray(g.pixel_assignment, np.int64).copy()
    out.merges_done = g.merges_done
    for rid, r in g.regions.items():
        out.regions[rid] = ref.Region(rid, r.pixel_count, r.band_sums.copy(), set(r.adjacency), list(r.pixels))
    return out


def _same_graph(a, b):
    assert (a.width, a.height, a.bands) == (b.width, b.height, b.bands)
    assert sorted(a.regions) == sorted(b.regions)
    assert np.array_equal(np.asarray(a.pixel_assignment), np.asarray(b.pixel_assignment))
    for rid in a.regions:
        x, y = a.regions[rid], b.regions[rid]
        assert x.pixel_count == y.pixel_count, rid
        assert np.array_equal(np.asarray(x.band_sums).view(np.uint64), np.asarray(y.band_sums).view(np.uint64)), rid
        assert set(x.adjacency) == set(y.adjacency), rid
        assert list(x.pixels) == list(y.pixels), rid


@pytest.mark.parametrize("conn", [4, 8])
def test_stitch_equals_reference(ref, conn):
    import paper_2106_12942_b200 as b200

    rng = np.random.default_rng(conn)
    quads = []
    for k in range(4):
        s = rng.normal(0, 5, size=(3, 6, 6)).astype(np.float32)
        g = b200.init_region_graph(b200.HyperImage(6, 6, 3, s), conn)
        for _ in range(int(rng.integers(0, 20))):  # arbitrary merges (not HSEG's) via the shared semantics
            ids = sorted(g.regions)
            a = int(rng.choice(ids))
            nb = sorted(g.regions[a].adjacency)
            if nb:
                b200.merge_regions(g, a, int(rng.choice(nb)), 0.0, b200.MergeKind.ADJACENT)
        quads.append(g)
    got = b200.stitch(quads, conn)
    exp = ref.stitch([_as_ref_graph(ref, g) for g in quads], conn)
    _same_graph(got, exp)
    with pytest.raises(b200.ShapeMismatch):
        b200.stitch(quads[:3], conn)


def test_init_from_presegmentation_equals_reference(ref):
    import paper_2106_12942_b200 as b200

    rng = np.random.default_rng(1)
    for conn in (4, 8):
        s = rng.normal(100, 30, size=(5, 8, 8)).astype(np.float32)
        lab = rng.integers(0, 6, size=(8, 8)) * 10 + 3
        got = b200.init_from_presegmentation(b200.HyperImage(8, 8, 5, s), b200.LabelMap(8, 8, lab), conn)
        exp = ref.init_from_presegmentation(ref.HyperImage(8, 8, 5, s), ref.LabelMap(8, 8, lab), conn)
        _same_graph(got, exp)


def test_assemble_result_equals_reference(ref):
    import paper_2106_12942_b200 as b200

    s = np.random.default_rng(2).normal(0, 5, size=(2, 4, 4)).astype(np.float32)
    g = b200.init_region_graph(b200.HyperImage(4, 4, 2, s), 8)
    root0 = g.copy()
    recs = [b200.merge_regions(g, 0, 1, 1.5, b200.MergeKind.ADJACENT),
            b200.merge_regions(g, 2, 3, 2.5, b200.MergeKind.NON_ADJACENT)]
    params = b200.RhsegParams(b200.HsegParams(0.21, 14), 1)
    got = b200.assemble_result(params, {b200.SectionId(1, 0, 0): recs}, root0, g, False)
    rparams = ref.RhsegParams(ref.HsegParams(0.21, 14), 1)
    exp = sys.modules["rhseg.recursive"].assemble_result(
        rparams, {ref.SectionId(1, 0, 0): recs}, _as_ref_graph(ref, root0), _as_ref_graph(ref, g), False)
    assert [r for r in got.flat_log()] == [r for r in exp.flat_log()]
    assert np.array_equal(got.labels.labels, exp.labels.labels)
    assert got.root_hierarchy.initial_region_count == exp.root_hierarchy.initial_region_count


def test_record_list_equals_reference_records(ref):
    from paper_2106_12942_b200.recursive import RecordList

    rl = RecordList(np.array([0, 2], np.int32), np.array([1, 3], np.int32), np.array([0.5, 1.5]),
                    np.array([0, 1], np.uint8))
    exp = [ref.MergeRecord(0, 0, 1, 0.5, ref.MergeKind.ADJACENT), ref.MergeRecord(1, 2, 3, 1.5, ref.MergeKind.NON_ADJACENT)]
    assert rl == exp
    exp[1] = ref.MergeRecord(1, 2, 3, 1.25, ref.MergeKind.NON_ADJACENT)
    assert rl != exp
