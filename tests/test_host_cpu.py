"""CPU-only checks: the C-ABI library loads and exports every declared symbol,
the host-side types mirror the reference's semantics, the synthetic generator
is byte-identical to the reference's, and the product path refuses to run
without a device (no silent CPU fallback)."""

import ctypes
import hashlib
import json
import os
import re

import numpy as np
import pytest

import paper_2106_12942_b200 as rh
from paper_2106_12942_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "rhseg_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char \*)\s*\*?\s*(rhseg_\w+)\s*\(", hdr, re.M)))


def test_header_declares_the_abi():
    syms = declared_symbols()
    for s in ("rhseg_scan_adjacent", "rhseg_scan_nonadjacent", "rhseg_hseg_graph", "rhseg_run_device",
              "rhseg_run_host", "rhseg_result_log", "rhseg_last_error"):
        assert s in syms
    assert set(syms) == set(_lib.EXPORTS)


def test_library_loads_and_exports_every_symbol():
    L = _lib.load()
    for s in declared_symbols():
        assert hasattr(L, s), s
    assert L.rhseg_abi_version() == 1


def test_no_device_means_loud_failure():
    """Without a GPU the product path raises; it never computes on the CPU."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    h = ctypes.c_void_p()
    assert _lib.load().rhseg_ctx_create(0, ctypes.byref(h)) == _lib.RHSEG_E_CUDA
    img, _ = rh.gen_synthetic(8, 2, 2, 2, 1.0, 1)
    with pytest.raises(rh.DeviceError):
        rh.rhseg_run(img, rh.RhsegParams(rh.HsegParams(0.21, 2)))
    counts = np.ones(2)
    d = np.empty(2)
    j = np.empty(2, np.int64)
    with pytest.raises(rh.DeviceError):
        rh.scan_adjacent(0, 2, counts, np.array([[0.0], [2.0]]), np.array([0, 1, 2]), np.array([1, 0]), d, j)


def test_synth_matches_reference_hashes():
    spec = json.load(open(os.path.join(ROOT, "tests", "golden", "synth_hashes.json")))
    for c in spec["cases"]:
        if c["args"][0] > 200:
            continue
        img, gt = rh.gen_synthetic(*c["args"])
        assert hashlib.sha256(img.samples.tobytes()).hexdigest() == c["samples_sha256"], c["args"]
        assert hashlib.sha256(gt.labels.astype(np.int64).tobytes()).hexdigest() == c["labels_sha256"]


def test_params_validation_like_reference():
    with pytest.raises(ValueError):
        rh.HsegParams(spectral_weight=1.5)
    with pytest.raises(ValueError):
        rh.HsegParams(target_regions=0)
    with pytest.raises(ValueError):
        rh.HsegParams(measure="euclid")
    with pytest.raises(ValueError):
        rh.RhsegParams(levels=0)
    assert rh.RhsegParams(rh.HsegParams(0.3, 7)).section_target_regions == 7
    with pytest.raises(ValueError):
        rh.make_strategy("gpu")


def test_sections_and_log_order():
    assert rh.log_order(2) == [rh.SectionId(2, 0, 0), rh.SectionId(2, 0, 1), rh.SectionId(2, 1, 0),
                               rh.SectionId(2, 1, 1), rh.SectionId(1, 0, 0)]
    assert rh.SectionId(1, 0, 0).children() == [rh.SectionId(2, 0, 0), rh.SectionId(2, 0, 1),
                                                rh.SectionId(2, 1, 0), rh.SectionId(2, 1, 1)]
    img = rh.HyperImage(8, 8, 1, np.arange(64, dtype=np.float32))
    tasks = rh.partition(img, 3)
    assert len(tasks) == 16 and tasks[5].origin == (2, 2)
    assert np.array_equal(tasks[5].image.samples[0], img.samples[0, 2:4, 2:4])
    with pytest.raises(rh.IndivisibleImage):
        rh.partition(rh.HyperImage(6, 6, 1, np.zeros(36, np.float32)), 3)


def test_graph_types_and_merge_semantics():
    img = rh.HyperImage(3, 3, 2, np.arange(18, dtype=np.float32))
    g = rh.init_region_graph(img, 8)
    assert g.region(4).adjacency == {0, 1, 2, 3, 5, 6, 7, 8}
    g4 = rh.init_region_graph(img, 4)
    assert g4.region(4).adjacency == {1, 3, 5, 7}
    rec = rh.merge_regions(g, 5, 1, 1.5, rh.MergeKind.ADJACENT)
    assert (rec.survivor_id, rec.absorbed_id, rec.step) == (1, 5, 0)
    assert g.region(1).pixel_count == 2 and 5 not in g.regions
    assert np.array_equal(g.region(1).band_sums, img.pixel_matrix()[1] + img.pixel_matrix()[5])
    g.check_invariants(img.samples.astype(np.float64).sum(axis=(1, 2)))
    with pytest.raises(rh.SelfMerge):
        rh.merge_regions(g, 1, 1, 0.0, rh.MergeKind.ADJACENT)
    with pytest.raises(rh.DeadRegion):
        rh.merge_regions(g, 5, 2, 0.0, rh.MergeKind.ADJACENT)


def test_dense_renumber_first_occurrence():
    assert rh.dense_renumber(np.array([7, 7, 3, 9, 3, 7])).tolist() == [0, 0, 1, 2, 1, 0]


def test_from_arrays_roundtrip():
    counts = np.array([2, 0, 1, 1])
    sums = np.arange(8, dtype=np.float64).reshape(4, 2)
    bits = np.zeros((4, 1), np.uint32)
    for a, b in ((0, 2), (2, 3)):
        bits[a, 0] |= 1 << b
        bits[b, 0] |= 1 << a
    g = rh.RegionGraph.from_arrays(2, 2, counts, sums, bits, np.array([0, 0, 2, 3]))
    assert sorted(g.regions) == [0, 2, 3]
    assert g.region(2).adjacency == {0, 3} and list(g.region(0).pixels) == [0, 1]
    g.check_invariants()


def test_record_list_is_lazy_sequence():
    from paper_2106_12942_b200.recursive import RecordList

    rl = RecordList(np.array([0, 2]), np.array([1, 3]), np.array([0.5, 1.0]), np.array([0, 1], np.uint8))
    assert len(rl) == 2 and rl[1].absorbed_id == 3 and rl[1].kind == rh.MergeKind.NON_ADJACENT
    assert rl == [rh.MergeRecord(0, 0, 1, 0.5, rh.MergeKind.ADJACENT),
                  rh.MergeRecord(1, 2, 3, 1.0, rh.MergeKind.NON_ADJACENT)]


def test_first_context_call_does_not_deadlock():
    """_lib.context() as the very first library call (what smoke() does) must
    reach the device check, not self-deadlock on the module lock."""
    import subprocess
    import sys

    code = ("import sys; sys.path.insert(0, %r)\n"
            "from paper_2106_12942_b200 import _lib, errors\n"
            "try:\n    _lib.context(0)\nexcept (errors.DeviceError, errors.ExtensionMissing):\n    pass\n"
            "print('ok')\n") % ROOT
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120,
                         env={**os.environ, "CUDA_VISIBLE_DEVICES": ""})
    assert out.returncode == 0 and out.stdout.strip() == "ok", out.stderr
