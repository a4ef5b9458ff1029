"""CPU-only checks of the measurement plumbing: both bench arms print the same config
dict, the committed CPU-baseline plan is read back correctly, the section-parallel CPU
leg (one leaf per thread) performs exactly the merges of the single-leaf leg, and the
loop-variant names the roofline keys on are the C ABI's (rhseg_b200.h)."""

import os
import re
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import bench  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_2106_12942_b200 import _lib  # noqa: E402


def test_config_dict_identical_across_arms_and_workloads():
    for name in bench.WORKLOADS:
        c = bench.config_of(name)
        assert c == bench.config_of(name)
        bands, edge, _ = bench.cube_shape(name)
        assert c["edge"] == edge and c["bands"] == bands
        spec, crop, levels, w, t, st = bench.WORKLOADS[name]
        assert (c["levels"], c["spectral_weight"], c["target_regions"]) == (levels, w, t)
        assert "parallelism" not in c  # arm-specific details live in "execution"


def test_full_cpu_plan_reads_the_committed_measurement():
    fp = bench.full_cpu_plan("c4")
    assert fp is not None and fp["cores"] >= 1 and fp["value"] > 0
    assert fp["best"] in ("within", "sections")
    assert fp["value"] == max(fp["within"], fp["sections"])
    c1 = bench.full_cpu_plan("c1")
    assert c1 is not None and c1["single_core"] < c1["value"]
    assert bench.full_cpu_plan("no-such-workload") is None


def test_section_parallel_leaves_match_single_leaf_runs():
    oracle.build()
    oracle.set_measure("sqrt-bsmse")
    rng = np.random.default_rng(5)
    cube = rng.normal(100, 10, size=(6, 16, 16)).astype(np.float32)
    origins = [(0, 0), (0, 8), (8, 0), (8, 8)]
    for w in (0.0, 0.5):
        par = oracle.run_leaves(cube, origins, 8, w, 3)
        oracle.set_threads(1)
        seq = [oracle.run_leaf(cube, r, c, 8, w, 3) for r, c in origins]
        assert list(par) == seq == [61] * 4


def test_loop_variant_names_follow_the_abi():
    hdr = open(os.path.join(ROOT, "include", "rhseg_b200.h")).read()
    codes = {m[0]: int(m[1]) for m in re.findall(r"#define (RHSEG_LOOP_\w+) (\d+)", hdr)}
    assert set(codes.values()) == set(_lib.LOOP_NAMES)
    assert _lib.LOOP_NAMES[codes["RHSEG_LOOP_APO"]] == "APO"
    assert _lib.LOOP_NAMES[codes["RHSEG_LOOP_ADJACENT"]].startswith("adjacent")
    assert _lib.LOOP_NAMES[codes["RHSEG_LOOP_GRID"]] == "grid"


def test_grid_loop_sections_have_no_fixed_region_limit():
    """The 16384-region section limit is gone from the drop-in contract (sections above a
    cluster's capacity run on the grid loop); only device memory for D bounds a section."""
    hdr = open(os.path.join(ROOT, "include", "rhseg_b200.h")).read()
    m = re.search(r"#define RHSEG_E_TOO_LARGE \d+\s*/\*(.*?)\*/", hdr)
    assert m and "16384" not in m.group(1) and "memory" in m.group(1)
    api = open(os.path.join(ROOT, "paper_2106_12942_b200", "csrc", "rhseg_api.cu")).read()
    assert "launch_grid_loop" in api and "max_regions" in api
