"""Sections above the shared-memory loops' capacity (16384 regions: one CTA, or a 16-CTA
cluster) run on the grid loop (csrc/grid_loop.cu): a group of co-resident CTAs per
section, state in HBM, one group barrier per merge. The reference runs any section size
(/root/reference/pkg/src/rhseg/sections.py:57-79), so these tests hold the grid loop to the
same bar as every other loop: the oracle's exact incremental HSEG, bit for bit.

Every device call goes through the C ABI (librhseg_b200.so)."""

import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2106_12942_b200 as rh
from paper_2106_12942_b200 import _lib
from test_gpu_full_parity import assert_flat_equal, device_flat

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _oracle_inc(oracle, samples, levels, w, t, st, measure="sqrt-bsmse"):
    oracle.set_threads(os.cpu_count() or 1)
    oracle.set_measure(measure)
    oracle.set_incremental(True)
    try:
        return oracle.rhseg_run(samples, levels, w, t, st)
    finally:
        oracle.set_incremental(False)
        oracle.set_measure("sqrt-bsmse")


def _host_ram_gb():
    try:
        import psutil

        return psutil.virtual_memory().available / 2**30
    except Exception:  # pragma: no cover
        return 0.0


def _run_and_check(oracle, img, levels, w, t, st, measure="sqrt-bsmse", grid_level=None):
    res = rh.rhseg_run(img, rh.RhsegParams(rh.HsegParams(w, t, measure), levels, st))
    if grid_level is not None:
        info = _lib.level_info(_lib.context(0).handle, grid_level)
        assert info["loop"] == "grid", info
    ref = _oracle_inc(oracle, img.samples, levels, w, t, st, measure)
    assert_flat_equal(device_flat(res), ref, f"{img.width}x{img.width}x{img.bands} L={levels} w={w} {measure}")
    assert np.array_equal(res.labels.labels, ref["labels"])
    assert res.converged_early == ref["converged_early"]
    return res


@pytest.mark.parametrize("w", [0.5, 0.0, 1.0])
def test_grid_loop_160x160_hseg_vs_oracle(w, oracle):
    """One 160x160 section (25600 regions > 16384) merged down to 8 regions: every record
    (survivor, absorbed, dissimilarity bits, kind), labels and convergence equal the
    oracle's; w = 0 runs the adjacency-only stage."""
    img, _ = rh.gen_synthetic(160, 8, 4, 6, 3.0, 160)
    _run_and_check(oracle, img, 1, w, 8, 8, grid_level=1)


@pytest.mark.parametrize("measure", ["sam", "euclidean"])
def test_grid_loop_extension_measures_vs_oracle(measure, oracle):
    img, _ = rh.gen_synthetic(136, 6, 4, 6, 3.0, 7)
    _run_and_check(oracle, img, 1, 0.21, 5, 5, measure=measure, grid_level=1)


def test_grid_loop_upper_level_above_cluster_capacity_vs_oracle(oracle):
    """RHSEG with section_target_regions 6000: the four 96x96 leaves (9216 regions, cluster
    loop) stop at 6000 regions each, so the root section holds 24000 regions and runs on the
    grid loop; leaves, root, labels all equal the oracle's."""
    img, _ = rh.gen_synthetic(192, 8, 4, 6, 3.0, 192)
    _run_and_check(oracle, img, 2, 0.21, 10, 6000, grid_level=1)


def test_grid_loop_hseg_graph_b2(oracle):
    """The B2 seam (hseg_run on a caller's RegionGraph) above 16384 regions: a 130x130 grid
    graph through rhseg_hseg_graph, records equal to the oracle's hseg_graph."""
    img, _ = rh.gen_synthetic(130, 5, 4, 6, 3.0, 3)
    g = rh.init_region_graph(img, 8)
    h = rh.hseg_run(g, rh.HsegParams(0.3, 40))
    assert _lib.level_info(_lib.context(0).handle, 1)["loop"] == "grid"
    oracle.set_threads(os.cpu_count() or 1)
    ref = _oracle_inc(oracle, img.samples, 1, 0.3, 40, 40)
    assert [(r.survivor_id, r.absorbed_id) for r in h.records] == list(
        zip(ref["log_survivor"].tolist(), ref["log_absorbed"].tolist()))
    got = np.array([r.dissimilarity for r in h.records])
    assert np.array_equal(got.view(np.uint64), ref["log_dissim"].view(np.uint64))
    assert [int(r.kind) for r in h.records] == ref["log_kind"].tolist()


def test_grid_loop_256x256_single_section_vs_oracle(oracle):
    """an L = 1 256x256 HSEG (65536 regions, a 34 GB D on the device and
    in the oracle's host memory) bit-exact against the oracle."""
    if _host_ram_gb() < 48:
        pytest.skip("the oracle's dense D for 65536 regions needs ~40 GB of host memory")
    img, _ = rh.gen_synthetic(256, 4, 4, 6, 3.0, 256)
    _run_and_check(oracle, img, 1, 0.5, 16, 16, grid_level=1)


_FORCED = r"""
import os, sys, numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, os.path.join({root!r}, "tests"))
import paper_2106_12942_b200 as rh
from paper_2106_12942_b200 import _lib
from oracle import oracle
from test_gpu_full_parity import assert_flat_equal, device_flat
oracle.build(); oracle.set_threads(os.cpu_count() or 1); oracle.set_incremental(True)
cases = [((64, 32, 4, 6, 3.0, 2), 1, 0.5, 2, 2),       # BASELINE config 1 (one 4096-region section)
         ((60, 12, 4, 6, 3.0, 60), 2, 0.21, 5, 9),
         ((60, 12, 4, 6, 3.0, 60), 2, 0.0, 5, 9),
         ((96, 16, 4, 6, 3.0, 9), 1, 1.0, 3, 3)]
for spec, L, w, t, st in cases:
    img, _ = rh.gen_synthetic(*spec)
    res = rh.rhseg_run(img, rh.RhsegParams(rh.HsegParams(w, t), L, st), executor=rh.B200Executor(cluster=16))
    loops = [_lib.level_info(_lib.context(0).handle, l)["loop"] for l in range(1, L + 1)]
    assert "grid" in loops, loops
    ref = oracle.rhseg_run(img.samples, L, w, t, st)
    assert_flat_equal(device_flat(res), ref, str(spec))
    assert np.array_equal(res.labels.labels, ref["labels"])
print("forced grid ok")
"""


def test_grid_loop_forced_on_cluster_sections_vs_oracle():
    """RHSEG_GRID=1 routes every multi-CTA section to the grid loop: BASELINE config 1 and
    small multi-level runs (forced 16-CTA sections, so the grid loop sees sections with
    fewer chunks than CTAs, w = 0, w = 1) equal the oracle. A subprocess, because the
    library reads the switch once."""
    env = dict(os.environ, RHSEG_GRID="1")
    out = subprocess.run([sys.executable, "-c", _FORCED.format(root=ROOT)], env=env, capture_output=True, text=True,
                         timeout=900)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert "forced grid ok" in out.stdout
