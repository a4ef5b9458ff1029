"""Drop-in semantics of the host seams on the device path (B2 stop_check, the
per-section helpers run_leaf / run_upper_levels / assemble_result)."""

import numpy as np
import pytest

import paper_2106_12942_b200 as rh

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("stop_at", [1, 2, 7, 40, 10**9])
def test_stop_check_called_before_every_step(stop_at):
    """engine.py:351-363: stop_check runs before each step with the graph at that step
    boundary; True ends the run with `interrupted` and exactly the steps done so far."""
    img, _ = rh.gen_synthetic(16, 6, 4, 6, 3.0, 9)
    full_g = rh.init_region_graph(img, 8)
    full = rh.hseg_run(full_g, rh.HsegParams(0.21, 5))
    g = rh.init_region_graph(img, 8)
    seen = []

    def stop():
        seen.append(g.live_count)
        return len(seen) >= stop_at

    h = rh.hseg_run(g, rh.HsegParams(0.21, 5), stop_check=stop)
    done = min(stop_at - 1, len(full.records))
    assert len(h.records) == done
    assert h.interrupted == (stop_at - 1 < len(full.records))
    # each call saw the graph after exactly the previous steps
    assert seen == [256 - k for k in range(len(seen))]
    assert [(r.survivor_id, r.absorbed_id, r.dissimilarity) for r in h.records] == [
        (r.survivor_id, r.absorbed_id, r.dissimilarity) for r in full.records[:done]]
    replay = rh.init_region_graph(img, 8)
    for r in full.records[:done]:
        rh.merge_regions(replay, r.survivor_id, r.absorbed_id, r.dissimilarity, r.kind)
    assert np.array_equal(g.pixel_assignment, replay.pixel_assignment)


def test_stop_check_on_converged_run():
    """A run that converges early (w = 0, disconnected graph) checks once more before
    the step that finds no pair, like the reference."""
    g = rh.init_region_graph(rh.HyperImage(2, 2, 1, np.array([[0, 0], [9, 9]], np.float32)), 4)
    for rid in list(g.regions):
        g.regions[rid].adjacency.clear()
    calls = []
    h = rh.hseg_run(g, rh.HsegParams(0.0, 1), stop_check=lambda: calls.append(1) and False)
    assert h.converged_early and not h.interrupted and len(calls) == 1


def test_per_section_helpers_equal_executor():
    """run_leaf + run_upper_levels + assemble_result (recursive.py:107-170, each section's
    HSEG through the B2 seam, host stitch) == the one-call device executor."""
    img, _ = rh.gen_synthetic(32, 8, 4, 6, 3.0, 21)
    params = rh.RhsegParams(rh.HsegParams(0.21, 5), 3, 9)
    exp = rh.rhseg_run(img, params)
    graphs, logs, conv, root0 = {}, {}, False, None
    for task in rh.partition(img, 3):
        g, recs, c, r0 = rh.run_leaf(task, params, rh.Sequential(), 8)
        graphs[task.section_id], logs[task.section_id] = g, recs
        conv |= c
    root0, c2 = rh.run_upper_levels(params, rh.Sequential(), 8, graphs, logs)
    got = rh.assemble_result(params, logs, root0, graphs[rh.SectionId(1, 0, 0)], conv | c2)
    assert list(got.flat_log()) == list(exp.flat_log())
    assert np.array_equal(got.labels.labels, exp.labels.labels)
