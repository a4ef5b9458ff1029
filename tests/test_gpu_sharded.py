"""The multi-GPU data path (partial subtree runs -> packed section states ->
reassembly on rank 0) replayed on one B200 with one private
context per rank: logs, labels and the root graph must be bit-identical to the
single-GPU run and to the CPU oracle, for every world size."""

import numpy as np
import pytest

import paper_2106_12942_b200 as rh
from paper_2106_12942_b200.distributed import emulate_sharded

pytestmark = pytest.mark.gpu


def _flat(res):
    a, b, d, k, sec = [], [], [], [], []
    for sid, recs in res.section_logs:
        aa, bb, dd, kk = recs.arrays()
        a.append(np.asarray(aa)); b.append(np.asarray(bb)); d.append(np.asarray(dd)); k.append(np.asarray(kk))
        sec += [(sid.level, sid.row, sid.col)] * len(aa)
    return (np.concatenate(a), np.concatenate(b), np.concatenate(d), np.concatenate(k), sec)


@pytest.mark.parametrize("world", [2, 4, 8, 16])
@pytest.mark.parametrize("w", [0.0, 0.21])
def test_sharded_equals_single(world, w, oracle):
    img, _ = rh.gen_synthetic(64, 12, 4, 6, 3.0, 64)
    params = rh.RhsegParams(rh.HsegParams(w, 6), 4, 12)
    single = rh.rhseg_run(img, params)
    shard = emulate_sharded(img, params, world)
    fa, fb = _flat(single), _flat(shard)
    assert fa[4] == fb[4]
    for x, y in zip(fa[:4], fb[:4]):
        assert np.array_equal(np.asarray(x).view(np.uint8), np.asarray(y).view(np.uint8))
    assert np.array_equal(single.labels.labels, shard.labels.labels)
    assert np.array_equal(single.graph.pixel_assignment, shard.graph.pixel_assignment)
    ref = oracle.rhseg_run(img.samples, 4, w, 6, 12)
    assert np.array_equal(fb[2].view(np.uint64), ref["log_dissim"].view(np.uint64))
    assert np.array_equal(shard.labels.labels, ref["labels"])


@pytest.mark.parametrize("world", [2, 4])
def test_torchrun_sharded_step(world, tmp_path):
    """The torch.distributed path itself (plan, export, gather, rank-0 upper
    levels, log gather + canonical reassembly) under torchrun; gloo stands in
    for NCCL because every rank shares the one GPU of the test box."""
    import json
    import os
    import socket
    import subprocess
    import sys

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = tmp_path / "res.json"
    worker = os.path.join(os.path.dirname(__file__), "sharded_worker.py")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", worker, str(out)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.loads(out.read_text())
    assert res["ok"] and res["records"] > 0 and res["world"] == world
