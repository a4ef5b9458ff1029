"""Host-side logic of the sharded (multi-GPU) RHSEG, on CPU: the subtree plan
 and the canonical-order reassembly of per-rank merge logs,
exercised across a real world-size-2 gloo process group. The per-rank log
pieces come from the CPU oracle, sliced by the plan exactly as the device
ranks would produce them."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2106_12942_b200.distributed import assemble_logs, block_sections, shard_plan


def test_plan_covers_every_subtree_once():
    for levels in (2, 3, 4, 7):
        for world in (1, 2, 4, 8, 16):
            top, blocks = shard_plan(levels, world)
            if world == 1:
                assert top == 1 and blocks == [(0, 0, 1, 1)]
                continue
            side = 1 << (top - 1)
            seen = []
            for b in blocks:
                if b is not None:
                    seen += block_sections(b, top, top)
            assert sorted(seen) == [(top, r, c) for r in range(side) for c in range(side)], (levels, world)
            # leaves of all blocks tile the leaf grid
            leaves = sorted(s for b in blocks if b is not None for s in block_sections(b, levels, top))
            ls = 1 << (levels - 1)
            assert leaves == [(levels, r, c) for r in range(ls) for c in range(ls)]


def test_plan_shapes():
    assert shard_plan(7, 2) == (2, [(0, 0, 1, 2), (1, 0, 1, 2)])
    assert shard_plan(7, 4)[0] == 2 and all(b[2:] == (1, 1) for b in shard_plan(7, 4)[1])
    top, blocks = shard_plan(7, 8)
    assert top == 3 and blocks[0] == (0, 0, 1, 2) and blocks[7] == (3, 2, 1, 2)
    assert shard_plan(1, 4) == (1, [(0, 0, 1, 1), None, None, None])
    assert shard_plan(2, 8)[0] == 2  # capped at levels: only 4 subtrees, 4 ranks idle
    assert sum(b is None for b in shard_plan(2, 8)[1]) == 4
    with pytest.raises(ValueError):
        shard_plan(7, 6)


def _slice_part(ref, keep):
    """(sections, a, b, d, k) for the sections in `keep` from a flat oracle log."""
    lev, row, col = ref["log_level"], ref["log_row"], ref["log_col"]
    secs, A, B, D, K = [], [], [], [], []
    off = 0
    seen = []
    for i in range(len(lev)):
        key = (int(lev[i]), int(row[i]), int(col[i]))
        if key in keep and key not in seen:
            seen.append(key)
    for key in seen:
        m = (lev == key[0]) & (row == key[1]) & (col == key[2])
        n = int(m.sum())
        secs.append((key[0], key[1], key[2], off, n))
        A.append(ref["log_survivor"][m]); B.append(ref["log_absorbed"][m])
        D.append(ref["log_dissim"][m]); K.append(ref["log_kind"][m])
        off += n
    cat = lambda xs, dt: np.concatenate(xs).astype(dt) if xs else np.zeros(0, dt)
    return secs, cat(A, np.int32), cat(B, np.int32), cat(D, np.float64), cat(K, np.uint8)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle

        levels = 3
        rng = np.random.default_rng(11)
        samples = rng.normal(0, 20, size=(5, 16, 16)).astype(np.float32)
        ref = oracle.rhseg_run(samples, levels, 0.21, 4, 7)
        top, blocks = shard_plan(levels, world)
        mine = set()
        for lv in range(levels, top - 1, -1):
            mine |= set(block_sections(blocks[rank], lv, top))
        part = _slice_part(ref, mine)
        got = [None] * world if rank == 0 else None
        dist.gather_object(part, got, dst=0)
        if rank == 0:
            upper = {(lv, r, c) for lv in range(top - 1, 0, -1) for r in range(1 << (lv - 1))
                     for c in range(1 << (lv - 1))}
            got.append(_slice_part(ref, upper))
            ids, a, b, d, k = assemble_logs(levels, got)
            ok = (np.array_equal(a, ref["log_survivor"]) and np.array_equal(b, ref["log_absorbed"])
                  and np.array_equal(d.view(np.uint64), ref["log_dissim"].view(np.uint64))
                  and np.array_equal(k, ref["log_kind"]))
            q.put(("ok" if ok else "mismatch", len(a), len(ref["log_dissim"])))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_log_reassembly(oracle):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    status, n, nref = q.get(timeout=5)
    assert status == "ok" and n == nref > 0
