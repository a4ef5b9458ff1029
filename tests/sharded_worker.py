"""torchrun worker for tests/test_gpu_sharded.py: the real torch.distributed
ShardedRhseg step (gloo backend, every rank on cuda:0 -- one GPU in the test
box) compared on rank 0 with the single-GPU executor, bit for bit."""

import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2106_12942_b200 as rh  # noqa: E402
from paper_2106_12942_b200.distributed import ShardedRhseg  # noqa: E402


def main():
    out = sys.argv[1]
    measure = sys.argv[2] if len(sys.argv) > 2 else "sqrt-bsmse"
    dist.init_process_group("gloo")
    rank = dist.get_rank()
    torch.cuda.set_device(0)
    img, _ = rh.gen_synthetic(64, 10, 4, 6, 3.0, 64)
    params = rh.RhsegParams(rh.HsegParams(0.21, 6, measure), 4, 12)
    cube = torch.from_numpy(np.ascontiguousarray(img.samples)).cuda()
    sh = ShardedRhseg(params, img.width, img.bands, 0)
    for _ in range(2):  # twice: buffers and contexts are reused across steps
        parts = sh.step(cube)
    if rank == 0:
        res = sh.result(parts)
        single = rh.rhseg_run(img, params)
        a = [tuple(r.values()) for r in res.flat_log()]
        b = [tuple(r.values()) for r in single.flat_log()]
        ok = a == b and np.array_equal(res.labels.labels, single.labels.labels)
        with open(out, "w") as f:
            json.dump({"ok": bool(ok), "records": len(a), "world": dist.get_world_size()}, f)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
