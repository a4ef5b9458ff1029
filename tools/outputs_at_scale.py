"""Time the host side of a C4 run: result collection + native output files."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_12942_b200 as rh  # noqa: E402
from bench import make_cube  # noqa: E402
from paper_2106_12942_b200 import outputs  # noqa: E402

samples = make_cube("c4")
img = rh.HyperImage(2048, 2048, 224, samples)
params = rh.RhsegParams(rh.HsegParams(0.21, 16), 7, 16)
ex = rh.B200Executor()
ex.execute(img, params)  # warm-up
t0 = time.perf_counter()
res = ex.execute(img, params)
t1 = time.perf_counter()
out = outputs.write_outputs(res, "/tmp/c4.pgm", "/tmp/c4.merges.jsonl")
t2 = time.perf_counter()
nrec = sum(len(r) for _, r in res.section_logs)
print(f"execute (device run + D2H + RhsegResult): {t1 - t0:.3f} s; native PGM + JSONL ({nrec} records, "
      f"{out['jsonl_bytes'] / 1e6:.0f} MB) + content hash: {t2 - t1:.3f} s; hash {out['content_hash']}")
