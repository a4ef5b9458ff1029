"""Small RHSEG runs for compute-sanitizer (racecheck / memcheck / synccheck):
w > 0 and w = 0, one CTA per section and a 4-CTA cluster, every measure."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_12942_b200 as rh  # noqa: E402

img, _ = rh.gen_synthetic(32, 6, 4, 6, 3.0, 9)
for measure in ("sqrt-bsmse", "sam", "euclidean"):
    for w in (0.21, 0.0):
        for cluster in (0, 4):
            rh.rhseg_run(img, rh.RhsegParams(rh.HsegParams(w, 4, measure), 2, 9),
                         executor=rh.B200Executor(cluster=cluster))
print("sanitize runs done")
