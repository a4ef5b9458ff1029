"""Per-phase cycle profile of the merge loop (RHSEG_PROFILE=1 lines on stderr) and
plain device timings of full RHSEG runs, per workload.

    RHSEG_PROFILE=1 python tools/profile_loop.py c4 c5w0 ...   # profile lines
    python tools/profile_loop.py --time c4 c3b ...             # device ms + phases
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2106_12942_b200 as rh  # noqa: E402
from bench import MEASURE_OF, WORKLOADS, _phase_ms_of, make_cube  # noqa: E402


def main():
    args = sys.argv[1:]
    timing = "--time" in args
    cluster = int(os.environ.get("RHSEG_CLUSTER", "0"))  # forced CTAs per section (0 = auto)
    names = [a for a in args if not a.startswith("--")]
    for name in names:
        spec, crop, levels, w, t, st = WORKLOADS[name]
        cube = torch.from_numpy(np.ascontiguousarray(make_cube(name))).cuda()
        bands, edge, _ = cube.shape
        ex = rh.B200Executor(device=0, cluster=cluster)
        params = rh.RhsegParams(rh.HsegParams(w, t, MEASURE_OF.get(name, "sqrt-bsmse")), levels, st)
        s = torch.cuda.Stream()
        res = []
        reps = 5 if timing else 1
        with torch.cuda.stream(s):
            for it in range(reps):
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record(s)
                ctx = ex.execute_device(cube.data_ptr(), edge, bands, params, stream=s.cuda_stream)
                e1.record(s)
                torch.cuda.synchronize()
                res.append((e0.elapsed_time(e1), _phase_ms_of(ctx).tolist()))
        keep = res[2:] if len(res) > 2 else res
        print(json.dumps({"workload": name, "ms": float(np.median([r[0] for r in keep])),
                          "phases": keep[-1][1]}), flush=True)
        del cube
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
