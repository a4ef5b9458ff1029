"""Device time of one workload for several forced CTAs-per-section values."""
import sys
import numpy as np
import torch
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_2106_12942_b200 as rh
from bench import WORKLOADS, MEASURE_OF, make_cube, _phase_ms_of

name = sys.argv[1]
spec, crop, levels, w, t, st = WORKLOADS[name]
cube = torch.from_numpy(np.ascontiguousarray(make_cube(name))).cuda()
bands, edge, _ = cube.shape
params = rh.RhsegParams(rh.HsegParams(w, t, MEASURE_OF.get(name, "sqrt-bsmse")), levels, st)
for C in [int(x) for x in sys.argv[2:]]:
    ex = rh.B200Executor(device=0, cluster=C)
    ts = []
    for it in range(4):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s = torch.cuda.current_stream()
        e0.record()
        ctx = ex.execute_device(cube.data_ptr(), edge, bands, params)
        e1.record()
        torch.cuda.synchronize()
        if it: ts.append(e0.elapsed_time(e1))
    print(name, "C=", C, "ms", round(float(np.median(ts)), 2), "phases", np.round(_phase_ms_of(ctx), 2).tolist(), flush=True)
