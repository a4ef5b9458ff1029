import sys, time, subprocess, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2106_12942_b200 as rh
from bench import make_cube, _phase_ms_of, ClockSampler
host = torch.empty((224, 2048, 2048), dtype=torch.float32, pin_memory=True)
make_cube("c4", out=host.numpy())
cube = host.cuda()
params = rh.RhsegParams(rh.HsegParams(0.21, 16), 7, 16)
ex = rh.B200Executor(device=0)
def run(label, stream, sampler=False):
    ts = []
    cm = ClockSampler(0) if sampler else None
    if cm: cm.__enter__()
    for it in range(5):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        ctx = ex.execute_device(cube.data_ptr(), 2048, 224, params, stream=stream)
        torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    if cm: cm.__exit__(None, None, None)
    print(label, [round(x*1e3) for x in ts], "phases", np.round(_phase_ms_of(ctx), 1).tolist(), flush=True)
s = torch.cuda.Stream()
run("ctx-stream", None)
run("torch-stream", s.cuda_stream)
run("ctx-stream+sampler", None, True)
run("torch-stream+sampler", s.cuda_stream, True)
run("ctx-stream again", None)
