"""A/B timing of library build variants (paper_2106_12942_b200/_lib/variants/lib_*.so)
on one workload: the cube is generated once into /dev/shm, each variant is timed in
its own process (device time of full RHSEG runs, CUDA events on one stream).

    python tools/ab_variants.py c4 A B C ...
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CHILD = r"""
import sys, json, numpy as np, torch
sys.path.insert(0, ROOT)
import paper_2106_12942_b200 as rh
from bench import MEASURE_OF, WORKLOADS, _phase_ms_of
spec, crop, levels, w, t, st = WORKLOADS[NAME]
cube_h = np.load(CUBE, mmap_mode='r')
cube = torch.from_numpy(np.ascontiguousarray(cube_h)).cuda()
bands, edge, _ = cube.shape
ex = rh.B200Executor(device=0)
params = rh.RhsegParams(rh.HsegParams(w, t, MEASURE_OF.get(NAME, 'sqrt-bsmse')), levels, st)
s = torch.cuda.Stream()
res = []
with torch.cuda.stream(s):
    for it in range(6):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record(s)
        ctx = ex.execute_device(cube.data_ptr(), edge, bands, params, stream=s.cuda_stream)
        e1.record(s); torch.cuda.synchronize()
        if it >= 2: res.append((e0.elapsed_time(e1), _phase_ms_of(ctx).tolist()))
print(json.dumps({"ms": float(np.median([r[0] for r in res])), "phases": res[-1][1]}))
"""


def main():
    name = sys.argv[1]
    variants = sys.argv[2:]
    from bench import make_cube
    import numpy as np

    cube = f"/dev/shm/rhseg_{name}.npy"
    if not os.path.exists(cube):
        np.save(cube, make_cube(name))
    for v in variants:
        lib = os.path.join(ROOT, "paper_2106_12942_b200", "_lib", "variants", f"lib_{v}.so") if v != "prod" else ""
        env = dict(os.environ, RHSEG_LIB_PATH=lib) if lib else dict(os.environ)
        code = CHILD.replace("ROOT", repr(ROOT)).replace("NAME", repr(name)).replace("CUBE", repr(cube))
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
        line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-400:]
        print(f"{v}: {line}", flush=True)


if __name__ == "__main__":
    main()
