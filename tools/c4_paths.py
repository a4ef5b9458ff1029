import sys
import torch
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import paper_2106_12942_b200 as rh
from bench import make_cube
host = torch.empty((224, 2048, 2048), dtype=torch.float32, pin_memory=True)
make_cube("c4", out=host.numpy())
params = rh.RhsegParams(rh.HsegParams(0.21, 16), 7, 16)
ex = rh.B200Executor(device=0)
mode = sys.argv[1]
if mode == "host":
    img = rh.HyperImage(2048, 2048, 224, host.numpy())
    for i in range(int(sys.argv[2]) if len(sys.argv) > 2 else 3):
        r = ex.execute(img, params); print("host run", i, len(r.section_logs), flush=True)
else:
    cube = host.cuda()
    for i in range(int(sys.argv[2]) if len(sys.argv) > 2 else 3):
        ctx = ex.execute_device(cube.data_ptr(), 2048, 224, params); torch.cuda.synchronize(); print("dev run", i, flush=True)
