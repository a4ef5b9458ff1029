#!/bin/bash
# Re-entry check of the restored HEAD: smoke, device time of every workload, GPU suite.
O=gpurun_out/r02/verify2
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; rc=$?; echo "smoke rc=$rc"
[ $rc -ne 0 ] && exit 1
timeout 300 python tools/profile_loop.py --time c1 c2 c3 c3b c4 c5w0 c5w1 > $O/times.jsonl 2>&1; echo "times rc=$?"
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "gpu suite rc=$?"
