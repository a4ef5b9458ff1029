#!/bin/bash
# Last check of the committed build: smoke, device time of every workload, the C4 bench line, GPU suite.
O=gpurun_out/r02/final3
mkdir -p $O
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; rc=$?; echo "smoke rc=$rc"
[ $rc -ne 0 ] && exit 1
timeout 400 python tools/profile_loop.py --time c1 c2 c3 c3b c4 c5w0 c5w1 > $O/times.jsonl 2>&1; echo "times rc=$?"
timeout 900 python bench.py --steps 5 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err; echo "bench rc=$?"
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "gpu suite rc=$?"
