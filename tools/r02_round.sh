#!/bin/bash
# Full GPU suite + C4 bench line + w=0 timings.
O=gpurun_out/r02/round
mkdir -p $O
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; rc=$?; echo "smoke rc=$rc"
[ $rc -ne 0 ] && exit 1
timeout 100 python tools/profile_loop.py --time c5w0 c5w1 c3b c2 c1 > $O/times.jsonl 2>&1; echo "times rc=$?"
RHSEG_PROFILE=1 timeout 100 python tools/profile_loop.py c5w0 > $O/profile_c5w0.txt 2>&1; echo "profile rc=$?"
timeout 900 python bench.py --steps 5 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err; echo "bench rc=$?"
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest gpu rc=$?"
