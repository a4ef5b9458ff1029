#!/bin/bash
O=gpurun_out/r02/stitch
mkdir -p $O
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; rc=$?; echo "smoke rc=$rc"
[ $rc -ne 0 ] && exit 1
timeout 300 python tools/profile_loop.py --time c4 c2 c5w0 > $O/times.jsonl 2>&1; echo "times rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_1run.csv python tools/c4_paths.py dev 1 > $O/l.log 2>&1; echo "launches rc=$?"
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "gpu suite rc=$?"
