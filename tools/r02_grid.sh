#!/bin/bash
# Grid loop (grid_loop.cu): parity against the oracle, C1 timing with RHSEG_GRID=1 vs the cluster loop.
O=gpurun_out/r02/grid
mkdir -p $O
free -g > $O/host_mem.txt; nproc >> $O/host_mem.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; rc=$?; echo "smoke rc=$rc"
[ $rc -ne 0 ] && exit 1
timeout 900 python -m pytest tests/test_gpu_grid.py -x -q -k "160 or extension or upper or b2 or forced" > $O/pytest_grid.log 2>&1; echo "grid tests rc=$?"
timeout 300 python tools/profile_loop.py --time c1 > $O/times_c1_cluster.jsonl 2>&1; echo "c1 cluster rc=$?"
RHSEG_GRID=1 timeout 300 python tools/profile_loop.py --time c1 > $O/times_c1_grid.jsonl 2>&1; echo "c1 grid rc=$?"
timeout 1200 python -m pytest tests/test_gpu_grid.py -x -q -k "256" > $O/pytest_grid256.log 2>&1; echo "grid 256 rc=$?"
