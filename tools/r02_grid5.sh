#!/bin/bash
# Grid loop: slot polling back-off A/B on C1 (RHSEG_GRID=1), ncu capture of the grid kernel, parity subset.
O=gpurun_out/r02/grid5
mkdir -p $O
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; rc=$?; echo "smoke rc=$rc"
[ $rc -ne 0 ] && exit 1
RHSEG_GRID=1 timeout 600 python tools/ab_variants.py c1 prod gt256 > $O/ab_c1_grid.txt 2>&1; echo "ab grid rc=$?"
RHSEG_PROFILE=1 RHSEG_GRID=1 timeout 300 python tools/profile_loop.py c1 > $O/profile_c1_grid.txt 2>&1; echo "profile rc=$?"
RHSEG_GRID=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"hseg_grid" -c 1 -f -o $O/grid_c1 python tools/profile_loop.py c1 > $O/ncu_grid.log 2>&1; echo "ncu rc=$?"
timeout 900 python -m pytest tests/test_gpu_grid.py -x -q -k "160 or forced" > $O/pytest_grid.log 2>&1; echo "grid tests rc=$?"
