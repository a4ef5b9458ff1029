#!/bin/bash
# Grid loop round 2 (smem live bits, batched rescans): parity, C1 timing over CTAs per
# section, per-phase profile; staged-rescan A/B of the APO loop on C4.
O=gpurun_out/r02/grid2
mkdir -p $O
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; rc=$?; echo "smoke rc=$rc"
[ $rc -ne 0 ] && exit 1
timeout 900 python -m pytest tests/test_gpu_grid.py -x -q -k "160 or extension or upper or b2 or forced" > $O/pytest_grid.log 2>&1; echo "grid tests rc=$?"
for g in 0 96 64 32 16; do
  RHSEG_GRID=1 RHSEG_GRID_CTAS=$g timeout 300 python tools/profile_loop.py --time c1 > $O/times_c1_grid_$g.jsonl 2>&1; echo "c1 grid G=$g rc=$?"
done
RHSEG_PROFILE=1 RHSEG_GRID=1 timeout 300 python tools/profile_loop.py c1 > $O/profile_c1_grid.txt 2>&1; echo "profile rc=$?"
timeout 1200 python tools/ab_variants.py c4 prod stg1 stg2 stg3 > $O/ab_c4.txt 2>&1; echo "ab rc=$?"
