#!/bin/bash
# APO rescans on the high words of D (RHSEG_RESCAN_HI): A/B + per-phase profile + parity.
O=gpurun_out/r02/hi
mkdir -p $O
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; rc=$?; echo "smoke rc=$rc"
[ $rc -ne 0 ] && exit 1
timeout 900 python tools/ab_variants.py c4 prod nohi prod nohi > $O/ab_c4.txt 2>&1; echo "ab c4 rc=$?"
timeout 600 python tools/ab_variants.py c3b prod nohi > $O/ab_c3b.txt 2>&1; echo "ab c3b rc=$?"
RHSEG_PROFILE=1 timeout 120 python tools/profile_loop.py c4 > $O/profile.txt 2>&1; echo "profile rc=$?"
timeout 1500 python -m pytest tests/test_gpu_full_parity.py -x -q > $O/pytest_full.log 2>&1; echo "full parity rc=$?"
