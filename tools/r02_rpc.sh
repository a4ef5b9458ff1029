#!/bin/bash
O=gpurun_out/r02/rpc
mkdir -p $O
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; rc=$?; echo "smoke rc=$rc"
[ $rc -ne 0 ] && exit 1
timeout 900 python tools/ab_variants.py c4 prod norpc prod norpc > $O/ab_c4.txt 2>&1; echo "ab rc=$?"
RHSEG_PROFILE=1 timeout 100 python tools/profile_loop.py c4 > $O/profile.txt 2>&1; echo "profile rc=$?"
timeout 600 python -m pytest tests/test_gpu_full_parity.py -x -q > $O/pytest_full.log 2>&1; echo "full parity rc=$?"
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "gpu suite rc=$?"
