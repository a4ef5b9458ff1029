#!/bin/bash
# APO loop re-cut + w=0 loop: parity gate, timings (A/B against the first variants), phase profile.
mkdir -p gpurun_out/r02
O=gpurun_out/r02/apo2
mkdir -p $O
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; rc=$?; echo "smoke rc=$rc"
[ $rc -ne 0 ] && exit 1
timeout 100 python tools/profile_loop.py --time c4 > $O/times_c4.jsonl 2>&1; rc=$?; echo "times c4 rc=$rc"
[ $rc -ne 0 ] && exit 1
timeout 200 python tools/profile_loop.py --time c3b c5w1 c2 c5w0 > $O/times.jsonl 2>&1; echo "times rc=$?"
RHSEG_PROFILE=1 timeout 200 python tools/profile_loop.py c4 c5w0 > $O/profile.txt 2>&1; echo "profile rc=$?"
timeout 500 python -m pytest tests/test_gpu_full_parity.py -x -q > $O/pytest_full.log 2>&1; echo "full parity rc=$?"
timeout 500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dropin.py -x -q > $O/pytest_parity.log 2>&1; echo "parity rc=$?"
RHSEG_ADJ_V1=1 timeout 100 python tools/profile_loop.py --time c5w0 > $O/times_v1.jsonl 2>&1; echo "times v1 rc=$?"
