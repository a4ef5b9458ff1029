#!/bin/bash
# w=0 loop: thread-per-neighbour row a', CTA width A/B, parity.
O=gpurun_out/r02/adj
mkdir -p $O
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; rc=$?; echo "smoke rc=$rc"
[ $rc -ne 0 ] && exit 1
timeout 100 python tools/profile_loop.py --time c5w0 > $O/times_auto.jsonl 2>&1; echo "auto rc=$?"
RHSEG_ADJ_NT=256 timeout 100 python tools/profile_loop.py --time c5w0 > $O/times_256.jsonl 2>&1; echo "256 rc=$?"
RHSEG_PROFILE=1 timeout 100 python tools/profile_loop.py c5w0 > $O/profile.txt 2>&1; echo "profile rc=$?"
timeout 400 python -m pytest tests/test_gpu_full_parity.py -x -q -k "w0" > $O/pytest_full.log 2>&1; echo "full parity rc=$?"
timeout 500 python -m pytest tests/test_gpu_parity.py -x -q > $O/pytest_parity.log 2>&1; echo "parity rc=$?"
