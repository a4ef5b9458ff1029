#!/bin/bash
O=gpurun_out/r02/c2
mkdir -p $O
for c in 0 1 2; do RHSEG_CLUSTER=$c timeout 200 python tools/profile_loop.py --time c2 > $O/c2_C$c.jsonl 2>&1; echo "c2 C=$c rc=$?"; done
RHSEG_CLUSTER=1 RHSEG_PROFILE=1 timeout 100 python tools/profile_loop.py c2 > $O/profile_C1.txt 2>&1
RHSEG_PROFILE=1 timeout 100 python tools/profile_loop.py c2 c1 > $O/profile_auto.txt 2>&1
