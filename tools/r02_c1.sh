#!/bin/bash
O=gpurun_out/r02/c1
mkdir -p $O
for c in 16 8 4; do RHSEG_CLUSTER=$c timeout 200 python tools/profile_loop.py --time c1 > $O/c1_C$c.jsonl 2>&1; echo "c1 C=$c rc=$?"; done
