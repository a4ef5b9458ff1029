#!/bin/bash
# ncu --set full (source counters) of the re-cut loops and the round-1 APO loop, C3b / C5w0 leaf levels.
O=gpurun_out/r02/ncu
mkdir -p $O
timeout 600 ncu --set full --import-source on --clock-control none -k regex:hseg_apo_kernel -c 1 -f -o $O/apo_v2_c3b python tools/profile_loop.py c3b > $O/apo_v2.log 2>&1; echo "apo v2 rc=$?"
RHSEG_APO_V1=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:hseg_loop_kernel -c 1 -f -o $O/apo_v1_c3b python tools/profile_loop.py c3b > $O/apo_v1.log 2>&1; echo "apo v1 rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:hseg_adj_kernel -c 1 -f -o $O/adj_c5w0 python tools/profile_loop.py c5w0 > $O/adj.log 2>&1; echo "adj rc=$?"
