#!/bin/bash
# compute-sanitizer over the late round-2 kernels: the APO loop with the gathered / dependency-free
# rescans and fused offers (default runs), and the grid loop (RHSEG_GRID=1 turns the 4-CTA-cluster
# sections of sanitize_run.py into grid sections; 4 CTAs per section keeps the spin-waits short).
O=gpurun_out/r02/sanitize2
mkdir -p $O
for tool in memcheck racecheck synccheck; do
  extra=""; [ $tool = racecheck ] && extra="--racecheck-report all"
  timeout 900 compute-sanitizer --tool $tool $extra --print-limit 50 python tools/sanitize_run.py > $O/$tool.txt 2>&1; echo "$tool rc=$?"
  RHSEG_GRID=1 RHSEG_GRID_CTAS=4 timeout 600 compute-sanitizer --tool $tool $extra --print-limit 50 python tools/sanitize_run.py > $O/${tool}_grid.txt 2>&1; echo "$tool grid rc=$?"
done
