#!/bin/bash
# compute-sanitizer over the round-2 kernels (APO loop with the merge beside the rescans,
# w=0 adj loop on both CTA widths, staged exact sums, 8x4 init, grid-wide stitch).
O=gpurun_out/r02/sanitize
mkdir -p $O
for tool in racecheck synccheck memcheck; do
  extra=""; [ $tool = racecheck ] && extra="--racecheck-report all"
  timeout 1200 compute-sanitizer --tool $tool $extra --print-limit 50 python tools/sanitize_run.py > $O/$tool.txt 2>&1; echo "$tool rc=$?"
  RHSEG_ADJ_NT=128 timeout 1200 compute-sanitizer --tool $tool $extra --print-limit 50 python tools/sanitize_run.py > $O/${tool}_adj128.txt 2>&1; echo "$tool adj128 rc=$?"
done
