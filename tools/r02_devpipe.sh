#!/bin/bash
# Device-resident leaf level in concurrent chunks (RHSEG_DEV_PIPE=1) vs one batch: A/B on C4 / C3b / C5w1 + parity.
O=gpurun_out/r02/devpipe
mkdir -p $O
for w in c4 c3b c5w1; do
  timeout 600 python tools/ab_variants.py $w prod > $O/ab_${w}_base.txt 2>&1; echo "$w base rc=$?"
  RHSEG_DEV_PIPE=1 timeout 600 python tools/ab_variants.py $w prod > $O/ab_${w}_pipe.txt 2>&1; echo "$w pipe rc=$?"
done
RHSEG_DEV_PIPE=1 timeout 1500 python -m pytest tests/test_gpu_full_parity.py -x -q -k "every_section" > $O/pytest_full_pipe.log 2>&1; echo "parity pipe rc=$?"
