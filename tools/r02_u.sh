#!/bin/bash
# APO rescans after the dependency fixes: D loads in flight per lane (RHSEG_RESCAN_U 4/6/8) + parity of prod.
O=gpurun_out/r02/u
mkdir -p $O
timeout 900 python tools/ab_variants.py c4 prod u6 u8 prod > $O/ab_c4.txt 2>&1; echo "ab c4 rc=$?"
timeout 600 python tools/ab_variants.py c3b prod u6 u8 > $O/ab_c3b.txt 2>&1; echo "ab c3b rc=$?"
timeout 1500 python -m pytest tests/test_gpu_full_parity.py -x -q > $O/pytest_full.log 2>&1; echo "full parity rc=$?"
