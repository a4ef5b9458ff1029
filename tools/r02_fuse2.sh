#!/bin/bash
# APO offers fused into the row-a' interval pass (RHSEG_APO_FUSE_OFFERS=1 variant vs prod): A/B + parity of the variant.
O=gpurun_out/r02/fuse2
mkdir -p $O
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; rc=$?; echo "smoke rc=$rc"
[ $rc -ne 0 ] && exit 1
timeout 900 python tools/ab_variants.py c4 prod fuse prod fuse > $O/ab_c4.txt 2>&1; echo "ab c4 rc=$?"
timeout 600 python tools/ab_variants.py c3b prod fuse > $O/ab_c3b.txt 2>&1; echo "ab c3b rc=$?"
RHSEG_LIB_PATH=$PWD/paper_2106_12942_b200/_lib/variants/lib_fuse.so timeout 1500 python -m pytest tests/test_gpu_full_parity.py -x -q > $O/pytest_full_fuse.log 2>&1; echo "full parity (fuse) rc=$?"
