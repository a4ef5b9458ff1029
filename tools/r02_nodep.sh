#!/bin/bash
# APO non-adjacent-only rescans with D loads independent of the adjacency words (RHSEG_N_NODEP): A/B + parity.
O=gpurun_out/r02/nodep
mkdir -p $O
timeout 900 python tools/ab_variants.py c4 prod nodep prod nodep > $O/ab_c4.txt 2>&1; echo "ab c4 rc=$?"
timeout 600 python tools/ab_variants.py c3b prod nodep > $O/ab_c3b.txt 2>&1; echo "ab c3b rc=$?"
RHSEG_LIB_PATH=$PWD/paper_2106_12942_b200/_lib/variants/lib_nodep.so timeout 1500 python -m pytest tests/test_gpu_full_parity.py -x -q > $O/pytest_full.log 2>&1; echo "full parity rc=$?"
