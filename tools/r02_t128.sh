#!/bin/bash
O=gpurun_out/r02/t128
mkdir -p $O
RHSEG_LIB_PATH=$PWD/paper_2106_12942_b200/_lib/variants/lib_t128.so timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_run.py > $O/memcheck.txt 2>&1; echo "memcheck rc=$?"
timeout 600 python tools/ab_variants.py c3b prod t128 > $O/ab_c3b.txt 2>&1; echo "ab rc=$?"
