#!/bin/bash
O=gpurun_out/r02/thr
mkdir -p $O
timeout 1200 python tools/ab_variants.py c4 prod sp34 sp14 cmp4 cmp16 prod > $O/ab_c4.txt 2>&1; echo "ab rc=$?"
