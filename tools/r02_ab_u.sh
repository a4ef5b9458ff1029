#!/bin/bash
O=gpurun_out/r02/ab_u
mkdir -p $O
timeout 900 python tools/ab_variants.py c4 prod u6 u8 u16 prod u8 > $O/ab_c4.txt 2>&1; echo "ab rc=$?"
