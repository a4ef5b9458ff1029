#!/bin/bash
O=gpurun_out/r02/ab_mb
mkdir -p $O
timeout 900 python tools/ab_variants.py c4 prod mb3 prod mb3 > $O/ab_c4.txt 2>&1; echo "ab rc=$?"
