#!/bin/bash
# A/B: 8x4 interval init vs 4x4; 128-thread loop CTAs (3/SM) vs 256 (2/SM). Parity on the new default.
O=gpurun_out/r02/ab2
mkdir -p $O
timeout 900 python tools/ab_variants.py c4 prod no84 t128 prod no84 t128 > $O/ab_c4.txt 2>&1; echo "ab rc=$?"
timeout 600 python -m pytest tests/test_gpu_full_parity.py -x -q > $O/pytest_full.log 2>&1; echo "full parity rc=$?"
