#!/bin/bash
# Grid loop for levels of few big sections (RHSEG_GRID=2: R0 >= 512 and >= 8 SMs per section): C2 / C1 / C3b times.
O=gpurun_out/r02/grid2x
mkdir -p $O
timeout 300 python tools/profile_loop.py --time c2 c1 c5w1 > $O/times_base.jsonl 2>&1; echo "base rc=$?"
RHSEG_GRID=2 timeout 300 python tools/profile_loop.py --time c2 c1 c5w1 > $O/times_grid2.jsonl 2>&1; echo "grid2 rc=$?"
RHSEG_GRID=2 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "synthetic_golden" > $O/pytest_golden_grid2.log 2>&1; echo "golden grid2 rc=$?"
