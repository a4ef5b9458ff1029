#!/bin/bash
# Round-2 baseline at HEAD: C4 bench line, per-phase loop profile, timings of every workload.
mkdir -p gpurun_out/r02
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02/smi.txt
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02/bench_c4_head.json 2> gpurun_out/r02/bench_c4_head.err
echo "bench rc=$?"
timeout 600 python tools/profile_loop.py --time c1 c2 c3 c3b c4 c5w0 c5w1 > gpurun_out/r02/times_head.jsonl 2>&1
echo "times rc=$?"
RHSEG_PROFILE=1 timeout 600 python tools/profile_loop.py c4 c5w0 c1 c5w1 > gpurun_out/r02/profile_head.txt 2>&1
echo "profile rc=$?"
