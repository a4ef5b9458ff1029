#!/bin/bash
# Final round-2 measurement of HEAD: device time of every workload, the C4 bench line (+ the
# reference arm), the ncu launch list of the bench command, DRAM bytes per heavy kernel, full
# ncu captures of the leaf-level APO loop, the interval init, the w=0 loop and the grid loop (C1).
O=gpurun_out/r02/final2
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; rc=$?; echo "smoke rc=$rc"
[ $rc -ne 0 ] && exit 1
timeout 400 python tools/profile_loop.py --time c1 c2 c3 c3b c4 c5w0 c5w1 > $O/times.jsonl 2>&1; echo "times rc=$?"
RHSEG_PROFILE=1 timeout 300 python tools/profile_loop.py c4 c1 c5w0 > $O/profile.txt 2>&1; echo "profile rc=$?"
timeout 900 python bench.py --steps 5 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_bench.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__inst_executed_pipe_fp64.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum --clock-control none --csv -k regex:"hseg_loop|hseg_adj|dinit_dense|dinit_iv84" -c 3 --log-file $O/traffic_c4.csv python tools/c4_paths.py dev 1 > $O/ncu_traffic.log 2>&1; echo "ncu traffic rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"hseg_loop_kernel" -c 1 -f -o $O/loop_c4 python tools/c4_paths.py dev 1 > $O/ncu_loop.log 2>&1; echo "ncu loop rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"dinit_iv84" -c 1 -f -o $O/dinit_c4 python tools/c4_paths.py dev 1 > $O/ncu_dinit.log 2>&1; echo "ncu dinit rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"hseg_grid" -c 1 -f -o $O/grid_c1 python tools/profile_loop.py c1 > $O/ncu_grid.log 2>&1; echo "ncu grid rc=$?"
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "gpu suite rc=$?"
