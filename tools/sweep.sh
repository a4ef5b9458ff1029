#!/bin/bash
# All BASELINE configs through bench.py (device + e2e), then sampled CPU baselines.
mkdir -p gpurun_out/sweep
for w in c1 c2 c3 c3b c4 c5w0 c5w1; do
  timeout 600 python bench.py --workload $w --steps 3 --no-cpu-baseline > gpurun_out/sweep/$w.json 2> gpurun_out/sweep/$w.err
  echo "$w rc=$?"
done
for w in c2 c3b c5w0 c5w1 c3; do
  timeout 300 python -c "
import sys, json; sys.path.insert(0, '.')
import bench
s = bench.make_cube('$w')
print(json.dumps(bench.cpu_sample('$w', s, seconds_hint=15.0)))" > gpurun_out/sweep/cpu_$w.json 2>&1
  echo "cpu $w rc=$?"
done
