#!/bin/bash
O=gpurun_out/r02/ncu_stitch
mkdir -p $O
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"stitch_kernel|leaf_init_kernel" -c 2 -f -o $O/stitch_c4 python tools/c4_paths.py dev 1 > $O/ncu.log 2>&1; echo "ncu rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_1run.csv python tools/c4_paths.py dev 1 > $O/l.log 2>&1; echo "launches rc=$?"
