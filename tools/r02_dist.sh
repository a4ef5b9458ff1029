#!/bin/bash
# The N>1 bench leg on one GPU: 2 ranks sharing the device over gloo (the driver's SCALE
# run uses NCCL, one rank per GPU); checks the JSON line carries every key.
O=gpurun_out/r02/dist
mkdir -p $O
RHSEG_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --workload c3b > $O/bench_n2_c3b.json 2> $O/bench_n2.err; echo "n2 rc=$?"
RHSEG_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --steps 1 --warmup 3 --workload c3b > $O/bench_ref_n2.json 2> $O/bench_ref_n2.err; echo "ref n2 rc=$?"
