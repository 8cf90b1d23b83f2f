#!/bin/bash
# One profiling session (run under gpurun): ncu --set full with source of the top kernels at C3
# and C4-8192, the launch list of the bench command, the bulk-reduce rate micro-benchmark and a
# 2-rank gloo run of the multi-GPU path. Usage: bash scripts/gpu_prof.sh TAG
TAG=${1:-r2}
O=gpurun_out
mkdir -p $O
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-sub"
timeout 300 python scripts/bulk_red_rate.py > $O/bulkred_$TAG.jsonl 2>&1
timeout 600 torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 \
  --dist-backend gloo --steps 3 --warmup 3 --no-e2e --config C2-c > $O/gloo2_$TAG.json 2> $O/gloo2_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C3_$TAG.csv \
  $B --config C3 > /dev/null 2>&1
for CFG in C3 C4-8192; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"fwd_kernel|bwd_" -c 4 \
    -o $O/prof_${CFG}_$TAG -f $B --config $CFG > $O/ncu_${CFG}_$TAG.log 2>&1
  tail -2 $O/ncu_${CFG}_$TAG.log
done
ls -la $O | tail -20
