#!/bin/bash
# One GPU session: tests, bench, ncu launch list, ncu --set full of our kernels.
# Usage (under gpurun): bash scripts/gpu_round.sh [config] [tag]
CFG=${1:-C3}
TAG=${2:-r1}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_$TAG.txt 2>&1
timeout 900 python bench.py --config $CFG --steps 10 --warmup 3 > gpurun_out/bench_${CFG}_$TAG.json 2> gpurun_out/bench_${CFG}_$TAG.err
tail -c 3000 gpurun_out/bench_${CFG}_$TAG.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${CFG}_$TAG.csv \
  python bench.py --config $CFG --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fwd_kernel|bwd_" -c 4 \
  -o gpurun_out/prof_${CFG}_$TAG -f python bench.py --config $CFG --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_${CFG}_$TAG.log 2>&1
tail -3 gpurun_out/ncu_${CFG}_$TAG.log
ls -la gpurun_out
