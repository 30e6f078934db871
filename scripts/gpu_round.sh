#!/bin/bash
# One gpurun call: GPU tests, the default bench line, the launch list of the pass kernels
# (ncu gpu__time_duration per launch, timed region only) and one --set full capture of each
# pass kernel of the headline workload.
# usage: bash scripts/gpu_round.sh <tag>
TAG=${1:-r}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
cat gpurun_out/bench_$TAG.json; tail -3 gpurun_out/bench_$TAG.err
CMD="python bench.py --steps 2 --warmup 3 --no-cpu --no-solve --no-cufft --no-plans"
KR='regex:k_row|k_y|k_z|k_p3|k_freq|k_col'
timeout 300 $CMD > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KR" --csv \
    --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
echo "ncu launches rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k "$KR" -s 10 -c 5 \
    -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu full rc=$?"
