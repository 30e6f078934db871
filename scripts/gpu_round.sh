#!/bin/bash
# One gpurun call: GPU tests, the default bench line, the launch list (ncu
# gpu__time_duration per launch) and one --set full capture of the pass kernels.
# usage: bash scripts/gpu_round.sh <tag>
TAG=${1:-r}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
cat gpurun_out/bench_$TAG.json; tail -3 gpurun_out/bench_$TAG.err
CMD="python bench.py --steps 3 --warmup 3 --no-cpu --no-solve --no-cufft"
timeout 300 $CMD > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
echo "ncu launches rc=$?"
CMD2="python bench.py --steps 3 --warmup 3 --no-cpu --no-solve --no-cufft"
timeout 300 $CMD2 > gpurun_out/plain2_$TAG.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_row|k_ytma|k_zmac" -s 5 -c 5 -o gpurun_out/prof_$TAG $CMD2 > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu full rc=$?"
