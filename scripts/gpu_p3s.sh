#!/bin/bash
# P3s / f4 round: new GPU tests, the thin-grid plan comparison, ncu of the P3s kernels (cfg3)
# and of pass C on the headline grid.
TAG=${1:-p3s}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_p3s.py tests/test_gpu_schur_direct.py tests/test_gpu_multiproc.py -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_$TAG.log
timeout 600 python -c "
import json, bench
print(json.dumps(bench.thin_grid_plans(0)))
" > gpurun_out/plans_$TAG.json 2> gpurun_out/plans_$TAG.err; echo "plans rc=$?"; cat gpurun_out/plans_$TAG.json; tail -3 gpurun_out/plans_$TAG.err
CMD3="python bench.py --workload cfg3 --nrhs 2 --steps 2 --warmup 3 --no-cpu --no-solve --no-cufft --no-plans"
timeout 300 $CMD3 > gpurun_out/cfg3_$TAG.json 2>&1; echo "cfg3 rc=$?"; cat gpurun_out/cfg3_$TAG.json | head -c 1500
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_p3" -s 9 -c 3 \
    -o gpurun_out/prof_p3_$TAG $CMD3 > gpurun_out/ncu_p3_$TAG.log 2>&1; echo "ncu p3 rc=$?"
CMD5="python bench.py --steps 1 --warmup 3 --no-cpu --no-solve --no-cufft --no-plans"
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:k_zpass" -s 6 -c 1 \
    -o gpurun_out/prof_zpass_$TAG $CMD5 > gpurun_out/ncu_zpass_$TAG.log 2>&1; echo "ncu zpass rc=$?"
