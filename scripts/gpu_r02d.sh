#!/bin/bash
TAG=${1:-r02d}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_extents.py tests/test_gpu_tucker.py -q -k "tucker or bench or blocked or cfg4" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --no-cpu --no-plans --no-cufft --steps 20 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; head -c 2200 gpurun_out/bench_$TAG.json; echo
KR='regex:k_spmvV|k_jacobi|k_residV|k_restrictG|k_prolongV|k_denseV|k_ddot|k_axpyV|k_xpbyV|k_fcg|k_kc_|k_pre_|k_zero'
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KR" --launch-skip 2000 --launch-count 1500 --csv \
   --log-file gpurun_out/solve4_launches_$TAG.csv python scripts/solve_profile.py cfg4 > gpurun_out/solve4_ncu_$TAG.log 2>&1
echo "ncu rc=$?"
