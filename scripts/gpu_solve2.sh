#!/bin/bash
TAG=${1:-s2}
mkdir -p gpurun_out
timeout 900 python scripts/solve_profile.py cfg3 cfg4 > gpurun_out/solve_$TAG.log 2>&1; echo "solve rc=$?"; cat gpurun_out/solve_$TAG.log
timeout 900 python -m pytest tests/test_gpu_multiproc.py tests/test_gpu_solve.py tests/test_gpu_config_scale.py tests/test_gpu_schur_direct.py -q > gpurun_out/pytest_solve_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_solve_$TAG.log
