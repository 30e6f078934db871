#!/bin/bash
# GPU AMG setup check: solve tests + config-scale tests, then time-to-L on cfg3 / cfg4
TAG=${1:-amg}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_solve.py tests/test_gpu_config_scale.py tests/test_gpu_schur_direct.py tests/test_gpu_multiproc.py tests/test_gpu_fp64.py -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_$TAG.log
timeout 1200 python scripts/solve_profile.py cfg3 cfg4 > gpurun_out/solve_$TAG.jsonl 2>&1; echo "solve rc=$?"; cat gpurun_out/solve_$TAG.jsonl
