#!/bin/bash
# Kernel-time breakdown of the port solve (PCG + K-cycle AMG inside FGMRES) on cfg3: the ncu
# launch list of the solve kernels after warm-up (per-launch gpu__time_duration).
TAG=${1:-solve}
mkdir -p gpurun_out
KR='regex:k_spmvV|k_jacobiV|k_residV|k_restrictG|k_prolongV|k_denseV|k_ddot|k_axpyV|k_xpbyV|k_fcg|k_kc_|k_pre_|k_zero|k_cdots|k_cupdate|k_csub|k_cscale|k_to_c64|k_row|k_y|k_z|k_p3'
timeout 600 python scripts/solve_profile.py cfg3 > gpurun_out/solve_plain_$TAG.log 2>&1; echo "plain rc=$?"; cat gpurun_out/solve_plain_$TAG.log
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KR" --launch-skip 3000 --launch-count 6000 --csv \
   --log-file gpurun_out/solve_launches_$TAG.csv python scripts/solve_profile.py cfg3 > gpurun_out/solve_ncu_$TAG.log 2>&1
echo "ncu rc=$?"
timeout 900 python scripts/solve_profile.py cfg4 > gpurun_out/solve_cfg4_$TAG.log 2>&1; echo "cfg4 rc=$?"; cat gpurun_out/solve_cfg4_$TAG.log
timeout 600 python -m pytest tests/test_gpu_multiproc.py tests/test_gpu_solve.py tests/test_gpu_config_scale.py -q > gpurun_out/pytest_solve_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_solve_$TAG.log
