#!/bin/bash
# pass C check (parity tests reaching k_zpass + headline bench), then the kernel-time breakdown
# of the cfg4 port solve (ncu launch list of ~3000 solve kernels after warm-up)
TAG=${1:-kv}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_extents.py tests/test_gpu_matvec.py tests/test_gpu_tucker.py -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --no-cpu --no-plans --no-cufft --no-solve --steps 20 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_$TAG.json'))
print(d['value'], d['ms_per_step'], d['roofline']['passes_ms_per_step'], d['roofline']['passes_frac'], d['roofline']['whole_matvec'], d['clocks'])"
KR='regex:k_spmvV|k_jacobiV|k_jacobi2V|k_residV|k_restrictG|k_prolongV|k_denseV|k_ddot|k_axpyV|k_xpbyV|k_fcg|k_kc_|k_pre_|k_zero|k_cdots|k_cupdate|k_csub|k_cscale|k_to_c64|k_row|k_y|k_z|k_p3|k_sys'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KR" --launch-skip 20000 --launch-count 3000 --csv \
   --log-file gpurun_out/solve_launches_$TAG.csv python scripts/solve_profile.py cfg4 > gpurun_out/solve_ncu_$TAG.log 2>&1
echo "ncu rc=$?"
