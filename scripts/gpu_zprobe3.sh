mkdir -p gpurun_out
TAG=${1:-q}
timeout 900 python -m pytest tests/test_gpu_tucker.py tests/test_gpu_matvec.py -x -q -k "ztma or tucker" > gpurun_out/zt_pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/zt_pytest_$TAG.log
timeout 600 python scripts/sweep.py --min-kz 64 > gpurun_out/zs_$TAG.log 2>&1; echo "sweep rc=$?"; cat gpurun_out/zs_$TAG.log | tail -4
