mkdir -p gpurun_out
TAG=${1:-q}
timeout 900 python -m pytest tests/test_gpu_matvec.py tests/test_gpu_slab.py -x -q -k "y2048 or max_extents or pruned or slab" > gpurun_out/zt_pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/zt_pytest_$TAG.log
timeout 300 python scripts/zprobe.py 1024 1024 16 4 2>&1 | tail -1
timeout 300 python scripts/zprobe.py 1024 1024 64 2 2>&1 | tail -1
timeout 300 python scripts/zprobe.py 2048 3 2 4 2>&1 | tail -1
