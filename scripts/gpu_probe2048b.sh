mkdir -p gpurun_out
TAG=${1:-q}
timeout 900 python -m pytest tests/test_gpu_matvec.py -x -q -k "y2048 or max_extents or pruned" > gpurun_out/zt_pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/zt_pytest_$TAG.log
for y in 0 1; do SVH_YTMA2048=$y timeout 300 python scripts/zprobe.py 1024 1024 16 4 2>&1 | tail -1; done
for y in 0 1; do SVH_YTMA2048=$y timeout 300 python scripts/zprobe.py 1024 1024 64 2 2>&1 | tail -1; done
