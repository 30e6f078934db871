mkdir -p gpurun_out
TAG=${1:-q}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 300 python scripts/zprobe.py 1024 1024 16 4 2>&1 | tail -1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_row|k_col|k_ytma" -s 5 -c 4 -o gpurun_out/p2048_$TAG python scripts/zprobe.py 1024 1024 16 4 > gpurun_out/p2048_$TAG.log 2>&1
echo "ncu rc=$?"
