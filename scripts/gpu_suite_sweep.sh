mkdir -p gpurun_out
TAG=${1:-s}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 900 python scripts/sweep.py --out gpurun_out/sweep_cfg5_$TAG.md > gpurun_out/sweep_$TAG.log 2>&1; echo "sweep rc=$?"; cat gpurun_out/sweep_cfg5_$TAG.md
