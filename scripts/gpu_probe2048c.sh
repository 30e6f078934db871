mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_matvec.py -x -q -k "max_extents or y2048" 2>&1 | tail -2
timeout 300 python scripts/zprobe.py 1024 1024 16 4 2>&1 | tail -1
timeout 300 python scripts/zprobe.py 1024 1024 64 2 2>&1 | tail -1
