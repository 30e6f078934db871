mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_matvec.py tests/test_gpu_tucker.py tests/test_gpu_slab.py -x -q -k "ztma or pruned or slab" 2>&1 | tail -2
timeout 300 python scripts/zprobe.py 1024 1024 64 2 2>&1 | tail -1
timeout 300 python scripts/zprobe.py 512 512 64 4 2>&1 | tail -1
timeout 300 python scripts/zprobe.py 128 128 128 8 2>&1 | tail -1
