mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_matvec.py tests/test_gpu_slab.py tests/test_gpu_tucker.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu --no-solve --no-cufft --steps 20 2> gpurun_out/bench.err | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), d['roofline']['passes_ms'], d['roofline']['whole_matvec']['frac'])"
