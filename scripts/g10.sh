mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_matvec.py tests/test_gpu_tucker.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
for m in "SVH_ZMAC=1 SVH_YTMA=1" "SVH_ZMAC=0 SVH_YTMA=1" "SVH_ZMAC=1 SVH_YTMA=0"; do
env $m timeout 600 python bench.py --no-cpu --no-solve --no-cufft --steps 10 2> gpurun_out/bench.err | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$m', round(d['ms_per_step'],3), d['roofline']['passes_ms'], d['roofline']['whole_matvec']['frac'])"
tail -2 gpurun_out/bench.err
done
