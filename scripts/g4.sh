mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_matvec.py tests/test_gpu_tucker.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu --no-solve --no-cufft > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
