mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_matvec.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
for m in "SVH_YQ=8" "SVH_YQ=4" "SVH_YQ=8 SVH_ZMAC=0"; do
env $m timeout 600 python bench.py --no-cpu --no-solve --no-cufft --steps 20 2> gpurun_out/bench.err | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$m', round(d['ms_per_step'],3), d['roofline']['passes_ms'], d['roofline']['whole_matvec']['frac'])"
tail -2 gpurun_out/bench.err
done
CMD="python bench.py --steps 1 --warmup 1 --no-cpu --no-solve --no-cufft --nrhs 16"
timeout 300 $CMD > gpurun_out/plain11.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_ytma|k_zmac|k_row" -s 5 -c 5 -o gpurun_out/prof_v11 $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"; tail -2 gpurun_out/ncu_full.log
