mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_matvec.py -x -q -k "max_extents or rejects" 2>&1 | tail -2
CMD="python bench.py --steps 3 --warmup 3 --no-cpu --no-solve --no-cufft"
SVH_NO_CLOCKS=1 timeout 300 $CMD > gpurun_out/plain45.log 2>&1 && \
SVH_NO_CLOCKS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_zmac2" -s 2 -c 1 -o gpurun_out/prof_v45 $CMD > gpurun_out/ncu45.log 2>&1
echo "ncu rc=$?"
