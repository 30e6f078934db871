mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-cpu --no-solve --no-cufft --nrhs 16"
timeout 300 $CMD > gpurun_out/plain8.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_ystage|k_freq" -s 3 -c 3 -o gpurun_out/prof_v8 $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"; tail -3 gpurun_out/ncu_full.log
