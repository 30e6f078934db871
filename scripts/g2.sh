mkdir -p gpurun_out
./scripts/micro/segbw > gpurun_out/segbw.txt 2>&1; cat gpurun_out/segbw.txt
CMD="python bench.py --steps 1 --warmup 1 --no-cpu --no-solve --no-cufft --nrhs 4"
timeout 300 $CMD > gpurun_out/plain2.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_row|k_col|k_freq" -s 5 -c 5 -o gpurun_out/prof_p5 $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"; tail -3 gpurun_out/ncu_full.log
