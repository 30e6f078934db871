mkdir -p gpurun_out
CMD="python scripts/solve_demo.py cfg3 inner_tol=1e-3"
timeout 300 $CMD > gpurun_out/solve_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 1500 --csv --log-file gpurun_out/solve_launches.csv $CMD > gpurun_out/ncu_solve.log 2>&1
echo "rc=$?"
