#!/bin/bash
# Round-2 batch: P3s / f4 / P2P tests, the thin-grid plan comparison, a cfg3 bench line (auto
# plan), ncu of the P3s kernels, time-to-L with AMG-PCG vs the sparse-direct Schur solve
# (cfg3, cfg4), and the f3 bend refinement study.
TAG=${1:-r02b}
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_p3s.py tests/test_gpu_schur_direct.py tests/test_gpu_multiproc.py -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/pytest_$TAG.log
timeout 600 python -c "
import json, bench
print(json.dumps(bench.thin_grid_plans(0)))
" > gpurun_out/plans_$TAG.json 2> gpurun_out/plans_$TAG.err; echo "plans rc=$?"; cat gpurun_out/plans_$TAG.json; tail -3 gpurun_out/plans_$TAG.err
CMD3="python bench.py --workload cfg3 --nrhs 2 --steps 20 --warmup 3 --no-cpu --no-solve --no-cufft --no-plans"
timeout 300 $CMD3 > gpurun_out/cfg3_$TAG.json 2>&1; echo "cfg3 rc=$?"; head -c 2500 gpurun_out/cfg3_$TAG.json; echo
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_p3" -s 12 -c 3 \
    -o gpurun_out/prof_p3_$TAG $CMD3 > gpurun_out/ncu_p3_$TAG.log 2>&1; echo "ncu p3 rc=$?"
for S in 0 1; do
  timeout 900 python scripts/solve_profile.py cfg3 cfg4 --schur $S > gpurun_out/solve_s${S}_$TAG.log 2>&1; echo "solve schur=$S rc=$?"
  cat gpurun_out/solve_s${S}_$TAG.log | tail -4
done
timeout 1200 python scripts/bend_refinement.py --out gpurun_out/bend_refinement_$TAG.md > gpurun_out/bend_$TAG.log 2>&1; echo "bend rc=$?"
tail -20 gpurun_out/bend_$TAG.log
