mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_solve.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python scripts/solve_demo.py cfg2 inner_tol=1e-3 2>&1 | tail -1 | cut -c1-200
timeout 300 python scripts/solve_demo.py cfg3 inner_tol=1e-3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['case'], d['solve_s'], d['L_pH'], d['stats'])"
SVH_NO_PCG_GRAPH=1 timeout 300 python scripts/solve_demo.py cfg3 inner_tol=1e-3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nograph', d['case'], d['solve_s'], d['stats']['inner_iterations'])"
