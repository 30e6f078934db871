timeout 900 python -m pytest tests/test_gpu_solve.py -x -q 2>&1 | tail -2
timeout 300 python scripts/solve_demo.py cfg3 inner_tol=1e-3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); st=d['stats']; print(d['case'], round(d['solve_s'],3), d['L_pH'], st['total_iterations'], st['inner_iterations'], round(st['t_matvec_s'],3), round(st['t_precond_s'],3))"
