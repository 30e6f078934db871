timeout 900 python -m pytest tests/test_gpu_matvec.py tests/test_gpu_tucker.py tests/test_gpu_slab.py -x -q 2>&1 | tail -2
timeout 600 python bench.py --no-cpu --no-solve --no-cufft --steps 20 2> /dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), d['value']/1e9, d['e2e'], d['roofline']['passes_ms'])"
