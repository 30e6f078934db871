SVH_ZMAC2=2 timeout 900 python -m pytest tests/test_gpu_matvec.py -x -q 2>&1 | tail -1
for m in 2 1; do
SVH_ZMAC2=$m timeout 600 python bench.py --no-cpu --no-solve --no-cufft 2> /dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('zmac2=$m', round(d['ms_per_step'],3), d['roofline']['passes_ms'], d['roofline']['frac'])"
done
