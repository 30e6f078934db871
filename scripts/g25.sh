timeout 900 python -m pytest tests/test_gpu_matvec.py -x -q 2>&1 | tail -1
for m in 1 0; do
SVH_ZPRE=$m timeout 600 python bench.py --no-cpu --no-solve --no-cufft --steps 10 2> /dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('zpre=$m', round(d['ms_per_step'],3), d['roofline']['passes_ms'])"
SVH_ZPRE=$m SVH_ZPROBE=2 timeout 600 python bench.py --no-cpu --no-solve --no-cufft --steps 10 2> /dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('zpre=$m probe2', round(d['ms_per_step'],3), d['roofline']['passes_ms'])"
done
