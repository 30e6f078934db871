for m in 0 1 2; do
SVH_ZPROBE=$m timeout 600 python bench.py --no-cpu --no-solve --no-cufft --steps 10 2> /dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('probe=$m', round(d['ms_per_step'],3), d['roofline']['passes_ms'])"
done
