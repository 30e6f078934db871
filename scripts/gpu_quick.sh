#!/bin/bash
# quick check of a matvec change: parity tests that reach the changed kernels, then the
# headline bench (no extras)
TAG=${1:-q}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_extents.py tests/test_gpu_matvec.py -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --no-cpu --no-plans --no-cufft --no-solve --steps 20 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_$TAG.json'))
print(d['value'], d['ms_per_step'], d['roofline']['passes_ms_per_step'], d['roofline']['passes_frac'], d['roofline']['whole_matvec'])"
