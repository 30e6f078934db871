mkdir -p gpurun_out
TAG=${1:-q}
SVH_ZMAC2=3 SVH_Z64=2 timeout 900 python -m pytest tests/test_gpu_matvec.py tests/test_gpu_tucker.py -x -q -k "ztma or small or pruned or config" > gpurun_out/zt_pytest_$TAG.log 2>&1; echo "pytest (opt-in) rc=$?"; tail -3 gpurun_out/zt_pytest_$TAG.log
for v in 1 3; do SVH_ZMAC2=$v timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu --no-solve --no-cufft > gpurun_out/zb_${TAG}_$v.json 2>/dev/null; echo "bench zmac2=$v rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/zb_${TAG}_$v.json')); print(d['ms_per_step'], d['roofline']['passes_ms'])"; done
for shp in "256 256 32 8" "512 512 32 4"; do for z in 0 2; do echo "== $shp z64=$z"; SVH_Z64=$z timeout 300 python scripts/zprobe.py $shp 2>&1 | tail -1; done; done
