mkdir -p gpurun_out
TAG=${1:-q}
timeout 900 python -m pytest tests/test_gpu_matvec.py -x -q -k "ztma or pruned" > gpurun_out/zt_pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/zt_pytest_$TAG.log
for shp in "64 64 64 16" "128 128 128 8" "256 256 256 2" "512 512 64 4" "1024 1024 64 2"; do
  echo "== $shp"; timeout 300 python scripts/zprobe.py $shp 2>&1 | tail -1
  SVH_ZQ=4 timeout 300 python scripts/zprobe.py $shp 2>&1 | tail -1
done
