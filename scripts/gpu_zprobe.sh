mkdir -p gpurun_out
TAG=${1:-z1}
timeout 900 python -m pytest tests/test_gpu_matvec.py -x -q -k "ztma or pruned" > gpurun_out/zt_pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/zt_pytest_$TAG.log
for q in 8; do
SVH_ZQ=$q timeout 600 python scripts/sweep.py --min-kz 33 --dense-only > gpurun_out/zs_${TAG}_q$q.log 2>&1; echo "sweep q=$q rc=$?"; head -4 gpurun_out/zs_${TAG}_q$q.log
done
timeout 300 python scripts/zprobe.py 128 8 > gpurun_out/zp_$TAG.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_ztma" -s 2 -c 1 -o gpurun_out/zprof_$TAG python scripts/zprobe.py 128 8 > gpurun_out/zncu_$TAG.log 2>&1
echo "ncu rc=$?"
