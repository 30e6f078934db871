mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_matvec.py -x -q -k "ztma or pruned or max_extents or small" > gpurun_out/zt_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/zt_pytest.log
timeout 600 python scripts/sweep.py --min-kz 33 --out gpurun_out/sweep_ztma.md > gpurun_out/zt_sweep.log 2>&1; echo "sweep rc=$?"; cat gpurun_out/zt_sweep.log | tail -8
