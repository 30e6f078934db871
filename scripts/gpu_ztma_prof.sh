mkdir -p gpurun_out
TAG=${1:-q}
timeout 300 python scripts/zprobe.py 128 128 128 8 > gpurun_out/zq1.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_ztma2" -s 2 -c 1 -o gpurun_out/zt2a_$TAG python scripts/zprobe.py 128 128 128 8 > gpurun_out/zt2a_$TAG.log 2>&1; echo "ncu a rc=$?"
timeout 300 python scripts/zprobe.py 512 512 64 4 > gpurun_out/zq2.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_ztma2|k_ytma|k_row" -s 4 -c 4 -o gpurun_out/zt2b_$TAG python scripts/zprobe.py 1024 1024 64 2 > gpurun_out/zt2b_$TAG.log 2>&1; echo "ncu b rc=$?"
python scripts/ncu_summary.py gpurun_out/zt2a_$TAG.ncu-rep gpurun_out/ncu_ztma2_128cube_$TAG.md > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/zt2b_$TAG.ncu-rep gpurun_out/ncu_1024x1024x64_$TAG.md > /dev/null 2>&1
rm -f gpurun_out/zt2b_$TAG.ncu-rep
ls -la gpurun_out
