TAG=${1:-r02g}
mkdir -p gpurun_out
OZIMMU_STATS=1 C5_DS=8 C5_SS=8 C5_IT=1 timeout 300 python tools/c5_sweep.py > gpurun_out/${TAG}_c5stats.txt 2>&1
tail -5 gpurun_out/${TAG}_c5stats.txt
C5_DS=8 C5_SS=8 C5_IT=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_oz_gemm -s 3 -c 1 -o gpurun_out/prof_c5d8_${TAG} python tools/c5_sweep.py > gpurun_out/ncu_c5d8_${TAG}.log 2>&1
echo ncu rc=$?
