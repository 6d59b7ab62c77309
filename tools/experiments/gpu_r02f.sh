TAG=${1:-r02f}
mkdir -p gpurun_out
for ws in 0 1; do for acc in 0 1; do
  if [ $ws = 1 ]; then export OZIMMU_NO_WAVE_SYNC=1; else unset OZIMMU_NO_WAVE_SYNC; fi
  OZIMMU_ACC2=$acc C5_DS=8,10 C5_SS=8,9 C5_IT=3 timeout 300 python tools/c5_sweep.py | sed "s/^/nows$ws acc$acc /"
done; done > gpurun_out/${TAG}_c5.txt 2>&1
unset OZIMMU_NO_WAVE_SYNC
cat gpurun_out/${TAG}_c5.txt
OZIMMU_NO_WAVE_SYNC=1 timeout 300 python tools/small_shapes.py --shapes 1024,2048,4096 | sed "s/^/nows /" > gpurun_out/${TAG}_small.txt 2>&1
cat gpurun_out/${TAG}_small.txt
