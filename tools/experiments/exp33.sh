for cfg in "TAG=default" "TAG=nosync OZIMMU_NO_WAVE_SYNC=1" "TAG=cl1 OZIMMU_CLUSTER=1" "TAG=cl1nosync OZIMMU_CLUSTER=1 OZIMMU_NO_WAVE_SYNC=1"; do
  env $cfg timeout 120 python tools/tiny_probe.py >> gpurun_out/exp33.log 2>&1
done
