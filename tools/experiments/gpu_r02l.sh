B="python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-cublas"
for cfg in "2 1" "4 1" "2 2" "1 1"; do
  set -- $cfg
  OZIMMU_CLUSTER_N=$1 OZIMMU_CLUSTER_M=$2 timeout 600 $B 2>/dev/null | tail -1 | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print('cln=$1 clm=$2', round(d['value'],2), d['clocks'], round(d['roofline']['gemm_ms'],2))"
done
OZIMMU_CLUSTER_N=4 timeout 900 python -m pytest tests/test_gpu_cluster.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2
