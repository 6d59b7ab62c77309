timeout 900 python -m pytest tests/test_gpu_split_fused.py tests/test_gpu_parity.py tests/test_gpu_zgemm.py -q -x 2>&1 | tail -2
for h in 0 1; do for b in 16 4 2; do
OZIMMU_SPLIT_HINTS=$h OZIMMU_SPLIT_BPS=$b python tools/split_bench.py --sizes 16384,2048 | grep contig | sed "s/^/hints$h bps$b /"
done; done
for h in 0 1; do for b in 0 3 2; do
OZIMMU_SPLIT_HINTS=$h OZIMMU_SPLIT_FUSED=1 OZIMMU_SPLIT_FUSED_BPS=$b python tools/split_bench.py --sizes 16384 | sed "s/^/fused hints$h bps$b /"
done; done
for b in 16 4; do
OZIMMU_SPLIT_BPS=$b timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_split_contig -s 3 -c 1 python tools/split_bench.py --sizes 16384 --it 3 2>&1 | grep -E "duration|dram__|lts__" | sed "s/^/ncu hints1 bps$b /"
done
OZIMMU_SPLIT_FUSED=1 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_split_fused -s 2 -c 2 python tools/split_bench.py --sizes 16384 --it 3 2>&1 | grep -E "duration|dram__|lts__" | sed "s/^/ncu fused /"
