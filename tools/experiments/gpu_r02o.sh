for b in 2 4 16; do
OZIMMU_SPLIT_BPS=$b timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:k_split_contig -s 3 -c 1 python tools/split_bench.py --sizes 16384 --it 3 2>&1 | grep -E "k_split|duration|dram__|lts__|sm__thr" | sed "s/^/bps$b /"
done
