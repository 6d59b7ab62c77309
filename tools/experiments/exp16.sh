for b in 2 3 4 6 8 16; do OZIMMU_SPLIT_BPS=$b timeout 300 python bench.py --steps 5 --no-e2e --no-cpu-baseline --no-cublas > gpurun_out/exp16_bps$b.log 2>&1; done
