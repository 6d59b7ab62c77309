V=paper_2306_11975_b200/variants
for lib in "" $V/libozimmu_minb5.so $V/libozimmu_minb6.so; do
OZIMMU_LIB=$lib OZIMMU_SPLIT_FUSED=1 python tools/split_bench.py --sizes 16384 | sed "s|^|fused [$lib] |"
done
