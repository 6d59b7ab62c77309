V=paper_2306_11975_b200/variants
for lib in $V/libozimmu_fminb4.so $V/libozimmu_fminb6.so; do
for b in -1 0; do
OZIMMU_LIB=$lib OZIMMU_SPLIT_FUSED=1 OZIMMU_SPLIT_FUSED_BPS=$b python tools/split_bench.py --sizes 16384,2048 | sed "s|^|$(basename $lib) bps$b |"
done; done
