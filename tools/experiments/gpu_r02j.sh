V=paper_2306_11975_b200/variants
for acc in 0 1; do
for lib in "" $V/libozimmu_nofma.so $V/libozimmu_nostore.so; do
  OZIMMU_LIB=$lib OZIMMU_ACC2=$acc OZIMMU_STATS=1 python tools/shape_stats.py 1048576 512 512 8 2 2>&1 | tail -2 | sed "s|^|[$lib acc$acc] |"
done; done
for lib in "" $V/libozimmu_nofma.so $V/libozimmu_nostore.so; do
  OZIMMU_LIB=$lib OZIMMU_STATS=1 python tools/shape_stats.py 1024 1024 1024 9 2 2>&1 | tail -2 | sed "s|^|[$lib] |"
done
