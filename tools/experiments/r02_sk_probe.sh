python -c "import __graft_entry__ as g; g.build()"
for sk in 0 1; do
  OZIMMU_SK=$sk OZIMMU_STATS=1 python tools/small_shapes.py --quick --shapes 1024 > gpurun_out/r02g_stats_sk$sk.txt 2>&1
done
OZIMMU_SK=1 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/r02g_sk_ncu.csv python tools/small_shapes.py --quick --shapes 1024 > /dev/null 2>&1
OZIMMU_SK=1 OZIMMU_CLUSTER=1 python tools/small_shapes.py --shapes 1024,2048 > gpurun_out/r02g_sk_cl1.txt 2>&1
