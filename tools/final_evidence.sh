# one round's evidence: GPU suite, smoke, ncu (launch list + full captures), bench lines,
# slicing / small-shape / ZGEMM-sweep probes.  usage: bash tools/final_evidence.sh TAG
TAG=${1:-r02x}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/final_tests_$TAG.log 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/final_smoke_$TAG.log 2>&1
bash tools/profile.sh $TAG > gpurun_out/profile_$TAG.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_c4_$TAG.log 2>&1
timeout 600 python bench.py --config C3 > gpurun_out/bench_c3_$TAG.log 2>&1
timeout 600 python bench.py --config C5 --no-cpu-baseline > gpurun_out/bench_c5_$TAG.log 2>&1
timeout 600 python bench.py --slices 0 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4auto_$TAG.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_$TAG.log 2>&1
timeout 300 python tools/split_bench.py --sizes 16384,8192,2048 > gpurun_out/split_$TAG.jsonl 2>&1
timeout 300 python tools/small_shapes.py > gpurun_out/small_$TAG.jsonl 2>&1
C5_SS=8,9,12 timeout 900 python tools/c5_sweep.py > gpurun_out/c5sweep_$TAG.jsonl 2>&1
