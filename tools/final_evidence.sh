# one round's evidence: GPU suite, smoke, ncu (launch list + full captures), bench lines
TAG=${1:-r01d}
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/final_tests_$TAG.log 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/final_smoke_$TAG.log 2>&1
bash tools/profile.sh $TAG > gpurun_out/profile_$TAG.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_c4_$TAG.log 2>&1
timeout 600 python bench.py --config C3 > gpurun_out/bench_c3_$TAG.log 2>&1
timeout 600 python bench.py --config C5 --no-cpu-baseline > gpurun_out/bench_c5_$TAG.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_$TAG.log 2>&1
