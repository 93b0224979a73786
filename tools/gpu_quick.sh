mkdir -p gpurun_out
TAG=${TAG:-x}
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_$TAG.log 2>&1
timeout 900 python tools/sweep.py --set c2 --out gpurun_out/sweep_c2_$TAG.jsonl > gpurun_out/sweep_c2_$TAG.log 2>&1
