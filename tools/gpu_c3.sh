mkdir -p gpurun_out
TAG=${TAG:-c3}
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "graph" > gpurun_out/pytest_graph_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_graph_$TAG.log
timeout 900 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_c3_$TAG.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_c3_$TAG.log
timeout 900 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu --no-graph > gpurun_out/bench_c3ng_$TAG.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_c3ng_$TAG.log
