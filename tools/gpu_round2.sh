mkdir -p gpurun_out
TAG=${TAG:-r1b}
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c2_$TAG.log 2>&1
timeout 900 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu --add-mode direct --no-e2e > gpurun_out/bench_c3_direct_$TAG.log 2>&1
timeout 900 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_c3_binned_$TAG.log 2>&1
