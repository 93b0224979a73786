# GPU test suite + smoke + default bench + configs[4] per-rank bench.
mkdir -p gpurun_out
TAG=${TAG:-suite}
timeout 1800 python -m pytest tests -q -m gpu -x --durations=8 > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_$TAG.log
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c5_$TAG.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_c5_$TAG.log
