# Final: whole GPU suite (junit), parity junit for the results table, smoke, bench lines.
mkdir -p gpurun_out
TAG=${TAG:-final}
timeout 1800 python -m pytest tests -q -m gpu --junitxml=gpurun_out/junit_gpu_$TAG.xml > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_$TAG.log
timeout 900 python bench.py --config c3 --steps 5 --no-cpu > gpurun_out/bench_c3_$TAG.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_c3_$TAG.log
