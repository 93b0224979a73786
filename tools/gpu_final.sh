# End-of-round validation on HEAD: GPU tests (junit), smoke, bench lines for configs[1] (default), [2], [4].
mkdir -p gpurun_out
TAG=${TAG:-final}
timeout 1800 python -m pytest tests -q -m gpu --junitxml=gpurun_out/junit_gpu_$TAG.xml > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_$TAG.log
timeout 900 python bench.py --config c3 --steps 5 --no-cpu > gpurun_out/bench_c3_$TAG.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_c3_$TAG.log
timeout 900 python bench.py --config c5 --steps 3 --no-cpu > gpurun_out/bench_c5_$TAG.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_c5_$TAG.log
timeout 900 python bench.py --impl reference --steps 3 > gpurun_out/bench_ref_$TAG.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_ref_$TAG.log
