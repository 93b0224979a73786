# Full-size parity (configs[2], configs[3]) + the configs[2] bench line.
mkdir -p gpurun_out
TAG=${TAG:-fs}
nproc > gpurun_out/nproc_$TAG.txt; free -g >> gpurun_out/nproc_$TAG.txt
timeout 1800 python -m pytest tests/test_gpu_fullsize.py -q -x --durations=5 > gpurun_out/pytest_fs_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_fs_$TAG.log
timeout 900 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_c3_$TAG.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_c3_$TAG.log
