# GPU parity suite + default bench + configs[1] sweep (profiles/r1_c2_sweep_roofline.md input).
mkdir -p gpurun_out
TAG=${TAG:-cs}
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py --no-cpu > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_$TAG.log
rm -f gpurun_out/sweep_c2_$TAG.jsonl
timeout 2400 python tools/sweep.py --set c2 --out gpurun_out/sweep_c2_$TAG.jsonl > gpurun_out/sweep_c2_$TAG.log 2>&1; echo "sweep rc=$?" >> gpurun_out/sweep_c2_$TAG.log
