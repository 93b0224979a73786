mkdir -p gpurun_out
TAG=${TAG:-r1d}
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 1800 python tools/sweep.py --set paper --n 268435456 --reps 3 --out gpurun_out/sweep_paper_$TAG.jsonl > gpurun_out/sweep_paper_$TAG.log 2>&1
