mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/sweep_c2_csbf.jsonl gpurun_out/sweep_c2_bbf.jsonl
timeout 900 python tools/sweep.py --set c2 --only-variant 4 --out gpurun_out/sweep_c2_csbf.jsonl > /dev/null 2>&1
timeout 900 python tools/sweep.py --set c2 --only-variant 1 --out gpurun_out/sweep_c2_bbf.jsonl > /dev/null 2>&1
