mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/sweep_c2_${TAG}.jsonl
timeout 2400 python tools/sweep.py --set c2 --out gpurun_out/sweep_c2_${TAG}.jsonl > /dev/null 2>&1
echo "sweep rc=$?" >> gpurun_out/pytest_gpu.log
