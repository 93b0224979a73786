# configs[1] sweep + iso-FPR sweep + GPU parity junit on the final kernels (one run).
mkdir -p gpurun_out
TAG=${TAG:-sf}
rm -f gpurun_out/sweep_c2_$TAG.jsonl gpurun_out/sweep_c2iso_$TAG.jsonl
timeout 2400 python tools/sweep.py --set c2 --out gpurun_out/sweep_c2_$TAG.jsonl > gpurun_out/sweep_c2_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/sweep_c2_$TAG.log
timeout 1800 python tools/sweep.py --set c2iso --out gpurun_out/sweep_c2iso_$TAG.jsonl > gpurun_out/sweep_c2iso_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/sweep_c2iso_$TAG.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu --junitxml=gpurun_out/junit_parity_$TAG.xml > gpurun_out/pytest_parity_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_parity_$TAG.log
