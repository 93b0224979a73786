# Inputs of tools/results_table.py: parity junit + iso-FPR sweep on the current kernels.
mkdir -p gpurun_out
TAG=${TAG:-res}
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu --junitxml=gpurun_out/junit_parity_$TAG.xml > gpurun_out/pytest_parity_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_parity_$TAG.log
rm -f gpurun_out/sweep_c2iso_$TAG.jsonl
timeout 1500 python tools/sweep.py --set c2iso --out gpurun_out/sweep_c2iso_$TAG.jsonl > gpurun_out/sweep_c2iso_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/sweep_c2iso_$TAG.log
