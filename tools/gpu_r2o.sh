timeout 900 python -m pytest -x -q tests/test_gpu_parity.py > gpurun_out/pytest_parity_r2o.log 2>&1
bash tools/gpu.sh bench r2o
