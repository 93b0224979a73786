timeout 900 python -m pytest -x -q tests/test_gpu_parity.py > gpurun_out/pytest_parity_r2q.log 2>&1
bash tools/gpu.sh bench r2q
timeout 1200 python tools/sweep.py --set c2 --out gpurun_out/sweep_c2_r2q.jsonl > /dev/null 2> gpurun_out/sweep_c2_r2q.err
timeout 900 python tools/sweep.py --set c2iso --out gpurun_out/sweep_c2iso_r2q.jsonl > /dev/null 2> gpurun_out/sweep_c2iso_r2q.err
