for b in base tma1 tma2; do KEXP_CPS=32 ./tools/kexp/kexp_$b > gpurun_out/kexp_${b}_def_r2i.jsonl 2>&1; done
timeout 900 python -m pytest -x -q tests/test_gpu_parity.py -k "binned or partitioned or cuda_graph or auto_add" > gpurun_out/pytest_bin_r2i.log 2>&1
timeout 900 python -m pytest -x -q tests/test_gpu_fullsize.py::test_configs2_full_size_sampled "tests/test_gpu_scale.py::test_configs3_every_schedule_full_size" >> gpurun_out/pytest_bin_r2i.log 2>&1
bash tools/gpu.sh bench r2i
timeout 1200 python tools/sweep.py --set c2 --out gpurun_out/sweep_c2_r2i.jsonl > /dev/null 2> gpurun_out/sweep_c2_r2i.err
