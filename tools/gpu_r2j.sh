for b in base ktc kta; do KEXP_CPS=32 ./tools/kexp/kexp_$b > gpurun_out/kexp_${b}_def_r2j.jsonl 2>&1; KEXP_CPS=32 ./tools/kexp/kexp_$b csbf > gpurun_out/kexp_${b}_csbf_r2j.jsonl 2>&1; done
timeout 900 python -m pytest -x -q tests/test_gpu_parity.py -k "binned or cuda_graph" > gpurun_out/pytest_bin_r2j.log 2>&1
bash tools/gpu.sh bench r2j --no-cpu --no-e2e --steps 20
