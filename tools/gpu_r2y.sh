timeout 900 python -m pytest -x -q tests/test_gpu_probes.py > gpurun_out/pytest_probes_r2y.log 2>&1
for b in base ksm0 pf1 ksm0l2pf4; do KEXP_CPS=32 ./tools/kexp/kexp_$b > gpurun_out/kexp_${b}_def_r2y.jsonl 2>&1; KEXP_CPS=32 ./tools/kexp/kexp_$b csbf > gpurun_out/kexp_${b}_csbf_r2y.jsonl 2>&1; done
