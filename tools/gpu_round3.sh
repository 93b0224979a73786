# full validation + measurement session
mkdir -p gpurun_out
TAG=${TAG:-r1c}
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 600 python bench.py > gpurun_out/bench_$TAG.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 > gpurun_out/bench_ref_$TAG.log 2>&1
timeout 900 python tools/sweep.py --set c2iso --out gpurun_out/sweep_c2iso_$TAG.jsonl > gpurun_out/sweep_c2iso_$TAG.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bulk_kernel -s 4 -c 2 -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-probe > gpurun_out/ncu_full_$TAG.log 2>&1
