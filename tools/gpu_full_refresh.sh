# After a kernel change: parity (junit), smoke, bench, configs[1] sweep, paper grid.
mkdir -p gpurun_out
TAG=${TAG:-fr}
timeout 1800 python -m pytest tests -q -m gpu -x --junitxml=gpurun_out/junit_gpu_$TAG.xml > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_$TAG.log
rm -f gpurun_out/sweep_c2_$TAG.jsonl gpurun_out/sweep_paper_$TAG.jsonl
timeout 2400 python tools/sweep.py --set c2 --out gpurun_out/sweep_c2_$TAG.jsonl > gpurun_out/sweep_c2_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/sweep_c2_$TAG.log
timeout 1500 python tools/sweep.py --set paper --n 268435456 --reps 3 --out gpurun_out/sweep_paper_$TAG.jsonl > gpurun_out/sweep_paper_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/sweep_paper_$TAG.log
