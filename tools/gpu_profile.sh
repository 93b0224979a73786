# Profiling session for profiles/: ncu launch list of the default bench command,
# one --set full capture of the headline add + contains kernels, the bench line.
mkdir -p gpurun_out
TAG=${TAG:-prof}
timeout 900 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_$TAG.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/launches_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bulk_kernel -s 4 -c 2 -o gpurun_out/prof_$TAG \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-probe --no-graph > gpurun_out/ncu_full_$TAG.log 2>&1
