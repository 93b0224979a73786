mkdir -p gpurun_out
for v in A B; do
  if [ $v = B ]; then export BF200_LIB=$PWD/paper_2512_15595_b200/libbf200_minb4.so; fi
  timeout 900 python tools/sweep.py --set c2 --out gpurun_out/sweep_c2_ab$v.jsonl > gpurun_out/sweep_ab$v.log 2>&1
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/bench_ab$v.log 2>&1
done
