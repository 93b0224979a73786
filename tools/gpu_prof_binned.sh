mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --csv --log-file gpurun_out/launches_binned.csv python bench.py --config c3 --n 268435456 --add-mode binned --steps 1 --warmup 3 --no-cpu --no-e2e --no-probe > gpurun_out/ncu_binned.log 2>&1
timeout 900 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu --no-e2e --add-mode binned > gpurun_out/bench_c3_binned.log 2>&1
timeout 900 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu --no-e2e --add-mode direct > gpurun_out/bench_c3_direct.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/bench_c2.log 2>&1
