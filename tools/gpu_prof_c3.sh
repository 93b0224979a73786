mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x -k "concurrent or binned or partitioned" > gpurun_out/pytest_conc.log 2>&1
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__warps_issue_stalled_long_scoreboard_per_warp_active.pct,sm__warps_active.avg.pct_of_peak_sustained_active,l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed"
timeout 900 ncu $M --clock-control none --csv --log-file gpurun_out/launches_c3n28.csv python bench.py --config c3 --n 268435456 --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
