mkdir -p gpurun_out
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_red_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_red_lookup_miss.sum"
for R in 8 32; do
timeout 900 ncu $M --clock-control none --csv --log-file gpurun_out/launches_binned_1g_$R.csv python bench.py --config c3 --m-bits 8589934592 --n 268435456 --add-mode binned --range-mib $R --steps 1 --warmup 3 --no-cpu --no-e2e --no-probe > /dev/null 2>&1
done
