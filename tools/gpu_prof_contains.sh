# source-level stall attribution of the SBF 256/64 contains kernel at k=16 and k=8
mkdir -p gpurun_out
for k in 16 8; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bulk_kernel -s 3 -c 1 \
  -o gpurun_out/prof_con_k$k python bench.py --k $k --steps 1 --warmup 3 --no-e2e --no-cpu --no-probe --no-graph \
  > gpurun_out/prof_con_k$k.log 2>&1
done
