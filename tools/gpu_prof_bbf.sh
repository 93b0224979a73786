# ncu --set full of the BBF kernels (C2 rows BBF 256/64 k8, BBF 256/32 k8, BBF 128/64 k8)
mkdir -p gpurun_out
for cfg in "256 64 8" "256 32 8" "128 64 8"; do
  set -- $cfg
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:bulk_kernel -s 2 -c 2 \
    -o gpurun_out/prof_bbf_$1_$2_$3 python bench.py --variant BBF --B $1 --S $2 --k $3 --steps 1 --warmup 3 \
    --no-e2e --no-cpu --no-probe --no-graph > gpurun_out/prof_bbf_$1_$2_$3.log 2>&1
done
