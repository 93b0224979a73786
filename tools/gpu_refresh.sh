# Re-run the configs[3] grid (HBM and L2), the paper's Table 1/2 grid and the
# optimisation ablation on the current kernels.
mkdir -p gpurun_out
TAG=${TAG:-rf}
for set in c4 c4l2 paper ablation; do
  rm -f gpurun_out/sweep_${set}_$TAG.jsonl
  extra=""
  [ "$set" = "paper" ] && extra="--n 268435456 --reps 3"
  timeout 2400 python tools/sweep.py --set $set $extra --out gpurun_out/sweep_${set}_$TAG.jsonl > gpurun_out/sweep_${set}_$TAG.log 2>&1
  echo "rc=$?" >> gpurun_out/sweep_${set}_$TAG.log
done
