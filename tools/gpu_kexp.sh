# Run every built experiment binary (tools/kexp/kexp_*) on the GPU; ARGS passed through.
mkdir -p gpurun_out
TAG=${TAG:-kx}
for b in tools/kexp/kexp_*; do
  echo "== $(basename $b)" >> gpurun_out/kexp_$TAG.log
  timeout 300 $b $ARGS >> gpurun_out/kexp_$TAG.log 2>&1
done
