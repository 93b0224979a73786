mkdir -p gpurun_out
TAG=${TAG:-r1}
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > gpurun_out/sanitize_${tool}_$TAG.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_${tool}_$TAG.log
done
