# GPU-box jobs (run under gpurun from the repo root):
#   bash tools/gpu.sh JOB [TAG] [extra args]
# JOB:
#   suite     pytest -m gpu (junit), smoke, default bench
#   bench     default bench line only (extra args go to bench.py)
#   launches  ncu launch list (gpu__time_duration per launch) of the default bench command
#   prof      ncu --set full of the bench's bulk kernels (extra args go to bench.py)
#   sanitize  compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_run.py
#   profbin   ncu --set full of the binned add's bin + apply kernels (configs[2], one 2^31-key batch)
#   profbc    ncu --set full of the binned contains' kernels (bin with slots, range lookup, unbin)
# Everything lands in gpurun_out/ with the TAG in its name.
set -u
JOB=${1:-suite}
TAG=${2:-r2}
shift 2 2>/dev/null || shift $#
mkdir -p gpurun_out
case "$JOB" in
suite)
  timeout 2400 python -m pytest tests -q -m gpu -x --durations=15 --junitxml=gpurun_out/junit_gpu_$TAG.xml \
    > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
  echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
  timeout 900 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_$TAG.log
  ;;
bench)
  timeout 1200 python bench.py "$@" > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_$TAG.log
  ;;
launches)
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu "$@" > gpurun_out/launches_$TAG.log 2>&1
  echo "ncu rc=$?" >> gpurun_out/launches_$TAG.log
  ;;
prof)
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:bulk_kernel -s 4 -c 2 \
    -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-probe --no-graph --no-hbm --no-fixed "$@" \
    > gpurun_out/prof_$TAG.log 2>&1
  echo "ncu rc=$?" >> gpurun_out/prof_$TAG.log
  ;;
profbin)
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"bin_range_kernel|apply_kernel" -c 2 \
    -o gpurun_out/profbin_$TAG python bench.py --config c3 --steps 1 --warmup 0 --no-e2e --no-cpu --no-probe --no-graph "$@" \
    > gpurun_out/profbin_$TAG.log 2>&1
  echo "ncu rc=$?" >> gpurun_out/profbin_$TAG.log
  ;;
profbc)
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"lookup_kernel|unbin_kernel" -c 2 \
    -o gpurun_out/profbc_$TAG python tools/binned_contains_prof.py > gpurun_out/profbc_$TAG.log 2>&1
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:bin_range_kernel -s 4 -c 1 \
    -o gpurun_out/profbcbin_$TAG python tools/binned_contains_prof.py >> gpurun_out/profbc_$TAG.log 2>&1
  echo "ncu rc=$?" >> gpurun_out/profbc_$TAG.log
  ;;
sanitize)
  for tool in memcheck racecheck synccheck; do
    timeout 2400 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py \
      > gpurun_out/sanitize_${tool}_$TAG.log 2>&1
    echo "rc=$?" >> gpurun_out/sanitize_${tool}_$TAG.log
  done
  ;;
*)
  echo "unknown job $JOB"; exit 2 ;;
esac
