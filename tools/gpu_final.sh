# Final validation on the current kernels: suite, sanitizers, tables, ncu evidence.
TAG=${1:-r2z}
bash tools/gpu.sh suite $TAG
[ "${SKIP_SAN:-0}" = 1 ] || bash tools/gpu.sh sanitize $TAG
timeout 1500 python tools/c3_variants.py gpurun_out/c3_variants_$TAG > gpurun_out/c3_variants_$TAG.log 2>&1
timeout 1500 python tools/sweep.py --set c4 --out gpurun_out/sweep_c4_$TAG.jsonl > /dev/null 2> gpurun_out/sweep_c4_$TAG.err
timeout 900 python tools/sweep.py --set c4l2 --out gpurun_out/sweep_c4l2_$TAG.jsonl > /dev/null 2> gpurun_out/sweep_c4l2_$TAG.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-hbm --no-fixed --no-probe > gpurun_out/launches_$TAG.log 2>&1
bash tools/gpu.sh prof $TAG
bash tools/gpu.sh profbin $TAG
