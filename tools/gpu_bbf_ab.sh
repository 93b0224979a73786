# parity + BBF rows (C2 geometry) after a kernel change
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
: > gpurun_out/bbf_ab.jsonl
for cfg in "BBF 256 64 8" "BBF 256 64 16" "BBF 256 32 8" "BBF 128 64 8" "SBF 256 64 8"; do
  set -- $cfg
  timeout 300 python bench.py --variant $1 --B $2 --S $3 --k $4 --steps 20 --warmup 5 --no-e2e --no-cpu --no-probe \
    | tail -1 >> gpurun_out/bbf_ab.jsonl
done
