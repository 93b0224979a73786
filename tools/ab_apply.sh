# A/B of the binned add / contains phase-2 launch forms (per-range launches vs
# one all-ranges launch with per-range tickets): bash tools/ab_apply.sh
mkdir -p gpurun_out
BF200_LOOKUP_CPS=8 BF200_APPLY_CPS=8 BF200_APPLY_CHUNK=1 timeout 900 python -m pytest tests -q -m gpu -x -k "binned or routed or configs2" > gpurun_out/ab2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab2_tests.log
run() {  # tag, env...
  tag=$1; shift
  env "$@" timeout 600 python bench.py --config c3 --steps 5 --warmup 3 --no-e2e --no-cpu --no-probe > gpurun_out/ab2_$tag.log 2>&1
  grep '^{' gpurun_out/ab2_$tag.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$tag', d['value'], d.get('add_gkeys_s'), d.get('contains_gkeys_s'), d.get('kernel_ms'))" >> gpurun_out/ab2_summary.log 2>&1
}
run base X=0
run a8c1 BF200_APPLY_CPS=8 BF200_APPLY_CHUNK=1
run a8c2 BF200_APPLY_CPS=8 BF200_APPLY_CHUNK=2
run a4c1 BF200_APPLY_CPS=4 BF200_APPLY_CHUNK=1
run l8c8 BF200_LOOKUP_CPS=8 BF200_LOOKUP_CHUNK=8
run l8c2 BF200_LOOKUP_CPS=8 BF200_LOOKUP_CHUNK=2
run l4c8 BF200_LOOKUP_CPS=4 BF200_LOOKUP_CHUNK=8
run l16c8 BF200_LOOKUP_CPS=16 BF200_LOOKUP_CHUNK=8
run base2 X=0
