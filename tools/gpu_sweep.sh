mkdir -p gpurun_out
TAG=${TAG:-r1}
timeout 900 python tools/sweep.py --set c2 --out gpurun_out/sweep_c2_$TAG.jsonl > gpurun_out/sweep_c2.log 2>&1; echo "c2 rc=$?" >> gpurun_out/sweep_c2.log
timeout 900 python tools/sweep.py --set c4l2 --reps 3 --out gpurun_out/sweep_c4l2_$TAG.jsonl > gpurun_out/sweep_c4l2.log 2>&1; echo "c4l2 rc=$?" >> gpurun_out/sweep_c4l2.log
timeout 1200 python tools/sweep.py --set c4 --reps 3 --out gpurun_out/sweep_c4_$TAG.jsonl > gpurun_out/sweep_c4.log 2>&1; echo "c4 rc=$?" >> gpurun_out/sweep_c4.log
