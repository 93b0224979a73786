# round-2 validation + tables on the final launch policy (waves)
bash tools/gpu.sh suite r2h
timeout 1200 python tools/sweep.py --set c2 --out gpurun_out/sweep_c2_r2h.jsonl > /dev/null 2> gpurun_out/sweep_c2_r2h.err
timeout 900 python tools/sweep.py --set c2iso --out gpurun_out/sweep_c2iso_r2h.jsonl > /dev/null 2> gpurun_out/sweep_c2iso_r2h.err
timeout 1500 python tools/c3_variants.py gpurun_out/c3_variants_r2h > gpurun_out/c3_variants_r2h.log 2>&1
timeout 1500 python tools/sweep.py --set c4 --out gpurun_out/sweep_c4_r2h.jsonl > /dev/null 2> gpurun_out/sweep_c4_r2h.err
timeout 900 python tools/sweep.py --set c4l2 --out gpurun_out/sweep_c4l2_r2h.jsonl > /dev/null 2> gpurun_out/sweep_c4l2_r2h.err
bash tools/gpu.sh sanitize r2h
