for b in base sma128 sma128k8 smak8; do KEXP_CPS=32 ./tools/kexp/kexp_$b bbf128 > gpurun_out/kexp_${b}_bbf_r2s.jsonl 2>&1; done
