for b in base am4 cm4 bm4; do KEXP_CPS=32 ./tools/kexp/kexp_$b > gpurun_out/kexp_${b}_def_r2r.jsonl 2>&1; KEXP_CPS=32 ./tools/kexp/kexp_$b csbf > gpurun_out/kexp_${b}_csbf_r2r.jsonl 2>&1; done
