timeout 900 python -m pytest tests -q -m gpu -k "cbf" > gpurun_out/pytest_cbf.log 2>&1
python - > gpurun_out/cbf_bench.log 2>&1 <<'PY'
import torch, json, statistics
from paper_2512_15595_b200 import bf
n=1<<28; dev=torch.device('cuda:0')
keys=torch.empty(n,dtype=torch.int64,device=dev); bf.bf_keygen(keys,n,0)
out=torch.empty(n//32,dtype=torch.int32,device=dev)
for m in (1<<28, 1<<32):
    f=bf.Filter(m,16,256,64,bf.BF_CBF)
    e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    for op in ('add','contains'):
        ts=[]
        for r in range(4):
            if op=='add': f.clear()
            e0.record(); (f.add(keys) if op=='add' else f.contains(keys,out)); e1.record(); torch.cuda.synchronize()
            if r: ts.append(e0.elapsed_time(e1))
        print(json.dumps({"m_bits":m,"op":op,"gkeys_s":n/statistics.median(ts)/1e6}))
PY
