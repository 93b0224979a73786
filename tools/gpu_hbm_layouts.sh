python - > gpurun_out/hbm_layouts.log 2>&1 <<'PY'
import torch, json, statistics
from paper_2512_15595_b200 import bf
dev=torch.device('cuda:0'); n=1<<28
keys=torch.empty(n,dtype=torch.int64,device=dev); bf.bf_keygen(keys,n,0)
out=torch.empty(n//32,dtype=torch.int32,device=dev)
e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
for m in (1<<33, 1<<36):
    for k in (16,):
        f=bf.Filter(m,k,256,64,"SBF"); f.add(keys); torch.cuda.synchronize()
        for th,ph in ((1,4),(2,2),(4,1)):
            for kpt in (1,2,4):
                try: f.set_layout(1,th,ph,kpt,0)
                except bf.BFError: continue
                ts=[]
                for r in range(4):
                    e0.record(); f.contains(keys,out); e1.record(); torch.cuda.synchronize()
                    if r: ts.append(e0.elapsed_time(e1))
                print(json.dumps({"m_gib":m/8/2**30,"k":k,"theta":th,"phi":ph,"kpt":kpt,"gkeys_s":round(n/statistics.median(ts)/1e6,2)}),flush=True)
        del f
PY
