timeout 900 python -m pytest tests -q -m gpu -x -k "hybrid or 2pow32" > gpurun_out/pytest_hybrid.log 2>&1
python - > gpurun_out/hybrid_perf.log 2>&1 <<'PY'
import torch, json, statistics
from paper_2512_15595_b200 import bf
dev=torch.device('cuda:0'); n=1<<26
keys=torch.empty(n,dtype=torch.int64,device=dev); bf.bf_keygen(keys,n,0)
e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
for (v,B,S,k,z) in [(3,256,64,8,0),(3,256,64,16,0),(3,256,32,8,0),(3,128,64,8,0),(3,512,64,16,0),(3,1024,64,16,0),(1,256,64,8,0),(4,256,32,8,2),(4,1024,64,16,4)]:
    for m in (1<<28, 1<<33):
        f=bf.Filter(m,k,B,S,v,z=z)
        res={}
        for mode,name in ((bf.BF_ADD_DIRECT,"direct"),(bf.BF_ADD_HYBRID,"hybrid")):
            try: f.set_add_mode(mode)
            except bf.BFError as ex: res[name]=str(ex)[:40]; continue
            ts=[]
            for r in range(6):
                f.clear(); e0.record(); f.add(keys); e1.record(); torch.cuda.synchronize()
                if r: ts.append(e0.elapsed_time(e1))
            res[name]=round(n/statistics.median(ts)/1e6,2)
        print(json.dumps({"v":v,"B":B,"S":S,"k":k,"z":z,"m_mib":m>>23,**res}),flush=True)
        del f
PY
