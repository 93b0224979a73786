python - > gpurun_out/n4_probe.log 2>&1 <<'PY'
import torch, json
from paper_2512_15595_b200 import bf
dev=torch.device('cuda:0')
n=1<<26
for mbytes in (32<<20, 1<<30):
    buf=torch.zeros(mbytes,dtype=torch.uint8,device=dev)
    for B in (64,128,256,512,1024):
        b=mbytes*8//B
        e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
        res={}
        for name,fn in (("red_lsu", lambda: bf.bf_probe_rng(buf,b,B,1,max(1,B//64),n)),("red_bulk", lambda: bf.bf_probe_rng(buf,b,B,2,1,n)),("hybrid", lambda: bf.bf_probe_rng(buf,b,B,3,1,n)),("read", lambda: bf.bf_probe_rng(buf,b,B,0,1,n))):
            fn(); torch.cuda.synchronize(); best=1e9
            for _ in range(5):
                e0.record(); fn(); e1.record(); torch.cuda.synchronize(); best=min(best,e0.elapsed_time(e1))
            res[name]=round(n/best/1e6,2)
        print(json.dumps({"bytes":mbytes,"B":B,**res}), flush=True)
    # correctness of the bulk OR: all ones pattern appears
    print("nonzero bytes", int((buf!=0).sum()))
PY
