import torch, sys
sys.path.insert(0, '.')
from paper_2512_15595_b200 import bf
dev = torch.device('cuda:0')
m, n = 1 << 36, 1 << 31
keys = torch.empty(n, dtype=torch.int64, device=dev)
bf.bf_keygen(keys, n, 0)
f = bf.Filter(m, 8, 256, 64, "SBF")
f.add(keys)
out = torch.empty((n + 31) // 32, dtype=torch.int32, device=dev)
for mode in (bf.BF_CONTAINS_BINNED, bf.BF_CONTAINS_DIRECT, bf.BF_CONTAINS_BINNED):
    f.set_contains_mode(mode)
    f.contains(keys, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); f.contains(keys, out); e1.record(); torch.cuda.synchronize()
    print(mode, f.contains_mode(), round(n / (e0.elapsed_time(e1) * 1e-3) / 1e9, 2), 'Gkeys/s', flush=True)
