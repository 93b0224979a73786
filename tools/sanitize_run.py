"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck): every kernel family once, on small inputs, checked against the
oracle.  Usage: compute-sanitizer --tool memcheck python tools/sanitize_run.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from oracle.bfo import OracleFilter  # noqa: E402
from paper_2512_15595_b200 import bf  # noqa: E402

dev = torch.device("cuda:0")
keys = synth.keys(0, 10_003)
q = np.concatenate([keys[:3000], synth.negatives(3001)])
kd = torch.from_numpy(keys.view(np.int64)).to(dev)
qd = torch.from_numpy(q.view(np.int64)).to(dev)
ok = True
for v, B, S, k, z, mode in [(3, 256, 64, 8, 0, bf.BF_ADD_DIRECT), (3, 256, 64, 8, 0, bf.BF_ADD_BINNED),
                            (1, 256, 64, 8, 0, bf.BF_ADD_DIRECT), (4, 256, 32, 8, 2, bf.BF_ADD_DIRECT),
                            (3, 1024, 64, 16, 0, bf.BF_ADD_DIRECT), (3, 512, 32, 16, 0, bf.BF_ADD_DIRECT),
                            (3, 256, 64, 8, 0, bf.BF_ADD_HYBRID), (0, 1 << 20, 0, 7, 0, bf.BF_ADD_DIRECT)]:
    m = (1 << 20) if v else B
    o = OracleFilter(v, m, B=B if v else 256, S=S if v else 64, k=k, z=z)
    o.add(keys)
    f = bf.Filter(m, k, B if v else 256, S if v else 64, v, z=z)
    f.set_add_mode(mode, 1 << 14, 4096)
    f.add(kd)
    out = f.contains(qd)
    torch.cuda.synchronize()
    got = f.data().cpu().numpy()
    ok &= np.array_equal(got[:o.nbytes], o.bytes()) and np.array_equal(out.cpu().numpy().view(np.uint32), o.contains(q))
# routing + scatter
P, cap = 3, 8192
parts = [bf.bf_create_part(1 << 20, 8, 256, 64, 3, 0, P, p) for p in range(P)]
recs = torch.empty(P * cap, dtype=torch.int64, device=dev)
idx = torch.empty(P * cap, dtype=torch.int64, device=dev)
cnt = torch.empty(P, dtype=torch.int64, device=dev)
bf.bf_route(parts[0], kd, kd.numel(), 0, recs, None, cap, cnt)
for p in range(P):
    bf.bf_add_routed(parts[p], recs[p * cap:], cnt[p:], 1, cap)
bf.bf_route(parts[0], qd, qd.numel(), 0, recs, idx, cap, cnt)
res = torch.empty(P * cap, dtype=torch.uint8, device=dev)
for p in range(P):
    bf.bf_contains_routed(parts[p], recs[p * cap:], cnt[p:], 1, cap, res[p * cap:])
outp = torch.zeros((q.size + 31) // 32, dtype=torch.int32, device=dev)
bf.bf_scatter_results(idx, res, cnt, P, cap, outp)
buf = torch.empty(4096, dtype=torch.int64, device=dev)
bf.bf_keygen(buf, 4095, 7)
dst = torch.zeros(1 << 12, dtype=torch.uint8, device=dev)
src = torch.ones(3 << 12, dtype=torch.uint8, device=dev)
bf.bf_or_fold(dst, src, 3, 1 << 12, 1 << 12)
# peer-memory OR merge, 3 virtual ranks on this device (ragged 4-byte tail)
pb = [torch.from_numpy(np.random.default_rng(r).integers(0, 256, 4096 + 12, dtype=np.uint8)).to(dev) for r in range(3)]
want_or = np.bitwise_or.reduce(np.stack([t.cpu().numpy() for t in pb]), axis=0)
for r in range(3):
    bf.bf_p2p_or_merge([t.data_ptr() for t in pb], r, 4096 + 12)
torch.cuda.synchronize()
ok &= all(np.array_equal(t.cpu().numpy(), want_or) for t in pb)
o = OracleFilter(3, 1 << 20, B=256, S=64, k=8)
o.add(keys)
ok &= np.array_equal(outp.cpu().numpy().view(np.uint32), o.contains(q))
for h in parts:
    bf.bf_destroy(h)
print("sanitize workload ok" if ok else "sanitize workload MISMATCH")
sys.exit(0 if ok else 1)
