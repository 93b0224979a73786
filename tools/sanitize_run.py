"""End-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck): every kernel family once, checked against the oracle.  The bulk
keys are 2^22 + 37 (SAN_N overrides): the launch grid is capped at the
occupancy grid, so every warp runs several tiles and the steady-state paths
(cross-tile key pipeline, cp.async key double buffer, shared-memory staging
reuse, ragged-tail hand-off) are under the tools, not only the first tile.
Usage: compute-sanitizer --tool racecheck python tools/sanitize_run.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from oracle.bfo import OracleFilter  # noqa: E402
from paper_2512_15595_b200 import bf  # noqa: E402

dev = torch.device("cuda:0")
N = int(os.environ.get("SAN_N", (1 << 22) + 37))
keys = synth.keys(0, N)
q = np.concatenate([keys[:N // 3], synth.negatives(N // 3 + 1)])
kd = torch.from_numpy(keys.view(np.int64)).to(dev)
qd = torch.from_numpy(q.view(np.int64)).to(dev)
ok = True
for v, B, S, k, z, mode in [(3, 256, 64, 8, 0, bf.BF_ADD_DIRECT), (3, 256, 64, 8, 0, bf.BF_ADD_BINNED),
                            (1, 256, 64, 8, 0, bf.BF_ADD_DIRECT), (4, 256, 32, 8, 2, bf.BF_ADD_DIRECT),
                            (3, 1024, 64, 16, 0, bf.BF_ADD_DIRECT), (3, 512, 32, 16, 0, bf.BF_ADD_DIRECT),
                            (1, 256, 64, 16, 0, bf.BF_ADD_DIRECT), (1, 256, 32, 11, 0, bf.BF_ADD_DIRECT),
                            (2, 64, 64, 8, 0, bf.BF_ADD_DIRECT),
                            (3, 256, 64, 8, 0, bf.BF_ADD_HYBRID), (0, 1 << 20, 0, 7, 0, bf.BF_ADD_DIRECT)]:
    m = (1 << 26) + 3 * 256 if v else B
    o = OracleFilter(v, m, B=B if v else 256, S=S if v else 64, k=k, z=z)
    o.add(keys, threads=os.cpu_count())
    f = bf.Filter(m, k, B if v else 256, S if v else 64, v, z=z)
    f.set_add_mode(mode, 1 << 20, 1 << 20)  # binned: 8 ranges x 5 batches
    if mode == bf.BF_ADD_BINNED:  # and the binned contains (same ranges and batches)
        f.set_contains_mode(bf.BF_CONTAINS_BINNED)
    f.add(kd)
    out = f.contains(qd)
    torch.cuda.synchronize()
    got = f.data().cpu().numpy()
    good = np.array_equal(got[:o.nbytes], o.bytes()) and \
        np.array_equal(out.cpu().numpy().view(np.uint32), o.contains(q, threads=os.cpu_count()))
    print(f"variant={v} B={B} S={S} k={k} z={z} mode={mode} contains_binned={f.contains_mode()[1] if v else 0}: "
          f"{'ok' if good else 'MISMATCH'}", flush=True)
    ok &= good
# routing + scatter
P = 3
cap = ((N // P) * 11 // 10 + 4096 + 127) // 128 * 128
parts = [bf.bf_create_part(1 << 26, 8, 256, 64, 3, 0, P, p) for p in range(P)]
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
o = OracleFilter(3, 1 << 26, B=256, S=64, k=8)
o.add(keys, threads=os.cpu_count())
ok &= np.array_equal(outp.cpu().numpy().view(np.uint32), o.contains(q, threads=os.cpu_count()))
for h in parts:
    bf.bf_destroy(h)
print("sanitize workload ok" if ok else "sanitize workload MISMATCH")
sys.exit(0 if ok else 1)
