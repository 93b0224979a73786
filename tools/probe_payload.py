"""RED payload experiment: random-block red.or at 1/2/4 lanes x 8 B per block (32 MiB, L2)."""
import json
import torch
from paper_2512_15595_b200 import bf
dev = torch.device("cuda:0")
nbytes = 32 << 20
buf = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
n = 1 << 26
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for B in (64, 128, 256, 512):
    b = nbytes * 8 // B
    for red, lanes in [(0, 1), (1, 1), (1, 2), (1, 4), (1, 8), (1, 16)]:
        if red == 1 and lanes * 64 > B:
            continue
        ts = []
        for r in range(6):
            e0.record()
            bf.bf_probe_rng(buf, b, B, red, lanes, n)
            e1.record()
            torch.cuda.synchronize()
            if r:
                ts.append(e0.elapsed_time(e1))
        ts.sort()
        print(json.dumps({"B": B, "red": red, "lanes": lanes, "gblocks_s": round(n / ts[2] / 1e6, 2)}), flush=True)
