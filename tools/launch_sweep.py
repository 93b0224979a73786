"""Product add / contains vs the launch shape (bf_set_launch: CTAs per SM;
0 = persistent grid at occupancy, above occupancy = waves).
Usage (GPU box): python tools/launch_sweep.py [--m-bits M] [--n N] [--cfg V,B,S,k,z] ..."""
import argparse
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_15595_b200 import bf  # noqa: E402


def timed(fn, reps=7):
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0.record(st)
        fn()
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m-bits", type=int, default=1 << 28)
    ap.add_argument("--n", type=int, default=1 << 26)
    ap.add_argument("--cfg", action="append", default=[])
    ap.add_argument("--cps", default="0,1,2,3,4,6,8,12,16,24,32")
    a = ap.parse_args()
    cfgs = [tuple(int(x) for x in c.split(",")) for c in a.cfg] or [(3, 256, 64, 8, 0)]
    dev = torch.device("cuda:0")
    keys = torch.empty(a.n, dtype=torch.int64, device=dev)
    bf.bf_keygen(keys, a.n, 0)
    out = torch.empty((a.n + 31) // 32, dtype=torch.int32, device=dev)
    for v, B, S, k, z in cfgs:
        f = bf.Filter(a.m_bits, k, B, S, v, z=z)
        f.set_add_mode(bf.BF_ADD_DIRECT)
        f.set_contains_mode(bf.BF_CONTAINS_DIRECT)
        f.add(keys)
        for op in (1, 0):
            occ = bf.bf_get_launch(f.handle, op)[1]
            for cps in [int(x) for x in a.cps.split(",")]:
                f.set_launch(op, cps)
                ms = timed((lambda: f.contains(keys, out)) if op else (lambda: f.add(keys)))
                print(json.dumps({"cfg": [v, B, S, k, z], "m_bits": a.m_bits, "n": a.n,
                                  "op": "contains" if op else "add", "ctas_per_sm": cps, "occupancy": occ,
                                  "ms": round(ms, 4), "gkeys_s": round(a.n / (ms * 1e-3) / 1e9, 3)}), flush=True)
            f.set_launch(op, 0)
        del f


if __name__ == "__main__":
    main()
