"""Binned vs direct add and contains on the configs[2] filter (8 GiB SBF
256/64 k=8), one 2^31-key call each, CUDA events.  Usage (GPU box):
python tools/binned_contains_prof.py  (prints one JSON line)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_15595_b200 import bf  # noqa: E402


def timed(fn, reps=3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    best = None
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1)
        best = t if best is None else min(best, t)
    return best


def main():
    dev = torch.device("cuda:0")
    m, n = 1 << 36, 1 << 31
    keys = torch.empty(n, dtype=torch.int64, device=dev)
    bf.bf_keygen(keys, n, 0)
    f = bf.Filter(m, 8, 256, 64, "SBF")
    out = torch.empty((n + 31) // 32, dtype=torch.int32, device=dev)
    res = {"range_cps": os.environ.get("BF_EXP_RANGE_CPS", "default")}

    def add():
        f.clear()
        f.add(keys)
    f.set_add_mode(bf.BF_ADD_BINNED)
    res["add_binned"] = round(n / (timed(add) * 1e-3) / 1e9, 2)
    for mode, name in ((bf.BF_CONTAINS_BINNED, "contains_binned"), (bf.BF_CONTAINS_DIRECT, "contains_direct")):
        f.set_contains_mode(mode)
        res[name] = round(n / (timed(lambda: f.contains(keys, out)) * 1e-3) / 1e9, 2)
        assert int((out != -1).sum().item()) == 0
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
