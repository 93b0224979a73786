"""Binned add / contains vs the range size on a large filter (configs[4]'s
per-rank share by default: 32 GiB SBF 256/64 k=8, 2^31 keys), CUDA events.
Usage (GPU box): python tools/binned_range_sweep.py [--log2-bytes 35] [--log2-n 31]"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_15595_b200 import bf  # noqa: E402
from binned_contains_prof import timed  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log2-bytes", type=int, default=35)
    ap.add_argument("--log2-n", type=int, default=31)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    m, n = 8 << a.log2_bytes, 1 << a.log2_n
    keys = torch.empty(n, dtype=torch.int64, device=dev)
    bf.bf_keygen(keys, n, 0)
    out = torch.empty((n + 31) // 32, dtype=torch.int32, device=dev)
    f = bf.Filter(m, 8, 256, 64, "SBF")

    def add():
        f.clear()
        f.add(keys)
    f.set_contains_mode(bf.BF_CONTAINS_DIRECT)
    add()
    res = {"filter_bytes": m // 8, "n": n,
           "contains_direct": round(n / (timed(lambda: f.contains(keys, out)) * 1e-3) / 1e9, 2)}
    for rb in [int(x) << 20 for x in os.environ.get("RANGES_MIB", "16,32,64").split(",")]:
        f.set_add_mode(bf.BF_ADD_BINNED, rb, 0)
        f.set_contains_mode(bf.BF_CONTAINS_BINNED)
        res[f"add_binned@{rb >> 20}MiB"] = round(n / (timed(add) * 1e-3) / 1e9, 2)
        res[f"contains_binned@{rb >> 20}MiB"] = round(n / (timed(lambda: f.contains(keys, out)) * 1e-3) / 1e9, 2)
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
