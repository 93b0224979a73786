"""HBM random-access probes vs the L2 fetch granularity.

For an 8 GiB buffer (configs[2]'s filter size, far beyond the 126 MB L2):
GUPS-style random loads of 8 / 32 / 64 bytes with and without the .L2::64B /
.L2::128B fill hints, random 8-byte red.or updates, the filter-geometry probes
(32-byte block loads, 4-lane RED.64 per block), and the product kernels
(configs[2] SBF 256/64 k=8 contains, direct add) -- each under
cudaLimitMaxL2FetchGranularity = driver default, 32, 64 and 128 bytes.

Prints one JSON line per (granularity, probe) with G accesses/s (median of
`reps` CUDA-event-timed launches, L2 flushed by the buffer size itself).
Usage (GPU box): python tools/hbm_probes.py [--gib 8] [--n 2^28] > out.jsonl
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_15595_b200 import bf  # noqa: E402


def timed(fn, reps):
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
    ap.add_argument("--gib", type=int, default=8)
    ap.add_argument("--n", type=int, default=1 << 28)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--grans", default="0,32,64,128")
    ap.add_argument("--no-product", action="store_true")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    nbytes = a.gib << 30
    n = a.n
    buf = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
    keys = torch.empty(n, dtype=torch.int64, device=dev)
    bf.bf_keygen(keys, n, 0)
    out = torch.empty((n + 31) // 32, dtype=torch.int32, device=dev)
    f = None
    if not a.no_product:
        f = bf.Filter(nbytes * 8, 8, 256, 64, "SBF")
        f.set_add_mode(bf.BF_ADD_DIRECT)
        f.add(keys)
    base = bf.bf_get_l2_fetch_granularity()
    probes = [
        ("gups_read_8", lambda: bf.bf_probe_gups(buf, nbytes, 8, 0, 0, n)),
        ("gups_read_8_L2_64B", lambda: bf.bf_probe_gups(buf, nbytes, 8, 0, 1, n)),
        ("gups_read_8_L2_128B", lambda: bf.bf_probe_gups(buf, nbytes, 8, 0, 2, n)),
        ("gups_read_32", lambda: bf.bf_probe_gups(buf, nbytes, 32, 0, 0, n)),
        ("gups_read_32_L2_64B", lambda: bf.bf_probe_gups(buf, nbytes, 32, 0, 1, n)),
        ("gups_read_64", lambda: bf.bf_probe_gups(buf, nbytes, 64, 0, 0, n)),
        ("gups_read_64_L2_64B", lambda: bf.bf_probe_gups(buf, nbytes, 64, 0, 1, n)),
        ("gups_update_8", lambda: bf.bf_probe_gups(buf, nbytes, 8, 1, 0, n)),
        ("block_read_rng_B256", lambda: bf.bf_probe_rng(buf, nbytes // 32, 256, 0, 1, n)),
        ("block_red_rng_B256_4lanes", lambda: bf.bf_probe_rng(buf, nbytes // 32, 256, 1, 4, n)),
        ("block_red_rng_B64_1lane", lambda: bf.bf_probe_rng(buf, nbytes // 8, 64, 1, 1, n)),
        ("block_read_keys_B256", lambda: bf.bf_probe_read(buf, nbytes // 32, 256, keys, out)),
        ("block_red_keys_B256_4lanes", lambda: bf.bf_probe_red(buf, nbytes // 32, 256, 4, keys)),
    ]
    if f is not None:
        probes += [("product_contains_sbf256_k8", lambda: f.contains(keys, out)),
                   ("product_add_direct_sbf256_k8", lambda: f.add(keys))]
    for g in [int(x) for x in a.grans.split(",")]:
        bf.bf_set_l2_fetch_granularity(g)
        eff = bf.bf_get_l2_fetch_granularity()
        for name, fn in probes:
            ms = timed(fn, a.reps)
            print(json.dumps({"probe": name, "gran_set": g, "gran_effective": eff, "gran_default": base,
                              "buffer_gib": a.gib, "n": n, "ms": round(ms, 4),
                              "g_per_s": round(n / (ms * 1e-3) / 1e9, 3)}), flush=True)
    bf.bf_set_l2_fetch_granularity(0)


if __name__ == "__main__":
    main()
