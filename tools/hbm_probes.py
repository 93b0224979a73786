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
    ap.add_argument("--sweep", action="store_true", help="MLP x CTAs sweep at the default granularity")
    ap.add_argument("--sweep2", action="store_true", help="fine CTA sweep at MLP 1/2, product KPT/CTA variants")
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
        f.set_contains_mode(bf.BF_CONTAINS_DIRECT)
        f.add(keys)
    base = bf.bf_get_l2_fetch_granularity()
    if a.sweep2:
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        for rep in range(2):
            for mlp in (1, 2):
                for cps in (8, 9, 10, 11, 12, 14, 16, 20, 24, 32):
                    ms = timed(lambda: bf.bf_probe_gups(buf, nbytes, 32, 0, 1, n, mlp, cps * sms), 9)
                    print(json.dumps({"probe": "gups_read_32_L2_64B", "rep": rep, "mlp": mlp, "ctas_per_sm": cps,
                                      "n": n, "ms": round(ms, 4), "g_per_s": round(n / (ms * 1e-3) / 1e9, 3)}), flush=True)
            ms = timed(lambda: bf.bf_probe_read(buf, nbytes // 32, 256, keys, out), 9)
            print(json.dumps({"probe": "block_read_keys_B256", "rep": rep, "n": n, "ms": round(ms, 4),
                              "g_per_s": round(n / (ms * 1e-3) / 1e9, 3)}), flush=True)
        if f is not None:
            for kpt in (4,):
                f.set_layout(1, 1, 4, kpt, 0)
                occ = bf.bf_get_launch(f.handle, 1)[1]
                for cps in sorted({1, 2, occ, 4, 6, 8, 10, 12, 16, 24, 32}):
                    f.set_launch(1, cps)
                    ms = timed(lambda: f.contains(keys, out), 9)
                    print(json.dumps({"probe": "product_contains_sbf256_k8", "kpt": kpt, "ctas_per_sm": cps,
                                      "occupancy": occ, "n": n, "ms": round(ms, 4),
                                      "g_per_s": round(n / (ms * 1e-3) / 1e9, 3)}), flush=True)
                f.set_launch(1, 0)
            occ = bf.bf_get_launch(f.handle, 0)[1]
            for cps in sorted({1, 2, occ, 8, 10, 12, 16, 24, 32}):
                f.set_launch(0, cps)
                ms = timed(lambda: f.add(keys), 5)
                print(json.dumps({"probe": "product_add_direct_sbf256_k8", "ctas_per_sm": cps, "occupancy": occ,
                                  "n": n, "ms": round(ms, 4), "g_per_s": round(n / (ms * 1e-3) / 1e9, 3)}), flush=True)
            f.set_launch(0, 0)
        for mlp in (1, 8):  # updates, fine CTA sweep
            for cps in (8, 10, 12, 16, 24):
                ms = timed(lambda: bf.bf_probe_gups(buf, nbytes, 8, 1, 0, n, mlp, cps * sms), 5)
                print(json.dumps({"probe": "gups_update_8", "mlp": mlp, "ctas_per_sm": cps, "n": n, "ms": round(ms, 4),
                                  "g_per_s": round(n / (ms * 1e-3) / 1e9, 3)}), flush=True)
        return
    if a.sweep:
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        for name, ab, red, hint in (("gups_read_8", 8, 0, 0), ("gups_read_32_L2_64B", 32, 0, 1),
                                    ("gups_update_8", 8, 1, 0)):
            for mlp in (1, 2, 4, 8, 16):
                for cps in (1, 2, 4, 8):
                    ms = timed(lambda: bf.bf_probe_gups(buf, nbytes, ab, red, hint, n, mlp, cps * sms), a.reps)
                    print(json.dumps({"probe": name, "mlp": mlp, "ctas_per_sm": cps, "threads_in_flight": cps * sms * 256,
                                      "accesses_in_flight": cps * sms * 256 * mlp, "buffer_gib": a.gib, "n": n,
                                      "ms": round(ms, 4), "g_per_s": round(n / (ms * 1e-3) / 1e9, 3)}), flush=True)
        if f is not None:
            occ = [bf.bf_get_launch(f.handle, op)[1] for op in (0, 1)]
            for op, name, fn in ((1, "product_contains_sbf256_k8", lambda: f.contains(keys, out)),
                                 (0, "product_add_direct_sbf256_k8", lambda: f.add(keys))):
                for cps in range(1, occ[op] + 1):
                    f.set_launch(op, cps)
                    ms = timed(fn, a.reps)
                    print(json.dumps({"probe": name, "ctas_per_sm": cps, "occupancy": occ[op], "n": n,
                                      "ms": round(ms, 4), "g_per_s": round(n / (ms * 1e-3) / 1e9, 3)}), flush=True)
                f.set_launch(op, 0)
        return
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
