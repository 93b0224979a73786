#!/usr/bin/env python
"""Schedule / configuration sweeps (BASELINE.json configs[1] and configs[3]).

For every filter configuration selected and every compiled schedule (Θ, Φ,
KPT, hash variant), time bulk add (into a cleared filter) and bulk contains
(of the inserted keys) with CUDA events, median of --reps launches, and print
one JSON line per (config, op, schedule).  Results are identical for every
schedule (tests/test_gpu_parity.py); this only measures speed.

    python tools/sweep.py --set c2      # configs[1]: 32 MiB, every block/k row, default layouts x KPT
    python tools/sweep.py --set c4      # configs[3] grid: SBF 256/32 k=8,16, all Θ/Φ/KPT/hash variants
    python tools/sweep.py --set c4l2    # the same grid on a 32 MiB (L2) filter
"""
from __future__ import annotations

import argparse
import importlib.util
import json
import os
import statistics
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def instances():
    spec = importlib.util.spec_from_file_location(
        "gen_instances", os.path.join(ROOT, "paper_2512_15595_b200", "csrc", "gen_instances.py"))
    g = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(g)
    return g.instances()


def c_iso(variant, B, S, k, z):
    """bits/key at FPR 1e-4 (profiles/iso_fpr_table.json, written from the
    exact model by tools/make_iso_table.py)."""
    tab = json.load(open(os.path.join(ROOT, "profiles", "iso_fpr_table.json")))["c4"]["rows"]
    for r in tab:
        if (r["variant"], r["B"], r["S"], r["k"], r["z"]) == (variant, B, S, k, z):
            return r["c_iso"]
    raise KeyError((variant, B, S, k, z))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--set", default="c2", choices=["c2", "c2iso", "c4", "c4l2", "one", "paper", "ablation"])
    ap.add_argument("--n", type=int, default=1 << 26)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--cfg", default=None, help="v,B,S,k,z for --set one")
    ap.add_argument("--out", default=None)
    ap.add_argument("--only-variant", type=int, default=None, help="restrict c2 to one variant id")
    ap.add_argument("--no-probe", action="store_true", help="c2: skip the per-row probes")
    a = ap.parse_args()

    import torch

    from paper_2512_15595_b200 import bf

    dev = torch.device("cuda:0")
    if a.set == "c2iso":
        return iso_sweep(a, torch, bf, dev)
    if a.set == "paper":
        return paper_tables(a, torch, bf, dev)
    if a.set == "ablation":
        return hash_ablation(a, torch, bf, dev)
    inst = instances()
    groups = defaultdict(list)
    for op, v, B, S, k, z, th, ph, kpt, hv in inst:
        groups[(v, B, S, k, z)].append((op, th, ph, kpt, hv))
    if a.set == "c2":
        sel = {c: s for c, s in groups.items() if 4 <= c[3] <= 16 and c[1] <= 256
               and (a.only_variant is None or c[0] == a.only_variant)}
        m_of = lambda c: 1 << 28  # noqa: E731
        n = a.n
    elif a.set in ("c4", "c4l2"):
        sel = {c: s for c, s in groups.items() if c[:3] == (3, 256, 32) and c[3] in (8, 16)}
        if a.set == "c4":
            # m = c_iso(1e-4) * 2^30 bits (~3.3 GiB, b not a power of two)
            m_of = lambda c: int(c_iso(c[0], c[1], c[2], c[3], c[4]) * (1 << 30))  # noqa: E731
            n = 1 << 30
        else:
            m_of = lambda c: 1 << 28  # noqa: E731
            n = 1 << 30
    else:
        c = tuple(int(x) for x in a.cfg.split(","))
        sel = {c: groups[c]}
        m_of = lambda c: 1 << 28  # noqa: E731
        n = a.n

    keys = torch.empty(n, dtype=torch.int64, device=dev)
    bf.bf_keygen(keys, n, 0)
    out = torch.empty((n + 31) // 32, dtype=torch.int32, device=dev)
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fh = open(a.out, "a") if a.out else None
    for cfg, scheds in sorted(sel.items()):
        v, B, S, k, z = cfg
        m = m_of(cfg)
        f = bf.Filter(m, k, B, S, v, z=z)
        # like-for-like Θ sweep: the direct add and contains for every
        # schedule (the binned add / contains are separate rows below)
        f.set_add_mode(bf.BF_ADD_DIRECT)
        f.set_contains_mode(bf.BF_CONTAINS_DIRECT)
        for op, th, ph, kpt, hv in sorted(scheds):
            f.set_layout(op, th, ph, kpt, hv)
            ts = []
            for r in range(a.reps + 1):
                if op == 0:
                    f.clear()
                e0.record(st)
                if op == 0:
                    f.add(keys)
                else:
                    f.contains(keys, out)
                e1.record(st)
                torch.cuda.synchronize()
                if r:
                    ts.append(e0.elapsed_time(e1))
            t = statistics.median(ts)
            rec = {"set": a.set, "variant": v, "B": B, "S": S, "k": k, "z": z, "m_bits": m, "n": n,
                   "op": "add" if op == 0 else "contains", "theta": th, "phi": ph, "kpt": kpt, "hv": hv,
                   "ms": round(t, 4), "gkeys_s": round(n / (t * 1e-3) / 1e9, 3)}
            print(json.dumps(rec), flush=True)
            if fh:
                fh.write(json.dumps(rec) + "\n")
        if a.set == "c2" and not a.no_probe:  # live, geometry- and payload-matched probes of this row
            rec = row_probes(bf, torch, dev, cfg, m, keys, out, a.reps)
            print(json.dumps(rec), flush=True)
            if fh:
                fh.write(json.dumps(rec) + "\n")
        # restore default and check all-true after the sweep (sanity)
        f.set_layout(0, 0, 0)
        f.set_layout(1, 0, 0)
        if m // 8 >= (96 << 20):  # HBM-resident: the binned add, default schedule, as its own row
            f.set_add_mode(bf.BF_ADD_BINNED)
            ts = []
            for r in range(a.reps + 1):
                f.clear()
                e0.record(st)
                f.add(keys)
                e1.record(st)
                torch.cuda.synchronize()
                if r:
                    ts.append(e0.elapsed_time(e1))
            t = statistics.median(ts)
            lay = f.layout(0)
            rec = {"set": a.set, "variant": v, "B": B, "S": S, "k": k, "z": z, "m_bits": m, "n": n,
                   "op": "add_binned", "theta": lay["theta"], "phi": lay["phi"], "kpt": lay["kpt"], "hv": 0,
                   "ms": round(t, 4), "gkeys_s": round(n / (t * 1e-3) / 1e9, 3)}
            print(json.dumps(rec), flush=True)
            if fh:
                fh.write(json.dumps(rec) + "\n")
            f.set_add_mode(bf.BF_ADD_DIRECT)
            f.set_contains_mode(bf.BF_CONTAINS_BINNED)  # the binned contains, as its own row
            ts = []
            for r in range(a.reps + 1):
                e0.record(st)
                f.contains(keys, out)
                e1.record(st)
                torch.cuda.synchronize()
                if r:
                    ts.append(e0.elapsed_time(e1))
            t = statistics.median(ts)
            rec = {"set": a.set, "variant": v, "B": B, "S": S, "k": k, "z": z, "m_bits": m, "n": n,
                   "op": "contains_binned", "theta": 1, "phi": B // S, "kpt": 4, "hv": 0,
                   "ms": round(t, 4), "gkeys_s": round(n / (t * 1e-3) / 1e9, 3)}
            print(json.dumps(rec), flush=True)
            if fh:
                fh.write(json.dumps(rec) + "\n")
            f.set_contains_mode(bf.BF_CONTAINS_DIRECT)
        f.clear()
        f.add(keys)
        f.contains(keys, out)
        torch.cuda.synchronize()
        if n % 32 == 0:
            assert int((out != -1).sum()) == 0, f"false negatives in {cfg}"
        del f


def row_probes(bf, torch, dev, cfg, m, keys, out, reps):
    """The row's roofline denominators, measured live on a buffer of the
    filter's size in two launch shapes (8 and 32 CTAs per SM):
    contains -- R_read(B): one random block load per key (key-stream and
    in-register forms); add -- R_red with the add's own RED pattern
    (bf_probe_pattern_records + bf_probe_red_records: precomputed (block,
    word-hit mask) records, s words for SBF/RBBF, the words of k draws for
    BBF, z words for CSBF, one group instruction per key) and the generic
    in-register block RED (all words)."""
    v, B, S, k, z = cfg
    nbytes = m // 8
    buf = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
    Bp = max(64, B)
    b = nbytes * 8 // Bp
    bb = nbytes * 8 // B
    n = keys.numel()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count

    def best(fn):
        fn()
        ts = []
        for _ in range(reps):
            e0.record(st)
            fn()
            e1.record(st)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return min(ts)

    res = {}
    recs = torch.empty(n, dtype=torch.int64, device=dev)
    bf.bf_probe_pattern_records(recs, n, bb, B, S, v, k, z, 1)
    for cps in (8, 32):
        bf.bf_set_probe_launch(cps)
        thr = sms * cps * 256
        n_rng = -(-n // (thr * 4)) * thr * 4
        res[f"read_keys@{cps}"] = n / best(lambda: bf.bf_probe_read(buf, b, Bp, keys, out)) / 1e6
        res[f"read_rng@{cps}"] = n_rng / best(lambda: bf.bf_probe_rng(buf, b, Bp, 0, 1, n)) / 1e6
        res[f"red_pattern@{cps}"] = n / best(lambda: bf.bf_probe_red_records(buf, B, S, recs, n)) / 1e6
    bf.bf_set_probe_launch(0)
    del buf, recs
    res = {kk: round(vv, 3) for kk, vv in res.items()}
    return {"set": "c2", "variant": v, "B": B, "S": S, "k": k, "z": z, "m_bits": m, "n": n, "op": "probe",
            "read": max(vv for kk, vv in res.items() if kk.startswith("read")),
            "red": max(vv for kk, vv in res.items() if kk.startswith("red")), "forms": res}


# the paper's Table 1 (1 GB) and Table 2 (32 MB), G keys/s
PAPER = {
    ("1GB", "contains"): {64: [48.69], 128: [48.54, 44.62], 256: [47.79, 43.74, 41.64],
                          512: [25.35, 40.66, 40.15, 33.66], 1024: [12.81, 36.01, 36.96, 33.38, 24.54]},
    ("1GB", "add"): {64: [22.43], 128: [13.57, 22.26], 256: [7.59, 13.65, 22.10],
                     512: [4.58, 7.72, 15.31, 20.75], 1024: [2.88, 5.02, 8.53, 15.41, 15.61]},
    ("32MB", "contains"): {64: [155.89], 128: [149.50, 51.58], 256: [141.88, 51.57, 50.40],
                           512: [104.55, 50.20, 50.35, 45.34], 1024: [44.87, 48.95, 48.69, 45.22, 42.11]},
    ("32MB", "add"): {64: [125.19], 128: [66.07, 121.45], 256: [33.91, 63.25, 111.88],
                      512: [17.10, 20.67, 35.56, 72.41], 1024: [8.19, 10.37, 11.55, 18.91, 39.22]},
}


def paper_tables(a, torch, bf, dev):
    """The paper's layout tables on this B200: SBF, S=64, k=16, B = 64..1024
    (B=64 is the RBBF), every Θ with Φ = s/Θ (KPT: best of 1/2/4), a 32 MiB
    (L2) and a 1 GiB (HBM) filter; add uses the paper's direct method (plus
    one binned row at 1 GiB)."""
    n = a.n
    keys = torch.empty(n, dtype=torch.int64, device=dev)
    bf.bf_keygen(keys, n, 0)
    out = torch.empty((n + 31) // 32, dtype=torch.int32, device=dev)
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fh = open(a.out, "a") if a.out else None

    def timeit(fn, reps, pre=None):
        ts = []
        for r in range(reps + 1):
            if pre:
                pre()
            e0.record(st)
            fn()
            e1.record(st)
            torch.cuda.synchronize()
            if r:
                ts.append(e0.elapsed_time(e1))
        return statistics.median(ts)

    for size, m in (("32MB", 1 << 28), ("1GB", 1 << 33)):
        for B in (64, 128, 256, 512, 1024):
            s = B // 64
            v = 2 if B == 64 else 3
            f = bf.Filter(m, 16, B, 64, v)
            f.set_contains_mode(bf.BF_CONTAINS_DIRECT)  # the paper's direct lookup for every Θ
            for op in ("add", "contains"):
                for ti, th in enumerate([1 << i for i in range(s.bit_length())]):
                    best = None
                    for kpt in (1, 2, 4):
                        try:
                            f.set_layout(0 if op == "add" else 1, th, s // th, kpt, 0)
                        except bf.BFError:
                            continue
                        if op == "add":
                            f.set_add_mode(bf.BF_ADD_DIRECT)
                            t = timeit(lambda: f.add(keys), a.reps, pre=f.clear)
                        else:
                            f.set_add_mode(bf.BF_ADD_DIRECT)
                            f.clear()
                            f.add(keys)
                            t = timeit(lambda: f.contains(keys, out), a.reps)
                        g = n / (t * 1e-3) / 1e9
                        if best is None or g > best[0]:
                            best = (g, kpt)
                    if best is None:
                        continue
                    rec = {"set": "paper", "size": size, "m_bits": m, "B": B, "S": 64, "k": 16, "op": op,
                           "theta": th, "phi": s // th, "kpt": best[1], "gkeys_s": round(best[0], 2),
                           "paper_gkeys_s": PAPER[(size, op)][B][ti], "n": n}
                    print(json.dumps(rec), flush=True)
                    if fh:
                        fh.write(json.dumps(rec) + "\n")
            if size == "1GB":
                f.set_layout(0, 0, 0)
                f.set_add_mode(bf.BF_ADD_BINNED)
                t = timeit(lambda: f.add(keys), a.reps, pre=f.clear)
                rec = {"set": "paper", "size": size, "m_bits": m, "B": B, "S": 64, "k": 16, "op": "add_binned",
                       "theta": f.layout(0)["theta"], "phi": f.layout(0)["phi"], "kpt": f.layout(0)["kpt"],
                       "gkeys_s": round(n / (t * 1e-3) / 1e9, 2), "n": n}
                print(json.dumps(rec), flush=True)
                if fh:
                    fh.write(json.dumps(rec) + "\n")
                f.set_contains_mode(bf.BF_CONTAINS_BINNED)
                t = timeit(lambda: f.contains(keys, out), a.reps)
                rec = {"set": "paper", "size": size, "m_bits": m, "B": B, "S": 64, "k": 16, "op": "contains_binned",
                       "theta": 1, "phi": s, "kpt": 4, "gkeys_s": round(n / (t * 1e-3) / 1e9, 2), "n": n}
                print(json.dumps(rec), flush=True)
                if fh:
                    fh.write(json.dumps(rec) + "\n")
            del f
        # the paper's GPU CBF baseline (k=16): P:L392 (32 MB) 13.43 add / 42.64 contains,
        # P:L352 (1 GB) 1.45 / 8.84
        f = bf.Filter(m, 16, 256, 64, bf.BF_CBF)
        ta = timeit(lambda: f.add(keys), a.reps, pre=f.clear)
        tc = timeit(lambda: f.contains(keys, out), a.reps)
        paper = {"32MB": (13.43, 42.64), "1GB": (1.45, 8.84)}[size]
        for op, t, pv in (("add", ta, paper[0]), ("contains", tc, paper[1])):
            rec = {"set": "paper", "size": size, "m_bits": m, "B": 0, "S": 32, "k": 16, "op": "cbf_" + op,
                   "theta": 1, "phi": 1, "kpt": 1, "gkeys_s": round(n / (t * 1e-3) / 1e9, 2),
                   "paper_gkeys_s": pv, "n": n}
            print(json.dumps(rec), flush=True)
            if fh:
                fh.write(json.dumps(rec) + "\n")
        del f


def hash_ablation(a, torch, bf, dev):
    """The paper's optimisation breakdown (Fig. 9) on SBF 256/64
    k=16: GPU CBF -> SBF with iterative single-hash draws (one XXH64 per draw,
    P:L223) -> double hashing -> multiplicative hashing, each at the
    unoptimised layout (Θ=1, KPT=1) and at the optimised one (add Θ=s with
    cooperation, KPT=4)."""
    n = a.n
    keys = torch.empty(n, dtype=torch.int64, device=dev)
    bf.bf_keygen(keys, n, 0)
    out = torch.empty((n + 31) // 32, dtype=torch.int32, device=dev)
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fh = open(a.out, "a") if a.out else None

    def timeit(fn, pre=None):
        ts = []
        for r in range(a.reps + 1):
            if pre:
                pre()
            e0.record(st)
            fn()
            e1.record(st)
            torch.cuda.synchronize()
            if r:
                ts.append(e0.elapsed_time(e1))
        return n / (statistics.median(ts) * 1e-3) / 1e9

    def emit(rec):
        print(json.dumps(rec), flush=True)
        if fh:
            fh.write(json.dumps(rec) + "\n")

    for size, m in (("32MB", 1 << 28), ("1GB", 1 << 33)):
        f = bf.Filter(m, 16, 256, 64, bf.BF_CBF)
        emit({"set": "ablation", "size": size, "step": "gpu_cbf", "add": round(timeit(lambda: f.add(keys), f.clear), 2),
              "contains": round(timeit(lambda: f.contains(keys, out)), 2)})
        del f
        for scheme, name in ((2, "sbf_iterative"), (1, "sbf_double"), (0, "sbf_multiplicative")):
            f = bf.Filter(m, 16, 256, 64, "SBF", scheme=scheme)
            f.set_add_mode(bf.BF_ADD_DIRECT)
            f.set_contains_mode(bf.BF_CONTAINS_DIRECT)  # the paper's lookup at every step
            for lay_name, add_lay, con_lay in (("theta1_kpt1", (1, 4, 1), (1, 4, 1)),
                                               ("optimised", (4, 1, 4) if scheme != 2 else (1, 4, 1),
                                                (1, 4, 4) if scheme != 2 else (1, 4, 1))):
                try:
                    f.set_layout(0, add_lay[0], add_lay[1], add_lay[2], 0)
                    f.set_layout(1, con_lay[0], con_lay[1], con_lay[2], 0)
                except bf.BFError:
                    continue
                emit({"set": "ablation", "size": size, "step": name, "layout": lay_name,
                      "add": round(timeit(lambda: f.add(keys), f.clear), 2),
                      "contains": round(timeit(lambda: f.contains(keys, out)), 2)})
            del f


def iso_sweep(a, torch, bf, dev):
    """configs[1] at iso FPR 1e-3: per row, add n_iso keys (profiles/
    iso_fpr_table.json) into a cleared 32 MiB filter, query 2^26 absent keys;
    report both throughputs and the measured FPR against the exact model."""
    import math

    import numpy as np

    import synth
    tab = json.load(open(os.path.join(ROOT, "profiles", "iso_fpr_table.json")))["c2"]
    m, Q = tab["m_bits"], 1 << 26
    neg = torch.empty(Q, dtype=torch.int64, device=dev)
    bf.bf_keygen(neg, Q, synth.NEG_BASE)
    out = torch.empty(Q // 32, dtype=torch.int32, device=dev)
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fh = open(a.out, "a") if a.out else None
    for row in tab["rows"]:
        v, B, S, k, z, n = row["variant"], row["B"], row["S"], row["k"], row["z"], row["n_iso"]
        keys = torch.empty(n, dtype=torch.int64, device=dev)
        bf.bf_keygen(keys, n, 0)
        f = bf.Filter(m, k, B, S, v, z=z)
        ta, tc = [], []
        for r in range(a.reps + 1):
            f.clear()
            e0.record(st)
            f.add(keys)
            e1.record(st)
            torch.cuda.synchronize()
            if r:
                ta.append(e0.elapsed_time(e1))
            e0.record(st)
            f.contains(neg, out)
            e1.record(st)
            torch.cuda.synchronize()
            if r:
                tc.append(e0.elapsed_time(e1))
        fp = int(np.unpackbits(out.cpu().numpy().view(np.uint8)).sum())
        p = row["fpr_model"]
        rec = {"set": "c2iso", "variant": v, "B": B, "S": S, "k": k, "z": z, "m_bits": m, "n_iso": n,
               "c_iso": round(row["c_iso"], 3), "add_gkeys_s": round(n / statistics.median(ta) / 1e6, 3),
               "contains_gkeys_s": round(Q / statistics.median(tc) / 1e6, 3), "fpr": fp / Q,
               "fpr_model": p, "fpr_z": round((fp - Q * p) / math.sqrt(Q * p * (1 - p)), 2),
               "layout_add": f.layout(0), "layout_contains": f.layout(1)}
        print(json.dumps(rec), flush=True)
        if fh:
            fh.write(json.dumps(rec) + "\n")
        del f, keys


if __name__ == "__main__":
    main()
