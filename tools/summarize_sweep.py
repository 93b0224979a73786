"""Summarise a configs[1] (C2) sweep (tools/sweep.py --set c2 jsonl) against the
random-access probes (profiles/r1_probe_red_payload.jsonl).

Per row (variant, B, S, k, z): the best add / contains schedule, the default
schedule's rate, and the best rate as % of the probe with the same geometry
(SURVEY 8(d) "% of roofline"):
  contains: R_read(B)   -- one random block load per key
  add:      R_red(payload) -- one random sector RED per key carrying the
            row's payload (words with bits x S/8 bytes); the probe at 8 and
            16 bytes per sector runs at the same rate, 32 bytes is slower
            (the L1->XBAR path, profiles/r1_probe_red_payload.jsonl).

Usage: python tools/summarize_sweep.py SWEEP.jsonl [PROBE.jsonl] > out.md
"""
from __future__ import annotations

import json
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "paper_2512_15595_b200", "csrc"))
from gen_instances import default_add  # noqa: E402

NAMES = {1: "BBF", 2: "RBBF", 3: "SBF", 4: "CSBF"}


def probes(path):
    read, red = {}, {}
    for line in open(path):
        d = json.loads(line)
        if d["red"] == 0:
            read[d["B"]] = d["gblocks_s"]
        elif d["lanes"] * 64 == d["B"]:  # every word of the block: payload B/8 (one key per s lanes)
            red[d["B"] // 8] = d["gblocks_s"]
    return read, red


def payload(v, B, S, k, z):
    s = B // S
    if v == 4:
        words = z
    elif v == 1:
        words = min(k, s)
    else:
        words = s
    return words * S // 8


def red_bound(red, nbytes):
    # probe rates exist for 8/16/32/64-byte payloads (B = 64..512, all lanes)
    for p in sorted(red):
        if nbytes <= p:
            return red[p], p
    return red[max(red)], max(red)


def main():
    sweep = sys.argv[1]
    probe = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "profiles", "r1_probe_red_payload.jsonl")
    read, red = probes(probe)
    rows = defaultdict(dict)
    for line in open(sweep):
        d = json.loads(line)
        key = (d["variant"], d["B"], d["S"], d["k"], d["z"])
        sc = (d["theta"], d["phi"], d["kpt"], d["hv"])
        rows[key].setdefault(d["op"], {})[sc] = d["gkeys_s"]
    print(f"# C2 sweep summary: `{os.path.basename(sweep)}`\n")
    print("32 MiB (L2-resident) filter, 2^26 keys; Gkeys/s, CUDA-event median of 5 launches. "
          "Schedules (Θ, Φ, KPT, hash variant). % = best / probe with the same geometry "
          "(contains: R_read(B); add: R_red at the row's bytes per sector).\n")
    print("| variant | B/S | k | z | add best | sched | add default | % R_red (payload) "
          "| contains best | sched | contains default | % R_read |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|")
    pa, pc = [], []
    for key in sorted(rows, key=lambda c: (NAMES[c[0]], c[1], c[2], c[4], c[3])):
        v, B, S, k, z = key
        r = rows[key]
        s = B // S
        ta, pa_ = default_add(v, B, S, z)
        tc = max(1, B // 256)
        add, con = r.get("add", {}), r.get("contains", {})
        ba = max(add.items(), key=lambda x: x[1]) if add else (None, 0)
        bc = max(con.items(), key=lambda x: x[1]) if con else (None, 0)
        da = add.get((ta, pa_, 4, 0), float("nan"))
        dc = con.get((tc, s // tc, 4, 0), float("nan"))
        rb, pl = red_bound(red, payload(v, B, S, k, z))
        rr = read.get(max(B, 64), float("nan"))  # a 32-bit block is one sector read too
        fa, fc = 100 * ba[1] / rb, 100 * bc[1] / rr
        pa.append(fa)
        pc.append(fc)
        print(f"| {NAMES[v]} | {B}/{S} | {k} | {z} | {ba[1]:.1f} | {ba[0]} | {da:.1f} | {fa:.0f}% ({pl} B) "
              f"| {bc[1]:.1f} | {bc[0]} | {dc:.1f} | {fc:.0f}% |")
    print(f"\nRows: {len(pa)}. add: median {sorted(pa)[len(pa) // 2]:.0f}% of R_red, "
          f"{sum(x >= 85 for x in pa)} rows >= 85%. contains: median {sorted(pc)[len(pc) // 2]:.0f}% of R_read, "
          f"{sum(x >= 85 for x in pc)} rows >= 85%.")
    print(f"\nProbes (G blocks/s): R_read {dict(sorted(read.items()))}; R_red by payload bytes "
          f"{dict(sorted(red.items()))}.")


if __name__ == "__main__":
    main()
