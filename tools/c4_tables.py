"""Render the configs[3] grid (tools/sweep.py --set c4 / c4l2 rows): the
paper-table form (each Θ with the maximal Φ = s/Θ, best KPT, hash variant 0)
and the hash-variant ablation (H0 immediates/registers, H1
constant-bank table, H2 shared-memory table, H3 per-lane re-hash) at KPT=1.

Usage: python tools/c4_tables.py SWEEP_C4.jsonl SWEEP_C4L2.jsonl > profiles/r1_c4_tables.md
"""
import json
import os
import sys
from collections import defaultdict


def render(path, title):
    rows = [json.loads(l) for l in open(path)]
    s = rows[0]["B"] // rows[0]["S"]
    print(f"## {title} (`{os.path.basename(path)}`)\n")
    m = rows[0]["m_bits"]
    print(f"SBF {rows[0]['B']}/{rows[0]['S']}, m = {m} bits ({m / 8 / 2**30:.2f} GiB at k=8), n = {rows[0]['n']} keys; "
          "G keys/s, CUDA-event median.\n")
    best = defaultdict(float)
    hv = {}
    for r in rows:
        if r["hv"] == 0 and r["phi"] == s // r["theta"]:
            key = (r["k"], r["op"], r["theta"])
            best[key] = max(best[key], r["gkeys_s"])
        if r["kpt"] == 1:
            hv[(r["k"], r["op"], r["theta"], r["phi"], r["hv"])] = r["gkeys_s"]
    thetas = sorted({r["theta"] for r in rows})
    binned = {(r["k"], r["op"][:-len("_binned")]): r["gkeys_s"] for r in rows if r["op"].endswith("_binned")}
    print("Every Θ column is the direct kernel (like for like); the binned add / contains (round 2b; default "
          "schedule) are their own column.\n")
    print("| k | op | " + " | ".join(f"Θ={t}" for t in thetas) + " | binned |")
    print("|---|---|" + "---|" * len(thetas) + "---|")
    for k in sorted({r["k"] for r in rows}):
        for op in ("contains", "add"):
            extra = f"{binned[(k, op)]:.2f}" if (k, op) in binned else "—"
            print(f"| {k} | {op} | " + " | ".join(f"{best.get((k, op, t), 0):.2f}" for t in thetas) + f" | {extra} |")
    print("\nHash variants at KPT=1 (H0 immediates/registers, H1 constant table, H2 smem table, H3 per-lane re-hash):\n")
    print("| k | op | layout | H0 | H1 | H2 | H3 |\n|---|---|---|---|---|---|---|")
    for k in sorted({r["k"] for r in rows}):
        for op, t, p in (("contains", 1, s), ("add", s, 1), ("contains", 4, s // 4)):
            vals = [hv.get((k, op, t, p, h)) for h in range(4)]
            if any(v is not None for v in vals):
                print(f"| {k} | {op} | Θ={t},Φ={p} | " + " | ".join(f"{v:.2f}" if v is not None else "—" for v in vals) + " |")
    print()


if __name__ == "__main__":
    print("# configs[3] grid on one B200 (tools/sweep.py --set c4 / c4l2)\n")
    render(sys.argv[1], "configs[3]: SBF 256/32 at FPR 1e-4 (HBM-resident)")
    render(sys.argv[2], "configs[3] grid on a 32 MiB (L2-resident) filter")
