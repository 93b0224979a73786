"""Render the paper's Table 1/2 grid (tools/sweep.py --set paper rows) as
markdown: ours (best KPT) vs the paper's B200 numbers (Table 1,
1 GiB; Table 2, 32 MiB), plus the GPU CBF baseline and the binned
add.  Also renders the optimisation ablation (--set ablation) if given.

Usage: python tools/paper_tables.py SWEEP_PAPER.jsonl [SWEEP_ABLATION.jsonl] > profiles/r1_paper_tables.md
"""
from __future__ import annotations

import json
import os
import sys
from collections import defaultdict


def main(paper, ablation=None):
    best = defaultdict(lambda: (0.0, None))
    cbf = {}
    for line in open(paper):
        d = json.loads(line)
        if d["op"].startswith("cbf_"):
            cbf[(d["size"], d["op"])] = d
            continue
        key = (d["size"], d["op"], d["B"], d["theta"])
        if d["gkeys_s"] > best[key][0]:
            best[key] = (d["gkeys_s"], d.get("paper_gkeys_s"))
    print(f"# The paper's Table 1 / Table 2 grid on this B200 (`{os.path.basename(paper)}`)\n")
    print("SBF, S=64, k=16 (B=64 is the RBBF), 2^28 keys, every Θ with Φ = s/Θ, best KPT of 1/2/4,")
    print("CUDA-event median of 3 launches. Cells: **ours** (paper, P:L326-336 / P:L371-381), G keys/s.")
    print("add / contains = the paper's method (direct red.global.or / block loads); `add_binned`, "
          "`contains_binned` = our binned add and binned contains (bf_binned.cuh).\n")
    thetas = (1, 2, 4, 8, 16)
    for size, title in (("32MB", "Table 2: 32 MiB (L2-resident) filter"), ("1GB", "Table 1: 1 GiB (HBM-resident) filter")):
        print(f"## {title}\n")
        print("| op | B | " + " | ".join(f"Θ={t}" for t in thetas) + " |")
        print("|---|---|" + "---|" * len(thetas))
        wins = total = 0
        for op in ("contains", "add", "add_binned", "contains_binned"):
            for B in (64, 128, 256, 512, 1024):
                cells = []
                any_cell = False
                for t in thetas:
                    v, pv = best.get((size, op, B, t), (0.0, None))
                    if not v:
                        cells.append("")
                        continue
                    any_cell = True
                    if pv:
                        total += 1
                        wins += v > pv
                        cells.append(f"**{v:.1f}** ({pv})")
                    else:
                        cells.append(f"**{v:.1f}**")
                if any_cell:
                    print(f"| {op} | {B} | " + " | ".join(cells) + " |")
        print(f"\nCells above the paper's number: {wins}/{total}.\n")
        a, c = cbf.get((size, "cbf_add")), cbf.get((size, "cbf_contains"))
        if a and c:
            print(f"GPU CBF baseline (k=16; NEXT N3): cbf_add **{a['gkeys_s']}** (paper {a['paper_gkeys_s']}), "
                  f"cbf_contains **{c['gkeys_s']}** (paper {c['paper_gkeys_s']}).")
            if size == "32MB":
                print("Contains issues k=16 independent random 4-byte loads per key, so it is bound by the "
                      "L1->XBAR request rate (~290 G requests/s / 16 = 18 G keys/s); the paper's 42.64 is not "
                      "reachable with 16 independent requests per key on this chip.")
            print()
    if ablation:
        rows = [json.loads(line) for line in open(ablation)]
        print(f"## Optimisation breakdown (P:L430-442; `{os.path.basename(ablation)}`)\n")
        print("SBF 256/64 k=16, 2^28 keys, G keys/s.\n")
        print("| step | layout | 32 MiB add | 32 MiB contains | 1 GiB add | 1 GiB contains |")
        print("|---|---|---|---|---|---|")
        keys = []
        for r in rows:
            k = (r["step"], r.get("layout", ""))
            if k not in keys:
                keys.append(k)
        for k in keys:
            def cell(size, op):
                for r in rows:
                    if (r["step"], r.get("layout", "")) == k and r["size"] == size:
                        return f"{r[op]}"
                return "—"
            print(f"| {k[0]} | {k[1]} | {cell('32MB', 'add')} | {cell('32MB', 'contains')} | "
                  f"{cell('1GB', 'add')} | {cell('1GB', 'contains')} |")
        print()


if __name__ == "__main__":
    main(*sys.argv[1:3])
