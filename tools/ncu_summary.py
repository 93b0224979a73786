#!/usr/bin/env python
"""Summarise ncu output into profiles/ (tracked).

    python tools/ncu_summary.py launches gpurun_out/launches_r1.csv  > profiles/r1_launches.md
    python tools/ncu_summary.py full gpurun_out/prof_r1.ncu-rep [N_KEYS] > profiles/r1_ncu_full.md
"""
from __future__ import annotations

import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("launch__registers_per_thread", "registers/thread"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1TEX throughput %"),
    ("l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed", "L1->XBAR request cycles %"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "L1 LSU data wavefronts %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("lts__t_tag_requests.avg.pct_of_peak_sustained_elapsed", "L2 tag requests %"),
    ("lts__t_requests_srcunit_tex_op_read.sum", "L2 read requests"),
    ("lts__t_requests_srcunit_tex_op_red.sum", "L2 RED requests"),
    ("lts__t_sectors_srcunit_tex_op_red.sum", "L2 RED sectors"),
    ("lts__t_sector_hit_rate.pct", "L2 sector hit rate %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    d = defaultdict(list)
    for r in rows[hi + 1:]:
        d[r[ki]].append(float(r[vi].replace(",", "")) * (1e-3 if r[ui] == "ns" else 1.0))
    tot = sum(sum(v) for v in d.values())
    print(f"# ncu launch list: {path}\n")
    print("Per-launch gpu__time_duration (cold-cache, serialised by ncu; compare shares, not absolutes).\n")
    print("| kernel | launches | mean us | total us | share |")
    print("|---|---|---|---|---|")
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        print(f"| `{k[:110]}` | {len(v)} | {sum(v) / len(v):.1f} | {sum(v):.1f} | {100 * sum(v) / tot:.1f}% |")


PER_KEY = [  # (metric, label, multiplier): per-key evidence (SURVEY 8(d) "ncu evidence per design choice")
    ("smsp__inst_executed.sum", "thread instructions / key", 32),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "L1 global-load requests (warp instructions) / key", 1),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "L1 global-load sectors / key", 1),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_red.sum", "L1 RED requests (warp instructions) / key", 1),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_red.sum", "L1 RED sectors / key", 1),
    ("lts__t_requests_srcunit_tex_op_read.sum", "L2 read requests / key", 1),
    ("lts__t_requests_srcunit_tex_op_red.sum", "L2 RED requests / key (1.0 = Θ lanes coalesced into one request)", 1),
    ("lts__t_sectors_srcunit_tex_op_red.sum", "L2 RED sectors / key", 1),
    ("dram__bytes_read.sum", "DRAM bytes read / key", 1),
    ("dram__bytes_write.sum", "DRAM bytes written / key", 1),
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "inst": 1, "request": 1, "sector": 1}


def full(path, n_keys=None):
    """n_keys: one count, or "ADD:CONTAINS" (per-key rows use the launch's own count)."""
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    print(f"# ncu --set full summary: {path}\n")
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        print(f"## `{name}`\n")
        print("| metric | value |")
        print("|---|---|")
        for key, label in KEYS:
            if key in h:
                i = h.index(key)
                print(f"| {label} (`{key}`) | {r[i]} {units[i]} |")
        if n_keys:
            na, _, nc = str(n_keys).partition(":")
            nk = float(na) if name.rstrip().endswith(", 1>(Params)") else float(nc or na)
            for key, label, mul in PER_KEY:
                if key in h:
                    i = h.index(key)
                    try:
                        v = float(r[i].replace(",", "")) * SCALE.get(units[i], 1) * mul / nk
                    except ValueError:
                        continue
                    print(f"| {label} (n = {int(nk)}) | {v:.3f} |")
        items = []
        for i, c in enumerate(h):
            if c.startswith("smsp__pcsamp_warps_issue_stalled_") and not c.endswith("_not_issued"):
                try:
                    items.append((float(r[i].replace(",", "")), c))
                except ValueError:
                    pass
        tot = sum(v for v, _ in items) or 1.0
        print("\nTop stall reasons (PC sampling):\n")
        for v, c in sorted(items, reverse=True)[:6]:
            print(f"- {c.replace('smsp__pcsamp_warps_issue_stalled_', '')}: {100 * v / tot:.1f}%")
        print()


def traffic(path, n_keys, out_json):
    """profiles/ncu_traffic.json: dram read+write bytes per launch per kernel
    (the `traffic` field of bench.py's roofline object)."""
    import json
    import os
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    acc = defaultdict(list)
    for r in rows[2:]:
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        b = float(r[h.index("dram__bytes_read.sum")].replace(",", "")) * scale[rows[1][h.index("dram__bytes_read.sum")]] + \
            float(r[h.index("dram__bytes_write.sum")].replace(",", "")) * scale[rows[1][h.index("dram__bytes_write.sum")]]
        acc[r[h.index("Kernel Name")]].append(b)
    old = json.load(open(out_json)) if os.path.exists(out_json) else {"kernels": {}}
    old["source"] = "ncu --set full captures (dram__bytes_read.sum + dram__bytes_write.sum per launch), one entry per kernel and key count"
    # n_keys: one count for every kernel, or "ADD:CONTAINS" (bulk_kernel<..., 1> is add)
    na, _, nc = str(n_keys).partition(":")
    nc = nc or na
    for k, v in acc.items():
        n = int(na) if k.rstrip().endswith(", 1>(Params)") else int(nc)
        old["kernels"][f"{k} [n={n}]"] = {"dram_bytes_per_launch": sum(v) / len(v), "n": n,
                                          "dram_bytes_per_key": sum(v) / len(v) / n,
                                          "capture": os.path.basename(path)}
    json.dump(old, open(out_json, "w"), indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "traffic":
        traffic(sys.argv[2], sys.argv[3], sys.argv[4])
    else:
        {"launches": launches, "full": full}[sys.argv[1]](*sys.argv[2:])
