#!/usr/bin/env python
"""Per-instruction view of an ncu capture (SASS page): instruction mix
weighted by executed warp instructions, and the hottest instructions by
stall samples.  python tools/ncu_sass_hot.py REP [N_KEYS] [TOP]"""
import csv
import io
import subprocess
import sys
from collections import Counter


def main():
    rep = sys.argv[1]
    nkeys = float(sys.argv[2]) if len(sys.argv) > 2 else None
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    lines = raw.splitlines()
    kernels = []
    cur = None
    for ln in lines:
        if ln.startswith('"Kernel Name"'):
            cur = [ln]
            kernels.append(cur)
        elif cur is not None:
            cur.append(ln)
    for block in kernels:
        name = next(csv.reader(io.StringIO(block[0])))[1]
        rows = list(csv.reader(io.StringIO("\n".join(block[1:]))))
        h = rows[0]
        iS, iW, iT = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Thread Instructions Executed")
        mix, samples = Counter(), []
        tot_t = tot_s = 0
        for r in rows[1:]:
            if len(r) <= iT:
                continue
            op = r[iS].strip().split()[0] if r[iS].strip() else "?"
            if op.startswith("@"):
                op = r[iS].strip().split()[1]
            op = op.split(".")[0]
            t = float(r[iT] or 0)
            s = float(r[iW] or 0)
            mix[op] += t
            tot_t += t
            tot_s += s
            samples.append((s, r[iS].strip(), t))
        print(f"## `{name[:140]}`\n")
        scale = nkeys if nkeys else 1.0
        unit = "thread instructions / key" if nkeys else "thread instructions"
        print(f"total {tot_t / scale:.1f} {unit}\n")
        print("| opcode | " + unit + " | share |\n|---|---|---|")
        for op, t in mix.most_common(18):
            print(f"| {op} | {t / scale:.2f} | {100 * t / tot_t:.1f}% |")
        print(f"\nHottest instructions (share of {int(tot_s)} stall samples):\n")
        for s, src, t in sorted(samples, reverse=True)[:top]:
            print(f"- {100 * s / max(tot_s, 1):5.1f}%  `{src}`")
        print()


if __name__ == "__main__":
    main()
