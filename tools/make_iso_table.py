#!/usr/bin/env python
"""Write profiles/iso_fpr_table.json: for every configs[1] sweep row (and the
configs[2]/[3] variants) the bits-per-key c_iso at the target FPR and the
exact-model FPR at the resulting load, from the oracle's exact ideal-hash
model (oracle/fpr_model.py).  Stored expected values come
only from this script, which calls only oracle/.

    python tools/make_iso_table.py
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import fpr_model as M  # noqa: E402

BBF, RBBF, SBF, CSBF = 1, 2, 3, 4
ROWS = [(RBBF, 32, 32, 0), (RBBF, 64, 64, 0), (SBF, 64, 32, 0), (SBF, 128, 64, 0),
        (SBF, 128, 32, 0), (SBF, 256, 64, 0), (SBF, 256, 32, 0), (BBF, 128, 64, 0),
        (BBF, 256, 64, 0), (CSBF, 256, 32, 2), (CSBF, 256, 32, 4), (CSBF, 256, 64, 2)]


def valid(v, B, S, k, z):
    s = B // S
    return not ((v == SBF and k % s) or (v == CSBF and k % z))


def n_iso(v, B, S, k, z, m_bits, target):
    """Largest n with exact-model FPR <= target (bisection on n)."""
    b = m_bits // B
    lo, hi = 1, m_bits // 2
    while hi - lo > max(1, lo // 20000):
        mid = (lo + hi) // 2
        if M.fpr_exact(v, mid, b, B, S, k, z) <= target:
            lo = mid
        else:
            hi = mid
    return lo


# the sweep's 3 extra rows (gen_instances.C2_EXTRA): one-word BBF, BBF with 32-bit words
EXTRA = [(BBF, 64, 64, 8, 0), (BBF, 256, 32, 8, 0), (BBF, 256, 32, 11, 0)]
# configs[2]: the five variants compared at 8 GiB / 2^32 keys
C3 = [(RBBF, 64, 64, 6, 0), (SBF, 256, 64, 8, 0), (CSBF, 256, 32, 8, 4), (CSBF, 256, 32, 8, 2), (BBF, 256, 64, 8, 0)]


def main():
    path = os.path.join(ROOT, "profiles", "iso_fpr_table.json")
    if "--add-missing" in sys.argv and os.path.exists(path):
        out = json.load(open(path))
        have = {(r["variant"], r["B"], r["S"], r["k"], r["z"]) for r in out["c2"]["rows"]}
        m = out["c2"]["m_bits"]
        for v, B, S, k, z in EXTRA:
            if (v, B, S, k, z) in have:
                continue
            n = n_iso(v, B, S, k, z, m, 1e-3)
            out["c2"]["rows"].append({"variant": v, "B": B, "S": S, "k": k, "z": z, "n_iso": n,
                                      "c_iso": m / n, "fpr_model": M.fpr_exact(v, n, m // B, B, S, k, z),
                                      "fill_model": M.fill_exact(v, n, m // B, B, S, k, z)})
            print("extra", v, B, S, k, z, n, flush=True)
        m3, n3 = 1 << 36, 1 << 32
        out["c3"] = {"m_bits": m3, "n": n3, "rows": []}
        for v, B, S, k, z in C3:
            f = M.fpr_exact(v, n3, m3 // B, B, S, k, z)
            out["c3"]["rows"].append({"variant": v, "B": B, "S": S, "k": k, "z": z, "fpr_model": f,
                                      "fill_model": M.fill_exact(v, n3, m3 // B, B, S, k, z)})
            print("c3", v, B, S, k, z, f, flush=True)
        json.dump(out, open(path, "w"), indent=1)
        print("wrote", path)
        return
    out = {"_source": "tools/make_iso_table.py (oracle/fpr_model.py exact ideal-hash model)",
           "c2": {"m_bits": 1 << 28, "target_fpr": 1e-3, "rows": []}}
    m = 1 << 28
    for v, B, S, z in ROWS:
        for k in range(4, 17):
            if not valid(v, B, S, k, z):
                continue
            n = n_iso(v, B, S, k, z, m, 1e-3)
            f = M.fpr_exact(v, n, m // B, B, S, k, z)
            out["c2"]["rows"].append({"variant": v, "B": B, "S": S, "k": k, "z": z, "n_iso": n,
                                      "c_iso": m / n, "fpr_model": f,
                                      "fill_model": M.fill_exact(v, n, m // B, B, S, k, z)})
            print(v, B, S, k, z, n, round(m / n, 2), f, flush=True)
    # configs[3]: SBF 256/32 at FPR 1e-4, c_iso for a large filter (b = 2^20 blocks)
    out["c4"] = {"target_fpr": 1e-4, "rows": []}
    for k in (8, 16):
        n = n_iso(SBF, 256, 32, k, 0, 256 << 20, 1e-4)
        out["c4"]["rows"].append({"variant": SBF, "B": 256, "S": 32, "k": k, "z": 0,
                                  "c_iso": (256 << 20) / n})
        print("c4", k, (256 << 20) / n, flush=True)
    path = os.path.join(ROOT, "profiles", "iso_fpr_table.json")
    json.dump(out, open(path, "w"), indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
