"""Schedule autotuning: the paper's grid search over layouts, at run time.

The paper picks, per filter configuration, the (Θ, Φ) layout that runs
fastest (Tables 1-2: every Θ with Φ = s/Θ).  The library's
defaults are rules distilled from those tables (bf_create); `autotune` instead
times every schedule compiled for the filter's (variant, B, S, k, z) -- each
valid (Θ, Φ) with Θ·Φ <= s and KPT in {1, 2, 4} (hash variant 0) -- on
synthetic keys of the caller's batch size and keeps the fastest.  Results do
not depend on the schedule (every compiled schedule is bit-exact with the
oracle), so this only changes speed.

Argument marshalling and timing only: the kernels are the library's.
"""
from __future__ import annotations

import statistics

from . import bf, layout


def candidate_layouts(s: int):
    """Every (Θ, Φ, KPT) the ABI accepts for a block of s words (the layout
    algebra of layout.py; KPT 1/2/4)."""
    return [(t, p, kpt) for t, p in layout.enumerate_layouts(s) for kpt in (1, 2, 4)]


def autotune(f: "bf.Filter", op: int, n: int = 1 << 24, reps: int = 5, allow_clear: bool = False,
             stream=None) -> dict:
    """Time every compiled schedule of `op` (0 add, 1 contains) on `n`
    synthetic keys and set the fastest on `f`.

    contains leaves the filter unchanged.  add writes into the filter, so it
    needs `allow_clear=True`: the filter is cleared before every timed add and
    after tuning (tune an empty filter, or a scratch filter of the same
    geometry).  Returns {"layout": (Θ, Φ, KPT), "gkeys_s": rate, "tried":
    {layout: rate}}."""
    import torch
    if op == 0 and not allow_clear:
        raise ValueError("tuning add writes into the filter: pass allow_clear=True (the filter is cleared)")
    dev = torch.device("cuda", torch.cuda.current_device())
    keys = torch.empty(n, dtype=torch.int64, device=dev)
    bf.bf_keygen(keys, n, 0x7A5E << 40, stream)  # synthetic keys (DESIGN.md section 5 generator)
    out = torch.empty((n + 31) // 32, dtype=torch.int32, device=dev)
    st = torch.cuda.current_stream() if stream is None else stream
    before = f.layout(op)
    tried = {}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for lay in candidate_layouts(f.s):
        try:
            f.set_layout(op, *lay, 0)
        except bf.BFError:
            continue  # not compiled for this configuration
        ts = []
        for r in range(reps + 1):
            if op == 0:
                f.clear(st)
            e0.record(st)
            if op == 0:
                f.add(keys, st)
            else:
                f.contains(keys, out, st)
            e1.record(st)
            e1.synchronize()
            if r:
                ts.append(e0.elapsed_time(e1))
        tried[lay] = n / (statistics.median(ts) * 1e-3) / 1e9
    if op == 0:
        f.clear(st)
    if not tried:  # nothing specialized: keep what bf_create chose (the generic kernel)
        return {"layout": (before["theta"], before["phi"], before["kpt"]), "gkeys_s": None, "tried": {}}
    best = max(tried, key=tried.get)
    f.set_layout(op, *best, 0)
    return {"layout": best, "gkeys_s": tried[best], "tried": tried}
