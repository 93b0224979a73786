"""bench.py's host-side helpers on the CPU: the FPR count over a bit range,
the false-negative guard, the workload resolution (iso-FPR load from the
oracle-written table), the probes' access rounding and the roofline object."""
import importlib.util
import os
import random

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


B = _bench()


def test_popcount_bits_matches_numpy():
    rng = np.random.default_rng(3)
    words = rng.integers(0, 2**32, 1000, dtype=np.uint64).astype(np.uint32)
    t = torch.from_numpy(words.view(np.int32).copy())
    bits = np.unpackbits(words.view(np.uint8), bitorder="little")
    for _ in range(200):
        lo = random.randrange(0, 32000)
        hi = random.randrange(lo, 32001)
        assert B.popcount_bits(torch, t, lo, hi) == int(bits[lo:hi].sum()), (lo, hi)


def test_check_positives():
    n = 1000
    out = torch.full(((n + 31) // 32,), -1, dtype=torch.int32)
    out[-1] = (1 << (n % 32)) - 1  # tail bits past n are zero
    assert B.check_positives(torch, out, n)
    out[5] = out[5] & ~(1 << 7)
    assert not B.check_positives(torch, out, n)
    out[5] = -1
    out[-1] = (1 << (n % 32)) - 2  # first key of the last word missing
    assert not B.check_positives(torch, out, n)


def test_default_workload_is_configs1_at_iso_fpr():
    cfg = B.resolve("c2")
    assert cfg["m_bits"] == 1 << 28 and (cfg["variant"], cfg["B"], cfg["S"], cfg["k"]) == ("SBF", 256, 64, 8)
    # n_iso from profiles/iso_fpr_table.json (written from oracle/ only), a multiple of 128
    assert cfg["n"] == 15973888 and cfg["n_neg"] == cfg["n"] and cfg["n"] % 128 == 0
    assert abs(cfg["iso"]["fpr_model"] - 1e-3) < 1e-5
    c3 = B.resolve("c3")
    assert c3["n"] == 1 << 32 and c3["n_neg"] == 1 << 28 and c3["residency"] == "HBM"


def test_rng_probe_access_rounding_and_roofline_fields():
    assert B._rng_accesses(100, 64) == 128 and B._rng_accesses(128, 64) == 128
    r = B.kernel_roofline("bf_contains", 200.0, 250.0, "probe", 256)
    assert r["bound"] == "l2" and r["unit"] == "GB/s" and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    assert r["algorithmic_bytes_per_key"] == 32


def test_phase_rooflines():
    """Each binned phase against its own bound: streaming phases divide the
    algorithmic bytes rate by the copy peak, the per-range phases their key
    rate by the range probe; phases without a timed span are left out."""
    cfg = {"n": 1 << 32, "n_neg": 1 << 28}
    phases = {"bin": (20.0, 2), "apply": (35.0, 2), "bin_slots": (25.0, 3), "lookup": (22.0, 3), "unbin": (0.0, 0)}
    probes = {"apply_range": {"range_mib": 32, "forms": {"red_rng@32": 128.0}, "best": 128.0, "best_form": "red_rng@32"},
              "lookup_range": {"range_mib": 64, "forms": {"read_rng@32": 270.0}, "best": 270.0,
                               "best_form": "read_rng@32"}}
    r = B.phase_rooflines(phases, probes, cfg, 6500.0)
    assert set(r) == {"bin", "apply", "bin_slots", "lookup"}
    g_bin = (1 << 32) / 20e-3 / 1e9
    assert abs(r["bin"]["achieved_gkeys_s"] - round(g_bin, 3)) < 1e-3
    assert abs(r["bin"]["frac"] - round(g_bin * 16 / 6500.0, 4)) < 1e-4 and r["bin"]["bound"] == "hbm"
    g_app = (1 << 32) / 35e-3 / 1e9
    assert r["apply"]["bound"] == "l2" and abs(r["apply"]["frac"] - round(g_app / 128.0, 4)) < 1e-4
    g_look = ((1 << 32) + (1 << 28)) / 22e-3 / 1e9
    assert abs(r["lookup"]["frac"] - round(g_look / 270.0, 4)) < 1e-4
    assert abs(r["bin_slots"]["frac"] - round(((1 << 32) + (1 << 28)) / 25e-3 / 1e9 * 20 / 6500.0, 4)) < 1e-4
