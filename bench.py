#!/usr/bin/env python
"""Benchmark of the bulk add / contains hot path (arXiv 2512.15595) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c2|c2n|c1|c3|c5] [--variant SBF --B 256 --S 64 --k 8 --z 0]

One step = one pass of the whole hot path over one batch of synthetic keys
resident in HBM:
    bf_clear -> bf_add(n_add positives) -> [N>1: OR-merge of the partial filters]
             -> bf_contains(the n_add positives + n_neg negatives)
(N=1: the step is captured once in a CUDA graph and replayed; per-kernel times
come from eager steps with CUDA events on the launching stream).

Default workload (the headline `value`): BASELINE.json configs[1] at iso FPR --
the 32 MiB L2-resident SBF 256/64 k=8 filter loaded with n_iso = 15,973,888
keys, the count at which the exact ideal-hash model gives FPR 1e-3
(profiles/iso_fpr_table.json, written from oracle/ only; reading 14:
2^26 keys in 32 MiB is 4 bits/key, FPR 16%), contains on those n_iso
positives plus n_iso negatives (positives + negatives).  The
FPR is measured from the timed contains' own output on the negatives.
value = (add keys + contains keys) over all ranks / max-over-ranks time.

Two more legs in the same line at N=1: `hbm` = configs[2] at full size (8 GiB
HBM-resident filter, 2^32 keys added, 2^32 positives + 2^28 negatives looked
up), and `fixed_load` = configs[1] as literally written (2^26 keys into the
32 MiB filter, 4 bits/key).  Each leg carries its own live roofline probes.

Rank 0 prints one JSON line.  `--impl reference` times the CPU oracle (the
only reference that exists: the paper released no code) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

NEG_BASE = 1 << 62  # negative key indices (synth.NEG_BASE)

CONFIGS = {
    # BASELINE.json configs[1] at iso FPR 1e-3 (the default): 32 MiB, n_iso keys
    "c2": dict(workload="configs[1] at iso FPR 1e-3: L2-resident 32 MiB filter, SBF B=256 S=64 k=8, "
                        "n_iso keys added (exact model), contains on n_iso positives + n_iso negatives",
               m_bits=1 << 28, n="iso", neg="same", variant="SBF", B=256, S=64, k=8, z=0, residency="L2"),
    # configs[1] as written: 2^26 keys (4 bits/key), 2^26 positives + 2^26 negatives
    "c2n": dict(workload="configs[1] fixed load: L2-resident 32 MiB filter, 2^26 keys (4 bits/key), SBF B=256 S=64 "
                         "k=8, contains on 2^26 positives + 2^26 negatives",
                m_bits=1 << 28, n=1 << 26, neg="same", variant="SBF", B=256, S=64, k=8, z=0, residency="L2"),
    # configs[0]: 2 MiB filter, 2^20 keys (the oracle's seconds-scale case).
    "c1": dict(workload="configs[0]: 16 Mbit filter, 2^20 keys, SBF B=256 S=64 k=8, 2^20 positives + 2^20 negatives",
               m_bits=1 << 24, n=1 << 20, neg="same", variant="SBF", B=256, S=64, k=8, z=0, residency="L2"),
    # configs[2]: HBM-resident 8 GiB filter, 2^32 keys (16 bits/key, model FPR 1.28e-3); FPR on 2^28 negatives
    "c3": dict(workload="configs[2]: HBM-resident 8 GiB filter, 2^32 keys, SBF B=256 S=64 k=8, contains on 2^32 "
                        "positives + 2^28 negatives",
               m_bits=1 << 36, n=1 << 32, neg=1 << 28, variant="SBF", B=256, S=64, k=8, z=0, residency="HBM"),
    # configs[4]: one rank's share of the 8-GPU job -- a 32 GiB replica and
    # 2^34 / 8 = 2^31 keys per rank (weak scaling).
    "c5": dict(workload="configs[4] per rank: 32 GiB replica, 2^31 keys per rank (2^34 at 8 GPUs), SBF B=256 S=64 "
                        "k=8, contains on the rank's positives + 2^27 negatives",
               m_bits=1 << 38, n=1 << 31, neg=1 << 27, variant="SBF", B=256, S=64, k=8, z=0, residency="HBM"),
}

VARIANT_IDS = {"BBF": 1, "RBBF": 2, "SBF": 3, "CSBF": 4}

# BASELINE.json "metric" (both arms report it; config.workload names the configuration)
METRIC = "bulk add & contains Gkeys/s at iso-FPR (L2-/HBM-resident), % of roofline"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c2")
    ap.add_argument("--variant", default=None)
    ap.add_argument("--B", type=int, default=None)
    ap.add_argument("--S", type=int, default=None)
    ap.add_argument("--k", type=int, default=None)
    ap.add_argument("--z", type=int, default=None)
    ap.add_argument("--n", type=int, default=None, help="keys added per rank (override)")
    ap.add_argument("--m-bits", dest="m_bits", type=int, default=None, help="filter bits (override)")
    ap.add_argument("--range-mib", type=int, default=0, help="binned add: filter MiB per range (0: library default)")
    ap.add_argument("--l2-fetch", type=int, default=0, help="cudaLimitMaxL2FetchGranularity for the run (0: default)")
    ap.add_argument("--merge", choices=["alltoall", "allgather", "nvls", "p2p", "route"], default="alltoall")
    ap.add_argument("--add-mode", choices=["auto", "direct", "binned"], default="auto")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-probe", action="store_true")
    ap.add_argument("--no-hbm", action="store_true", help="skip the configs[2] HBM leg")
    ap.add_argument("--no-fixed", action="store_true", help="skip the configs[1] fixed-load leg")
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="time eager launches instead of replays of one captured step (CUDA graph, N=1 default)")
    a = ap.parse_args()
    a.warmup = max(3, a.warmup)
    return a, resolve(a.config, a)


def resolve(name, a=None):
    """Concrete workload of a config (+ command-line overrides)."""
    cfg = dict(CONFIGS[name])
    cfg["name"] = name
    if a is not None:
        for key in ("variant", "B", "S", "k", "z", "n", "m_bits"):
            if getattr(a, key, None) is not None:
                cfg[key] = getattr(a, key)
    cfg["iso"] = None
    if cfg["n"] == "iso":
        row = iso_row(cfg)
        if row is None:
            raise SystemExit(f"no iso-FPR row for {cfg}: pass --n")
        cfg["iso"] = row
        cfg["n"] = int(row["n_iso"]) // 128 * 128
    cfg["n_neg"] = cfg["n"] if cfg["neg"] == "same" else int(cfg["neg"])
    return cfg


def iso_row(cfg):
    """The exact-model iso-FPR row (profiles/iso_fpr_table.json, written by
    tools/make_iso_table.py from oracle/ only) for this geometry."""
    try:
        tab = json.load(open(os.path.join(ROOT, "profiles", "iso_fpr_table.json")))["c2"]
    except (OSError, KeyError):
        return None
    if tab.get("m_bits") != cfg["m_bits"]:
        return None
    vid = VARIANT_IDS[cfg["variant"]]
    row = next((r for r in tab["rows"] if (r["variant"], r["B"], r["S"], r["k"], r["z"]) ==
                (vid, cfg["B"], cfg["S"], cfg["k"], cfg["z"])), None)
    if row is not None:
        row = dict(row, target_fpr=tab["target_fpr"])
    return row


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d.get("hbm_gbs", 6650.0)), "measured", d
    return 6650.0, "fallback", {}


class ClockSampler:
    """SM clock, power and throttle reasons sampled DURING the measured region
    (NVML in-process every 5 ms; nvidia-smi as a fallback).  mark() starts the
    timed sub-window, so the summary reports samples inside it separately."""
    BITS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
            "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, local_rank: int):
        self.local_rank = local_rank
        self.rows = []  # (t, sm_mhz, max_mhz, power_w, reasons set)
        self.t_mark = None
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml
            import torch
            pynvml.nvmlInit()
            pr = torch.cuda.get_device_properties(local_rank)
            try:
                bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
                h = pynvml.nvmlDeviceGetHandleByPciBusId(bus.encode())
            except Exception:
                h = pynvml.nvmlDeviceGetHandleByIndex(local_rank)
            self._nvml = (pynvml, h)
        except Exception:
            self._nvml = None

    def _sample_nvml(self):
        nv, h = self._nvml
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        pw = nv.nvmlDeviceGetPowerUsage(h) / 1000.0
        try:
            bits = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        except Exception:
            bits = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
        return (float(sm), float(mx), pw, {k for k, v in self.BITS.items() if bits & v})

    def _sample_smi(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        out = subprocess.run(["nvidia-smi", f"--id={self.local_rank}", f"--query-gpu={q}",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True,
                             timeout=5).stdout.strip().split(",")
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        return (float(out[0]), float(out[1]), float(out[2]),
                {names[i] for i in range(4) if out[3 + i].strip() == "Active"})

    def _run(self):
        while not self._stop.is_set():
            try:
                r = self._sample_nvml() if self._nvml else self._sample_smi()
                self.rows.append((time.perf_counter(),) + r)
            except Exception:
                pass
            self._stop.wait(0.005 if self._nvml else 0.1)

    def mark(self):
        self.t_mark = time.perf_counter()

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        rows = self.rows
        timed = [r for r in rows if self.t_mark is not None and r[0] >= self.t_mark]
        return {"sm_mhz": statistics.median(r[1] for r in rows),
                "sm_max_mhz": max(r[2] for r in rows),
                "reasons": sorted(set().union(*(r[4] for r in rows))),
                "samples": len(rows), "samples_in_timed_region": len(timed),
                "sm_mhz_timed_region": statistics.median(r[1] for r in timed) if timed else None,
                "power_w_max": max(r[3] for r in rows),
                "window": "untimed graph replays (>= 0.3 s clock soak) + the timed region",
                "source": "nvml" if self._nvml else "nvidia-smi"}


# --------------------------------------------------------------------- reference
def run_reference(a, cfg, rank, world):
    """The CPU oracle as it stands, on the host cores, on the same workload
    (the paper published no code)."""
    if rank != 0:
        return
    import numpy as np

    import synth
    from oracle.bfo import OracleFilter

    cores = os.cpu_count() or 1
    v = VARIANT_IDS[cfg["variant"]]
    sample = min(cfg["n"], 1 << 26)
    nneg = min(cfg["n_neg"], sample)
    keys = synth.positives(sample)
    q = np.concatenate([keys, synth.negatives(nneg)])
    f = OracleFilter(v, cfg["m_bits"], B=cfg["B"], S=cfg["S"], k=cfg["k"], z=cfg["z"])
    f.add(keys[:4096], threads=cores)  # warm the page tables
    for _ in range(max(1, a.warmup // 3)):
        f.add(keys[:1 << 16], threads=cores)
    times = []
    for _ in range(min(a.steps, 10)):
        t0 = time.perf_counter()
        f.add(keys, threads=cores)
        f.contains(q, threads=cores)
        times.append(time.perf_counter() - t0)
    t = statistics.median(times)
    value = (sample + q.size) / t / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "Gkeys/s",
        "n_gpus": world, "steps": len(times), "warmup": a.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": config_block(cfg, world, extra={"keys_per_rank": sample, "negatives_per_rank": nneg,
                                                   "parallelism": f"CPU oracle, {cores} host threads"}),
        "cpu_baseline": {"value": value, "unit": "Gkeys/s", "cores": cores, "kind": "oracle",
                         "sample": f"add {sample} + contains {q.size} keys ({sample} positives + {nneg} negatives) "
                                   "of the same workload (filter at full size)"},
        "e2e": {"value": value, "unit": "Gkeys/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(cfg):
    import numpy as np

    import synth
    from oracle.bfo import OracleFilter
    cores = os.cpu_count() or 1
    v = VARIANT_IDS[cfg["variant"]]
    sample = min(cfg["n"], 1 << 26)
    nneg = min(cfg["n_neg"], sample)
    keys = synth.positives(sample)
    q = np.concatenate([keys, synth.negatives(nneg)])
    f = OracleFilter(v, cfg["m_bits"], B=cfg["B"], S=cfg["S"], k=cfg["k"], z=cfg["z"])
    f.add(keys[:1 << 16], threads=cores)
    t0 = time.perf_counter()
    f.add(keys, threads=cores)
    f.contains(q, threads=cores)
    t = time.perf_counter() - t0
    # one thread (T=1 and T=all host cores), a 2^22-key sample
    s1 = min(sample, 1 << 22)
    g = OracleFilter(v, cfg["m_bits"], B=cfg["B"], S=cfg["S"], k=cfg["k"], z=cfg["z"])
    t1 = time.perf_counter()
    g.add(keys[:s1], threads=1)
    g.contains(keys[:s1], threads=1)
    t1 = time.perf_counter() - t1
    return {"value": (sample + q.size) / t / 1e9, "unit": "Gkeys/s", "cores": cores, "kind": "oracle",
            "sample": f"add {sample} + contains {q.size} keys ({sample} positives + {nneg} negatives) of the same "
                      f"workload (full-size filter), {t:.2f} s on {cores} threads",
            "single_thread": {"value": 2 * s1 / t1 / 1e9, "unit": "Gkeys/s",
                              "sample": f"add {s1} + contains {s1} keys, {t1:.2f} s on 1 thread"},
            "host_cpu": _cpu_model()}


def _cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def config_block(cfg, world, extra=None):
    out = {"workload": cfg["workload"], "variant": cfg["variant"], "B": cfg["B"], "S": cfg["S"], "k": cfg["k"],
           "z": cfg["z"], "m_bits": cfg["m_bits"], "keys_added_per_rank": cfg["n"],
           "negatives_per_rank": cfg["n_neg"], "keys_per_step": (2 * cfg["n"] + cfg["n_neg"]) * world,
           "bits_per_key": round(cfg["m_bits"] / (cfg["n"] * world), 3)}
    if cfg.get("iso"):
        out["iso_fpr"] = {"target": cfg["iso"]["target_fpr"], "n_iso": cfg["iso"]["n_iso"],
                          "fpr_exact_model": cfg["iso"]["fpr_model"], "source": "profiles/iso_fpr_table.json"}
    out.update(extra or {})
    return out


# --------------------------------------------------------------------- ours
def popcount_bits(torch, words, lo_bit, hi_bit):
    """Number of set bits in [lo_bit, hi_bit) of a packed LSB-first int32
    tensor (bit i = bit i%8 of byte i/8 on this little-endian layout),
    counted on the device with a 256-entry table."""
    if hi_bit <= lo_bit:
        return 0
    by = words.view(torch.uint8)
    lut = torch.tensor([bin(i).count("1") for i in range(256)], dtype=torch.int32, device=by.device)
    seg = by[lo_bit // 8:(hi_bit + 7) // 8]
    tot = 0
    for c in range(0, seg.numel(), 1 << 26):  # bounded temporaries
        tot += int(lut[seg[c:c + (1 << 26)].long()].sum().item())
    if lo_bit % 8:
        tot -= bin(int(seg[0].item()) & ((1 << (lo_bit % 8)) - 1)).count("1")
    if hi_bit % 8:
        tot -= bin(int(seg[-1].item()) >> (hi_bit % 8)).count("1")
    return tot


def check_positives(torch, out, n_pos):
    """Every inserted key must be found (no false negatives): the
    first n_pos result bits are all set."""
    full = n_pos // 32
    if full and int((out[:full] != -1).sum().item()) != 0:
        return False
    if n_pos % 32:
        mask = (1 << (n_pos % 32)) - 1
        if (int(out[full].item()) & 0xFFFFFFFF) & mask != mask:
            return False
    return True


class Leg:
    """One workload: filter, keys on the device, the step, its timing."""

    def __init__(self, bf, torch, cfg, a, rank, world, dev, bfdist=None):
        self.bf, self.torch, self.cfg, self.a = bf, torch, cfg, a
        self.rank, self.world, self.dev, self.bfdist = rank, world, dev, bfdist
        n, nneg = cfg["n"], cfg["n_neg"]
        self.f = bf.Filter(cfg["m_bits"], cfg["k"], cfg["B"], cfg["S"], cfg["variant"], z=cfg["z"])
        self.f.set_add_mode({"auto": bf.BF_ADD_AUTO, "direct": bf.BF_ADD_DIRECT,
                             "binned": bf.BF_ADD_BINNED}[a.add_mode], a.range_mib << 20)
        # one query array: positives (this rank's shard, also the add input) then negatives
        self.q = torch.empty(n + nneg, dtype=torch.int64, device=dev)
        bf.bf_keygen(self.q[:n], n, rank * n)
        bf.bf_keygen(self.q[n:], nneg, NEG_BASE + rank * nneg)
        self.keys = self.q[:n]
        self.out = torch.empty((n + nneg + 31) // 32, dtype=torch.int32, device=dev)
        self.stream = torch.cuda.current_stream()
        self.pf = None
        if world > 1 and a.merge == "route":  # E3: route keys to block-range owners, gather the ranges
            self.pf = bfdist.PartitionedFilter(cfg["m_bits"], cfg["k"], cfg["B"], cfg["S"],
                                               VARIANT_IDS[cfg["variant"]], z=cfg["z"])

    def step(self, ev=None):
        f = self.f
        if ev:
            ev[0].record(self.stream)
        f.clear()
        if self.pf is not None:
            self.pf.clear()
        if ev:
            ev[1].record(self.stream)
        if self.pf is not None:
            self.pf.add(self.keys)
        else:
            f.add(self.keys)
        if ev:
            ev[2].record(self.stream)
        if self.pf is not None:
            self.pf.gather_into(f.data(), self.cfg["B"] // 8)
        elif self.world > 1:
            self.bfdist.MERGES[self.a.merge](f.data())
        if ev:
            ev[3].record(self.stream)
        f.contains(self.q, self.out)
        if ev:
            ev[4].record(self.stream)

    def run(self, steps, warmup, graph, clk=None):
        torch, bf = self.torch, self.bf
        for _ in range(warmup):
            self.step()
        torch.cuda.synchronize()
        assert check_positives(torch, self.out, self.cfg["n"]), "false negative in bench output (warm-up)"
        if self.world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()
        n_eager = max(steps, 5)
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(n_eager)]
        t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g = None
        launches_per_step = None
        if graph and self.world == 1:
            # per-kernel times from eager steps, then the timed region replays
            # one captured step (launch overhead removed)
            for i in range(n_eager):
                self.step(evs[i])
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            cap = torch.cuda.Stream()
            cap.wait_stream(self.stream)
            lc0 = bf.bf_launch_count()
            with torch.cuda.stream(cap):
                with torch.cuda.graph(g, stream=cap):
                    self.step()
            launches_per_step = bf.bf_launch_count() - lc0
            self.stream.wait_stream(cap)
            g.replay()
            torch.cuda.synchronize()
            if clk is not None:  # clock soak: untimed replays for >= 0.3 s under the sampler
                t0 = time.perf_counter()
                while time.perf_counter() - t0 < 0.3:
                    for _ in range(8):
                        g.replay()
                    torch.cuda.synchronize()
        launches0 = bf.bf_launch_count()
        if clk is not None:
            clk.mark()
        t_start.record(self.stream)
        for i in range(steps):
            if g is not None:
                g.replay()
            else:
                self.step(evs[i])
        t_end.record(self.stream)
        torch.cuda.synchronize()
        launches = bf.bf_launch_count() - launches0
        if g is not None:
            launches = launches_per_step * steps  # each replay runs the captured kernels of one step
        assert check_positives(torch, self.out, self.cfg["n"]), "false negative in bench output (timed steps)"
        ms_local = t_start.elapsed_time(t_end) / steps
        used = evs[:n_eager] if g is not None else evs[:steps]
        t = {name: statistics.mean(e[i].elapsed_time(e[i + 1]) for e in used)
             for i, name in enumerate(("clear", "add", "merge", "contains"))}
        per_step = [e[0].elapsed_time(e[4]) for e in used]
        rel = (statistics.stdev(per_step) / statistics.mean(per_step) / len(per_step) ** 0.5
               if len(per_step) > 1 else None)
        ms = ms_local
        if self.world > 1:
            import torch.distributed as dist
            tt = torch.tensor([ms_local], device=self.dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms = float(tt.item())
            dist.barrier()
        n, nneg = self.cfg["n"], self.cfg["n_neg"]
        fp = popcount_bits(torch, self.out, n, n + nneg)
        return {"ms": ms, "t": t, "rel_stderr": rel, "launches": launches, "graph": g is not None,
                "value": (2 * n + nneg) * self.world / (ms * 1e-3) / 1e9,
                "add_gkeys_s": n / (t["add"] * 1e-3) / 1e9,
                "contains_gkeys_s": (n + nneg) / (t["contains"] * 1e-3) / 1e9,
                "fp": fp}

    def phase_pass(self):
        """One eager step with the library's phase timing on, after the timed
        region (bf_set_phase_timing: CUDA events around each binned phase's
        launches on the stream that runs them): {phase: (ms, spans)}."""
        f = self.f
        f.set_phase_timing(True)
        self.step()
        self.torch.cuda.synchronize()
        t = f.phase_times()
        f.set_phase_timing(False)
        return t

    def free(self):
        del self.f, self.q, self.keys, self.out
        self.torch.cuda.empty_cache()


def best_time(torch, fn, reps=5):
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    best = None
    for _ in range(reps):
        e0.record(st)
        fn()
        e1.record(st)
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1)
        best = t if best is None else min(best, t)
    return best


def _rng_accesses(n, unit):
    """The in-register probes run whole iterations of the grid: the number of
    accesses they really make for a request of n."""
    return -(-n // unit) * unit


def run_probes_l2(bf, torch, cfg, dev, n=1 << 26, sizes=None, buf=None):
    """R_read / R_red on a buffer of the filter's size and block geometry
    (SURVEY 8(d) roofline probes), every form measured live on 2^26 keys
    (the asymptotic rate: no launch ramp or tail) and in two launch shapes
    (8 CTAs/SM persistent-style and 32 CTAs/SM waves, the product's shape):
    the key-stream forms (same key loads as the product, no hashing), the
    in-register address forms, for add the configuration's own RED pattern
    (precomputed block + word-hit records: the add's memory traffic without
    hashing) and the LSU+TMA form (half the warps OR whole blocks with
    cp.reduce.async.bulk, half issue RED.64s).  The denominator is the best
    of the forms and shapes (the strictest).

    `sizes` = {"add": n_add, "contains": n_query}: the same forms again at the
    timed kernels' own key counts in the product's launch shape (32 CTAs/SM),
    so that probe and kernel pay the same per-launch costs (CTA start-up of
    the ~4,700 wave CTAs, ramp, tail: ~11 us per launch measured with
    tools/kexp at any n >= 2^23); these are the `roofline` denominators and the
    2^26-key ones are reported beside them (`frac_asymptotic`).

    `buf`: the product filter's own word array (a uint8 view; the probes
    overwrite it after the timed region), so that probe and kernel access the
    same allocation -- the same physical pages, L2 slices and partitions (the
    probes on a fresh allocation of the same size measured up to 5% apart
    from box to box while the product kernels did not)."""
    B = max(64, cfg["B"])
    nbytes = cfg["m_bits"] // 8
    own = buf is not None
    if own:
        assert buf.numel() >= nbytes and buf.dtype == torch.uint8
        buf = buf[:nbytes]
    else:
        buf = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
    keys = torch.empty(n, dtype=torch.int64, device=dev)
    bf.bf_keygen(keys, n, 0)
    out = torch.empty((n + 31) // 32, dtype=torch.int32, device=dev)
    b = nbytes * 8 // B
    lanes = max(1, B // 64)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    recs = torch.empty(n, dtype=torch.int64, device=dev)  # the add's own RED pattern (word-hit records)
    bf.bf_probe_pattern_records(recs, n, nbytes * 8 // cfg["B"], cfg["B"], cfg["S"], VARIANT_IDS[cfg["variant"]],
                                cfg["k"], cfg["z"], 1)
    res = {}
    for cps in (8, 32):
        bf.bf_set_probe_launch(cps)
        thr = sms * cps * 256
        forms = {"read_keys": (lambda: bf.bf_probe_read(buf, b, B, keys, out), n),
                 "red_pattern": (lambda: bf.bf_probe_red_records(buf, cfg["B"], cfg["S"], recs, n), n),
                 "read_rng": (lambda: bf.bf_probe_rng(buf, b, B, 0, 1, n), _rng_accesses(n, thr * 4)),
                 "red_keys": (lambda: bf.bf_probe_red(buf, b, B, lanes, keys), n),
                 "red_rng": (lambda: bf.bf_probe_rng(buf, b, B, 1, lanes, n), _rng_accesses(n, thr // lanes))}
        if B >= 128:
            forms["red_lsu_tma"] = (lambda: bf.bf_probe_rng(buf, b, B, 3, lanes, n), _rng_accesses(n, thr))
        for name, (fn, acc) in forms.items():
            res[f"{name}@{cps}"] = round(acc / (best_time(torch, fn) * 1e-3) / 1e9, 3)
    bf.bf_set_probe_launch(0)
    read = {k: v for k, v in res.items() if k.startswith("read_")}
    red = {k: v for k, v in res.items() if k.startswith("red_")}
    res["read"], res["read_form"] = max(read.values()), max(read, key=read.get)
    res["red"], res["red_form"] = max(red.values()), max(red, key=red.get)
    for op, nk in (sizes or {}).items():
        if nk > n:
            continue
        bf.bf_set_probe_launch(32)
        thr = sms * 32 * 256
        if op == "contains":
            forms = {"read_keys": (lambda: bf.bf_probe_read(buf, b, B, keys[:nk], out), nk),
                     "read_rng": (lambda: bf.bf_probe_rng(buf, b, B, 0, 1, nk), _rng_accesses(nk, thr * 4))}
        else:
            forms = {"red_pattern": (lambda: bf.bf_probe_red_records(buf, cfg["B"], cfg["S"], recs[:nk], nk), nk),
                     "red_keys": (lambda: bf.bf_probe_red(buf, b, B, lanes, keys[:nk]), nk),
                     "red_rng": (lambda: bf.bf_probe_rng(buf, b, B, 1, lanes, nk), _rng_accesses(nk, thr // lanes))}
            if B >= 128:
                forms["red_lsu_tma"] = (lambda: bf.bf_probe_rng(buf, b, B, 3, lanes, nk), _rng_accesses(nk, thr))
        same = {f"{name}@32": round(acc / (best_time(torch, fn) * 1e-3) / 1e9, 3) for name, (fn, acc) in forms.items()}
        res[f"{op}_n"] = nk
        res[f"{op}_same_n"] = same
        res[f"{op}_best_same_n"] = max(same.values())
        res[f"{op}_best_same_n_form"] = max(same, key=same.get)
    bf.bf_set_probe_launch(0)
    res["read_name"] = (f"R_read^L2(B={B}): one {B // 8}-byte block load per key, no hash, 2^26 keys; best of "
                        + " / ".join(f"{k} {v}" for k, v in read.items()) + " Gkeys/s (form@CTAs per SM)")
    res["red_name"] = (f"R_red^L2(B={B}): {lanes} lanes x RED.64 into one block per key, no hash, 2^26 keys; best of "
                       + " / ".join(f"{k} {v}" for k, v in red.items()) + " Gkeys/s (form@CTAs per SM)")
    res["buffer"] = "the product filter's own allocation" if own else "a fresh allocation of the filter's size"
    del buf, keys, out, recs
    torch.cuda.empty_cache()
    return res


def run_probes_hbm(bf, torch, cfg, n):
    """The HBM random-access speed of light (P:L340 footnote) on a
    buffer of the filter's size: GUPS-style random loads (8 B, and the 32 B
    block with the .L2::64B fill hint the product uses), random 8 B updates,
    and the filter-geometry block probes, in the persistent-style (8 CTAs/SM)
    and the wave (32 CTAs/SM) launch shapes; the best form is the roofline."""
    dev = torch.device("cuda", torch.cuda.current_device())
    nbytes = cfg["m_bits"] // 8
    buf = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
    B = cfg["B"]
    b = nbytes * 8 // B
    lanes = max(1, B // 64)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    res = {}
    for cps in (8, 32):
        bf.bf_set_probe_launch(cps)
        thr = sms * cps * 256
        forms = {"gups_read_8": (lambda: bf.bf_probe_gups(buf, nbytes, 8, 0, 0, n), _rng_accesses(n, thr * 8)),
                 "gups_read_8_l2_64B": (lambda: bf.bf_probe_gups(buf, nbytes, 8, 0, 1, n), _rng_accesses(n, thr * 8)),
                 "block_read_32_l2_64B": (lambda: bf.bf_probe_gups(buf, nbytes, 32, 0, 1, n), _rng_accesses(n, thr * 8)),
                 "block_read_rng": (lambda: bf.bf_probe_rng(buf, b, B, 0, 1, n), _rng_accesses(n, thr * 4)),
                 "gups_update_8": (lambda: bf.bf_probe_gups(buf, nbytes, 8, 1, 0, n), _rng_accesses(n, thr * 8)),
                 "block_red_rng": (lambda: bf.bf_probe_rng(buf, b, B, 1, lanes, n), _rng_accesses(n, thr // lanes))}
        for name, (fn, acc) in forms.items():
            res[f"{name}@{cps}"] = round(acc / (best_time(torch, fn, 3) * 1e-3) / 1e9, 3)
    bf.bf_set_probe_launch(0)
    pick = lambda pre: max(v for k, v in res.items() if k.startswith(pre))  # noqa: E731
    res["read"] = max(pick("block_read_32_l2_64B"), pick("block_read_rng"))
    res["read_gups"] = pick("gups_read_8")
    res["update_gups"] = pick("gups_update_8")
    res["block_red"] = pick("block_red_rng")
    res["paper_gups"] = {"read": 52.9, "update": 23.7, "source": "P:L428 (B200)"}
    del buf
    torch.cuda.empty_cache()
    return res


def run_probes_range(bf, torch, cfg, buf, n=1 << 26):
    """The L2 bounds of the binned paths' per-range kernels, on views of the
    product filter's own allocation (after the timed region): the apply ORs
    records into one L2-resident range of the binned add (32 MiB, the
    library default) -- R_red of that range (LSU REDs of the block's lanes,
    and the LSU+TMA form); the lookup tests records against one range of the
    binned contains (64 MiB) -- R_read of that range (in-register block
    loads).  Launch shapes 8 and 32 CTAs/SM; the best form is the bound."""
    B = cfg["B"]
    lanes = max(1, B // 64)
    sms = torch.cuda.get_device_properties(buf.device).multi_processor_count
    res = {}
    for name, mib in (("apply_range", 32), ("lookup_range", 64)):
        view = buf[: mib << 20]
        b = (mib << 20) * 8 // B
        forms = {}
        for cps in (8, 32):
            bf.bf_set_probe_launch(cps)
            thr = sms * cps * 256
            if name == "apply_range":
                fl = {"red_rng": (lambda: bf.bf_probe_rng(view, b, B, 1, lanes, n), _rng_accesses(n, thr // lanes))}
                if B >= 128:
                    fl["red_lsu_tma"] = (lambda: bf.bf_probe_rng(view, b, B, 3, lanes, n), _rng_accesses(n, thr))
            else:
                fl = {"read_rng": (lambda: bf.bf_probe_rng(view, b, B, 0, 1, n), _rng_accesses(n, thr * 4))}
            for fn_name, (fn, acc) in fl.items():
                forms[f"{fn_name}@{cps}"] = round(acc / (best_time(torch, fn) * 1e-3) / 1e9, 3)
        bf.bf_set_probe_launch(0)
        best = max(forms, key=forms.get)
        res[name] = {"range_mib": mib, "forms": forms, "best": forms[best], "best_form": best}
    return res


def phase_rooflines(phases, range_probes, cfg, hbm_peak):
    """Each binned phase against its own bound: bin / bin-with-slots / unbin
    against HBM streaming (their algorithmic bytes per key over the measured
    copy peak), apply / lookup against the L2 probe of their range
    (run_probes_range) in Gkeys/s, shown as GB/s of 32-byte sectors."""
    n, nneg = cfg["n"], cfg["n_neg"]
    nq = n + nneg
    out = {}
    spec = {"bin": (n, 16.0, "hbm", "key 8 B in + record 8 B out"),
            "apply": (n, None, "l2", "apply_range"),
            "bin_slots": (nq, 20.0, "hbm", "key 8 B in + record 8 B + slot 4 B out"),
            "lookup": (nq, None, "l2", "lookup_range"),
            "unbin": (nq, 4.125, "hbm", "slot 4 B in + 1/8 B result out (+ the result-bit gather from L2)")}
    for ph, (keys, bpk, bound, what) in spec.items():
        ms, spans = phases.get(ph, (0.0, 0))
        if spans == 0 or ms <= 0:
            continue
        g = keys / (ms * 1e-3) / 1e9
        o = {"bound": bound, "ms": round(ms, 4), "spans": spans, "achieved_gkeys_s": round(g, 3)}
        if bound == "hbm":
            o.update({"achieved": round(g * bpk, 1), "peak": hbm_peak, "unit": "GB/s",
                      "frac": round(g * bpk / hbm_peak, 4), "algorithmic_bytes_per_key": bpk,
                      "peak_kind": "MEASURED_PEAKS.json hbm_gbs (copy)", "bytes": what})
        else:
            pr = range_probes[what]
            o.update({"achieved": round(g * 32, 1), "peak": round(pr["best"] * 32, 1), "unit": "GB/s",
                      "frac": round(g / pr["best"], 4), "algorithmic_bytes_per_key": 32,
                      "peak_gkeys_s": pr["best"],
                      "peak_kind": f"measured live: L2 probe on a {pr['range_mib']} MiB range of the filter's own "
                                   f"allocation, best of {pr['forms']}"})
        out[ph] = o
    return out


PHASE_KERNELS = {"bin": "bin_range_kernel", "apply": "apply_kernel, one launch per range",
                 "bin_slots": "bin_range_kernel<..., SLOTS>", "lookup": "lookup_kernel, one launch per range",
                 "unbin": "unbin_kernel"}


def sector_bytes(B):
    return max(32, B // 8)


def kernel_roofline(name, gkeys, probe_gkeys, probe_name, B, traffic=None, same_n_gkeys=None, n=None):
    """The binding roofline of an L2-resident kernel: the random 32-byte-sector
    rate of the L2 for its access pattern, measured live (probe), expressed
    as GB/s of block sectors.  The denominator is the best probe form at the
    kernel's own key count and launch shape when measured (same per-launch
    costs), else the asymptotic (2^26-key) one; both fractions are kept."""
    sb = sector_bytes(B)
    peak = same_n_gkeys if same_n_gkeys else probe_gkeys
    d = {"bound": "l2", "achieved": round(gkeys * sb, 1), "peak": round(peak * sb, 1), "unit": "GB/s",
         "frac": round(gkeys / peak, 4), "traffic": traffic, "kernel": name,
         "algorithmic_bytes_per_key": sb, "achieved_gkeys_s": round(gkeys, 3),
         "peak_gkeys_s": round(peak, 3), "peak_kind": "measured live (probe, same run)",
         "probe": probe_name}
    if same_n_gkeys:
        d["peak_kind"] = (f"measured live (probe, same run): best probe form at the kernel's own key count ({n}) "
                          "and launch shape (32 CTAs/SM)")
        d["peak_asymptotic_gkeys_s"] = round(probe_gkeys, 3)
        d["frac_asymptotic"] = round(gkeys / probe_gkeys, 4)
    return d


def ncu_traffic(f, op, n_launch):
    """dram bytes per launch of this kernel from the committed ncu --set full
    capture of the same command (profiles/ncu_traffic.json), if present."""
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        lay = f.layout(op)
        lgs = (f.B // f.S).bit_length() - 1
        head = (f"Cfg<{f.variant}, {f.S}, {lgs}, {f.k}, {f.z}, {lay['theta']}, {lay['phi']}, "
                f"{lay['kpt']}, {lay['hash_variant']}")
        tail = f">, {1 if op == 0 else 0}>"
        sigs = (head + tail, head + ", 0" + tail)
        hit = [v for k, v in tr["kernels"].items() if any(sg in k for sg in sigs) and v.get("n") == n_launch]
        if hit:
            return hit[0]["dram_bytes_per_launch"], hit[0].get("capture")
    except Exception:
        pass
    return None, None


def leg_result(leg, r, probes, cfg, world, hbm_peak):
    """JSON block of one leg."""
    n, nneg = cfg["n"], cfg["n_neg"]
    f = leg.f
    fpr = r["fp"] / nneg if nneg else None
    res = {"workload": cfg["workload"], "value": round(r["value"], 3), "unit": "Gkeys/s",
           "ms_per_step": round(r["ms"], 4), "keys_per_step": (2 * n + nneg) * world,
           "add_gkeys_s": round(r["add_gkeys_s"], 3), "contains_gkeys_s": round(r["contains_gkeys_s"], 3),
           "kernel_ms": {k: round(v, 4) for k, v in r["t"].items()},
           "step_rel_stderr": round(r["rel_stderr"], 5) if r["rel_stderr"] is not None else None,
           "gpu_launches": r["launches"], "cuda_graph": r["graph"],
           "layout_add": f.layout(0), "layout_contains": f.layout(1),
           "add_path": "binned" if f.add_mode()[1] else "direct",
           "contains_path": "binned" if f.contains_mode()[1] else "direct",
           "fpr": {"measured": fpr, "false_positives": r["fp"], "negatives": nneg,
                   "source": "the timed contains' own output bits on the negatives"}}
    if cfg.get("iso"):
        p = cfg["iso"]["fpr_model"]
        res["fpr"]["exact_model"] = p
        res["fpr"]["z"] = round((r["fp"] - nneg * p) / (nneg * p * (1 - p)) ** 0.5, 2)
    if cfg["residency"] == "L2" and probes:
        tr_a, cap_a = ncu_traffic(f, 0, n)
        tr_c, cap_c = ncu_traffic(f, 1, n + nneg)
        ka = kernel_roofline("bf_add", r["add_gkeys_s"], probes["red"], probes["red_name"], cfg["B"], tr_a,
                             probes.get("add_best_same_n"), probes.get("add_n"))
        kc = kernel_roofline("bf_contains", r["contains_gkeys_s"], probes["read"], probes["read_name"], cfg["B"], tr_c,
                             probes.get("contains_best_same_n"), probes.get("contains_n"))
        if cap_a:
            ka["traffic_source"] = f"ncu --set full capture {cap_a} (dram__bytes_read.sum + dram__bytes_write.sum)"
        if cap_c:
            kc["traffic_source"] = f"ncu --set full capture {cap_c} (dram__bytes_read.sum + dram__bytes_write.sum)"
        dom = "add" if r["t"]["add"] >= r["t"]["contains"] else "contains"
        res["roofline"] = ka if dom == "add" else kc
        res["roofline_kernels"] = {"add": ka, "contains": kc}
        res["probes"] = probes
        # HBM context: an L2-resident filter moves only keys + results through HBM
        hb = (8.0 * (2 * n + nneg) + (n + nneg) / 8.0) / (r["ms"] * 1e-3) / 1e9
        res["hbm_context"] = {"achieved": round(hb, 1), "peak": hbm_peak, "unit": "GB/s",
                              "frac": round(hb / hbm_peak, 4),
                              "note": "keys (8 B) + result bits over the whole step; the filter never leaves L2"}
    elif cfg["residency"] == "HBM" and probes:
        cg = r["contains_gkeys_s"]
        sb = sector_bytes(cfg["B"])
        tr_c, cap_c = ncu_traffic(f, 1, n + nneg)
        if res["contains_path"] == "binned":
            # bin: key in + record and slot out; lookup: record in + each filter line once per batch;
            # unbin: slot in (+ result-bit gather, L2) + result bits out
            batch = min(n + nneg, 1 << 31)
            apc = 8 + 8 + 4 + 8 + (cfg["m_bits"] / 8) / batch + 4 + 1 / 8
            kc = {"bound": "hbm", "achieved": round(cg * apc, 1), "peak": hbm_peak, "unit": "GB/s",
                  "frac": round(cg * apc / hbm_peak, 4), "traffic": None,
                  "kernel": "bf_contains (binned: bin + per-range lookup + unbin)",
                  "algorithmic_bytes_per_key": round(apc, 3), "achieved_gkeys_s": round(cg, 3),
                  "peak_kind": "MEASURED_PEAKS.json hbm_gbs (copy)",
                  "note": "streaming bound: key 8 B + record 8+8 B + slot 4+4 B + filter once per batch + result bits",
                  "vs_random_read_probe": round(cg / probes["read"], 4), "random_read_probe_gkeys_s": probes["read"]}
        else:
            kc = {"bound": "hbm", "achieved": round(cg * (8 + sb + 1 / 8), 1), "unit": "GB/s",
                  "peak": round(probes["read"] * (8 + sb + 1 / 8), 1), "frac": round(cg / probes["read"], 4),
                  "traffic": tr_c, "kernel": "bf_contains", "algorithmic_bytes_per_key": 8 + sb + 1 / 8,
                  "achieved_gkeys_s": round(cg, 3), "peak_gkeys_s": probes["read"],
                  "peak_kind": "measured live: HBM random block-read probe (same buffer size, same loads)",
                  "vs_gups_read": round(cg / probes["read_gups"], 4),
                  "vs_copy_peak": round(cg * (8 + sb + 1 / 8) / hbm_peak, 4)}
            if cap_c:
                kc["traffic_source"] = f"ncu --set full capture {cap_c}"
        ag = r["add_gkeys_s"]
        if res["add_path"] == "binned":
            # bin: key in + record out; apply: record in + each filter line read and written once per batch
            batch = min(n, 1 << 31)
            apb = 8 + 8 + 8 + 2 * (cfg["m_bits"] / 8) / batch
            ka = {"bound": "hbm", "achieved": round(ag * apb, 1), "peak": hbm_peak, "unit": "GB/s",
                  "frac": round(ag * apb / hbm_peak, 4), "traffic": None, "kernel": "bf_add (binned: bin + apply)",
                  "algorithmic_bytes_per_key": round(apb, 3), "achieved_gkeys_s": round(ag, 3),
                  "peak_kind": "MEASURED_PEAKS.json hbm_gbs (copy)",
                  "note": "streaming bound: key 8 B + record write 8 B + record read 8 B + filter read+write per batch"}
        else:
            ka = {"bound": "hbm", "achieved_gkeys_s": round(ag, 3), "peak_gkeys_s": probes["block_red"],
                  "frac": round(ag / probes["block_red"], 4), "kernel": "bf_add (direct)",
                  "peak_kind": "measured live: HBM random block-RED probe"}
        dom = "add" if r["t"]["add"] >= r["t"]["contains"] else "contains"
        res["roofline"] = ka if dom == "add" else kc
        res["roofline_kernels"] = {"add": ka, "contains": kc}
        res["probes"] = probes
        if r.get("phases") and r.get("range_probes"):
            ph = phase_rooflines(r["phases"], r["range_probes"], cfg, hbm_peak)
            if ph:
                # the step's dominant kernel is the phase with the most time:
                # it carries the leg's roofline; the whole-path streaming
                # figures stay in roofline_kernels
                top = max(ph, key=lambda k: ph[k]["ms"])
                res["roofline_phases"] = ph
                res["roofline"] = dict(ph[top], kernel=f"{top} phase ({PHASE_KERNELS[top]})",
                                       traffic=None, dominant_by="phase time in one eager step (bf_phase_times)")
                res["range_probes"] = r["range_probes"]
    return res


def run_ours(a, cfg, rank, world, local_rank):
    import torch

    from paper_2512_15595_b200 import bf
    from paper_2512_15595_b200 import dist as bfdist

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    if a.l2_fetch:
        bf.bf_set_l2_fetch_granularity(a.l2_fetch)
    hbm_peak, peak_kind, _ = load_peaks()

    leg = Leg(bf, torch, cfg, a, rank, world, dev, bfdist)
    with ClockSampler(local_rank) as clk:
        r = leg.run(a.steps, a.warmup, a.graph, clk)
    if cfg["residency"] == "HBM":
        r["phases"] = leg.phase_pass()
        if not a.no_probe and rank == 0:
            r["range_probes"] = run_probes_range(bf, torch, cfg, leg.f.data())
    probes = None
    if not a.no_probe and rank == 0:
        if cfg["residency"] == "L2":
            probes = run_probes_l2(bf, torch, cfg, dev, sizes={"add": cfg["n"], "contains": cfg["n"] + cfg["n_neg"]},
                                   buf=leg.f.data())
        else:
            probes = run_probes_hbm(bf, torch, cfg, 1 << 28)
    e2e = None
    if not a.no_e2e:
        e2e = run_e2e(bf, torch, leg, cfg, world)
    main = leg_result(leg, r, probes, cfg, world, hbm_peak) if rank == 0 else None
    leg.free()
    del leg

    extra = {}
    if world == 1 and a.config == "c2" and rank == 0:
        sub_steps = max(3, min(a.steps, 10))
        for key, name, skip in (("fixed_load", "c2n", a.no_fixed), ("hbm", "c3", a.no_hbm)):
            if skip:
                continue
            c = resolve(name, None)
            free, _ = torch.cuda.mem_get_info()
            # filter + probe buffer + keys + binned-add scratch + slack
            need = c["m_bits"] // 8 * 2 + (c["n"] + c["n_neg"]) * 8 + (19 << 30)
            if free < need:
                extra[key] = {"skipped": f"needs {need >> 30} GiB of device memory, {free >> 30} free"}
                continue
            lg = Leg(bf, torch, c, a, rank, world, dev, bfdist)
            rr = lg.run(sub_steps, 3, a.graph)
            if c["residency"] == "HBM":
                rr["phases"] = lg.phase_pass()
                if not a.no_probe:
                    rr["range_probes"] = run_probes_range(bf, torch, c, lg.f.data())
            pr = None
            if not a.no_probe:
                pr = (run_probes_l2(bf, torch, c, dev, sizes={"add": c["n"], "contains": c["n"] + c["n_neg"]},
                                    buf=lg.f.data())
                      if c["residency"] == "L2"
                      else run_probes_hbm(bf, torch, c, 1 << 28))
            extra[key] = leg_result(lg, rr, pr, c, world, hbm_peak)
            extra[key]["steps"] = sub_steps
            lg.free()
            del lg

    if rank != 0:
        return
    n = cfg["n"]
    res = {
        "metric": METRIC,
        "value": main["value"], "unit": "Gkeys/s", "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": main["ms_per_step"], "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u64", "data": "synthetic",
        "config": config_block(cfg, world, extra={
            "parallelism": f"dp{world} (replicated filter)", "merge": a.merge if world > 1 else None,
            "layout_add": main["layout_add"], "layout_contains": main["layout_contains"],
            "add_path": main["add_path"], "contains_path": main["contains_path"], "cuda_graph": main["cuda_graph"],
            "l2_fetch_granularity": bf.bf_get_l2_fetch_granularity(),
            "l2": f"inputs larger than L2 ({(2 * n + cfg['n_neg']) * 8 >> 20} MiB of keys streamed per step, "
                  f"evict-first); filter {cfg['residency']}-resident by design"}),
        "add_gkeys_s": main["add_gkeys_s"], "contains_gkeys_s": main["contains_gkeys_s"],
        "kernel_ms": main["kernel_ms"], "step_rel_stderr": main["step_rel_stderr"],
        "fpr": main["fpr"],
        "roofline": main.get("roofline"),
        "roofline_kernels": main.get("roofline_kernels"),
        "roofline_phases": main.get("roofline_phases"),
        "range_probes": main.get("range_probes"),
        "hbm_context": main.get("hbm_context"),
        "probes": main.get("probes"),
        "gpu_launches": main["gpu_launches"],
        "clocks": clk.summary(),
    }
    for key in ("roofline_phases", "range_probes"):
        if res[key] is None:
            del res[key]
    res.update(extra)
    if e2e:
        res["e2e"] = e2e
    if not a.no_cpu and world == 1:
        res["cpu_baseline"] = cpu_baseline(cfg)
    print(json.dumps(res), flush=True)


def run_e2e(bf, torch, leg, cfg, world, steps=3):
    """The same step end to end through the C ABI's host-buffer calls
    (bf_add_host + bf_contains_host: keys in pinned host memory, results
    back in pinned host memory, every host<->device copy inside the timed
    region; the library streams each call's keys through double-buffered
    device staging, copies overlapped with the kernels).  Wall clock,
    synchronized.  Bound: the PCIe host->device rate (every key crosses
    once), measured here with a pinned copy of the same size."""
    n, nneg = cfg["n"], cfg["n_neg"]
    hq = torch.empty(n + nneg, dtype=torch.int64, pin_memory=True)
    hq.copy_(leg.q.cpu())
    hk = hq[:n]
    hout = torch.empty((n + nneg + 31) // 32, dtype=torch.int32, pin_memory=True)
    f = leg.f

    def one():
        f.clear()
        f.add_host(hk)
        f.contains_host(hq, hout)

    one()
    torch.cuda.synchronize()
    ts = []
    for _ in range(steps):
        t0 = time.perf_counter()
        one()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    t = statistics.median(ts)
    ok = check_positives(torch, hout, n)
    assert ok, "false negative in the e2e result"
    # PCIe H2D reference: one pinned copy of all the step's key bytes
    dbuf = torch.empty(n + nneg, dtype=torch.int64, device=leg.dev)
    dbuf.copy_(hq, non_blocking=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dbuf[:n].copy_(hk, non_blocking=True)
    dbuf.copy_(hq, non_blocking=True)
    torch.cuda.synchronize()
    t_pcie = time.perf_counter() - t0
    del dbuf
    h2d = (2 * n + nneg) * 8
    return {"value": round((2 * n + nneg) * world / t / 1e9, 3), "unit": "Gkeys/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": ((n + nneg + 31) // 32) * 4,
            "ms_per_step": round(t * 1e3, 3),
            "path": "C ABI host-buffer calls: bf_clear + bf_add_host(pinned keys) + bf_contains_host(pinned "
                    "positives + negatives -> pinned result bits); wall clock, synchronized",
            "pcie_bound": {"h2d_gb_s": round(h2d / t_pcie / 1e9, 2), "gkeys_s": round((2 * n + nneg) / t_pcie / 1e9, 3),
                           "frac": round(t_pcie / t, 4),
                           "note": "torch pinned H2D copy of the same bytes; every key must cross PCIe once"}}


def main():
    a, cfg = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", a.gpus))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if world != a.gpus and "WORLD_SIZE" in os.environ:
        world = int(os.environ["WORLD_SIZE"])
    if a.impl == "reference":
        run_reference(a, cfg, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(a, cfg, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
