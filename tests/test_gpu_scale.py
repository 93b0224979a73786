"""Parity at scale (SURVEY 8(d) "Parity at scale"): the
CUDA path's steady-state code runs here, not only its first tile.

* Every compiled schedule (variant x B x S x k x z x Θ x Φ x KPT x hash
  variant) on 2^22 + 37 keys: the bulk kernels' grid is capped at the
  occupancy grid (<= 8 CTAs x 148 SMs x 8 warps), so every warp runs >= 3
  tiles -- the cross-tile key pipeline (knext), the cp.async double buffer of
  the key-staged contains, the shared-memory staging reuse of the BBF add,
  and the ragged-tail hand-off (n mod 128 = 37) all execute.  b is not a
  power of two and the filter is about half full (m = n k / ln 2), so a wrong
  bit cannot hide in a saturated block.  Whole filter after add; every
  result bit of a 2^22-key query (positives interleaved with negatives).
* Every configs[1] row (97 = the sweep's 94 + 3 extra geometries) at the
  bench size: 2^26 keys into the 32 MiB filter with the default schedules the
  sweep times; whole filter, all 2^26 positives found, 2^22 negatives
  answered as the oracle answers.
* configs[3] (SBF 256/32, k = 8 and 16, ~3.3 GiB, 2^30 keys): every compiled
  Θ/Φ/KPT/hash-variant add schedule with the direct add (and the binned
  add), every contains schedule; the whole filter equals the oracle's (the
  comparison runs on the device against the oracle's uploaded bytes), all
  2^30 positives found, 2^24 negatives answered as the oracle answers.

Every expected value comes from oracle/ on keys made by synth/ on the host.
"""
import importlib.util
import math
import os
from collections import defaultdict
from functools import lru_cache

import numpy as np
import pytest

import synth
from oracle.bfo import SBF, OracleFilter

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
THREADS = os.cpu_count() or 4


def _gen():
    spec = importlib.util.spec_from_file_location(
        "gen_instances", os.path.join(ROOT, "paper_2512_15595_b200", "csrc", "gen_instances.py"))
    g = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(g)
    return g


GEN = _gen()


def _groups():
    grp = defaultdict(list)
    for op, v, B, S, k, z, theta, phi, kpt, hv in GEN.instances():
        grp[(v, B, S, k, z)].append((op, theta, phi, kpt, hv))
    return sorted(grp.items())


GROUPS = _groups()
N_MT = (1 << 22) + 37  # n mod 128 = 37: a ragged last tile for every KPT


@lru_cache(maxsize=None)
def _keys(base, n):
    return synth.keys(base, n)


def _query_mt():
    """2^22 + 11 keys: the even-indexed inserted keys interleaved with
    negatives by a fixed permutation (mixed answers in every tile)."""
    pos = _keys(1000, N_MT)[::2]
    neg = synth.negatives(N_MT - pos.size + 11, offset=77)
    q = np.concatenate([pos, neg])
    return q[np.random.default_rng(5).permutation(q.size)]


def _dev(torch, a, dev):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).to(dev)


def _odd_blocks(m_bits, B):
    b = max(3, m_bits // B)
    return b | 1 if b & (b - 1) else b + 1  # never a power of two


@pytest.mark.parametrize("cfg,scheds", GROUPS, ids=[f"v{c[0]}_B{c[1]}_S{c[2]}_k{c[3]}_z{c[4]}" for c, _ in GROUPS])
def test_every_compiled_schedule_multitile(bflib, cuda, cfg, scheds):
    import torch
    bf = bflib
    v, B, S, k, z = cfg
    b = _odd_blocks(int(N_MT * k / math.log(2)), B)  # ~half-full filter
    m = b * B
    keys = _keys(1000, N_MT)
    query = _query_mt()
    o = OracleFilter(v, m, B=B, S=S, k=k, z=z)
    o.add(keys, threads=THREADS)
    want = torch.from_numpy(o.bytes()).to(cuda)
    want_res = torch.from_numpy(o.contains(query, threads=THREADS).view(np.int32)).to(cuda)
    kd, qd = _dev(torch, keys, cuda), _dev(torch, query, cuda)
    f = bf.Filter(m, k, B, S, variant=v, z=z)
    assert f.b == b and f.b & (f.b - 1)
    # every warp gets >= 3 tiles: the launch grid (<= occupancy grid) holds
    # at most 8 CTAs/SM x 148 SMs x 8 warps = 9472 warps; 2^22 keys are
    # >= 32768 tiles of 32*KPT (KPT <= 4)
    assert N_MT // (32 * 4) >= 3 * 8 * 148 * 8
    f.set_add_mode(bf.BF_ADD_DIRECT)
    for op, theta, phi, kpt, hv in scheds:
        if op != 0:
            continue
        f.set_layout(0, theta, phi, kpt, hv)
        f.clear()
        f.add(kd)
        got = f.data()
        assert torch.equal(got, want), f"add schedule Θ={theta} Φ={phi} kpt={kpt} hv={hv}"
    f.set_layout(0, 0, 0)
    f.clear()
    f.add(kd)
    assert torch.equal(f.data(), want)
    out = torch.empty((query.size + 31) // 32 + 1, dtype=torch.int32, device=cuda)
    for op, theta, phi, kpt, hv in scheds:
        if op != 1:
            continue
        f.set_layout(1, theta, phi, kpt, hv)
        out.fill_(-1)
        f.contains(qd, out)
        nw = want_res.numel()
        assert torch.equal(out[:nw], want_res), f"contains schedule Θ={theta} Φ={phi} kpt={kpt} hv={hv}"
        assert int(out[nw].item()) == -1, "wrote past ceil(n/32) words"


def _query_runs(pos, n_neg):
    """Queries in runs that decide whether a warp's 32 keys can all fail
    early (the BBF contains' grouped early exit, tuning::EXIT_GROUP): 2^20
    negatives (all-negative warps: the exit taken), 2^20 negatives with a
    positive at every index = 13 mod 32 (key slot 1 of lanes 3/11/19/27 of a
    128-key tile, so some warp calls keep one live lane and the others exit),
    2^18 positives (no exit), a ragged tail of 1,007 negatives."""
    neg = synth.negatives(n_neg, offset=4242)
    a = neg[: 1 << 20]
    b = neg[1 << 20: 2 << 20].copy()
    b[13::32] = pos[: b[13::32].size]
    c = pos[: 1 << 18]
    d = neg[2 << 20: (2 << 20) + 1007]
    return np.concatenate([a, b, c, d])


BBF_GROUPS = [(c, s) for c, s in GROUPS if c[0] == 1]


@pytest.mark.parametrize("cfg,scheds", BBF_GROUPS, ids=[f"v{c[0]}_B{c[1]}_S{c[2]}_k{c[3]}_z{c[4]}" for c, _ in BBF_GROUPS])
def test_bbf_contains_runs_of_negatives(bflib, cuda, cfg, scheds):
    """Every compiled BBF contains schedule on the run-structured query of
    _query_runs, against a half-full filter (every drawn bit set with
    probability ~1/2, so an all-negative warp fails within a few draw groups
    while a warp with one positive lane runs all k draws): every result bit
    equals the oracle's, including the false positives."""
    import torch
    bf = bflib
    v, B, S, k, z = cfg
    n = 1 << 20
    b = _odd_blocks(int(n * k / math.log(2)), B)
    m = b * B
    keys = _keys(3000, n)
    query = _query_runs(keys, (2 << 20) + 1007)
    o = OracleFilter(v, m, B=B, S=S, k=k, z=z)
    o.add(keys, threads=THREADS)
    want_res = torch.from_numpy(o.contains(query, threads=THREADS).view(np.int32)).to(cuda)
    kd, qd = _dev(torch, keys, cuda), _dev(torch, query, cuda)
    f = bf.Filter(m, k, B, S, variant=v, z=z)
    f.add(kd)
    assert torch.equal(f.data(), torch.from_numpy(o.bytes()).to(cuda))
    out = torch.empty((query.size + 31) // 32 + 1, dtype=torch.int32, device=cuda)
    ran = 0
    for op, theta, phi, kpt, hv in scheds:
        if op != 1:
            continue
        f.set_layout(1, theta, phi, kpt, hv)
        out.fill_(-1)
        f.contains(qd, out)
        nw = want_res.numel()
        assert torch.equal(out[:nw], want_res), f"contains schedule Θ={theta} Φ={phi} kpt={kpt} hv={hv}"
        assert int(out[nw].item()) == -1, "wrote past ceil(n/32) words"
        ran += 1
    assert ran > 0


def test_generic_kernel_multitile(bflib, cuda):
    """The runtime-parameter kernel (grid-stride, one key per thread) over
    many grid strides, ragged tail: SBF 512/32 k=16 (no specialization)."""
    import torch
    bf = bflib
    v, B, S, k = 3, 512, 32, 16
    n = (1 << 22) + 5
    m = _odd_blocks(int(n * k / math.log(2)), B) * B
    keys = _keys(31, n)
    o = OracleFilter(v, m, B=B, S=S, k=k)
    o.add(keys, threads=THREADS)
    f = bf.Filter(m, k, B, S, variant=v)
    assert f.layout(0)["specialized"] == 0
    f.add(_dev(torch, keys, cuda))
    assert torch.equal(f.data(), torch.from_numpy(o.bytes()).to(cuda))
    q = _query_mt()
    got = f.contains(_dev(torch, q, cuda))
    assert torch.equal(got, torch.from_numpy(o.contains(q, threads=THREADS).view(np.int32)).to(cuda))


C2 = GEN.c2_rows()


@pytest.mark.parametrize("row", C2, ids=[f"v{r[0]}_B{r[1]}_S{r[2]}_k{r[3]}_z{r[4]}" for r in C2])
def test_configs1_row_full_size(bflib, cuda, row):
    """One configs[1] row at the size bench.py / tools/sweep.py time it:
    2^26 keys, 32 MiB, the default schedules."""
    import torch
    bf = bflib
    v, B, S, k, z = row
    m, n = 1 << 28, 1 << 26
    f = bf.Filter(m, k, B, S, variant=v, z=z)
    assert f.layout(0)["specialized"] and f.layout(1)["specialized"]
    kd = torch.empty(n, dtype=torch.int64, device=cuda)
    bf.bf_keygen(kd, n, 0)
    f.add(kd)
    out = f.contains(kd)
    negs = _keys(synth.NEG_BASE, 1 << 22)
    got_neg = f.contains(_dev(torch, negs, cuda))
    keys = _keys(0, n)
    o = OracleFilter(v, m, B=B, S=S, k=k, z=z)
    o.add(keys, threads=THREADS)
    assert torch.equal(f.data(), torch.from_numpy(o.bytes()).to(cuda))
    assert int((out != -1).sum().item()) == 0  # every inserted key found
    want = torch.from_numpy(o.contains(negs, threads=THREADS).view(np.int32)).to(cuda)
    assert torch.equal(got_neg, want)


def _c4_scheds(k):
    return sorted({(op, th, ph, kpt, hv) for op, v, B, S, kk, z, th, ph, kpt, hv in GEN.instances()
                   if (v, B, S, kk, z) == (SBF, 256, 32, k, 0)})


@pytest.mark.parametrize("k", [8, 16])
def test_configs3_every_schedule_full_size(bflib, cuda, k):
    """configs[3]'s Θ/Φ/KPT/hash-variant grid at full size."""
    import json

    import torch
    bf = bflib
    tab = json.load(open(os.path.join(ROOT, "profiles", "iso_fpr_table.json")))["c4"]["rows"]
    row = next(r for r in tab if (r["variant"], r["B"], r["S"], r["k"]) == (SBF, 256, 32, k))
    m, n = int(row["c_iso"] * (1 << 30)), 1 << 30
    free, _ = torch.cuda.mem_get_info()
    if free < 2 * (m // 8) + n * 8 + (4 << 30):
        pytest.skip("not enough device memory for configs[3]")
    o = OracleFilter(SBF, m, B=256, S=32, k=k)
    chunk = 1 << 26
    for off in range(0, n, chunk):
        o.add(synth.keys(off, chunk), threads=THREADS)
    want = torch.from_numpy(o.bytes()).to(cuda)
    negs = synth.negatives(1 << 24)
    want_neg = torch.from_numpy(o.contains(negs, threads=THREADS).view(np.int32)).to(cuda)
    del o
    f = bf.Filter(m, k, 256, 32, "SBF")
    assert f.b & (f.b - 1)
    keys = torch.empty(n, dtype=torch.int64, device=cuda)
    bf.bf_keygen(keys, n, 0)
    nd = _dev(torch, negs, cuda)
    scheds = _c4_scheds(k)
    assert len([s for s in scheds if s[0] == 0]) >= 10 and len([s for s in scheds if s[0] == 1]) >= 10
    f.set_add_mode(bf.BF_ADD_DIRECT)
    for op, th, ph, kpt, hv in scheds:
        if op == 0:
            f.set_layout(0, th, ph, kpt, hv)
            f.clear()
            f.add(keys)
            assert torch.equal(f.data(), want), f"add Θ={th} Φ={ph} kpt={kpt} hv={hv}"
    f.set_layout(0, 0, 0)
    f.set_add_mode(bf.BF_ADD_BINNED)
    f.clear()
    f.add(keys)
    assert f.add_mode()[1] == 1 and torch.equal(f.data(), want), "binned add"
    for op, th, ph, kpt, hv in scheds:
        if op == 1:
            f.set_layout(1, th, ph, kpt, hv)
            assert torch.equal(f.contains(nd), want_neg), f"contains Θ={th} Φ={ph} kpt={kpt} hv={hv}"
            out = f.contains(keys)
            assert int((out != -1).sum().item()) == 0, f"false negative, contains Θ={th} Φ={ph} kpt={kpt} hv={hv}"
