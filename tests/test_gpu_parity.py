"""GPU parity: the CUDA path (through the C ABI) reproduces the CPU oracle
bit-exactly -- the whole filter bit array after bulk add, and every packed
result bit of bulk contains -- on the same seeded keys (synth/), for every
compiled schedule (variant x B x S x k x z x Θ x Φ x KPT x hash variant), the
generic runtime-parameter kernel, and the edge cases (empty, ragged, unaligned
inputs, non-power-of-two block counts, repeated adds, clear, seeds)."""
import importlib.util
import os
from collections import defaultdict

import numpy as np
import pytest

import synth
from oracle.bfo import OracleFilter, unpack_bits

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _instances():
    spec = importlib.util.spec_from_file_location(
        "gen_instances", os.path.join(ROOT, "paper_2512_15595_b200", "csrc", "gen_instances.py"))
    g = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(g)
    return g.instances()


def _groups():
    grp = defaultdict(list)
    for op, v, B, S, k, z, theta, phi, kpt, hv in _instances():
        grp[(v, B, S, k, z)].append((op, theta, phi, kpt, hv))
    return sorted(grp.items())


GROUPS = _groups()


def _to_dev(torch, a, dev):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).to(dev)


def _gpu_bytes(f):
    return f.data().cpu().numpy()


def _gpu_contains(torch, f, qd):
    out = f.contains(qd)
    torch.cuda.synchronize()
    return out.cpu().numpy().view(np.uint32)


# keys spanning several tiles with a ragged tail; small filter -> real collisions
N_ADD, N_NEG = 6 * 1024 + 37, 4 * 1024 + 5


@pytest.mark.parametrize("cfg,scheds", GROUPS, ids=[f"v{c[0]}_B{c[1]}_S{c[2]}_k{c[3]}_z{c[4]}" for c, _ in GROUPS])
def test_every_compiled_schedule_matches_oracle(bflib, cuda, cfg, scheds):
    import torch
    bf = bflib
    v, B, S, k, z = cfg
    m = B * 997  # b = 997 blocks: not a power of two, heavy fill
    keys = synth.keys(1000, N_ADD)
    query = np.concatenate([keys[::3], synth.negatives(N_NEG)])
    o = OracleFilter(v, m, B=B, S=S, k=k, z=z)
    o.add(keys)
    want_bytes = o.bytes()
    want_res = o.contains(query)
    kd, qd = _to_dev(torch, keys, cuda), _to_dev(torch, query, cuda)
    f = bf.Filter(m, k, B, S, variant=v, z=z)
    for op, theta, phi, kpt, hv in scheds:
        f.set_layout(op, theta, phi, kpt, hv)
        lay = f.layout(op)
        assert lay["specialized"] == 1 and (lay["theta"], lay["phi"], lay["kpt"]) == (theta, phi, kpt)
        if op == 0:
            f.clear()
            f.add(kd)
            torch.cuda.synchronize()
            got = _gpu_bytes(f)
            assert np.array_equal(got, want_bytes), f"add schedule Θ={theta} Φ={phi} kpt={kpt} hv={hv}"
    # contains schedules on the oracle-equal filter
    f.set_layout(0, 0, 0)
    f.clear()
    f.add(kd)
    for op, theta, phi, kpt, hv in scheds:
        if op == 1:
            f.set_layout(1, theta, phi, kpt, hv)
            got = _gpu_contains(torch, f, qd)
            assert np.array_equal(got, want_res), f"contains schedule Θ={theta} Φ={phi} kpt={kpt} hv={hv}"


GENERIC = [  # no specialized instantiation -> generic runtime kernel
    (3, 512, 32, 16, 0), (3, 1024, 32, 32, 0), (4, 1024, 32, 16, 4), (1, 512, 32, 20, 0),
    (3, 256, 64, 20, 0), (2, 64, 64, 25, 0), (4, 512, 32, 16, 8), (1, 32, 32, 3, 0),
    (3, 128, 32, 32, 0), (4, 256, 64, 8, 1),
    (2, 32, 32, 1, 0), (1, 64, 64, 1, 0), (1, 1024, 64, 7, 0), (4, 1024, 32, 16, 16),  # k=1, 1024-bit BBF, z=16
]


@pytest.mark.parametrize("cfg", GENERIC, ids=[f"v{c[0]}_B{c[1]}_S{c[2]}_k{c[3]}_z{c[4]}" for c in GENERIC])
def test_generic_kernel_matches_oracle(bflib, cuda, cfg):
    import torch
    bf = bflib
    v, B, S, k, z = cfg
    m = B * 1531
    keys = synth.keys(7, N_ADD)
    query = np.concatenate([keys[::2], synth.negatives(N_NEG)])
    o = OracleFilter(v, m, B=B, S=S, k=k, z=z)
    o.add(keys)
    f = bf.Filter(m, k, B, S, variant=v, z=z)
    assert f.layout(0)["specialized"] == 0 and f.layout(1)["specialized"] == 0
    f.add(_to_dev(torch, keys, cuda))
    torch.cuda.synchronize()
    assert np.array_equal(_gpu_bytes(f), o.bytes())
    assert np.array_equal(_gpu_contains(torch, f, _to_dev(torch, query, cuda)), o.contains(query))


EDGE_CFGS = [(3, 256, 64, 8, 0), (1, 256, 64, 8, 0), (4, 256, 32, 8, 2), (2, 64, 64, 6, 0)]


@pytest.mark.parametrize("cfg", EDGE_CFGS)
@pytest.mark.parametrize("n", [0, 1, 31, 32, 33, 127, 128, 129, 1000, 4096 + 3])
def test_sizes_and_tails(bflib, cuda, cfg, n):
    import torch
    bf = bflib
    v, B, S, k, z = cfg
    m = (1 << 16) + 3 * B
    keys = synth.keys(50, n)
    query = np.concatenate([keys, synth.negatives(n + 7)])
    o = OracleFilter(v, m, B=B, S=S, k=k, z=z)
    o.add(keys)
    f = bf.Filter(m, k, B, S, variant=v, z=z)
    f.add(_to_dev(torch, keys, cuda))
    torch.cuda.synchronize()
    assert np.array_equal(_gpu_bytes(f), o.bytes())
    qd = _to_dev(torch, query, cuda)
    out = torch.full(((query.size + 31) // 32 + 2,), -1, dtype=torch.int32, device=cuda)
    bf.bf_contains(f.handle, qd, out, query.size)
    torch.cuda.synchronize()
    got = out.cpu().numpy().view(np.uint32)
    nw = (query.size + 31) // 32
    assert np.array_equal(got[:nw], o.contains(query))
    assert (got[nw:] == 0xFFFFFFFF).all(), "wrote past ceil(n/32) words"
    if query.size % 32:
        assert got[nw - 1] >> (query.size % 32) == 0, "tail bits must be zero"


@pytest.mark.parametrize("cfg", EDGE_CFGS)
@pytest.mark.parametrize("off", [1, 2])
def test_unaligned_keys_idempotence_clear_seed(bflib, cuda, cfg, off):
    """Key arrays 8-byte aligned (off=1: scalar key loads, no cp.async key
    staging) and 16- but not 32-byte aligned (off=2: staging on, the 256-bit
    key loads off) give the oracle's bits, for several seeds and layouts."""
    import torch
    bf = bflib
    v, B, S, k, z = cfg
    m = 1 << 18
    keys = synth.keys(3, 10001)
    buf = _to_dev(torch, np.concatenate([np.zeros(off, np.uint64), keys]), cuda)
    kd = buf[off:]
    assert kd.data_ptr() % 32 != 0 and kd.data_ptr() % 16 == (0 if off == 2 else 8)
    for seed in (0, 1, 0xDEADBEEF):
        o = OracleFilter(v, m, B=B, S=S, k=k, z=z, seed=seed)
        o.add(keys)
        f = bf.Filter(m, k, B, S, variant=v, z=z, seed=seed)
        for kpt in (1, 2, 4):
            for op in (0, 1):
                try:
                    f.set_layout(op, *((B // S, 1) if op == 0 else (1, B // S)), kpt, 0)
                except bf.BFError:
                    continue
            f.clear()
            f.add(kd)
            f.add(kd)  # idempotent
            torch.cuda.synchronize()
            assert np.array_equal(_gpu_bytes(f), o.bytes())
            q = np.concatenate([keys[:999], synth.negatives(1001)])
            qbuf = _to_dev(torch, np.concatenate([np.zeros(off, np.uint64), q]), cuda)
            assert np.array_equal(_gpu_contains(torch, f, qbuf[off:]), o.contains(q))
        f.clear()
        torch.cuda.synchronize()
        assert not _gpu_bytes(f).any()


def test_streams_and_concurrent_adds(bflib, cuda):
    """Two adds of disjoint halves on two streams == one add of all (OR commutes)."""
    import torch
    bf = bflib
    keys = synth.keys(11, 200_003)
    o = OracleFilter(3, 1 << 22, B=256, S=64, k=8)
    o.add(keys)
    f = bf.Filter(1 << 22, 8, 256, 64, "SBF")
    kd = _to_dev(torch, keys, cuda)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    with torch.cuda.stream(s1):
        f.add(kd[:100_000])
    with torch.cuda.stream(s2):
        f.add(kd[100_000:])
    torch.cuda.synchronize()
    assert np.array_equal(_gpu_bytes(f), o.bytes())


def test_host_buffer_path(bflib, cuda):
    """bf_add_host / bf_contains_host (chunked, double-buffered) == oracle,
    across a chunk boundary (chunks are 2^23 keys)."""
    import torch
    bf = bflib
    n = (1 << 23) + 12345
    keys = synth.keys(0, n)
    o = OracleFilter(3, 1 << 26, B=256, S=64, k=8)
    o.add(keys, threads=8)
    hk = torch.from_numpy(keys.view(np.int64)).pin_memory()
    f = bf.Filter(1 << 26, 8, 256, 64, "SBF")
    f.add_host(hk)
    assert np.array_equal(_gpu_bytes(f), o.bytes())
    q = np.concatenate([keys[:1 << 22], synth.negatives((1 << 23) + 999)])
    hq = torch.from_numpy(q.view(np.int64)).pin_memory()
    out = f.contains_host(hq)
    assert np.array_equal(out.numpy().view(np.uint32), o.contains(q, threads=8))


def test_keygen_matches_synth(bflib, cuda):
    import torch
    bf = bflib
    for base, n in [(0, 1), (0, 1000), (5, 1001), (synth.NEG_BASE, 4099)]:
        out = torch.empty(n, dtype=torch.int64, device=cuda)
        bf.bf_keygen(out, n, base)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().view(np.uint64), synth.keys(base, n))
    # unaligned output
    buf = torch.empty(1001, dtype=torch.int64, device=cuda)
    bf.bf_keygen(buf[1:], 1000, 42)
    torch.cuda.synchronize()
    assert np.array_equal(buf[1:].cpu().numpy().view(np.uint64), synth.keys(42, 1000))


@pytest.mark.parametrize("nsrc,nbytes", [(1, 8), (2, 4096), (3, 1 << 20), (8, (1 << 20) + 8)])
def test_or_fold(bflib, cuda, nsrc, nbytes):
    import torch
    bf = bflib
    rng = np.random.default_rng(nsrc)
    stride = nbytes + 64 if nbytes % 16 else nbytes
    src = rng.integers(0, 256, nsrc * stride, dtype=np.uint8)
    want = np.zeros(nbytes, np.uint8)
    for r in range(nsrc):
        want |= src[r * stride: r * stride + nbytes]
    sd = torch.from_numpy(src).to(cuda)
    dst = torch.zeros(nbytes, dtype=torch.uint8, device=cuda)
    bf.bf_or_fold(dst, sd, nsrc, stride, nbytes)
    torch.cuda.synchronize()
    assert np.array_equal(dst.cpu().numpy(), want)
    # in place into source 0
    bf.bf_or_fold(sd, sd, nsrc, stride, nbytes)
    torch.cuda.synchronize()
    assert np.array_equal(sd[:nbytes].cpu().numpy(), want)


def test_probes_run(bflib, cuda):
    import torch
    bf = bflib
    keys = torch.empty(1 << 16, dtype=torch.int64, device=cuda)
    bf.bf_keygen(keys, keys.numel(), 0)
    buf = torch.zeros(1 << 20, dtype=torch.uint8, device=cuda)
    out = torch.empty(keys.numel() // 32, dtype=torch.int32, device=cuda)
    bf.bf_probe_read(buf, (1 << 20) // 32, 256, keys, out)
    bf.bf_probe_red(buf, (1 << 20) // 32, 256, 4, keys)
    torch.cuda.synchronize()
    assert buf.any()
    n0 = bf.bf_launch_count()
    bf.bf_probe_read(buf, (1 << 20) // 32, 256, keys, out)
    assert bf.bf_launch_count() == n0 + 1


def test_configs0_full_size(bflib, cuda):
    """BASELINE configs[0] exactly: 2^20 keys into a 16 Mbit filter, B=256,
    S=64, k=8, BBF and SBF; contains on 2^20 positives + 2^20 negatives."""
    import torch
    bf = bflib
    n = 1 << 20
    pos, neg = synth.positives(n), synth.negatives(n)
    q = np.concatenate([pos, neg])
    for v in (1, 3):
        o = OracleFilter(v, 1 << 24, B=256, S=64, k=8)
        o.add(pos, threads=8)
        f = bf.Filter(1 << 24, 8, 256, 64, variant=v)
        f.add(_to_dev(torch, pos, cuda))
        torch.cuda.synchronize()
        assert np.array_equal(_gpu_bytes(f), o.bytes())
        got = _gpu_contains(torch, f, _to_dev(torch, q, cuda))
        assert np.array_equal(got, o.contains(q, threads=8))
        assert unpack_bits(got, 2 * n)[:n].all()


def test_configs1_bench_workload_full_size(bflib, cuda):
    """The bench workload (configs[1]: 32 MiB SBF 256/64 k=8, 2^26 keys) in the
    launch configuration bench.py times: full bit array + all 2^26 results."""
    import torch
    bf = bflib
    n = 1 << 26
    kd = torch.empty(n, dtype=torch.int64, device=cuda)
    bf.bf_keygen(kd, n, 0)
    f = bf.Filter(1 << 28, 8, 256, 64, "SBF")
    f.add(kd)
    out = f.contains(kd)
    torch.cuda.synchronize()
    keys = synth.keys(0, n)
    o = OracleFilter(3, 1 << 28, B=256, S=64, k=8)
    o.add(keys, threads=os.cpu_count())
    assert np.array_equal(_gpu_bytes(f), o.bytes())
    assert (out.cpu().numpy().view(np.uint32) == 0xFFFFFFFF).all()  # all positives
    negs = synth.negatives(1 << 22)
    got = _gpu_contains(torch, f, _to_dev(torch, negs, cuda))
    assert np.array_equal(got, o.contains(negs, threads=os.cpu_count()))


def test_large_filter_offsets_sampled(bflib, cuda):
    """An 8 GiB filter (configs[2]'s size; word offsets beyond 2^32 bytes):
    oracle-built block ranges at the start, middle and end match exactly."""
    import torch
    bf = bflib
    m = 1 << 36
    n = 1 << 24
    free, _ = torch.cuda.mem_get_info()
    if free < (m // 8) + (1 << 30):
        pytest.skip("not enough device memory")
    kd = torch.empty(n, dtype=torch.int64, device=cuda)
    bf.bf_keygen(kd, n, 0)
    f = bf.Filter(m, 8, 256, 64, "SBF")
    f.add(kd)
    torch.cuda.synchronize()
    keys = synth.keys(0, n)
    o = OracleFilter(3, m, B=256, S=64, k=8, allocate=False)
    b = o.b
    data = f.data()
    for lo in (0, b // 2 - 1000, b - 4096):
        hi = lo + 4096
        want = o.add_range(keys, lo, hi, threads=os.cpu_count())
        got = data[lo * 32: hi * 32].cpu().numpy()
        assert np.array_equal(got, want), lo
    q = keys[:1 << 20]
    out = f.contains(_to_dev(torch, q, cuda))
    torch.cuda.synchronize()
    assert (out.cpu().numpy().view(np.uint32) == 0xFFFFFFFF).all()


BINNED_CFGS = [(3, 256, 64, 8, 0), (1, 256, 64, 8, 0), (4, 256, 32, 8, 4), (2, 64, 64, 6, 0), (3, 256, 32, 16, 0)]


@pytest.mark.parametrize("cfg", BINNED_CFGS)
@pytest.mark.parametrize("range_bytes,batch,misalign", [(1 << 16, 0, 0), (1 << 15, 30_000, 0), (3 << 14, 7_777, 0),
                                                         (1 << 10, 0, 0), (1 << 16, 0, 1)])
def test_binned_add_matches_oracle(bflib, cuda, cfg, range_bytes, batch, misalign):
    """BF_ADD_BINNED (hash once, bin by filter range, apply range-major) builds
    exactly the oracle's filter, across several ranges, batches and a ragged
    last range; 1 KiB ranges give R > 512 buckets (several per bin-kernel
    thread); misalign = keys 8 bytes off a 32-byte boundary (the bin kernel's
    scalar key path)."""
    import torch
    bf = bflib
    v, B, S, k, z = cfg
    m = (1 << 22) + 5 * B  # b not a power of two; last range partial
    keys = synth.keys(321, 100_003)
    o = OracleFilter(v, m, B=B, S=S, k=k, z=z)
    o.add(keys)
    f = bf.Filter(m, k, B, S, variant=v, z=z)
    f.set_add_mode(bf.BF_ADD_BINNED, range_bytes, batch)
    if misalign:
        kd = torch.empty(keys.size + 1, dtype=torch.int64, device=cuda)
        kd[1:].copy_(_to_dev(torch, keys, cuda))
        f.add(kd[1:])
    else:
        f.add(_to_dev(torch, keys, cuda))
    torch.cuda.synchronize()
    assert f.add_mode() == (bf.BF_ADD_BINNED, 1)
    assert np.array_equal(_gpu_bytes(f), o.bytes())
    q = np.concatenate([keys[:5000], synth.negatives(5000)])
    assert np.array_equal(_gpu_contains(torch, f, _to_dev(torch, q, cuda)), o.contains(q))


def test_binned_add_bucket_overflow(bflib, cuda):
    """Keys concentrated in one range overflow its bucket; the overflow is
    OR-ed in directly and the filter is still exact."""
    import torch
    bf = bflib
    m, B = 1 << 22, 256
    o_geom = OracleFilter(3, m, B=B, S=64, k=8, allocate=False)
    cand = synth.keys(9, 200_000)
    b = o_geom.b
    per_range = (1 << 15) // (B // 8)
    hot = np.array([key for key in cand if o_geom.pattern(int(key))[0] < per_range], dtype=np.uint64)
    keys = np.concatenate([hot, cand[:20_000]])
    assert hot.size > 4000 and b // per_range == 16
    o = OracleFilter(3, m, B=B, S=64, k=8)
    o.add(keys)
    f = bf.Filter(m, 8, B, 64, "SBF")
    f.set_add_mode(bf.BF_ADD_BINNED, 1 << 15, 0)
    f.add(_to_dev(torch, keys, cuda))
    torch.cuda.synchronize()
    assert np.array_equal(_gpu_bytes(f), o.bytes())


@pytest.mark.parametrize("cfg", BINNED_CFGS)
@pytest.mark.parametrize("range_bytes,batch,misalign", [(1 << 16, 0, 0), (1 << 15, 30_000, 0), (3 << 14, 7_777, 0),
                                                         (1 << 10, 0, 0), (1 << 16, 0, 1)])
def test_binned_contains_matches_oracle(bflib, cuda, cfg, range_bytes, batch, misalign):
    """BF_CONTAINS_BINNED (bin the queries by filter range with their record
    slots, test range by range, gather back to key order) answers exactly as
    the oracle: several ranges, batches that are not multiples of 128 (cut
    to whole result words), a ragged last range and result word, R > 512
    buckets, keys off a 32-byte boundary."""
    import torch
    bf = bflib
    v, B, S, k, z = cfg
    m = (1 << 22) + 5 * B
    keys = synth.keys(321, 100_003)
    o = OracleFilter(v, m, B=B, S=S, k=k, z=z)
    o.add(keys)
    f = bf.Filter(m, k, B, S, variant=v, z=z)
    f.add(_to_dev(torch, keys, cuda))
    f.set_add_mode(bf.BF_ADD_AUTO, range_bytes, batch)
    f.set_contains_mode(bf.BF_CONTAINS_BINNED)
    q = np.concatenate([keys[:60_001], synth.negatives(60_013)])
    if misalign:
        qd = torch.empty(q.size + 1, dtype=torch.int64, device=cuda)
        qd[1:].copy_(_to_dev(torch, q, cuda))
        qd = qd[1:]
    else:
        qd = _to_dev(torch, q, cuda)
    got = _gpu_contains(torch, f, qd)
    assert f.contains_mode() == (bf.BF_CONTAINS_BINNED, 1)
    assert np.array_equal(got, o.contains(q))


def test_phase_timing_of_binned_paths(bflib, cuda):
    """bf_set_phase_timing / bf_phase_times (measurement hook): one timed span
    per batch and phase, positive times, nothing recorded while off or for
    direct calls, and the timed binned add / contains still match the
    oracle."""
    import torch
    bf = bflib
    v, B, S, k, z = 3, 256, 64, 8, 0
    m = (1 << 22) + 5 * B
    keys = synth.keys(777, 100_003)
    q = np.concatenate([keys[:50_000], synth.negatives(50_011)])
    o = OracleFilter(v, m, B=B, S=S, k=k, z=z)
    o.add(keys)
    f = bf.Filter(m, k, B, S, variant=v, z=z)
    f.set_add_mode(bf.BF_ADD_BINNED, 1 << 16, 40_000)  # 3 batches of keys, 3 of queries
    f.set_contains_mode(bf.BF_CONTAINS_BINNED)
    kd, qd = _to_dev(torch, keys, cuda), _to_dev(torch, q, cuda)
    f.add(kd)  # not timed
    assert all(t == (0.0, 0) for t in f.phase_times().values())
    f.clear()
    f.set_phase_timing(True)
    f.add(kd)
    got = _gpu_contains(torch, f, qd)
    t = f.phase_times()
    assert t["bin"][1] == 3 and t["apply"][1] == 3, t
    assert t["bin_slots"][1] == 3 and t["lookup"][1] == 3 and t["unbin"][1] == 3, t
    assert all(ms > 0 for ms, _ in t.values()), t
    assert np.array_equal(_gpu_bytes(f), o.bytes())
    assert np.array_equal(got, o.contains(q))
    assert all(v == (0.0, 0) for v in f.phase_times().values())  # forgotten after reading
    f.set_add_mode(bf.BF_ADD_DIRECT)
    f.add(kd)  # the direct path records nothing
    assert all(v == (0.0, 0) for v in f.phase_times().values())
    f.set_phase_timing(False)


def test_binned_contains_bucket_overflow(bflib, cuda):
    """Queries concentrated in one range overflow its bucket; those keys are
    looked up directly (slot marker) and every answer is still exact."""
    import torch
    bf = bflib
    m, B = 1 << 22, 256
    o_geom = OracleFilter(3, m, B=B, S=64, k=8, allocate=False)
    cand = synth.keys(9, 200_000)
    per_range = (1 << 15) // (B // 8)
    hot = np.array([key for key in cand if o_geom.pattern(int(key))[0] < per_range], dtype=np.uint64)
    keys = cand[:50_000]
    o = OracleFilter(3, m, B=B, S=64, k=8)
    o.add(keys)
    f = bf.Filter(m, 8, B, 64, "SBF")
    f.add(_to_dev(torch, keys, cuda))
    f.set_add_mode(bf.BF_ADD_AUTO, 1 << 15, 0)
    f.set_contains_mode(bf.BF_CONTAINS_BINNED)
    q = np.concatenate([hot, hot, keys[:20_000], synth.negatives(7)])
    assert hot.size > 4000
    got = _gpu_contains(torch, f, _to_dev(torch, q, cuda))
    assert f.contains_mode()[1] == 1
    assert np.array_equal(got, o.contains(q))


def test_binned_contains_auto_policy(bflib, cuda):
    """AUTO takes the binned lookup only for a filter >= 96 MiB queried with at
    least one key per block; answers equal the direct path's."""
    import torch
    bf = bflib
    m = 1 << 30  # 128 MiB, b = 2^22 blocks of 256 bits
    f = bf.Filter(m, 8, 256, 64, "SBF")
    kd = torch.empty(1 << 22, dtype=torch.int64, device=cuda)
    bf.bf_keygen(kd, kd.numel(), 5)
    f.add(kd)
    qd = torch.empty((1 << 22) + 77, dtype=torch.int64, device=cuda)
    bf.bf_keygen(qd, qd.numel(), 3)  # half overlap with the added keys
    small = f.contains(qd[:1024])
    assert f.contains_mode() == (bf.BF_CONTAINS_AUTO, 0)
    big = f.contains(qd)
    assert f.contains_mode() == (bf.BF_CONTAINS_AUTO, 1)
    f.set_contains_mode(bf.BF_CONTAINS_DIRECT)
    ref = f.contains(qd)
    assert f.contains_mode() == (bf.BF_CONTAINS_DIRECT, 0)
    torch.cuda.synchronize()
    assert torch.equal(big, ref) and torch.equal(small, ref[:32])
    assert int((ref == 0).sum()) < ref.numel()


def test_binned_add_large_filter_sampled(bflib, cuda):
    """Binned add on an 8 GiB filter (256 ranges of 32 MiB): sampled block
    ranges equal the oracle's."""
    import torch
    bf = bflib
    m, n = 1 << 36, 1 << 24
    free, _ = torch.cuda.mem_get_info()
    if free < (m // 8) + (1 << 31):
        pytest.skip("not enough device memory")
    kd = torch.empty(n, dtype=torch.int64, device=cuda)
    bf.bf_keygen(kd, n, 77)
    f = bf.Filter(m, 8, 256, 64, "SBF")
    f.set_add_mode(bf.BF_ADD_BINNED)
    f.add(kd)
    torch.cuda.synchronize()
    assert f.add_mode()[1] == 1
    keys = synth.keys(77, n)
    o = OracleFilter(3, m, B=256, S=64, k=8, allocate=False)
    data = f.data()
    for lo in (0, o.b // 3, o.b - 2048):
        hi = lo + 2048
        assert np.array_equal(data[lo * 32: hi * 32].cpu().numpy(),
                              o.add_range(keys, lo, hi, threads=os.cpu_count())), lo


def _iso_rows():
    import json
    path = os.path.join(ROOT, "profiles", "iso_fpr_table.json")
    return json.load(open(path))["c2"]["rows"]


@pytest.mark.parametrize("row", _iso_rows(), ids=lambda r: f"v{r['variant']}_B{r['B']}_S{r['S']}_k{r['k']}_z{r['z']}")
def test_iso_fpr_configs1_rows(bflib, cuda, row):
    """configs[1] at iso FPR 1e-3 (32 MiB, n_iso keys from the exact model,
    profiles/iso_fpr_table.json written by tools/make_iso_table.py from
    oracle/ only): the GPU's measured FPR on 2^24 absent keys is within 4
    binomial sigma of the exact ideal-hash model, and every inserted key is
    found."""
    import torch
    bf = bflib
    v, B, S, k, z = row["variant"], row["B"], row["S"], row["k"], row["z"]
    m, n, Q = 1 << 28, row["n_iso"], 1 << 24
    f = bf.Filter(m, k, B, S, variant=v, z=z)
    keys = torch.empty(n, dtype=torch.int64, device=cuda)
    bf.bf_keygen(keys, n, 0)
    f.add(keys)
    neg = torch.empty(Q, dtype=torch.int64, device=cuda)
    bf.bf_keygen(neg, Q, synth.NEG_BASE)
    out = f.contains(neg)
    pos = f.contains(keys)
    torch.cuda.synchronize()
    fp = int(np.unpackbits(out.cpu().numpy().view(np.uint8)).sum())
    p = row["fpr_model"]
    zz = (fp - Q * p) / np.sqrt(Q * p * (1 - p))
    assert abs(zz) <= 4.0, (fp, Q * p)
    got = np.unpackbits(pos.cpu().numpy().view(np.uint8), bitorder="little")[:n]
    assert got.all()


@pytest.mark.parametrize("m,k", [(1 << 20, 7), ((1 << 22) + 13, 16), (1 << 25, 16), (999_983, 1), (1 << 32, 4),
                                 ((1 << 33) + 7, 16)])
def test_cbf_matches_oracle(bflib, cuda, m, k):
    """GPU classical Bloom filter (NEXT N3; the paper's GPU CBF baseline,
    P:L352/P:L392) == the oracle's CBF, bits and results, incl. m = 2^32 and
    the 128-bit fast range above it (m = 2^33 + 7, the 1 GB baseline)."""
    import torch
    bf = bflib
    keys = synth.keys(5, 70_001)
    q = np.concatenate([keys[::3], synth.negatives(30_000)])
    o = OracleFilter(0, m, k=k)
    o.add(keys, threads=4)
    f = bf.Filter(m, k, 256, 64, bf.BF_CBF)
    assert f.layout(0)["specialized"] == 0
    f.add(_to_dev(torch, keys, cuda))
    torch.cuda.synchronize()
    got = _gpu_bytes(f)
    want = o.bytes()
    assert np.array_equal(got[:want.size], want) and not got[want.size:].any()
    assert np.array_equal(_gpu_contains(torch, f, _to_dev(torch, q, cuda)), o.contains(q, threads=4))


@pytest.mark.parametrize("P", [1, 2, 3, 8])
@pytest.mark.parametrize("cfg", [(3, 256, 64, 8, 0), (4, 256, 32, 8, 2), (1, 256, 64, 8, 0), (2, 64, 64, 6, 0)])
def test_partitioned_filter_single_gpu(bflib, cuda, cfg, P):
    """NEXT N1 kernels on one GPU with P virtual owners: bf_route bins the keys
    by owner, each part applies its bucket (bf_add_routed); the concatenated
    parts equal the oracle's filter, and routed lookups (bf_contains_routed +
    bf_scatter_results) equal the oracle's answers."""
    import torch
    bf = bflib
    v, B, S, k, z = cfg
    m = B * 40_009
    vz = bf.BF_CSBF_Z(z) if v == 4 else v
    parts = [bf.bf_create_part(m, k, B, S, vz, 0, P, p) for p in range(P)]
    try:
        keys = synth.keys(17, 120_001)
        o = OracleFilter(v, m, B=B, S=S, k=k, z=z)
        o.add(keys)
        kd = _to_dev(torch, keys, cuda)
        cap = ((120_001 // P) * 11 // 10 + 4096 + 127) // 128 * 128
        recs = torch.empty(P * cap, dtype=torch.int64, device=cuda)
        counts = torch.empty(P, dtype=torch.int64, device=cuda)
        bf.bf_route(parts[0], kd, kd.numel(), 0, recs, None, cap, counts)
        for p in range(P):
            bf.bf_add_routed(parts[p], recs[p * cap:], counts[p:], 1, cap)
        torch.cuda.synchronize()
        assert int(counts.sum()) == keys.size and int(counts.max()) <= cap
        got = np.concatenate([bf._device_view(*bf.bf_data(h)).cpu().numpy() for h in parts])
        assert np.array_equal(got, o.bytes())
        q = np.concatenate([keys[:30_000], synth.negatives(40_003)])
        qd = _to_dev(torch, q, cuda)
        idx = torch.empty(P * cap, dtype=torch.int64, device=cuda)
        bf.bf_route(parts[0], qd, qd.numel(), 0, recs, idx, cap, counts)
        res = torch.empty(P * cap, dtype=torch.uint8, device=cuda)
        for p in range(P):
            bf.bf_contains_routed(parts[p], recs[p * cap:], counts[p:], 1, cap, res[p * cap:])
        out = torch.zeros((q.size + 31) // 32, dtype=torch.int32, device=cuda)
        bf.bf_scatter_results(idx, res, counts, P, cap, out)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().view(np.uint32), o.contains(q))
    finally:
        for h in parts:
            bf.bf_destroy(h)


SCHEME_CFGS = [(3, 256, 64, 16), (3, 256, 64, 8), (1, 256, 64, 8), (2, 64, 64, 8)]


@pytest.mark.parametrize("scheme", [1, 2])
@pytest.mark.parametrize("cfg", SCHEME_CFGS)
def test_draw_schemes_match_oracle(bflib, cuda, cfg, scheme):
    """NEXT N3: the double-hashing and iterative draw schemes on the
    GPU == the oracle's, every compiled schedule (bits and answers)."""
    import torch
    bf = bflib
    v, B, S, k = cfg
    m = B * 3001
    keys = synth.keys(23, N_ADD)
    q = np.concatenate([keys[::3], synth.negatives(N_NEG)])
    o = OracleFilter(v, m, B=B, S=S, k=k, scheme=scheme)
    o.add(keys)
    kd, qd = _to_dev(torch, keys, cuda), _to_dev(torch, q, cuda)
    f = bf.Filter(m, k, B, S, variant=v, scheme=scheme)
    s = B // S
    scheds = [(0, 1, s, 1 if scheme == 2 else 4)] + ([(0, s, 1, 4)] if scheme == 1 and s > 1 else [])
    for op, th, ph, kpt in scheds:
        f.set_layout(op, th, ph, kpt, 0)
        f.clear()
        f.add(kd)
        torch.cuda.synchronize()
        assert np.array_equal(_gpu_bytes(f), o.bytes()), (op, th, ph, kpt)
    f.set_layout(1, 1, s, 1 if scheme == 2 else 4, 0)
    assert np.array_equal(_gpu_contains(torch, f, qd), o.contains(q))


def test_concurrent_binned_adds_and_host_calls(bflib, cuda):
    """Binned adds on two streams from two host threads share the filter's
    scratch: the library orders them; the result is the oracle's filter.
    Host-buffer calls from two threads are serialised per filter."""
    import threading

    import torch
    bf = bflib
    m = 1 << 24
    keys = synth.keys(31, 400_000)
    o = OracleFilter(3, m, B=256, S=64, k=8)
    o.add(keys, threads=8)
    f = bf.Filter(m, 8, 256, 64, "SBF")
    f.set_add_mode(bf.BF_ADD_BINNED, 1 << 16, 50_000)
    halves = [_to_dev(torch, keys[:200_000], cuda), _to_dev(torch, keys[200_000:], cuda)]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    torch.cuda.synchronize()

    def work(i):
        with torch.cuda.stream(streams[i]):
            f.add(halves[i])

    th = [threading.Thread(target=work, args=(i,)) for i in range(2)]
    [t.start() for t in th]
    [t.join() for t in th]
    torch.cuda.synchronize()
    assert np.array_equal(_gpu_bytes(f), o.bytes())

    g = bf.Filter(m, 8, 256, 64, "SBF")
    hk = [torch.from_numpy(keys[:200_000].view(np.int64)).pin_memory(),
          torch.from_numpy(keys[200_000:].view(np.int64)).pin_memory()]
    th = [threading.Thread(target=lambda i=i: g.add_host(hk[i])) for i in range(2)]
    [t.start() for t in th]
    [t.join() for t in th]
    torch.cuda.synchronize()
    assert np.array_equal(_gpu_bytes(g), o.bytes())


def test_max_block_count_2pow32(bflib, cuda):
    """b = 2^32 blocks (the largest filter the spec allows; block = h >> 32,
    the b mod 2^32 == 0 path): RBBF 32/32, a 16 GiB filter; sampled block
    ranges equal the oracle's and every inserted key is found."""
    import torch
    bf = bflib
    m = 1 << 37  # 2^32 blocks of 32 bits
    free, _ = torch.cuda.mem_get_info()
    if free < (m // 8) + (1 << 30):
        pytest.skip("not enough device memory")
    n = 1 << 22
    kd = torch.empty(n, dtype=torch.int64, device=cuda)
    bf.bf_keygen(kd, n, 99)
    f = bf.Filter(m, 5, 32, 32, "RBBF")
    assert f.b == 1 << 32
    f.add(kd)
    out = f.contains(kd)
    torch.cuda.synchronize()
    assert (out.cpu().numpy().view(np.uint32) == 0xFFFFFFFF).all()
    keys = synth.keys(99, n)
    o = OracleFilter(2, m, B=32, S=32, k=5, allocate=False)
    data = f.data()
    for lo in (0, (1 << 31) + 12345, (1 << 32) - 8192):
        hi = lo + 8192
        assert np.array_equal(data[lo * 4: hi * 4].cpu().numpy(), o.add_range(keys, lo, hi, threads=os.cpu_count())), lo


HYBRID_CFGS = [(3, 256, 64, 8, 0), (3, 256, 32, 16, 0), (1, 256, 64, 8, 0), (4, 256, 32, 8, 2), (3, 128, 64, 8, 0),
               (3, 512, 64, 16, 0), (3, 1024, 64, 16, 0), (4, 1024, 64, 16, 4)]


@pytest.mark.parametrize("cfg", HYBRID_CFGS)
def test_hybrid_add_matches_oracle(bflib, cuda, cfg):
    """BF_ADD_HYBRID (half the warps OR whole blocks through the TMA engine,
    half through cooperative red.global.or) builds the oracle's filter."""
    import torch
    bf = bflib
    v, B, S, k, z = cfg
    m = B * 20_011
    keys = synth.keys(41, 150_001)
    o = OracleFilter(v, m, B=B, S=S, k=k, z=z)
    o.add(keys, threads=4)
    f = bf.Filter(m, k, B, S, variant=v, z=z)
    f.set_add_mode(bf.BF_ADD_HYBRID)
    f.add(_to_dev(torch, keys, cuda))
    torch.cuda.synchronize()
    assert np.array_equal(_gpu_bytes(f), o.bytes())


@pytest.mark.parametrize("binned", [False, True, 2], ids=["direct", "binned", "binned_pipelined"])
def test_cuda_graph_capture_and_replay(bflib, cuda, binned):
    """bf_clear + bf_add + bf_contains are stream-ordered and capture-safe:
    one captured step replayed three times gives the oracle's bits and
    answers (bench.py times such replays), for the direct add and for the
    binned add (bin + one apply launch per range) that configs[2] uses."""
    import torch
    bf = bflib
    n = (1 << 18) + 7
    keys = synth.keys(3, n)
    o = OracleFilter(3, 1 << 22, B=256, S=64, k=8)
    o.add(keys)
    f = bf.Filter(1 << 22, 8, 256, 64, "SBF")
    if binned:
        # 8 ranges; "pipelined": 6 batches, bin of batch i+1 on the caller's
        # stream overlapping the apply of batch i on the filter's side stream
        # (a fork/join captured into the graph)
        f.set_add_mode(bf.BF_ADD_BINNED, 1 << 16, 50_000 if binned == 2 else 0)
    kd = _to_dev(torch, keys, cuda)
    out = torch.empty((n + 31) // 32, dtype=torch.int32, device=cuda)
    f.add(kd)  # warm-up (lazy module loading) outside the capture
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            f.clear()
            f.add(kd)
            f.contains(kd, out)
    for _ in range(3):
        out.fill_(0)
        g.replay()
    torch.cuda.synchronize()
    assert f.add_mode()[1] == int(bool(binned))
    assert np.array_equal(_gpu_bytes(f), o.bytes())
    assert np.array_equal(out.cpu().numpy().view(np.uint32), o.contains(keys))


@pytest.mark.parametrize("cfg,add_l,con_l", [
    ((3, 256, 64, 8, 0), (4, 1, 4), (1, 4, 4)),     # SBF: add Θ=s, contains Θ=1
    ((1, 256, 64, 8, 0), (4, 1, 4), (1, 4, 4)),     # BBF
    ((2, 64, 64, 8, 0), (1, 1, 4), (1, 1, 4)),      # RBBF
    ((4, 256, 32, 8, 2), (2, 4, 4), (1, 8, 4)),     # CSBF z < s: one lane per group
    ((4, 256, 32, 8, 4), (4, 2, 4), (1, 8, 4)),
    ((3, 1024, 64, 16, 0), (16, 1, 4), (4, 4, 4)),  # B > 256: contains Θ = B/256
])
def test_default_layouts(bflib, cuda, cfg, add_l, con_l):
    """The default schedules bf_create picks, all specialized kernels."""
    bf = bflib
    v, B, S, k, z = cfg
    f = bf.Filter(1 << 22, k, B, S, variant=v, z=z)
    for op, want in ((0, add_l), (1, con_l)):
        lay = f.layout(op)
        assert (lay["theta"], lay["phi"], lay["kpt"], lay["specialized"]) == (*want, 1), (op, lay)


def test_auto_add_path_threshold(bflib, cuda):
    """BF_ADD_AUTO takes the binned path for filters >= 96 MiB once the batch
    has one key per 64 filter bytes (include/bf.h), the direct path below;
    both give the oracle's bits on a sampled range."""
    import torch
    bf = bflib
    m = 1 << 31  # 256 MiB
    nb = (m // 8) // 64
    f = bf.Filter(m, 8, 256, 64, "SBF")
    for n, want in ((nb - 1, 0), (nb, 1)):
        f.clear()
        kd = torch.empty(n, dtype=torch.int64, device=cuda)
        bf.bf_keygen(kd, n, 5)
        f.add(kd)
        torch.cuda.synchronize()
        assert f.add_mode() == (bf.BF_ADD_AUTO, want), n
        o = OracleFilter(3, m, B=256, S=64, k=8, allocate=False)
        lo, hi = o.b // 2, o.b // 2 + 4096
        assert np.array_equal(_gpu_bytes(f)[lo * 32:hi * 32], o.add_range(synth.keys(5, n), lo, hi, threads=os.cpu_count()))


@pytest.mark.parametrize("cfg,m", [((3, 256, 64, 8, 0), 1), ((3, 256, 64, 8, 0), 256), ((2, 32, 32, 4, 0), 32),
                                   ((4, 256, 32, 8, 2), 100)])
def test_single_block_filter(bflib, cuda, cfg, m):
    """Degenerate geometry: b = ceil(m/B) = 1 (every key selects block 0; the
    filter saturates), incl. m < B (m_eff = B, reading 11)."""
    import torch
    bf = bflib
    v, B, S, k, z = cfg
    keys = synth.keys(23, 777)
    q = np.concatenate([keys[:100], synth.negatives(1000)])
    o = OracleFilter(v, m, B=B, S=S, k=k, z=z)
    o.add(keys)
    f = bf.Filter(m, k, B, S, variant=v, z=z)
    assert f.b == 1 and f.m_eff == B
    f.add(_to_dev(torch, keys, cuda))
    torch.cuda.synchronize()
    assert np.array_equal(_gpu_bytes(f), o.bytes())
    assert np.array_equal(_gpu_contains(torch, f, _to_dev(torch, q, cuda)), o.contains(q))


def test_autotune_picks_a_compiled_schedule_and_keeps_results(bflib, cuda):
    """paper_2512_15595_b200.tune.autotune (the paper's layout grid search at
    run time): the chosen schedule is one of the compiled ones, contains
    tuning leaves the filter untouched, add tuning leaves it empty, and the
    tuned filter still equals the oracle's."""
    import torch
    from paper_2512_15595_b200 import tune
    bf = bflib
    m, n = 1 << 24, 50_000
    keys = synth.keys(41, n)
    o = OracleFilter(4, m, B=256, S=32, k=8, z=2)
    o.add(keys)
    f = bf.Filter(m, 8, 256, 32, "CSBF", z=2)
    with pytest.raises(ValueError):
        tune.autotune(f, 0, n=1 << 16)
    r0 = tune.autotune(f, 0, n=1 << 18, reps=2, allow_clear=True)
    assert len(r0["tried"]) >= 2 and r0["layout"] in r0["tried"]
    assert (f.layout(0)["theta"], f.layout(0)["phi"], f.layout(0)["kpt"]) == r0["layout"]
    assert not _gpu_bytes(f).any()
    f.add(_to_dev(torch, keys, cuda))
    torch.cuda.synchronize()
    before = _gpu_bytes(f).copy()
    r1 = tune.autotune(f, 1, n=1 << 18, reps=2)
    assert r1["layout"] in r1["tried"] and np.array_equal(_gpu_bytes(f), before)
    assert np.array_equal(before, o.bytes())
    q = np.concatenate([keys[:999], synth.negatives(5000)])
    assert np.array_equal(_gpu_contains(torch, f, _to_dev(torch, q, cuda)), o.contains(q))
