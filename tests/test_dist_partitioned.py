"""Block-range partitioned filters (NEXT N1) over torch.distributed (gloo,
CPU, world sizes 2 and 3): the routing/exchange logic of
paper_2512_15595_b200.dist.PartitionedFilter -- fixed-count all_to_all of
record buckets and counts, owner-side apply/test, the inverse all_to_all of
result bytes and the scatter to key indices -- yields exactly the filter and
the answers of one unpartitioned filter.  The per-key kernels are emulated
here with the CPU oracle (test-only ops); the CUDA kernels behind bf_route /
bf_add_routed / bf_contains_routed / bf_scatter_results are checked against
the oracle in tests/test_gpu_parity.py::test_partitioned_filter_single_gpu."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class OracleRouteOps:
    """CPU stand-ins with the kernels' contract: a record is the raw key here
    (the owner recomputes its pattern), buckets/counts/cap as on the GPU."""

    def __init__(self, geom, P, part):
        self.g, self.P = geom, P
        self.lo = geom.b * part // P
        self.hi = geom.b * (part + 1) // P
        self.bits = np.zeros((self.hi - self.lo) * geom.B, dtype=np.uint8)

    def owner(self, blk):
        return next(p for p in range(self.P) if self.g.b * p // self.P <= blk < self.g.b * (p + 1) // self.P)

    def route(self, keys, cap, P, want_idx):
        recs = torch.zeros(P * cap, dtype=torch.int64)
        idx = torch.zeros(P * cap, dtype=torch.int64)
        counts = torch.zeros(P, dtype=torch.int64)
        for i, key in enumerate(keys.numpy().view(np.uint64)):
            o = self.owner(self.g.pattern(int(key))[0])
            j = int(counts[o])
            if j < cap:
                recs[o * cap + j] = int(np.int64(key.view(np.int64)))
                idx[o * cap + j] = i
            counts[o] += 1
        return recs, (idx if want_idx else None), counts

    def _walk(self, recv, rcounts, P, cap):
        for s in range(P):
            for j in range(min(int(rcounts[s]), cap)):
                key = int(np.int64(recv[s * cap + j]).view(np.uint64))
                blk, pos = self.g.pattern(key)
                assert self.lo <= blk < self.hi
                yield s * cap + j, [(blk - self.lo) * self.g.B + p for p in pos]

    def add_routed(self, recv, rcounts, P, cap):
        for _, bits in self._walk(recv, rcounts, P, cap):
            self.bits[bits] = 1

    def contains_routed(self, recv, rcounts, P, cap):
        res = torch.zeros(P * cap, dtype=torch.uint8)
        for slot, bits in self._walk(recv, rcounts, P, cap):
            res[slot] = int(self.bits[bits].all())
        return res

    def part_bytes(self):
        return torch.from_numpy(np.packbits(self.bits, bitorder="little"))

    def clear(self):
        self.bits[:] = 0

    def scatter(self, idx, res, counts, P, cap, n):
        out = np.zeros(n, dtype=np.uint8)
        for s in range(P):
            for j in range(min(int(counts[s]), cap)):
                if int(res[s * cap + j]):
                    out[int(idx[s * cap + j])] = 1
        return out


def _worker(rank, world, port, m_bits, results):
    import torch.distributed as dist

    import synth
    from oracle.bfo import OracleFilter
    from paper_2512_15595_b200.dist import PartitionedFilter

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        geom = OracleFilter(3, m_bits, B=256, S=64, k=8, allocate=False)
        ops = OracleRouteOps(geom, world, rank)
        pf = PartitionedFilter(m_bits, 8, 256, 64, 3, group=None, ops=ops)
        n = 1500 + 37 * rank  # ranks hold different key counts
        mine = synth.keys(10_000 * rank, n)
        pf.add(torch.from_numpy(mine.view(np.int64)))
        # the union of the parts is the unpartitioned filter of all keys
        parts = [None] * world
        dist.all_gather_object(parts, ops.bits)
        full = OracleFilter(3, m_bits, B=256, S=64, k=8)
        for r in range(world):
            full.add(synth.keys(10_000 * r, 1500 + 37 * r))
        want_bits = np.unpackbits(full.bytes(), bitorder="little")
        ok_bits = bool(np.array_equal(np.concatenate(parts), want_bits))
        # lookups of own keys + absent keys
        q = np.concatenate([mine[:700], synth.negatives(900, offset=rank * 1000)])
        got = pf.contains(torch.from_numpy(q.view(np.int64)))
        want = np.unpackbits(full.contains(q).view(np.uint8), bitorder="little")[: q.size]
        # E3: route-to-owner construction + all_gather of the parts = a replica
        words = torch.zeros(full.nbytes, dtype=torch.uint8)
        from paper_2512_15595_b200.dist import build_replicated_routed
        build_replicated_routed(pf, torch.from_numpy(mine.view(np.int64)), words, 256 // 8)
        ok_rep = bool(np.array_equal(words.numpy(), full.bytes()))
        results[rank] = (ok_bits and ok_rep, bool(np.array_equal(got, want)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_filter_matches_single(world):
    mgr = mp.Manager()
    results = mgr.dict()
    m_bits = 256 * 1003  # b = 1003 blocks: uneven parts
    mp.spawn(_worker, args=(world, _free_port(), m_bits, results), nprocs=world, join=True)
    assert dict(results) == {r: (True, True) for r in range(world)}


def _skew_worker(rank, world, port, m_bits, results):
    """Rank 0's shard lands entirely in owner 0's block range, so only rank 0
    overflows the first cap: every rank must agree to re-route (collective
    MAX of the counts) instead of rank 0 raising while the others wait in
    all_to_all, and no record may be dropped."""
    import torch.distributed as dist

    import synth
    from oracle.bfo import OracleFilter
    from paper_2512_15595_b200.dist import PartitionedFilter

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        geom = OracleFilter(3, m_bits, B=256, S=64, k=8, allocate=False)
        ops = OracleRouteOps(geom, world, rank)
        pf = PartitionedFilter(m_bits, 8, 256, 64, 3, group=None, ops=ops, slack=0.05, pad=0)
        cand = synth.keys(777, 4000)
        hot = np.array([k for k in cand if ops.owner(geom.pattern(int(k))[0]) == 0], dtype=np.uint64)
        mine = hot[:600] if rank == 0 else synth.keys(50_000 * rank, 600)
        pf.add(torch.from_numpy(mine.view(np.int64)))
        parts = [None] * world
        dist.all_gather_object(parts, ops.bits)
        full = OracleFilter(3, m_bits, B=256, S=64, k=8)
        full.add(hot[:600])
        for r in range(1, world):
            full.add(synth.keys(50_000 * r, 600))
        want_bits = np.unpackbits(full.bytes(), bitorder="little")
        q = np.concatenate([mine, synth.negatives(300, offset=rank * 1000)])
        got = pf.contains(torch.from_numpy(q.view(np.int64)))
        want = np.unpackbits(full.contains(q).view(np.uint8), bitorder="little")[: q.size]
        results[rank] = (bool(np.array_equal(np.concatenate(parts), want_bits)), bool(np.array_equal(got, want)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_bucket_overflow_is_agreed_collectively(world):
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_skew_worker, args=(world, _free_port(), 256 * 1003, results), nprocs=world, join=True)
    assert dict(results) == {r: (True, True) for r in range(world)}
