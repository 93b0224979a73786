"""Multi-GPU construction and lookup over torch.distributed (one process per GPU).

* Lookup (``contains``) shards naturally: every rank queries its own key shard
  against a full filter replica -- no collective on the data path.
* Construction (``add``) has one real exchange step: each rank builds a partial
  filter from its key shard, and the partials are OR-merged.  NCCL has no
  bitwise-OR reduction, so the merge is NCCL data movement + the OR-fold
  kernel (bf_or_fold):

  E1 ``allgather``  (the north_star's literal recipe): for each chunk of the
     filter, all_gather the P partial chunks and OR-fold them.  Receives
     (P-1)*M bytes per rank.
  E2 ``alltoall``  (bandwidth-optimal with the same primitives): all_to_all so
     rank r receives every rank's r-th range (a reduce-scatter by OR once
     folded), OR-fold it, then all_gather the merged ranges.  Receives
     2*(P-1)/P*M bytes per rank, 4x less than E1 at P=8.

  E4 ``nvls``  in-switch OR over NVLink SHARP (NvlsMerger, bf_mcast_*).
  p2p ``p2p``  one kernel per rank over CUDA-IPC peer mappings (P2pMerger,
     bf_p2p_or_merge): rank r loads its 1/P slice of every peer's partial
     straight over NVLink, ORs and stores it into every peer -- the
     reduce-scatter by OR and the all-gather fused, no staging, no fold pass.

The functions take the filter's word array as a flat uint8 tensor (a view of
bf_data) and an ``or_fold(dst, src2d)`` callable; the default is the CUDA
kernel.  (CPU/gloo tests pass a CPU fold to check the chunk and offset
arithmetic; the product path has no CPU fold.)
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def gpu_or_fold(dst: torch.Tensor, src2d: torch.Tensor) -> None:
    """dst[:] = OR over rows of src2d (CUDA, bf_or_fold)."""
    from . import bf
    nsrc, nbytes = src2d.shape
    bf.bf_or_fold(dst, src2d, nsrc, src2d.stride(0), nbytes)


def merge_allgather(words: torch.Tensor, group=None, chunk_bytes: int = 1 << 28,
                    or_fold=gpu_or_fold) -> None:
    """E1: in-place OR-merge of every rank's `words` via chunked all_gather."""
    P = dist.get_world_size(group)
    if P == 1:
        return
    M = words.numel()
    chunk = min(chunk_bytes, M)
    stage = torch.empty(P * chunk, dtype=words.dtype, device=words.device)
    for off in range(0, M, chunk):
        c = min(chunk, M - off)
        out = stage[: P * c]
        dist.all_gather_into_tensor(out, words[off:off + c], group=group)
        or_fold(words[off:off + c], out.view(P, c))


def merge_alltoall(words: torch.Tensor, group=None, or_fold=gpu_or_fold) -> None:
    """E2: in-place OR-merge via all_to_all (reduce-scatter by OR) + all_gather.

    The filter is viewed as P equal ranges (zero-padded to a multiple of P*64
    bytes); rank r receives range r of every partial, folds it, and the
    merged ranges are all-gathered back into a full replica."""
    P = dist.get_world_size(group)
    if P == 1:
        return
    M = words.numel()
    per = -(-M // P)
    per = -(-per // 64) * 64
    padded = per * P
    if padded != M:
        send = torch.zeros(padded, dtype=words.dtype, device=words.device)
        send[:M] = words
    else:
        send = words
    recv = torch.empty((P, per), dtype=words.dtype, device=words.device)
    dist.all_to_all_single(recv.view(-1), send, group=group)
    mine = torch.empty(per, dtype=words.dtype, device=words.device)
    or_fold(mine, recv)
    dist.all_gather_into_tensor(send, mine, group=group)  # send is free again
    if padded != M:
        words.copy_(send[:M])


class NvlsMerger:
    """E4: in-switch OR merge over NVLink SHARP (bf_mcast_*, include/bf.h).

    Collective constructor: rank 0 creates the multicast object and
    broadcasts its handle, every rank adds its device and binds a
    ``nbytes`` buffer of its own (``self.buf``, a uint8 device view).
    ``merge(words)``: copy the partial filter in, each rank ORs its 1/P slice
    of all copies inside the switch (multimem.ld_reduce.or + multimem.st),
    copy the merged filter back.  NVLink traffic per rank: M/P in + M/P out
    through the switch, against 2(P-1)/P*M for E2."""

    def __init__(self, nbytes: int, group=None, handle_type: int | None = None):
        from . import bf
        self.group = group
        self.P = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        ht = bf.BF_MCAST_POSIX_FD if handle_type is None else handle_type
        obj = [None]
        if self.rank == 0:
            self.m, blob = bf.bf_mcast_create(nbytes, self.P, ht, True)
            obj = [blob]
        if self.P > 1:
            dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group else 0, group=group)
        if self.rank != 0:
            self.m, _ = bf.bf_mcast_create(nbytes, self.P, ht, False, obj[0])
        bf.bf_mcast_add_device(self.m)
        self._barrier()
        uc = bf.bf_mcast_bind(self.m)
        self._barrier()
        self.nbytes = nbytes
        self.buf = bf._device_view(uc, nbytes)

    def _barrier(self):
        if self.P > 1:
            dist.barrier(group=self.group)

    def merge(self, words: torch.Tensor) -> None:
        from . import bf
        M = words.numel()
        assert M <= self.nbytes and M % 8 == 0
        self.buf[:M].copy_(words)
        torch.cuda.synchronize()
        self._barrier()
        bf.bf_mcast_or_reduce(self.m, self.rank, M)
        torch.cuda.synchronize()
        self._barrier()
        words.copy_(self.buf[:M])

    def close(self):
        from . import bf
        if getattr(self, "m", None):
            self._barrier()
            bf.bf_mcast_destroy(self.m)
            self.m = None


_nvls_cache: dict = {}


def merge_nvls(words: torch.Tensor, group=None) -> None:
    """E4 as a MERGES entry: one NvlsMerger per (group, size), kept for reuse."""
    key = (id(group), words.numel(), words.device.index)
    mg = _nvls_cache.get(key)
    if mg is None:
        mg = _nvls_cache[key] = NvlsMerger(words.numel(), group)
    mg.merge(words)


class P2pMerger:
    """OR merge over NVLink peer memory (bf_p2p_or_merge, include/bf.h).

    Collective constructor over the group: every rank exports the CUDA IPC
    handle of its filter allocation (``words`` must be the filter's whole
    word array, bf_data's view), all_gathers the handles and maps every
    peer's filter.  ``merge()``: a stream-ordered barrier (all_reduce of one
    element: every rank's adds are done), one kernel per rank that ORs its
    1/P slice of all P filters and writes it into all P, and a second barrier
    (every rank's stores into this filter are done before it is read).  No
    staging buffer, no separate fold pass; per rank (P-1)/P*M bytes read from
    peers and (P-1)/P*M written to them."""

    def __init__(self, words: torch.Tensor, group=None):
        from . import bf
        self.group = group
        self.P = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if self.P > bf.BF_P2P_MAX_RANKS:
            raise ValueError(f"p2p merge supports at most {bf.BF_P2P_MAX_RANKS} ranks")
        self.words = words
        self.nbytes = words.numel()
        mine = bf.bf_ipc_handle(words.data_ptr())
        handles = [None] * self.P
        dist.all_gather_object(handles, mine, group=group)
        self.peers = []
        self._opened = []
        for q, h in enumerate(handles):
            if q == self.rank:
                self.peers.append(words.data_ptr())
            else:
                p = bf.bf_ipc_open(h)
                self._opened.append(p)
                self.peers.append(p)
        self.flag = torch.zeros(1, dtype=torch.int32, device=words.device)

    def merge(self, words: torch.Tensor | None = None) -> None:
        from . import bf
        if words is not None and words.data_ptr() != self.words.data_ptr():
            raise ValueError("P2pMerger merges the filter it was built for")
        dist.all_reduce(self.flag, group=self.group)  # every rank's adds are done
        bf.bf_p2p_or_merge(self.peers, self.rank, self.nbytes)
        dist.all_reduce(self.flag, group=self.group)  # every rank's stores are done

    def close(self):
        from . import bf
        if self._opened:
            if self.words.is_cuda:
                torch.cuda.synchronize()
            dist.barrier(group=self.group)
            for p in self._opened:
                bf.bf_ipc_close(p)
            self._opened = []


_p2p_cache: dict = {}


def merge_p2p(words: torch.Tensor, group=None) -> None:
    """P2P merge as a MERGES entry: one P2pMerger per (group, filter), kept."""
    key = (id(group), words.data_ptr(), words.numel())
    mg = _p2p_cache.get(key)
    if mg is None:
        mg = _p2p_cache[key] = P2pMerger(words, group)
    mg.merge(words)


MERGES = {"allgather": merge_allgather, "alltoall": merge_alltoall, "nvls": merge_nvls, "p2p": merge_p2p}


def build_replicated(filt, keys: torch.Tensor, strategy: str = "alltoall", group=None) -> None:
    """Every rank adds its key shard, then the partial filters are OR-merged so
    every rank holds the filter of the union of all shards."""
    filt.add(keys)
    MERGES[strategy](filt.data(), group=group)


def build_replicated_routed(pf, keys: torch.Tensor, words: torch.Tensor, block_bytes: int) -> None:
    """E3: route every key to the owner of its block range
    (hash once, all_to_all of records), each owner builds its range, then the
    ranges are all-gathered into every rank's replica `words`.  Moves 8 B per
    key plus (P-1)/P of the filter per rank, instead of E2's 2(P-1)/P of the
    filter; no OR-fold (owners never overlap)."""
    pf.clear()
    pf.add(keys)
    pf.gather_into(words, block_bytes)


def lookup_sharded(filt, keys: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """Data-parallel lookup of this rank's shard against its replica (no
    communication)."""
    return filt.contains(keys, out)


# --------------------------------------------------------------------------
# Block-range partitioned filters (NEXT N1): filters larger than one GPU.
# Owner p of P ranks holds global blocks [floor(p*b/P), floor((p+1)*b/P)).
# add:      route (hash once, bin by owner) -> fixed-count all_to_all of the
#           record buckets (+ their counts) -> each owner ORs what it received.
# contains: route -> all_to_all -> owners test -> all_to_all of the result
#           bytes back -> each sender scatters the bits to its keys' indices.

class GpuRouteOps:
    """The CUDA kernels behind the C ABI (bf_route, bf_add_routed,
    bf_contains_routed, bf_scatter_results)."""

    def __init__(self, handle):
        from . import bf
        self.bf, self.h = bf, handle

    def route(self, keys, cap, P, want_idx):
        dev = keys.device
        recs = torch.empty(P * cap, dtype=torch.int64, device=dev)
        idx = torch.empty(P * cap, dtype=torch.int64, device=dev) if want_idx else None
        counts = torch.empty(P, dtype=torch.int64, device=dev)
        self.bf.bf_route(self.h, keys, keys.numel(), 0, recs, idx, cap, counts)
        return recs, idx, counts

    def add_routed(self, recv, rcounts, P, cap):
        self.bf.bf_add_routed(self.h, recv, rcounts, P, cap)

    def contains_routed(self, recv, rcounts, P, cap):
        res = torch.empty(P * cap, dtype=torch.uint8, device=recv.device)
        self.bf.bf_contains_routed(self.h, recv, rcounts, P, cap, res)
        return res

    def scatter(self, idx, res, counts, P, cap, n):
        out = torch.zeros((n + 31) // 32, dtype=torch.int32, device=idx.device)
        self.bf.bf_scatter_results(idx, res, counts, P, cap, out)
        return out

    def part_bytes(self):
        """This part's word array (a uint8 device view, no copy)."""
        ptr, nbytes = self.bf.bf_data(self.h)
        return self.bf._device_view(ptr, nbytes)

    def clear(self):
        self.bf.bf_clear(self.h)


class PartitionedFilter:
    """One rank's part of a block-range partitioned filter."""

    def __init__(self, m_bits: int, k: int, block_bits: int = 256, word_bits: int = 64, variant: int = 3,
                 z: int = 0, seed: int = 0, group=None, ops=None, slack: float = 0.05,
                 pad: int = 4096):
        from . import bf
        self.group = group
        self.P = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.slack, self.pad = slack, pad
        if ops is None:
            v = variant | (z << 8) if variant == bf.BF_CSBF else variant
            self.handle = bf.bf_create_part(m_bits, k, block_bits, word_bits, v, seed, self.P, self.rank)
            self.info = bf.bf_part_info(self.handle)
            ops = GpuRouteOps(self.handle)
        self.ops = ops

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            from . import bf
            bf.bf_destroy(h)
            self.handle = None

    def _cap(self, n: int) -> int:
        """Records per (sender, owner) bucket: the same on every rank (the
        all_to_all is fixed-count), a multiple of 128."""
        t = torch.tensor([n], dtype=torch.int64, device=self._dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        nmax = int(t.item())
        cap = int(nmax / self.P * (1 + self.slack)) + self.pad
        return (cap + 127) // 128 * 128

    def _exchange(self, send, P, cap):
        recv = torch.empty_like(send)
        dist.all_to_all_single(recv, send, group=self.group)
        return recv

    def _route_agreed(self, keys, want_idx):
        """Route, then agree COLLECTIVELY on whether any (sender, owner)
        bucket overflowed: every rank all-reduces (MAX) its largest count, so
        all ranks see the same number and either all proceed to the
        exchange or all re-route with a larger cap (a skewed or
        duplicate-heavy shard would otherwise raise on one rank while the
        others wait in all_to_all, or drop records: false negatives).
        bf_route counts every record, also those past cap, so one retry
        always suffices."""
        P, cap = self.P, self._cap(keys.numel())
        while True:
            recs, idx, counts = self.ops.route(keys, cap, P, want_idx)
            t = counts.max().reshape(1).to(torch.int64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
            need = int(t.item())
            if need <= cap:
                return recs, idx, counts, cap
            cap = (int(need * (1 + self.slack)) + 127) // 128 * 128

    def add(self, keys: torch.Tensor) -> None:
        self._dev = keys.device
        P = self.P
        recs, _, counts, cap = self._route_agreed(keys, False)
        recv = self._exchange(recs, P, cap)
        rcounts = self._exchange(counts, P, 1)
        self.ops.add_routed(recv, rcounts, P, cap)

    def clear(self) -> None:
        self.ops.clear()

    def gather_into(self, words: torch.Tensor, block_bytes: int) -> None:
        """E3's second half: all_gather every owner's block
        range into `words`, the full filter's word array on every rank, so
        that route-to-owner construction (``add``) yields a replica.  Parts
        differ by at most one block; each rank sends its part padded to the
        largest and the valid prefix of every part is copied to its offset
        floor(p*b/P)*block_bytes."""
        mine = self.ops.part_bytes()
        P = self.P
        b = words.numel() // block_bytes
        offs = [b * p // P * block_bytes for p in range(P + 1)]
        mx = max(offs[p + 1] - offs[p] for p in range(P))
        send = torch.zeros(mx, dtype=torch.uint8, device=words.device)
        send[:mine.numel()].copy_(mine)
        recv = torch.empty(P * mx, dtype=torch.uint8, device=words.device)
        dist.all_gather_into_tensor(recv, send, group=self.group)
        for p in range(P):
            words[offs[p]:offs[p + 1]].copy_(recv[p * mx:p * mx + offs[p + 1] - offs[p]])

    def contains(self, keys: torch.Tensor) -> torch.Tensor:
        self._dev = keys.device
        P = self.P
        recs, idx, counts, cap = self._route_agreed(keys, True)
        recv = self._exchange(recs, P, cap)
        rcounts = self._exchange(counts, P, 1)
        res = self.ops.contains_routed(recv, rcounts, P, cap)
        back = self._exchange(res, P, cap)  # result bytes return to the senders' slots
        return self.ops.scatter(idx, back, counts, P, cap, keys.numel())
