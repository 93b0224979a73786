"""Multi-process (torch.distributed, gloo, CPU) tests of the multi-GPU merge
logic in paper_2512_15595_b200/dist.py: every rank builds a partial filter
from its key shard, the partials are OR-merged (E1 chunked all_gather + fold,
E2 all_to_all + fold + all_gather), and every rank must end up with exactly
the filter one builder makes from all keys (north_star: "merges them with
ncclAllGather plus an OR-fold kernel").

The partial filters come from the CPU oracle and the OR-fold is a CPU torch
fold here (test-only); the product path uses the CUDA library for both
(tests/test_gpu_parity.py::test_or_fold covers the kernel)."""
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


def _cpu_fold(dst, src2d):
    acc = src2d[0].clone()
    for r in range(1, src2d.shape[0]):
        acc |= src2d[r]
    dst.copy_(acc)


def _worker(rank, world, port, strategy, m_bits, n, chunk, results):
    import torch.distributed as dist

    import synth
    from oracle.bfo import OracleFilter
    from paper_2512_15595_b200 import dist as bfdist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shard = synth.positives(n, rank, world)
        part = OracleFilter(3, m_bits, B=256, S=64, k=8)
        part.add(shard)
        words = torch.from_numpy(part.bytes())
        if strategy == "allgather":
            bfdist.merge_allgather(words, chunk_bytes=chunk, or_fold=_cpu_fold)
        else:
            bfdist.merge_alltoall(words, or_fold=_cpu_fold)
        full = OracleFilter(3, m_bits, B=256, S=64, k=8)
        full.add(synth.positives(n))
        results[rank] = bool(np.array_equal(words.numpy(), full.bytes()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("strategy,m_bits,chunk", [
    ("alltoall", 1 << 20, 0),              # M divisible by P*64
    ("alltoall", (1 << 20) + 256 * 7, 0),  # ragged: zero-padded ranges
    ("allgather", 1 << 20, 1 << 12),       # several chunks
    ("allgather", (1 << 20) + 256 * 7, 5000),  # ragged last chunk
])
def test_merge_equals_single_builder(world, strategy, m_bits, chunk):
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), strategy, m_bits, 30011, chunk or (1 << 28), results),
             nprocs=world, join=True)
    assert dict(results) == {r: True for r in range(world)}
