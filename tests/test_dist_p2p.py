"""Host logic of the peer-memory OR merge (dist.P2pMerger) with gloo at world
sizes 2 and 3: every rank exports its filter's IPC handle, gathers all, maps
the peers' (its own slot keeps the local pointer), and each merge is one
kernel launch for its own rank between two stream-ordered barriers.  The CUDA
calls are replaced by recorders (no GPU here); tests/test_gpu_p2p.py checks
the kernel itself."""
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, results):
    import torch.distributed as dist

    from paper_2512_15595_b200 import bf
    from paper_2512_15595_b200 import dist as bfdist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    calls = []
    bf.bf_ipc_handle = lambda ptr: f"{rank}:{ptr}".encode().ljust(bf.BF_IPC_HANDLE_BYTES, b"\0")
    bf.bf_ipc_open = lambda h: int(h.rstrip(b"\0").decode().split(":")[1]) + 10 ** 9
    bf.bf_ipc_close = lambda p: calls.append(("close", p))
    bf.bf_p2p_or_merge = lambda peers, r, n, stream=None: calls.append(("merge", list(peers), r, n))
    try:
        words = torch.zeros(4096 + 64 * rank, dtype=torch.uint8)
        m = bfdist.P2pMerger(words)
        ptrs = [None] * world
        dist.all_gather_object(ptrs, words.data_ptr())
        want = [ptrs[q] if q == rank else ptrs[q] + 10 ** 9 for q in range(world)]
        ok = m.peers == want and m.rank == rank and m.P == world
        m.merge(words)
        m.merge()
        ok = ok and calls == [("merge", want, rank, words.numel())] * 2
        m._opened and m.close()
        ok = ok and sorted(c[1] for c in calls if c[0] == "close") == sorted(p for q, p in enumerate(want) if q != rank)
        try:
            m.merge(torch.zeros(8, dtype=torch.uint8))
            ok = False
        except ValueError:
            pass
        results[rank] = ok
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_p2p_merger_host_logic(world):
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    assert dict(results) == {r: True for r in range(world)}
