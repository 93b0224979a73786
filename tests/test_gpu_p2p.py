"""OR merge over peer memory (bf_p2p_or_merge, include/bf.h).

One GPU here, so the P ranks are virtual: P filters on the same device, each
built from its key shard, and rank r's merge kernel launched for r = 0..P-1
(the ranks' slices are disjoint, so the order does not matter).  Afterwards
every filter must equal the oracle's filter of ALL keys -- the property the
multi-GPU merge must have.  The IPC mapping between processes is the CUDA
runtime's; here only the export and the documented same-process refusal are
exercised."""
import numpy as np
import pytest

import synth
from oracle.bfo import OracleFilter

pytestmark = pytest.mark.gpu


def _dev(torch, a, dev):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).to(dev)


@pytest.mark.parametrize("P", [2, 3, 8])
@pytest.mark.parametrize("cfg", [(3, 256, 64, 8, 0, 1 << 22), (4, 256, 32, 8, 2, (1 << 22) + 256 * 5),
                                 (2, 32, 32, 6, 0, (1 << 20) + 32 * 3)])
def test_p2p_merge_equals_single_builder(bflib, cuda, P, cfg):
    import torch
    bf = bflib
    v, B, S, k, z, m = cfg
    n = 50_021
    filters = []
    for r in range(P):
        f = bf.Filter(m, k, B, S, variant=v, z=z)
        f.add(_dev(torch, synth.positives(n, r, P), cuda))
        filters.append(f)
    torch.cuda.synchronize()
    nbytes = filters[0].nbytes()
    peers = [bf.bf_data(f.handle)[0] for f in filters]
    launches = bf.bf_launch_count()
    for r in range(P):
        bf.bf_p2p_or_merge(peers, r, nbytes)
    torch.cuda.synchronize()
    assert bf.bf_launch_count() - launches == P
    o = OracleFilter(v, m, B=B, S=S, k=k, z=z)
    o.add(synth.positives(n))
    want = o.bytes()
    for f in filters:
        assert np.array_equal(f.data().cpu().numpy(), want)


@pytest.mark.parametrize("P,nbytes", [(2, 4), (3, 16 * 5 + 12), (5, (1 << 20) + 4 * 3), (16, 4096)])
def test_p2p_merge_raw_buffers_and_tails(bflib, cuda, P, nbytes):
    import torch
    bf = bflib
    rng = np.random.default_rng(P * 1000 + nbytes)
    host = [rng.integers(0, 256, nbytes, dtype=np.uint8) & rng.integers(0, 256, nbytes, dtype=np.uint8)
            for _ in range(P)]
    bufs = [torch.from_numpy(h).to(cuda) for h in host]
    want = np.bitwise_or.reduce(np.stack(host), axis=0)
    for r in range(P):
        bf.bf_p2p_or_merge([b.data_ptr() for b in bufs], r, nbytes)
    torch.cuda.synchronize()
    for b in bufs:
        assert np.array_equal(b.cpu().numpy(), want)


def test_p2p_argument_validation_and_ipc(bflib, cuda):
    import torch
    bf = bflib
    a = torch.zeros(1024, dtype=torch.uint8, device=cuda)
    b = torch.zeros(1024, dtype=torch.uint8, device=cuda)
    ptrs = [a.data_ptr(), b.data_ptr()]
    for bad in (lambda: bf.bf_p2p_or_merge(ptrs, 2, 1024),            # rank >= nranks
                lambda: bf.bf_p2p_or_merge(ptrs, 0, 1022),            # bytes % 4
                lambda: bf.bf_p2p_or_merge([ptrs[0], ptrs[1] + 4], 0, 1000),  # misaligned
                lambda: bf.bf_p2p_or_merge(ptrs * 9, 0, 1024),        # > 16 ranks
                lambda: bf.bf_p2p_or_merge([ptrs[0], 0], 0, 1024)):   # null peer
        with pytest.raises(bf.BFError) as ei:
            bad()
        assert ei.value.code == bf.BF_EINVAL
    bf.bf_p2p_or_merge(ptrs, 0, 0)  # empty: no-op
    f = bf.Filter(1 << 20, 8, 256, 64, "SBF")
    h = bf.bf_ipc_handle(bf.bf_data(f.handle)[0])
    assert len(h) == bf.BF_IPC_HANDLE_BYTES and any(h)
    with pytest.raises(bf.BFError) as ei:  # IPC is between processes (documented)
        bf.bf_ipc_open(h)
    assert ei.value.code == bf.BF_ECUDA
