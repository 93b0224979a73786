"""The multi-GPU construction strategies on a one-rank NCCL group (the only
GPU topology here): E3 route-to-owner construction + all_gather of the block
ranges (dist.build_replicated_routed) through the CUDA routing kernels, and
the E1/E2/p2p merges, must leave the oracle's filter of all keys.  With P = 1
the exchanges are trivial; the P > 1 exchange logic is covered with gloo
(tests/test_dist_*.py) and the kernels with P virtual owners
(tests/test_gpu_parity.py, tests/test_gpu_p2p.py)."""
import socket

import numpy as np
import pytest

import synth
from oracle.bfo import OracleFilter

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl1(cuda):
    import torch.distributed as dist
    if not dist.is_nccl_available():
        pytest.skip("no NCCL")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=cuda)
    yield
    dist.destroy_process_group()


@pytest.mark.parametrize("strategy", ["route", "alltoall", "allgather", "p2p"])
def test_one_rank_strategies(bflib, cuda, nccl1, strategy):
    import torch
    from paper_2512_15595_b200 import dist as bfdist
    bf = bflib
    m, n = (1 << 22) + 256 * 3, 30_011
    keys = synth.keys(17, n)
    kd = torch.from_numpy(keys.view(np.int64)).to(cuda)
    f = bf.Filter(m, 8, 256, 64, "SBF")
    words = f.data()
    if strategy == "route":
        pf = bfdist.PartitionedFilter(m, 8, 256, 64, 3)
        bfdist.build_replicated_routed(pf, kd, words, 32)
    else:
        bfdist.build_replicated(f, kd, strategy)
    torch.cuda.synchronize()
    o = OracleFilter(3, m, B=256, S=64, k=8)
    o.add(keys)
    assert np.array_equal(words.cpu().numpy(), o.bytes())
