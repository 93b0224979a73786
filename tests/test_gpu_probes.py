"""Round-2 ABI on the GPU: the launch-shape control (results never depend on
it), the roofline probes' contracts (records of the add's RED pattern, GUPS
probes, probe launch shape) and the L2 fetch-granularity control."""
import numpy as np
import pytest

import synth
from oracle.bfo import OracleFilter

pytestmark = pytest.mark.gpu


def _dev(torch, a, dev):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).to(dev)


@pytest.mark.parametrize("cfg", [(3, 256, 64, 8, 0), (1, 256, 64, 16, 0), (2, 64, 64, 13, 0), (4, 256, 32, 8, 2)])
def test_launch_shape_never_changes_results(bflib, cuda, cfg):
    """bf_set_launch: 1 CTA/SM (persistent, under occupancy), the occupancy
    grid, the default waves and an oversized grid all give the oracle's bits."""
    import torch
    bf = bflib
    v, B, S, k, z = cfg
    m = B * 40_013
    n = (1 << 20) + 3
    keys = synth.keys(77, n)
    q = np.concatenate([keys[::5], synth.negatives(50_001)])
    o = OracleFilter(v, m, B=B, S=S, k=k, z=z)
    o.add(keys, threads=8)
    want, want_q = o.bytes(), o.contains(q, threads=8)
    f = bf.Filter(m, k, B, S, variant=v, z=z)
    kd, qd = _dev(torch, keys, cuda), _dev(torch, q, cuda)
    occ = [bf.bf_get_launch(f.handle, op)[1] for op in (0, 1)]
    assert bf.bf_get_launch(f.handle, 0)[0] == 32  # the default: waves of 32 CTAs per SM
    for cps in (1, occ[0], 0, 100):
        f.set_launch(0, cps)
        f.set_launch(1, cps)
        f.clear()
        f.add(kd)
        got = f.contains(qd)
        torch.cuda.synchronize()
        assert np.array_equal(f.data().cpu().numpy(), want), cps
        assert np.array_equal(got.cpu().numpy().view(np.uint32), want_q), cps
    with pytest.raises(bf.BFError):
        bf.bf_set_launch(f.handle, 0, 2000)


@pytest.mark.parametrize("cfg", [(3, 256, 64, 8, 0), (2, 64, 64, 6, 0), (1, 256, 64, 11, 0), (1, 128, 64, 16, 0),
                                 (4, 256, 32, 8, 2), (4, 256, 32, 8, 4)])
def test_pattern_records_follow_the_configuration(bflib, cuda, cfg):
    """bf_probe_pattern_records: block < b; the word-hit mask is all s words
    (SBF/RBBF), one word per group (CSBF), 1..min(k, s) words (BBF); the
    BBF mean matches s(1 - (1 - 1/s)^k) (k uniform word draws)."""
    import torch
    bf = bflib
    v, B, S, k, z = cfg
    s = B // S
    b, n = 1_000_003, 1 << 20
    recs = torch.empty(n, dtype=torch.int64, device=cuda)
    bf.bf_probe_pattern_records(recs, n, b, B, S, v, k, z, 5)
    torch.cuda.synchronize()
    r = recs.cpu().numpy().view(np.uint64)
    blk = (r >> np.uint64(32)).astype(np.int64)
    mask = (r & np.uint64(0xFFFFFFFF)).astype(np.uint64)
    assert blk.min() >= 0 and blk.max() < b
    assert (mask >> np.uint64(s) == 0).all()
    pc = np.array([bin(int(x)).count("1") for x in mask[:20000]])
    if v in (2, 3):
        assert (mask == (1 << s) - 1).all()
    elif v == 4:
        g = s // z
        for gi in range(z):
            grp = (mask[:20000] >> np.uint64(gi * g)) & np.uint64((1 << g) - 1)
            assert all(bin(int(x)).count("1") == 1 for x in grp)
    else:
        assert pc.min() >= 1 and pc.max() <= min(k, s)
        assert abs(pc.mean() - s * (1 - (1 - 1 / s) ** k)) < 0.02 * s
    buf = torch.zeros(b * B // 8, dtype=torch.uint8, device=cuda)
    bf.bf_probe_red_records(buf, B, S, recs, n)
    torch.cuda.synchronize()
    assert buf.any()


def test_gups_probes_and_probe_launch(bflib, cuda):
    import torch
    bf = bflib
    nbytes = 64 << 20
    buf = torch.zeros(nbytes, dtype=torch.uint8, device=cuda)
    for ab, red, hint in ((8, 0, 0), (8, 0, 1), (32, 0, 1), (64, 0, 0), (8, 1, 0)):
        for mlp, ctas in ((0, 0), (1, 148), (16, 0)):
            bf.bf_probe_gups(buf, nbytes, ab, red, hint, 1 << 20, mlp, ctas)
    torch.cuda.synchronize()
    assert buf.any()  # the update probe ORed bits in
    with pytest.raises(bf.BFError):
        bf.bf_probe_gups(buf, nbytes, 16, 0, 0, 1 << 20)  # 16-byte accesses are not a probe form
    with pytest.raises(bf.BFError):
        bf.bf_probe_gups(buf, nbytes, 8, 1, 1, 1 << 20)  # updates take no fill hint
    for cps in (8, 32, 0):
        bf.bf_set_probe_launch(cps)
        bf.bf_probe_rng(buf, nbytes // 32, 256, 0, 1, 1 << 20)
    torch.cuda.synchronize()
    with pytest.raises(bf.BFError):
        bf.bf_set_probe_launch(-1)


def test_l2_fetch_granularity_roundtrip(bflib, cuda):
    bf = bflib
    base = bf.bf_get_l2_fetch_granularity()
    for g in (32, 64, 128):
        bf.bf_set_l2_fetch_granularity(g)
        assert bf.bf_get_l2_fetch_granularity() in (g, base)  # the driver may keep its own value
    bf.bf_set_l2_fetch_granularity(0)
    assert bf.bf_get_l2_fetch_granularity() == base
    with pytest.raises(bf.BFError):
        bf.bf_set_l2_fetch_granularity(48)
