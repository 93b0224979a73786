"""The oracle's range-restricted add / contains (used to check multi-GiB GPU
filters on sampled block ranges) against the full oracle filter.

Pinned to the full filter's definition: bfo_add_range over [lo, hi) must equal
bytes [lo*B/8, hi*B/8) of the whole filter built from the same keys, also when
accumulated over key chunks (OR commutes); bfo_contains_range must
equal bfo_contains for keys whose block is in the range and report -1
for the others.
"""
import numpy as np
import pytest

import synth
from oracle.bfo import BBF, CSBF, SBF, OracleFilter, unpack_bits

CFGS = [(SBF, 256, 64, 8, 0), (BBF, 256, 32, 11, 0), (CSBF, 256, 32, 8, 2), (SBF, 64, 32, 4, 0)]


@pytest.mark.parametrize("cfg", CFGS)
def test_add_range_equals_full_filter_slice(cfg):
    v, B, S, k, z = cfg
    m = (1 << 20) + 3 * B
    keys = synth.keys(5, 60_000)
    full = OracleFilter(v, m, B=B, S=S, k=k, z=z)
    full.add(keys)
    geo = OracleFilter(v, m, B=B, S=S, k=k, z=z, allocate=False)
    bb = B // 8
    for lo, hi in ((0, 97), (geo.b // 2, geo.b // 2 + 1000), (geo.b - 5, geo.b)):
        want = full.bytes()[lo * bb:hi * bb]
        assert np.array_equal(geo.add_range(keys, lo, hi, threads=3), want)
        acc = np.zeros(want.size, dtype=np.uint8)  # chunked accumulation
        for c in range(0, keys.size, 7_001):
            acc |= geo.add_range(keys[c:c + 7_001], lo, hi)
        assert np.array_equal(acc, want)


@pytest.mark.parametrize("cfg", CFGS)
def test_contains_range_equals_contains_inside(cfg):
    v, B, S, k, z = cfg
    m = 1 << 18  # dense enough for false positives among the negatives
    keys = synth.keys(11, 20_000)
    full = OracleFilter(v, m, B=B, S=S, k=k, z=z)
    full.add(keys)
    q = np.concatenate([keys[:3000], synth.negatives(20_000)])
    want = unpack_bits(full.contains(q), q.size)
    lo, hi = full.b // 4, full.b // 4 + full.b // 3
    bb = B // 8
    got = full.contains_range(q, lo, hi, full.bytes()[lo * bb:hi * bb], threads=2)
    blk = np.array([full.pattern(int(x))[0] for x in q])
    inside = (blk >= lo) & (blk < hi)
    assert inside.sum() > 1000 and (~inside).sum() > 1000
    assert (got[~inside] == -1).all()
    assert np.array_equal(got[inside].astype(bool), want[inside])
    assert got[inside][:].min() >= 0 and want[inside].sum() > inside[:3000].sum()  # some FPs too
    with pytest.raises(ValueError):
        full.contains_range(q, lo, hi, np.zeros(3, dtype=np.uint8))
