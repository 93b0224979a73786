"""Pins of the oracle's block selection and bit patterns.

* SBF(B=256, S=32, k=8) is the Parquet split-block Bloom filter (Apple's
  split-block filter, cited by the paper for the SBF): the
  oracle's bit array must appear byte for byte in the file pyarrow writes.
  This pins XXH64 of the LE key, block = ((h>>32)*b)>>32, the 32-bit
  multiply-shift draws with SALT[0..7], the bit order and the block layout.
* Equivalences fixed by the definitions: RBBF == BBF(B=S) == SBF(s=1);
  BBF bytes independent of S; CSBF(z=s) == SBF.
* Invariants: no false negatives, idempotence, order/partition invariance,
  block confinement, SBF <= q bits per word, CSBF exactly one word per group.
* Uniformity of every draw and of the block index (chi-square).
"""
import io

import numpy as np
import pytest
from scipy import stats

import synth
from oracle import bfo
from oracle.bfo import BBF, CSBF, RBBF, SBF, OracleFilter, unpack_bits

pa = pytest.importorskip("pyarrow")
pq = pytest.importorskip("pyarrow.parquet")


def _parquet_bytes(keys, ndv, fpp):
    t = pa.table({"k": pa.array(keys, pa.uint64())})
    buf = io.BytesIO()
    pq.write_table(t, buf, bloom_filter_options={"k": {"ndv": ndv, "fpp": fpp}})
    return buf.getvalue()


@pytest.mark.parametrize("n,ndv,fpp,nbytes", [
    (5000, 5000, 0.01, 8192),
    (20000, 20000, 0.01, 32768),
    (1 << 16, 1 << 16, 0.001, 131072),
    (1 << 20, 1 << 20, 0.01, 1 << 21),   # configs[0] size: m = 2^24 bits, 2^20 keys
])
def test_sbf_256_32_8_equals_parquet_sbbf(n, ndv, fpp, nbytes):
    keys = synth.keys(0, n)
    data = _parquet_bytes(keys, ndv, fpp)
    f = OracleFilter(SBF, nbytes * 8, B=256, S=32, k=8)
    f.add(keys, threads=4)
    assert data.find(f.bytes().tobytes()) >= 0


def test_parquet_pin_high_keys():
    keys = synth.keys(12345, 20000)
    assert (keys >= np.uint64(1 << 63)).sum() > 5000
    data = _parquet_bytes(keys, 20000, 0.01)
    f = OracleFilter(SBF, 32768 * 8, B=256, S=32, k=8)
    f.add(keys)
    assert data.find(f.bytes().tobytes()) >= 0


def _build(variant, m, B, S, k, z=0, keys=None, threads=1):
    f = OracleFilter(variant, m, B=B, S=S, k=k, z=z)
    f.add(keys, threads=threads)
    return f


KEYS = synth.keys(0, 30000)


@pytest.mark.parametrize("W,k", [(32, 3), (32, 8), (64, 5), (64, 16)])
def test_rbbf_equals_bbf_equals_sbf_one_word(W, k):
    m = 1 << 18
    a = _build(RBBF, m, W, W, k, keys=KEYS).bytes()
    b = _build(BBF, m, W, W, k, keys=KEYS).bytes()
    c = _build(SBF, m, W, W, k, keys=KEYS).bytes()
    assert np.array_equal(a, b) and np.array_equal(a, c)


@pytest.mark.parametrize("B,k", [(64, 4), (128, 7), (256, 11)])
def test_bbf_independent_of_word_size(B, k):
    m = 1 << 18
    assert np.array_equal(_build(BBF, m, B, 32, k, keys=KEYS).bytes(),
                          _build(BBF, m, B, 64, k, keys=KEYS).bytes())


@pytest.mark.parametrize("B,S,k", [(256, 32, 8), (256, 64, 8), (128, 32, 8), (256, 64, 12)])
def test_csbf_with_z_equal_s_is_sbf(B, S, k):
    s = B // S
    m = (1 << 18) + B * 3  # non-power-of-two block count
    assert np.array_equal(_build(CSBF, m, B, S, k, z=s, keys=KEYS).bytes(),
                          _build(SBF, m, B, S, k, keys=KEYS).bytes())


CONFIGS = [
    (BBF, 256, 64, 8, 0), (BBF, 128, 32, 5, 0), (RBBF, 64, 64, 6, 0), (RBBF, 32, 32, 4, 0),
    (SBF, 256, 64, 8, 0), (SBF, 256, 32, 16, 0), (SBF, 128, 64, 4, 0), (SBF, 64, 32, 6, 0),
    (CSBF, 256, 32, 8, 2), (CSBF, 256, 32, 8, 4), (CSBF, 256, 64, 6, 2), (BBF, 1024, 64, 16, 0),
]


@pytest.mark.parametrize("cfg", CONFIGS)
def test_no_false_negatives_idempotence_order_partition(cfg):
    v, B, S, k, z = cfg
    m = 1 << 17
    f = _build(v, m, B, S, k, z, keys=KEYS)
    assert unpack_bits(f.contains(KEYS), KEYS.size).all()
    once = f.bytes()
    f.add(KEYS)
    assert np.array_equal(f.bytes(), once)
    rng = np.random.default_rng(3)
    g = _build(v, m, B, S, k, z, keys=rng.permutation(KEYS), threads=7)
    assert np.array_equal(g.bytes(), once)
    # contains answers are thread-count independent
    q = np.concatenate([KEYS[:1000], synth.negatives(5000)])
    assert np.array_equal(f.contains(q, threads=1), f.contains(q, threads=5))


@pytest.mark.parametrize("cfg", CONFIGS)
def test_single_key_structure(cfg):
    v, B, S, k, z = cfg
    s = B // S
    m = B * 37  # b = 37 blocks
    for key in synth.keys(99, 200):
        f = OracleFilter(v, m, B=B, S=S, k=k, z=z)
        f.add([key])
        bits = np.unpackbits(f.bytes(), bitorder="little").reshape(37, B)
        touched = np.nonzero(bits.any(axis=1))[0]
        blk, pos = f.pattern(int(key))
        assert list(touched) == [blk]                      # block confinement
        assert bits.sum() == len(set(pos)) and 1 <= bits.sum() <= k
        words = bits[blk].reshape(s, S).sum(axis=1)
        if v == SBF:
            q = k // s
            assert (words >= 1).all() and (words <= q).all()
        if v == CSBF:
            g = s // z
            per_group = (words.reshape(z, g) > 0).sum(axis=1)
            assert (per_group == 1).all()
            assert (words[words > 0] <= k // z).all()
        assert f.popcount() == bits.sum()
        assert unpack_bits(f.contains([key]), 1)[0]


def test_empty_filter_rejects_everything():
    f = OracleFilter(SBF, 1 << 16, B=256, S=64, k=8)
    assert not unpack_bits(f.contains(KEYS[:1000]), 1000).any()
    assert f.contains([]).size == 0


def test_validation_rules():
    ok = bfo.validate
    assert ok(SBF, 1 << 20, 256, 64, 16)
    assert not ok(SBF, 1 << 20, 256, 64, 10)      # k % s != 0
    assert ok(CSBF, 1 << 20, 1024, 64, 16, 4)
    assert not ok(CSBF, 1 << 20, 256, 64, 6, 4)   # k % z != 0
    assert not ok(RBBF, 1 << 20, 128, 64, 8)      # RBBF needs B == S
    assert not ok(BBF, 1 << 20, 256, 48, 8)       # S in {32, 64}
    assert not ok(BBF, 1 << 20, 96, 32, 8)        # B power of two
    assert not ok(BBF, 1 << 20, 256, 64, 0)
    assert not ok(BBF, 1 << 20, 256, 64, 33)
    assert not ok(BBF, 0, 256, 64, 8)


def test_draw_and_block_uniformity():
    """Every draw's top bits and the block index are uniform (chi-square)."""
    n = 200_000
    keys = synth.keys(777, n)
    f = OracleFilter(SBF, 7 * 256, B=256, S=32, k=32)  # b = 7, not a power of two
    blocks = np.empty(n, dtype=np.int64)
    pos = np.empty((n, 32), dtype=np.int64)
    for i, key in enumerate(keys[:n]):
        b, p = f.pattern(int(key))
        blocks[i] = b
        pos[i] = p
    assert stats.chisquare(np.bincount(blocks, minlength=7)).pvalue > 1e-4
    for j in range(32):
        bitpos = pos[:, j] % 32
        word = pos[:, j] // 32
        assert (word == j // 4).all()  # SBF contiguous draw->word map (q = 4)
        assert stats.chisquare(np.bincount(bitpos, minlength=32)).pvalue > 1e-5, j
