"""Pins of the oracle's hashing (XXH64) and salt tables.

Pinned against: the independent `xxhash` library (exact), the published
XXH64 reference value of the empty input, and the generation rule the salt
tables are declared to follow (DESIGN.md "Readings" item 2).
"""
import numpy as np
import pytest
import xxhash

import synth
from oracle import bfo


def test_xxh64_empty_published_vector():
    # xxHash reference: XXH64("", seed=0) = 0xEF46DB3751D8E999
    assert bfo.xxh64(b"", 0) == 0xEF46DB3751D8E999


@pytest.mark.parametrize("seed", [0, 1, 0x9E3779B97F4A7C15, 2**64 - 1])
def test_xxh64_all_lengths_vs_xxhash(seed):
    rng = np.random.default_rng(7)
    for L in list(range(0, 80)) + [127, 128, 129, 1000]:
        data = rng.integers(0, 256, L, dtype=np.uint8).tobytes()
        assert bfo.xxh64(data, seed) == xxhash.xxh64_intdigest(data, seed), (L, seed)


def test_xxh64_u64_keys_vs_xxhash():
    ks = synth.keys(0, 20000)
    extra = [0, 1, 2**63, 0x0123456789ABCDEF, 2**64 - 1]
    for key in list(ks) + extra:
        key = int(key)
        assert bfo.xxh64_u64(key, 0) == xxhash.xxh64_intdigest(key.to_bytes(8, "little"), 0)
        assert bfo.xxh64_u64(key, 1) == xxhash.xxh64_intdigest(key.to_bytes(8, "little"), 1)


def _rule_tables():
    """The stated generation rule: v_i = (mix64(0x5A17+i) >> 32) | 1, skipping
    repeats; SALT[8..63] then GSALT[0..15]; SALT[0..7] = Parquet SBBF salts."""
    parquet = [0x47B6137B, 0x44974D91, 0x8824AD5B, 0xA2B7289D,
               0x705495C7, 0x2DF1424B, 0x9EFC4947, 0x5C6BFB31]
    tab, ext, i = list(parquet), [], 0
    with np.errstate(over="ignore"):
        while len(ext) < 72:
            v = (int(synth.mix64(np.uint64(0x5A17 + i))) >> 32) | 1
            i += 1
            if v in tab or v in ext:
                continue
            ext.append(v)
    return parquet + ext[:56], ext[56:72]


def test_salt_tables_follow_rule():
    salt, gsalt = _rule_tables()
    assert bfo.salt_table() == salt
    assert bfo.gsalt_table() == gsalt
    allv = salt + gsalt
    assert all(v & 1 for v in allv), "salts must be odd (multiply-shift)"
    assert len(set(allv)) == len(allv)


def test_keygen_splitmix_first_outputs():
    # SplitMix64 (Steele/Lea/Flood; Vigna's reference) first outputs from state 0
    assert [int(x) for x in synth.keys(0, 3)] == [0xE220A8397B1DCDAF, 0x910A2DEC89025CC1,
                                                   0x975835DE1C9756CE]


def test_keygen_unique_and_disjoint():
    pos = synth.positives(1 << 18)
    neg = synth.negatives(1 << 18)
    assert np.unique(pos).size == pos.size
    assert np.intersect1d(pos, neg).size == 0
    # shards partition the positive set
    parts = [synth.positives(1 << 12, r, 3) for r in range(3)]
    assert np.array_equal(np.concatenate(parts), synth.positives(1 << 12))
