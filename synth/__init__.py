"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic (no hashing, no block
selection, no pattern generation).  It only produces the key sets the paper's
workloads are made of ("N unique, random uint64_t input keys"; P:L271:
"query N keys not present in the insertion set") and the workload recipes of
BASELINE.json configs[0..4].

Key generator (DESIGN.md "Readings" item 20): key(i) = mix64(i), the SplitMix64
output function, a bijection on uint64, so distinct indices give distinct keys.
Positives use i in [0, n); negatives use i in [NEG_BASE, NEG_BASE + Q) with
NEG_BASE = 2**62, so the two sets are disjoint by construction.  The CUDA
library implements the same counter-based generator (bf_keygen) so that
multi-GiB key sets can be made on the device; tests check both produce the
same keys.
"""
from __future__ import annotations

import numpy as np

NEG_BASE = 1 << 62
_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def mix64(x: np.ndarray) -> np.ndarray:
    """SplitMix64 output function on a uint64 array (wrapping arithmetic)."""
    z = np.asarray(x, dtype=np.uint64) + _GOLDEN
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def keys(base: int, n: int, chunk: int = 1 << 24) -> np.ndarray:
    """Keys mix64(base), ..., mix64(base + n - 1) as a uint64 array."""
    out = np.empty(n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        for lo in range(0, n, chunk):
            hi = min(n, lo + chunk)
            idx = np.arange(lo, hi, dtype=np.uint64) + np.uint64(base)
            out[lo:hi] = mix64(idx)
    return out


def positives(n: int, rank: int = 0, world: int = 1) -> np.ndarray:
    """Rank r's shard [r*n/P, (r+1)*n/P) of the positive set."""
    lo = rank * n // world
    hi = (rank + 1) * n // world
    return keys(lo, hi - lo)


def negatives(q: int, offset: int = 0) -> np.ndarray:
    """q keys from the negative index range, disjoint from every positive set."""
    return keys(NEG_BASE + offset, q)


# Workload recipes: BASELINE.json configs[0..4] made concrete.
# variant ids follow SPEC S:L272: 1 BBF, 2 RBBF, 3 SBF, 4 CSBF.
WORKLOADS = {
    # configs[0]: 2^20 keys into a 16 Mbit filter, 256-bit blocks of 64-bit
    # words, k=8; add then contains on 2^20 positives + 2^20 negatives.
    "c1": dict(m_bits=1 << 24, B=256, S=64, k=8, n_add=1 << 20, n_pos=1 << 20, n_neg=1 << 20,
               variants=[("BBF", 1, 0), ("SBF", 3, 0)]),
    # configs[1]: L2-resident 32 MiB filter, 2^26 keys (bench default: SBF 256/64 k=8).
    "c2": dict(m_bits=1 << 28, B=256, S=64, k=8, n_add=1 << 26, n_pos=1 << 26, n_neg=0,
               variants=[("SBF", 3, 0)]),
    # configs[2]: HBM-resident 8 GiB filter, 2^32 keys.
    "c3": dict(m_bits=1 << 36, B=256, S=64, k=8, n_add=1 << 32, n_pos=1 << 32, n_neg=0,
               variants=[("SBF", 3, 0)]),
}
