"""Exact ideal-hash false-positive-rate model for the blocked variants.

TEST INFRASTRUCTURE.  SURVEY.md Appendix B, derived from the variant
definitions:

* a key's block is uniform over the b blocks, so the number of keys in a given
  block is L ~ Binomial(n, 1/b)                       (BBF)
* the k draws of a key are i.i.d. uniform over the B bits of the block (BBF),
  q = k/s of them over each S-bit word (SBF), or q = k/z over one word
  chosen uniformly in each of z groups of g = s/z words (CSBF)
* a query is independent of the inserted keys.

E(T, W, q) = E[(X/W)^q] where X is the number of occupied cells after T
throws into W cells, by the occupancy recurrence
    P_{T+1}(x) = P_T(x) x/W + P_T(x-1) (W-x+1)/W.

Unconditional FPR:
    BBF   sum_i P(L=i) E(i k, B, k)
    SBF   sum_i P(L=i) E(i q, S, q)^s          (RBBF: s = 1)
    CSBF  sum_i P(L=i) [sum_j Bin(j; i, 1/g) E(j q, S, q)]^z
    CBF   E(k n, m, k)  (Eq. 1 is its large-m limit)

Filter-conditional FPR (given the actual popcounts):
    BBF   mean_blk (pc_blk/B)^k
    SBF   mean_blk prod_w (pc_w/S)^q
    CSBF  mean_blk prod_groups mean_{w in group} (pc_w/S)^q
    CBF   (pc/m)^k
"""
from __future__ import annotations

import math

import numpy as np
from scipy import stats

CBF, BBF, RBBF, SBF, CSBF = 0, 1, 2, 3, 4


def _load_pmf(n: int, b: int, tol: float = 1e-300):
    """P(L = i), L ~ Binomial(n, 1/b), on a window that holds all but a
    negligible (< 1e-15) part of the mass."""
    if b == 1:
        return np.array([n]), np.array([1.0])
    mean = n / b
    hi = int(min(n, mean + 60.0 * math.sqrt(mean + 1.0) + 60))
    lo = int(max(0, mean - 60.0 * math.sqrt(mean + 1.0) - 60))
    i = np.arange(lo, hi + 1)
    w = stats.binom.pmf(i, n, 1.0 / b)
    assert abs(w.sum() - 1.0) < 1e-12, "load window too narrow"
    keep = w > tol
    return i[keep], w[keep]


def occupancy_moments(T_max: int, W: int, q: int) -> np.ndarray:
    """E[(X_T/W)^q] and E[X_T/W] for T = 0..T_max (rows 0 and 1)."""
    p = np.zeros(W + 1)
    p[0] = 1.0
    x = np.arange(W + 1, dtype=np.float64)
    frac_q = (x / W) ** q
    out = np.empty((2, T_max + 1))
    out[0, 0] = frac_q @ p
    out[1, 0] = (x / W) @ p
    stay = x / W
    move = (W - x + 1) / W  # probability a throw moves x-1 -> x
    for t in range(1, T_max + 1):
        newp = p * stay
        newp[1:] += p[:-1] * move[1:]
        p = newp
        out[0, t] = frac_q @ p
        out[1, t] = (x / W) @ p
    return out


def fpr_exact(variant: int, n: int, b: int, B: int, S: int, k: int, z: int = 0,
              m_bits: int | None = None) -> float:
    """Unconditional FPR of a random filter with n keys (ideal hashing)."""
    if variant == CBF:
        m = int(m_bits)
        # E[(X/m)^k] for kn throws into m cells; the occupancy recurrence on
        # m cells is too large, so use the exact first-order form: X/m
        # concentrates (relative sd ~ m^-1/2) and E[(X/m)^k] = (E X/m)^k (1+O(k^2/m)).
        fill = 1.0 - (1.0 - 1.0 / m) ** (k * n)
        return fill ** k
    s = B // S
    i, w = _load_pmf(n, b)
    imax = int(i.max())
    if variant in (BBF,):
        mom = occupancy_moments(imax * k, B, k)[0]
        return float(w @ mom[i * k])
    if variant in (SBF, RBBF):
        q = k // s
        mom = occupancy_moments(imax * q, S, q)[0]
        return float(w @ mom[i * q] ** s)
    if variant == CSBF:
        g = s // z
        q = k // z
        mom = occupancy_moments(imax * q, S, q)[0]
        tot = 0.0
        for ii, wi in zip(i, w):
            j = np.arange(ii + 1)
            pj = stats.binom.pmf(j, ii, 1.0 / g) if g > 1 else (j == ii).astype(float)
            tot += wi * float(pj @ mom[j * q]) ** z
        return tot
    raise ValueError(variant)


def fill_exact(variant: int, n: int, b: int, B: int, S: int, k: int, z: int = 0,
               m_bits: int | None = None) -> float:
    """Expected fraction of set bits."""
    if variant == CBF:
        return 1.0 - (1.0 - 1.0 / int(m_bits)) ** (k * n)
    s = B // S
    i, w = _load_pmf(n, b)
    if variant == BBF:
        return float(w @ (1.0 - (1.0 - 1.0 / B) ** (i * k)))
    if variant in (SBF, RBBF):
        q = k // s
        return float(w @ (1.0 - (1.0 - 1.0 / S) ** (i * q)))
    if variant == CSBF:
        g = s // z
        q = k // z
        tot = 0.0
        for ii, wi in zip(i, w):
            j = np.arange(ii + 1)
            pj = stats.binom.pmf(j, ii, 1.0 / g) if g > 1 else (j == ii).astype(float)
            tot += wi * float(pj @ (1.0 - (1.0 - 1.0 / S) ** (j * q)))
        return tot
    raise ValueError(variant)


def _popcounts(bits_u8: np.ndarray, width: int) -> np.ndarray:
    """Popcount of consecutive `width`-bit groups of a little-endian bit array."""
    b = np.unpackbits(bits_u8, bitorder="little")
    return b.reshape(-1, width).sum(axis=1).astype(np.float64)


def fpr_conditional(variant: int, bits_u8: np.ndarray, B: int, S: int, k: int,
                    z: int = 0, m_bits: int | None = None) -> float:
    """FPR of THIS filter for an independent uniform query (ideal hashing)."""
    if variant == CBF:
        b = np.unpackbits(bits_u8, bitorder="little")[: int(m_bits)]
        return float((b.sum() / int(m_bits)) ** k)
    s = B // S
    if variant == BBF:
        pc = _popcounts(bits_u8, B)
        return float(np.mean((pc / B) ** k))
    pcw = _popcounts(bits_u8, S).reshape(-1, s)
    if variant in (SBF, RBBF):
        q = k // s
        return float(np.mean(np.prod((pcw / S) ** q, axis=1)))
    if variant == CSBF:
        g = s // z
        q = k // z
        per = ((pcw / S) ** q).reshape(-1, z, g).mean(axis=2)
        return float(np.mean(np.prod(per, axis=1)))
    raise ValueError(variant)


def putze_bound(variant: int, n: int, b: int, B: int, S: int, k: int, z: int = 0) -> float:
    """Putze/Lang Poisson closed form (P:L117 cites Putze) -- reported only."""
    s = B // S
    lam = n / b
    i = np.arange(0, int(lam + 20 * math.sqrt(lam + 1) + 20))
    w = stats.poisson.pmf(i, lam)
    if variant == BBF:
        return float(w @ (1.0 - (1.0 - 1.0 / B) ** (i * k)) ** k)
    q = k // (s if variant in (SBF, RBBF) else z)
    e = (1.0 - (1.0 - 1.0 / S) ** (i * q)) ** q
    if variant in (SBF, RBBF):
        return float(w @ e ** s)
    g = s // z
    return float(w @ (1.0 - (1.0 - 1.0 / S) ** (i * q / g)) ** (q * z))


def binom_z(count: int, trials: int, p: float) -> float:
    """Standardised deviation of a binomial count from trials * p."""
    sd = math.sqrt(trials * p * (1.0 - p))
    return (count - trials * p) / sd if sd > 0 else float("inf")
