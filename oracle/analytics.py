"""The paper's closed forms, Eq. 1-3 -- TEST INFRASTRUCTURE.

c = m/n bits per key; Eq. 1 f = (1 - e^{-kn/m})^k;
Eq. 2 k = c ln 2; Eq. 3 f_min = (1/2)^{c ln 2}.
The "space-error-rate-optimal number of distinct keys, obtained by solving
Eq. (3) for n" is n = m ln2 / k for the configured k (DESIGN.md
"Readings" item 13).
"""
from __future__ import annotations

import math

LN2 = math.log(2.0)


def fpr_eq1(m: float, n: float, k: int) -> float:
    """Eq. 1: f = (1 - exp(-k n / m))^k."""
    if m <= 0 or n < 0 or k < 1:
        raise ValueError("fpr_eq1 needs m > 0, n >= 0, k >= 1")
    return (1.0 - math.exp(-k * n / m)) ** k


def optimal_k_real(c: float) -> float:
    """Eq. 2: k = c ln 2."""
    return c * LN2


def optimal_k(c: float) -> int:
    """The integer neighbour of Eq. 2's k that minimises Eq. 1 at m/n = c."""
    kr = optimal_k_real(c)
    cands = sorted({max(1, math.floor(kr)), max(1, math.ceil(kr))})
    return min(cands, key=lambda k: fpr_eq1(c, 1.0, k))


def min_fpr(c: float) -> float:
    """Eq. 3: f_min = (1/2)^{c ln 2}."""
    return 0.5 ** (c * LN2)


def optimal_n(m_eff: int, k: int) -> int:
    """Eq. 3 solved for n at the configured k: n = round(m ln2 / k), at least 1."""
    return max(1, int(round(m_eff * LN2 / k)))


def capacity_for_fpr(m_eff: int, target: float):
    """Eq. 3 inverted: c = -ln f / (ln 2)^2, n = floor(m/c), k = optimal_k(c)."""
    if not 0.0 < target < 1.0:
        raise ValueError("target FPR must lie in (0, 1)")
    c = -math.log(target) / (LN2 * LN2)
    return c, int(math.floor(m_eff / c)), optimal_k(c)
