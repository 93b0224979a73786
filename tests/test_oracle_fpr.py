"""Statistical and closed-form pins of the oracle.

* Eq. 1-3 values (tests/golden/paper_equations.json, each cited).
* The exact occupancy model is itself pinned: closed form of E[X/W]
  (1-(1-1/W)^T), brute-force enumeration of all W^T throw sequences on tiny
  cases, and BBF with one block == CBF of B bits.
* The oracle's measured FPR matches the exact ideal-hash model (unconditional
  and filter-conditional) within |z| <= 4, its fill ratio matches the exact
  expectation, and Eq. 1 is a lower bound for the blocked variants (P:L117:
  "The false positive rate is notably higher than that of a CBF").
* CBF at the optimal load: measured FPR within 4 sigma of (1/2)^k (Eq. 3).
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

import synth
from oracle import analytics as A
from oracle import fpr_model as M
from oracle.bfo import BBF, CBF, CSBF, RBBF, SBF, OracleFilter, unpack_bits

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_equations.json")))


def test_equations_golden():
    for e in GOLD["eq1"]:
        assert A.fpr_eq1(e["m_over_n"], 1.0, e["k"]) == pytest.approx(e["fpr"], rel=e["rtol"])
    for e in GOLD["eq1_at_optimal_load"]:
        k = e["k"]
        assert A.fpr_eq1(1.0, math.log(2) / k, k) == pytest.approx(e["fpr"], rel=e["rtol"])
    for e in GOLD["optimal_k"]:
        assert A.optimal_k_real(e["c"]) == pytest.approx(e["k_real"], abs=e.get("atol", 0.006))
        if "k_int" in e:
            assert A.optimal_k(e["c"]) == e["k_int"]
    for e in GOLD["min_fpr"]:
        assert A.min_fpr(e["c"]) == pytest.approx(e["fpr"], rel=e["rtol"])
    for e in GOLD["optimal_n"]:
        assert abs(A.optimal_n(e["m"], e["k"]) - e["n"]) <= e["tol"]
    for e in GOLD["capacity_for_fpr"]:
        c, n, k = A.capacity_for_fpr(1 << 20, e["target"])
        assert c == pytest.approx(e["c"], abs=1e-3) and k == e["k"]
        assert A.min_fpr(c) == pytest.approx(e["target"], rel=1e-12)


def test_equation_identities():
    for c in np.linspace(1.0, 40.0, 79):
        k = A.optimal_k(c)
        for kk in (k - 1, k + 1):
            if kk >= 1:
                assert A.fpr_eq1(c, 1.0, k) <= A.fpr_eq1(c, 1.0, kk) + 1e-15
        # Eq. 1 at the (real) optimal k equals Eq. 3
        kr = A.optimal_k_real(c)
        assert (1 - math.exp(-kr / c)) ** kr == pytest.approx(A.min_fpr(c), rel=1e-9)


def test_occupancy_closed_form_and_brute_force():
    for W in (8, 32, 64):
        mom = M.occupancy_moments(300, W, 1)
        T = np.arange(301)
        assert np.allclose(mom[1], 1 - (1 - 1 / W) ** T, rtol=0, atol=1e-12)
    for W, T, q in [(4, 5, 3), (5, 4, 2), (3, 6, 4), (8, 3, 5)]:
        tot = 0.0
        for seq in itertools.product(range(W), repeat=T):
            tot += (len(set(seq)) / W) ** q
        assert M.occupancy_moments(T, W, q)[0][T] == pytest.approx(tot / W ** T, rel=1e-12)


def test_model_special_cases():
    # one block of B bits with n keys is a CBF of B bits for all purposes
    for n in (1, 5, 20):
        bbf = M.fpr_exact(BBF, n, 1, 256, 64, 8)
        mom = M.occupancy_moments(n * 8, 256, 8)[0][n * 8]
        assert bbf == pytest.approx(mom, rel=1e-12)
    # CSBF with z = s is SBF; RBBF (s = 1) is SBF with one word
    assert M.fpr_exact(CSBF, 1 << 20, 1 << 16, 256, 64, 8, z=4) == pytest.approx(
        M.fpr_exact(SBF, 1 << 20, 1 << 16, 256, 64, 8), rel=1e-10)
    assert M.fpr_exact(RBBF, 1 << 18, 1 << 16, 64, 64, 6) == pytest.approx(
        M.fpr_exact(SBF, 1 << 18, 1 << 16, 64, 64, 6), rel=1e-12)
    # larger blocks -> lower FPR, and every blocked variant is above Eq. 1
    m, n = 1 << 24, 1 << 20
    f64 = M.fpr_exact(SBF, n, m // 64, 64, 64, 8)
    f256 = M.fpr_exact(SBF, n, m // 256, 256, 64, 8)
    assert f64 > f256 > A.fpr_eq1(m, n, 8)


STAT_CASES = [
    # (variant, B, S, k, z) at configs[0]'s geometry: m = 2^24, n = 2^20 (c = 16)
    (BBF, 256, 64, 8, 0), (SBF, 256, 64, 8, 0), (CSBF, 256, 32, 8, 2), (RBBF, 64, 64, 8, 0),
    (SBF, 256, 32, 16, 0), (CSBF, 256, 32, 8, 4), (BBF, 128, 32, 7, 0),
]


@pytest.mark.parametrize("cfg", STAT_CASES)
def test_fpr_matches_exact_model(cfg):
    v, B, S, k, z = cfg
    m, n, Q = 1 << 24, 1 << 20, 1 << 22
    f = OracleFilter(v, m, B=B, S=S, k=k, z=z)
    f.add(synth.positives(n), threads=8)
    neg = synth.negatives(Q)
    fp = int(unpack_bits(f.contains(neg, threads=8), Q).sum())
    b = m // B
    p_unc = M.fpr_exact(v, n, b, B, S, k, z)
    p_cond = M.fpr_conditional(v, f.bytes(), B, S, k, z)
    assert abs(M.binom_z(fp, Q, p_unc)) <= 4.0, (fp, Q * p_unc)
    assert abs(M.binom_z(fp, Q, p_cond)) <= 4.0, (fp, Q * p_cond)
    assert fp / Q > A.fpr_eq1(m, n, k)
    fill = f.popcount() / f.nbits
    assert fill == pytest.approx(M.fill_exact(v, n, b, B, S, k, z), abs=1e-3)
    # every inserted key is found
    assert unpack_bits(f.contains(synth.positives(n)[:100000], threads=8), 100000).all()


def test_cbf_eq1_at_optimal_load():
    """P:L271 protocol on the CBF: n = m ln2/k, FPR ~ (1/2)^k (Eq. 3)."""
    m, k = 1 << 25, 16
    n = A.optimal_n(m, k)
    f = OracleFilter(CBF, m, k=k)
    f.add(synth.positives(n), threads=8)
    Q = 10_000_000
    fp = int(unpack_bits(f.contains(synth.negatives(Q), threads=8), Q).sum())
    assert abs(M.binom_z(fp, Q, 0.5 ** k)) <= 4.0, fp
    assert f.popcount() / m == pytest.approx(0.5, abs=2e-3)
    assert abs(M.binom_z(fp, Q, M.fpr_conditional(CBF, f.bytes(), 0, 64, k, m_bits=m))) <= 4.0


@pytest.mark.parametrize("scheme", [1, 2])
@pytest.mark.parametrize("cfg", [(SBF, 256, 64, 16, 0), (BBF, 256, 64, 8, 0), (RBBF, 64, 64, 8, 0)])
def test_draw_schemes_fpr_matches_exact_model(scheme, cfg):
    """The pattern-changing draw schemes of P:L223 (NEXT N3).  The iterative
    single hash (k chained XXH64 evaluations) behaves like ideal hashing:
    FPR within |z| <= 4 of the exact model.  Double hashing (draws in
    arithmetic progression, top bits) does not: its draws are correlated and
    its FPR sits 1.4-1.9x above the ideal model (the reason P:L225 gives for
    multiplicative hashing: "approximately uniform distribution of bits").
    Both have no false negatives and differ from the multiplicative scheme."""
    v, B, S, k, z = cfg
    m, n, Q = 1 << 24, 1 << 20, 1 << 22
    f = OracleFilter(v, m, B=B, S=S, k=k, z=z, scheme=scheme)
    f.add(synth.positives(n), threads=8)
    fp = int(unpack_bits(f.contains(synth.negatives(Q), threads=8), Q).sum())
    p = M.fpr_exact(v, n, m // B, B, S, k, z)
    if scheme == 2:
        assert abs(M.binom_z(fp, Q, p)) <= 4.0, (fp, Q * p)
    else:
        assert 1.2 < fp / (Q * p) < 2.5, (fp, Q * p)
    assert unpack_bits(f.contains(synth.positives(n)[:50000], threads=8), 50000).all()
    g = OracleFilter(v, m, B=B, S=S, k=k, z=z, scheme=0)
    g.add(synth.positives(n)[:1000])
    h = OracleFilter(v, m, B=B, S=S, k=k, z=z, scheme=scheme)
    h.add(synth.positives(n)[:1000])
    assert not np.array_equal(g.bytes(), h.bytes())


def test_cbf_large_m_positions():
    """CBF above 2^32 bits (the paper's 1 GB baseline): positions are
    the 128-bit fast range (d_j * m) >> 64 of d_j = h * C_j mod 2^64.
    Pinned by (i) the power-of-two special case, where the fast range is
    exactly the top log2(m) bits of d_j (h from the xxhash library, C_j from
    the stated constant rule), (ii) boundedness and uniformity over a
    non-power-of-two m (chi-square over 64 equal cells), and (iii) m <= 2^32
    keeping the 32-bit form (the existing CBF pins)."""
    import xxhash
    from scipy import stats
    k = 16
    m2 = 1 << 33
    g = OracleFilter(CBF, m2, k=k, allocate=False)
    C = [(int(synth.mix64(np.uint64(0xCBF + j))) | 1) for j in range(k)]
    for key in synth.keys(99, 300):
        h = xxhash.xxh64_intdigest(int(key).to_bytes(8, "little"), 0)
        _, pos = g.pattern(int(key))
        assert pos == [((h * c) % (1 << 64)) >> (64 - 33) for c in C]
    m = (1 << 33) + 12345
    g = OracleFilter(CBF, m, k=k, allocate=False)
    cells = np.zeros(64, np.int64)
    for key in synth.keys(7, 20_000):
        _, pos = g.pattern(int(key))
        assert max(pos) < m
        for p in pos:
            cells[p * 64 // m] += 1
    assert stats.chisquare(cells).pvalue > 1e-4
    assert any(p >= (1 << 32) for p in pos)  # the range above 2^32 is reached
    with pytest.raises(ValueError):
        OracleFilter(CBF, (1 << 38) + 1, k=k, allocate=False)
