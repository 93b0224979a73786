"""Θ/Φ vectorization layouts, host side.

Θ (horizontal) = lanes cooperating on one key; Φ (vertical) = contiguous words a
lane loads per step.  Valid iff both are powers of two and 1 <= Θ·Φ <= s
(P:L198).  Lane `lane` of a group handles, at step `step`, the Φ words
[step·Θ·Φ + lane·Φ, step·Θ·Φ + lane·Φ + Φ) -- "strided processing in
increments of Θ·Φ" (Fig. 2 caption).  The kernels use exactly this
map (csrc/bf_kernels.cuh, Cfg::word).
"""
from __future__ import annotations


def _pow2(x: int) -> bool:
    return x >= 1 and (x & (x - 1)) == 0


def validate_layout(theta: int, phi: int, s: int) -> str | None:
    """None if (Θ, Φ) is valid for s words per block, else the violated rule."""
    if not _pow2(theta):
        return f"Θ={theta} is not a power of two"
    if not _pow2(phi):
        return f"Φ={phi} is not a power of two"
    if theta * phi > s:
        return f"Θ·Φ={theta * phi} exceeds s={s}"
    return None


def enumerate_layouts(s: int) -> list[tuple[int, int]]:
    """All valid (Θ, Φ) for s words, ordered by Θ then Φ."""
    out = []
    t = 1
    while t <= s:
        p = 1
        while t * p <= s:
            out.append((t, p))
            p *= 2
        t *= 2
    return out


def word_assignment(theta: int, phi: int, s: int, lane: int, step: int) -> list[int]:
    """Words lane `lane` of a group handles at step `step`."""
    err = validate_layout(theta, phi, s)
    if err:
        raise ValueError(err)
    if not 0 <= lane < theta or not 0 <= step < s // (theta * phi):
        raise ValueError("lane or step out of range")
    base = step * theta * phi + lane * phi
    return list(range(base, base + phi))


def default_layout(op: str, s: int) -> tuple[int, int]:
    """The paper's best layouts for B <= 256: contains Θ=1, Φ=s;
    add Θ=s, Φ=1."""
    return (1, s) if op == "contains" else (s, 1)
