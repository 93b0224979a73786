"""Θ/Φ layout algebra against the paper's Fig. 2 layouts
(tests/golden/fig2_layouts.json, cited)."""
import json
import os

import pytest

from paper_2512_15595_b200 import layout as L

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "fig2_layouts.json")))


def test_fig2_layouts():
    s = GOLD["s"]
    for lay in GOLD["layouts"]:
        assert L.validate_layout(lay["theta"], lay["phi"], s) is None, lay["fig"]
        for lane, step, words in lay["assign"]:
            assert L.word_assignment(lay["theta"], lay["phi"], s, lane, step) == words, lay["fig"]


def test_enumeration_counts():
    assert len(L.enumerate_layouts(8)) == GOLD["n_valid_layouts_s8"]
    assert len(L.enumerate_layouts(4)) == GOLD["n_valid_layouts_s4"]
    assert L.enumerate_layouts(1) == [(1, 1)]


@pytest.mark.parametrize("s", [1, 2, 4, 8, 16, 32, 64])
def test_assignment_partitions_block(s):
    for theta, phi in L.enumerate_layouts(s):
        seen = []
        for step in range(s // (theta * phi)):
            for lane in range(theta):
                w = L.word_assignment(theta, phi, s, lane, step)
                assert w[0] % phi == 0 and w == list(range(w[0], w[0] + phi))
                seen += w
        assert sorted(seen) == list(range(s))


def test_invalid_layouts():
    assert L.validate_layout(3, 1, 8)
    assert L.validate_layout(4, 4, 8)
    assert L.validate_layout(1, 0, 8)
    with pytest.raises(ValueError):
        L.word_assignment(2, 2, 8, 2, 0)
