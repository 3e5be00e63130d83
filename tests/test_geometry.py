"""Window geometry pins (reading A7) -- oracle side and, independently, the C++ side.

The paper prints two worked group tables (Tables I-II).  In units of
pilot positions both are instances of the stride-grid window rule with edge
clamping: 3W = (N=100 pilots, b=3, s=1), 12W = (N=100, b=12, s=1).  The golden
files under tests/golden/ are the printed rows verbatim.
"""
import os

import numpy as np
import pytest

from oracle import window_table

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _rows(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            rows.append([c.strip() for c in line.split("|")])
    return rows


def _window_of(table, pos):
    for a, o, o_next in table:
        if o <= pos < o_next:
            return a, pos - a
    raise AssertionError(pos)


def test_table1_3w_groups_reproduced():
    """group g (1-based) -> weight id, input LS pilots."""
    table = window_table(100, 3, 1)
    for idx, out_tones, wid, in_tones in _rows("table1_3w_groups.txt"):
        g = int(idx)
        a, row = _window_of(table, g - 1)
        assert row + 1 == int(wid), (g, row)
        assert [12 * (a + j) + 1 for j in range(3)] == [int(v) for v in in_tones.split(",")]
        # output tones of group g start at pilot g-1's tone (3 outputs spaced 4 apart)
        assert int(out_tones.split(",")[0]) == 12 * (g - 1) + 1


def test_table2_12w_groups_reproduced():
    """groups 1-6 W(1..6) on the first window, interior W(6) sliding,
    groups 95-100 W(7..12) on the last (clamped) window."""
    table = window_table(100, 12, 1)
    for idx, out_tones, wid, in_tones in _rows("table2_12w_groups.txt"):
        g = int(idx)
        a, row = _window_of(table, g - 1)
        assert row + 1 == int(wid), (g, row, wid)
        start, step, end = (int(v) for v in in_tones.split(":"))
        assert (start, step, end) == (12 * a + 1, 12, 12 * (a + 11) + 1)
        if g != 100:  # row 100 printed 1190:1:1200, reading A8
            assert int(out_tones.split(":")[0]) == 12 * (g - 1) + 1


@pytest.mark.parametrize("N,b,s", [(72, 12, 12), (300, 50, 25), (1200, 100, 100), (1200, 150, 100),
                                   (3276, 126, 126), (1050, 100, 100), (7, 7, 3), (10, 4, 1),
                                   (5, 1, 1), (1, 1, 1), (1201, 150, 99), (13, 6, 5)])
def test_partition_and_bounds(N, b, s):
    table = window_table(N, b, s)
    assert len(table) == -(-(N - b) // s) + 1
    covered = np.zeros(N, int)
    for a, o, o_next in table:
        assert 0 <= a <= N - b
        assert o < o_next
        assert 0 <= o - a and o_next - a <= b     # kept rows inside the window
        covered[o:o_next] += 1
    assert (covered == 1).all()                   # kept ranges partition [0, N)
    assert table[0][1] == 0 and table[-1][2] == N


def test_survey_tilings():
    """config 2 = 11 windows (first keeps 37, last 38);
    config 4 = 12 windows (first 125, last 75 from rows [75, 150))."""
    t2 = window_table(300, 50, 25)
    assert len(t2) == 11 and t2[0][2] - t2[0][1] == 37 and t2[-1][2] - t2[-1][1] == 38
    t4 = window_table(1200, 150, 100)
    assert len(t4) == 12 and t4[0][2] == 125
    a, o, o_next = t4[-1]
    assert (o - a, o_next - a) == (75, 150)


def test_cpp_geometry_matches_oracle():
    """C++ ce_window_table (host-only, no GPU) vs the independent Python derivation."""
    ce = pytest.importorskip("paper_1802_05427_b200")
    for N, b, s in [(72, 12, 12), (300, 50, 25), (1200, 100, 100), (1200, 150, 100), (3276, 126, 126),
                    (1050, 100, 100), (7, 7, 3), (10, 4, 1), (100, 12, 1), (100, 3, 1), (1, 1, 1)]:
        assert ce.window_table(N, b, s) == window_table(N, b, s), (N, b, s)
