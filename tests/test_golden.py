"""Pins against the fixtures in tests/golden/ (each file cites its source passage).

The paper prints no entry values; what it does print for the model case is the list of
problem sizes N of the unit cube (Table "tab:runtimes") and the observed convergence rate
1.3 of the interior error.  These tests tie the input generator and the oracle to them.
"""
import os

import numpy as np
import pytest

from inputs.meshes import cube

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _rows(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return [ln.split() for ln in f if ln.strip() and not ln.startswith("#")]


def golden_value(name, key):
    return float(dict((r[0], r[1]) for r in _rows(name))[key])


@pytest.mark.parametrize("L,N", [(int(a), int(b)) for a, b in _rows("paper_table_runtimes_cube_N.txt")])
def test_cube_sizes_match_the_papers_table(L, N):
    V, Q = cube(L)
    assert Q.shape == (N, 4)
    assert V.shape == (N + 2, 3)                       # closed genus-0 quad mesh: V = F + 2


def test_unit_square_closed_form_decimal():
    from test_oracle_quads import UNIT_SQUARE
    assert abs(UNIT_SQUARE - golden_value("unit_square_self_integral.txt", "value")) < 1e-10


def test_paper_rate_fixture_is_the_one_the_convergence_tests_use():
    from test_oracle_quads import PAPER_RATE
    assert PAPER_RATE == golden_value("paper_cube_convergence_rate.txt", "rate")
