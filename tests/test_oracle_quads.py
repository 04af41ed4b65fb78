"""Pins of the oracle's quadrilateral mode (reading A25: the paper's model case, the unit
cube surface, §4).

Independent references: the unit-square self integral in closed form
4 ln(1+sqrt2) - (4/3)(sqrt2 - 1); square-pair integrals with the exact
rectangle potential and a graded outer rule (tests/_analytic.py, no triangle split); exact
integrals of the paper's quadratic f over squares; the exact interior solution U = f of
the Dirichlet problem (f harmonic) with the paper's measured convergence rate.
"""
import os

import numpy as np
import pytest

from inputs.meshes import cube
from _analytic import square_pair_integral

UNIT_SQUARE = 4.0 * np.log(1.0 + np.sqrt(2.0)) - 4.0 / 3.0 * (np.sqrt(2.0) - 1.0)   # 2.97320959824...
# the paper's observed interior-error rate on the cube (tests/golden/paper_cube_convergence_rate.txt)
with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "paper_cube_convergence_rate.txt")) as _f:
    PAPER_RATE = float(dict(ln.split() for ln in _f if ln.strip() and not ln.startswith("#"))["rate"])


def _square(V, q):
    a, b, c, d = V[q]
    return a, b - a, d - a


@pytest.mark.parametrize("L", [0, 1, 2, 3])
def test_cube_mesh(L):
    V, Q = cube(L)
    n = 2 ** L
    assert Q.shape == (6 * n * n, 4) and V.shape == (6 * n * n + 2, 3)      # Euler: V - E + F = 2
    assert np.array_equal(V * n, np.round(V * n))                            # exact lattice i / 2^L
    edges = {}
    for q in Q:
        for a in range(4):
            edges[(q[a], q[(a + 1) % 4])] = edges.get((q[a], q[(a + 1) % 4]), 0) + 1
    assert all(v == 1 for v in edges.values()) and all((b, a) in edges for (a, b) in edges)
    a, b, c = V[Q[:, 0]], V[Q[:, 1]], V[Q[:, 2]]
    nrm = np.cross(b - a, c - a)
    assert (np.einsum("ij,ij->i", nrm, V[Q].mean(axis=1) - 0.5) > 0).all()      # outward
    assert np.allclose(np.linalg.norm(nrm, axis=1), 1.0 / n ** 2, rtol=0, atol=1e-15)


def test_reference_reproduces_unit_square_closed_form():
    o, e1, e2 = np.zeros(3), np.array([1.0, 0, 0]), np.array([0, 1.0, 0])
    assert abs(square_pair_integral((o, e1, e2), (o, e1, e2)) - UNIT_SQUARE) <= 1e-12 * UNIT_SQUARE


def test_unit_square_self_entry(O):
    # cube(0): six unit faces; a_ii = (1/4pi) int_Q int_Q 1/|x-y|, within the Sauter-Schwab
    # (6 points) error of its two common-edge triangle pairs (A14)
    V, Q = cube(0)
    P = O.Problem(V, Q)
    a = P.entries([[i, i] for i in range(6)])
    assert np.all(a == a[0])
    assert abs(a[0] * 4 * np.pi - UNIT_SQUARE) <= 1e-6 * UNIT_SQUARE
    # scaling |Q|^(3/2): the h = 1/2 faces of cube(1)
    P1 = O.Problem(*cube(1))
    assert abs(P1.entries([[0, 0]])[0] * 4 * np.pi - UNIT_SQUARE / 8) <= 1e-6 * UNIT_SQUARE / 8


def test_square_pairs_vs_rectangle_potential(O):
    # all 24 x 24 pairs of cube(1): identical, coplanar and perpendicular (across a cube edge)
    # edge- and vertex-adjacent, separated on one face and on different faces
    V, Q = cube(1)
    P = O.Problem(V, Q)
    A = P.dense()
    assert np.array_equal(A, A.T)                                             # canonical order (A15)
    worst = {}
    for i in range(len(Q)):
        for j in range(len(Q)):
            ref = square_pair_integral(_square(V, Q[i]), _square(V, Q[j])) / (4 * np.pi)
            shared = len(set(Q[i]) & set(Q[j]))
            worst[shared] = max(worst.get(shared, 0.0), abs(A[i, j] - ref) / ref)
    assert set(worst) == {0, 1, 2, 4}
    assert worst[4] <= 1e-6            # identical: closed-form triangles + common-edge SS
    assert worst[2] <= 1e-5            # common edge (coplanar and 90 degrees): SS 6 points
    assert worst[1] <= 1e-5            # common vertex
    assert worst[0] <= 1e-9            # separated: tensor Gauss on both squares (A25, A14 bands)


def test_quad_matrix_spd_and_rhs_exact(O):
    V, Q = cube(2)
    P = O.Problem(V, Q)
    A = P.dense()
    np.linalg.cholesky(A)                                                     # SPD (single layer)
    # f = 4x^2 - 3y^2 - z^2 integrated exactly over each axis-aligned square
    f = P.rhs(1)
    lo, hi = V[Q].min(axis=1), V[Q].max(axis=1)
    exact = np.zeros(len(Q))
    for k, c in enumerate((4.0, -3.0, -1.0)):
        flat = hi[:, k] == lo[:, k]
        side = np.where(flat, 1.0, hi[:, k] - lo[:, k])
        mean_sq = np.where(flat, lo[:, k] ** 2, (hi[:, k] ** 3 - lo[:, k] ** 3) / (3 * side))
        exact += c * mean_sq
    area = np.prod(np.where(hi - lo == 0, 1.0, hi - lo), axis=1)
    assert np.allclose(P.geometry()[1], area, rtol=0, atol=1e-16)
    assert np.allclose(f, exact * area, rtol=1e-14, atol=1e-17)
    assert np.allclose(P.rhs(0), area, rtol=0, atol=1e-16)


def test_cube_interior_solution_converges_at_the_papers_rate(O):
    # V u = f on the cube surface, f harmonic -> the potential of u equals f inside;
    # worst-case error at fixed interior points decays like N^-1.3 (the paper's Fig. cube
    # convergence; 1.5 would need a smooth surface)
    X = 0.25 + 0.5 * np.random.default_rng(5).random((32, 3))
    fx = 4 * X[:, 0] ** 2 - 3 * X[:, 1] ** 2 - X[:, 2] ** 2
    err = []
    for L in (2, 3, 4):
        P = O.Problem(*cube(L))
        P.assemble(1e-6)
        x, it, rr, st = P.gmres(P.rhs(1), 1e-10)
        assert st == 0 and rr <= 1e-10
        err.append(np.abs(P.potential(x, X) - fx).max())
    assert err[2] < 1e-3
    rate = np.log(err[1] / err[2]) / np.log(4.0)                              # per N (N = 6 * 4^L)
    assert PAPER_RATE - 0.2 <= rate <= PAPER_RATE + 0.3, err
