"""Pins of the oracle's Galerkin entries (§2.2 a_ij read per A1; §4.1 quadrature;
rule set A14, arithmetic A15).

Independent references: 60-digit Gauss-Legendre (decimal module), exact monomial
integrals over the reference pair (measure preservation of the Sauter-Schwab maps),
the analytic triangle potential with a subdivided outer rule (Richardson-extrapolated),
the far-field asymptotics, and the unit-sphere identity V1 = 1.
"""
import numpy as np
import pytest

from inputs.meshes import icosphere
from _analytic import double_integral_semianalytic, gauss_legendre_decimal, triangle_potential


def _exact(tx, ty, level=5, rate=4):
    a = double_integral_semianalytic(tx, ty, level=level - 1, order=8)
    b = double_integral_semianalytic(tx, ty, level=level, order=8)
    return (rate * b - a) / (rate - 1)   # Richardson on the O(rate^-level) outer error
                                         # (4: edge-type singular set, 8: point singularity)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 6, 8, 10])
def test_gauss_legendre_correctly_rounded(O, n):
    x, w = O.gauss_legendre01(n)
    xr, wr = gauss_legendre_decimal(n)
    assert np.array_equal(x, xr) and np.array_equal(w, wr)


@pytest.mark.parametrize("kind", [0, 1, 2])
@pytest.mark.parametrize("expo", [(0, 0, 0, 0), (1, 0, 0, 0), (0, 1, 0, 0), (0, 0, 1, 0), (0, 0, 0, 1),
                                  (2, 1, 0, 3), (1, 1, 1, 1), (3, 2, 1, 0), (0, 3, 2, 2)])
def test_sauter_schwab_maps_preserve_measure(O, kind, expo):
    # int_{T^ x T^} x1^a x2^b y1^c y2^d = 1/((b+1)(a+b+2)) * 1/((d+1)(c+d+2)), exact for GL6
    a, b, c, d = expo
    exact = 1.0 / ((b + 1) * (a + b + 2)) / ((d + 1) * (c + d + 2))
    got = O.ss_reference_monomial(kind, 6, a, b, c, d)
    assert abs(got - exact) <= 1e-14 * max(1.0, abs(exact))


TRIS = {
    "equilateral": np.array([[0, 0, 0], [1, 0, 0], [0.5, 3 ** 0.5 / 2, 0]], float),
    "right_isosceles": np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0]], float),
    "scalene": np.array([[0, 0, 0], [2, 0, 0], [0.3, 0.7, 0]], float),
    "tilted": np.array([[0.1, -0.2, 0.3], [0.9, 0.1, 0.2], [0.2, 0.8, 0.7]], float),
}


@pytest.mark.parametrize("name", list(TRIS))
def test_selfterm_closed_form_vs_semianalytic(O, name):
    T = TRIS[name]
    closed = O.selfterm_closed(T)
    ref = _exact(T, T)
    assert abs(closed - ref) <= 2e-9 * ref
    if name == "equilateral":
        assert abs(closed - 0.75 * np.log(3.0)) <= 1e-15      # (3/4) ln 3
    # Sauter-Schwab identical-panel map converges to the same closed form
    assert abs(O.sauter_schwab(0, T, T, 16) - closed) <= 1e-11 * closed   # exponential convergence
    assert abs(O.sauter_schwab(0, T, T, 6) - closed) <= 2e-5 * closed


def _rot(rng):
    Q, R = np.linalg.qr(rng.normal(size=(3, 3)))
    return Q * np.sign(np.diag(R))


def _edge_pair(rng):
    """Well-shaped edge neighbours: apex heights 0.5-1 x |AB|, dihedral angle 60-180 deg."""
    Q = _rot(rng); o = rng.normal(size=3)
    A, B = np.zeros(3), np.array([1.0, 0, 0])
    a1, a2 = rng.uniform(0.0, np.pi), None
    a2 = a1 + rng.uniform(np.pi / 3, np.pi)
    Cx = np.array([rng.uniform(0.3, 0.7), *(rng.uniform(0.5, 1.0) * np.array([np.cos(a1), np.sin(a1)]))])
    Cy = np.array([rng.uniform(0.3, 0.7), *(rng.uniform(0.5, 1.0) * np.array([np.cos(a2), np.sin(a2)]))])
    f = lambda P: np.array([p @ Q.T + o for p in P])
    return f([A, B, Cx]), f([A, B, Cy])


def _vertex_pair(rng):
    """Well-shaped vertex neighbours sharing A, separated by a random rotation."""
    Q = _rot(rng); o = rng.normal(size=3)
    A = np.zeros(3)
    tx = np.array([A, [1.0, 0, 0], [0.5, 0.8, 0.0]])
    ang = rng.uniform(np.pi / 2, np.pi)
    R = np.array([[np.cos(ang), -np.sin(ang), 0], [np.sin(ang), np.cos(ang), 0], [0, 0, 1]])
    ty = tx @ R.T
    ty[1:, 2] += rng.uniform(-0.3, 0.3, size=2)
    return tx @ Q.T + o, ty @ Q.T + o


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_sauter_schwab_edge_vertex_vs_semianalytic(O, seed):
    rng = np.random.default_rng(seed)
    tx, ty = _edge_pair(rng)
    ref = _exact(tx, ty, 6)
    assert abs(O.sauter_schwab(1, tx, ty, 16) - ref) <= 1e-9 * ref
    assert abs(O.sauter_schwab(1, tx, ty, 6) - ref) <= 2e-5 * ref
    # coplanar edge neighbours (the sphere mesh case is nearly coplanar)
    A, B = np.zeros(3), np.array([1.0, 0, 0])
    tx = np.array([A, B, [0.4, 0.8, 0]]); ty = np.array([A, B, [0.6, -0.7, 0]])
    ref = _exact(tx, ty, 6)
    assert abs(O.sauter_schwab(1, tx, ty, 16) - ref) <= 1e-9 * ref
    tx, ty = _vertex_pair(rng)
    ref = _exact(tx, ty, 6, rate=8)
    assert abs(O.sauter_schwab(2, tx, ty, 24) - ref) <= 1e-10 * ref
    assert abs(O.sauter_schwab(2, tx, ty, 6) - ref) <= 5e-4 * ref


def test_singular_entries_on_sphere_mesh(O):
    # the rule actually used (n_s = 6, A14) on icosphere neighbours: near-equilateral,
    # nearly coplanar panels -> much better than the distorted random pairs above
    V, T = icosphere(3)
    P = O.Problem(V, T)
    t0 = set(T[0])
    shared = np.array([len(t0 & set(t)) for t in T])
    for j, rate in ((int(np.where(shared == 2)[0][0]), 4), (int(np.where(shared == 1)[0][0]), 8), (0, 4)):
        a = P.entries([[0, j]])[0]
        ref = _exact(V[T[0]], V[T[j]], 6, rate) * 0.07957747154594767
        assert abs(a - ref) <= 2e-7 * ref


def test_radon_rule_table(O):
    # A14's rho >= 8 rule: Radon's 7-point degree-5 formula (Stroud T2:5-1).  Pins: the table is
    # the correctly rounded exact one (60-digit decimal here), it integrates every monomial
    # s^i t^j of degree <= 5 over {0 <= t <= s <= 1} exactly, and not degree 6.
    from decimal import Decimal, getcontext
    from fractions import Fraction
    getcontext().prec = 60
    s, t, w = O.rule_table(3)
    assert len(s) == 7
    r15 = Decimal(15).sqrt()
    exp = [(Decimal(2) / 3, Decimal(1) / 3, Decimal(9) / 80)]
    for a, wt in (((6 - r15) / 21, (155 - r15) / 2400), ((6 + r15) / 21, (155 + r15) / 2400)):
        c = 1 - 2 * a
        for lam in ((a, a, c), (a, c, a), (c, a, a)):
            exp.append((1 - lam[0], lam[2], wt))
    for q in range(7):
        assert (s[q], t[q], w[q]) == tuple(float(v) for v in exp[q]), q
    for deg in range(7):
        for i in range(deg + 1):
            j = deg - i
            exact = Fraction(1, (j + 1) * (i + j + 2))          # int_0^1 int_0^s s^i t^j dt ds
            got = sum(w[q] * s[q] ** i * t[q] ** j for q in range(7))
            if deg <= 5:
                assert abs(got - float(exact)) <= 4e-16, (i, j)
            elif (i, j) == (0, 6):
                assert abs(got - float(exact)) > 1e-6


@pytest.mark.parametrize("rho,n,tol", [(1.5, 6, 1e-8), (3.0, 5, 1e-8), (6.0, 4, 1e-8), (10.0, 3, 2e-9)])
def test_regular_rule_vs_semianalytic(O, rho, n, tol):
    T = TRIS["tilted"]
    h = max(np.linalg.norm(T[1] - T[0]), np.linalg.norm(T[2] - T[1]), np.linalg.norm(T[0] - T[2]))
    rng = np.random.default_rng(int(rho * 10))
    d = rng.normal(size=3); d /= np.linalg.norm(d)
    R = np.linalg.qr(rng.normal(size=(3, 3)))[0]
    c = T.mean(axis=0)
    Ty = (T - c) @ R.T + c + rho * h * d
    ref = _exact(T, Ty)
    assert abs(O.regular_rule(T, Ty, n) - ref) <= tol * ref


def test_regular_far_field_asymptotics(O):
    # a_ij 4 pi |c_i - c_j| / (|T_i||T_j|) = 1 + O((h/d)^2)
    T = TRIS["tilted"]
    h = 1.0
    area = 0.5 * np.linalg.norm(np.cross(T[1] - T[0], T[2] - T[0]))
    for dist in (100.0, 1000.0):
        Ty = T + np.array([dist, 0.0, 0.0])
        I = O.regular_rule(T, Ty, 3)
        assert abs(I * dist / (area * area) - 1.0) < 10 * (h / dist) ** 2


def test_sphere_entries_symmetric_spd_and_row_sums(O):
    devs = []
    for L in (2, 3):
        V, T = icosphere(L)
        P = O.Problem(V, T)
        A = P.dense()
        assert np.array_equal(A, A.T)                          # canonical panel order: exact symmetry
        np.linalg.cholesky(A)                                  # SPD
        _, area, _ = P.geometry()
        devs.append(np.abs(A.sum(axis=1) / area - 1.0).max())  # V1 = 1 on the unit sphere
    assert devs[0] < 0.01 and devs[1] < devs[0] / 3            # O(h^2) geometric error


def test_entry_classes_on_sphere(O):
    V, T = icosphere(3)
    P = O.Problem(V, T)
    assert P.entry_class(5, 5) == 0
    # find an edge neighbour and a vertex neighbour of triangle 5
    t5 = set(T[5])
    shared = np.array([len(t5 & set(t)) for t in T])
    e = int(np.where(shared == 2)[0][0]); v = int(np.where(shared == 1)[0][0])
    assert P.entry_class(5, e) == 1 and P.entry_class(5, v) == 2
    c, _, h = P.geometry()
    far = int(np.argmax(np.linalg.norm(c - c[5], axis=1)))
    assert P.entry_class(5, far) == 3
    # regular entry matches the explicit regular rule on the same panels
    a = P.entries([[5, far]])[0]
    ref = O.regular_rule(V[T[5]], V[T[far]], 3) * 0.07957747154594767
    assert abs(a - ref) <= 1e-15 * abs(ref)
