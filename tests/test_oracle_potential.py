"""Pins of the oracle's single-layer potential (reading A23).

* one panel: the banded collapsed-Gauss rule against the closed-form triangle potential
  (tests/_analytic.py, Wilton/Graglia edge formula) in every rho band, and convergence in n;
* whole sphere: the exact density of V u = 1 is u = 1 (V1 = 1 on the unit sphere) and its
  potential is 1 inside; for the paper's f = 4x^2 - 3y^2 - z^2 (a harmonic degree-2
  polynomial) the potential of the solution is f itself inside.  The discrete
  potentials at interior points approach these closed forms as the mesh is refined.
"""
import numpy as np
import pytest

from _analytic import triangle_potential
from inputs.meshes import icosphere


def _band_order(rho):
    r2 = rho * rho
    return 6 if r2 < 4 else 5 if r2 < 16 else 4 if r2 < 64 else 3


@pytest.mark.parametrize("rho", [1.0, 1.5, 2.5, 3.5, 5.0, 7.5, 9.0, 20.0, 60.0])
def test_panel_potential_vs_closed_form(O, rho):
    tri = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.3, 0.8, 0.1]])
    c = tri.mean(axis=0)
    h = max(np.linalg.norm(tri[i] - tri[(i + 1) % 3]) for i in range(3))
    nrm = np.cross(tri[1] - tri[0], tri[2] - tri[0]); nrm /= np.linalg.norm(nrm)
    for d in (nrm, np.array([0.6, 0.48, 0.64]), np.array([-0.2, 0.9, -0.1])):
        x = c + rho * h * d / np.linalg.norm(d)
        exact = triangle_potential(x, tri)[0]
        n = _band_order(rho)
        assert abs(O.panel_potential(x, tri, n) - exact) <= 1e-8 * exact
        errs = [abs(O.panel_potential(x, tri, k) - exact) for k in (3, 4, 5, 6)]
        if rho <= 3.5:                                   # converging, not yet at round-off
            assert errs[0] > errs[1] > errs[2] > errs[3]


def test_sphere_interior_potential_closed_forms(O):
    rng = np.random.default_rng(3)
    X = rng.standard_normal((40, 3)); X /= np.linalg.norm(X, axis=1)[:, None]
    X *= rng.uniform(0.0, 0.6, size=(40, 1))
    f = 4 * X[:, 0] ** 2 - 3 * X[:, 1] ** 2 - X[:, 2] ** 2
    errs = {0: [], 1: []}
    for L in (2, 3, 4):
        V, T = icosphere(L)
        R = O.Problem(V, T)
        R.assemble(1e-6)
        for kind, exact in ((0, np.ones(len(X))), (1, f)):
            a, _, _, _ = R.gmres(R.rhs(kind), tol=1e-10, restart=100)
            errs[kind].append(np.abs(R.potential(a, X) - exact).max())
    for kind in (0, 1):
        e = errs[kind]
        assert e[0] > 4 * e[1] > 16 * e[2], e          # O(h^2) or better, per level
    assert errs[0][2] < 5e-6 and errs[1][2] < 5e-5
