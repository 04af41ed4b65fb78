"""Pins of the oracle's ACA (A11-A12), H-matvec, solvers (P:646,
P:667-668, A17) and RHS (A16).

References: exactly low-rank matrices (k in {r, r+1}, A12), the interpolation
property, H = A exactly when no block is admissible, the dense Galerkin
matrix (BJ: ||Hx - Ax|| <= 10 eps_aca), LAPACK Cholesky (numpy), and the
unit-sphere closed forms V1 = 1 and V Y_2 = Y_2 / 5.
"""
import numpy as np
import pytest

from inputs.meshes import icosphere, seeded_vector


@pytest.mark.parametrize("m,n", [(20, 20), (37, 20), (500, 37), (2000, 500)])
@pytest.mark.parametrize("r", [1, 3, 10])
def test_aca_exact_low_rank(O, m, n, r):
    rng = np.random.default_rng(m * 1000 + n + r)
    a = rng.standard_normal((m, r)); b = rng.standard_normal((n, r))
    A = a @ b.T
    U, V, piv = O.aca_matrix(A, 1e-6, 64)
    assert U.shape[1] in (r, r + 1)
    assert np.linalg.norm(A - U @ V.T) <= 1e-13 * np.linalg.norm(A) * max(1, r)


def test_aca_zero_and_rank_one(O):
    U, V, _ = O.aca_matrix(np.zeros((7, 9)), 1e-6, 64)
    assert U.shape[1] == 0
    a = np.arange(1, 8, dtype=float); b = np.linspace(-1, 2, 9)
    U, V, piv = O.aca_matrix(np.outer(a, b), 1e-6, 64)
    assert np.allclose(U @ V.T, np.outer(a, b), rtol=0, atol=1e-14 * 14)
    assert tuple(piv[0]) == (0, 8)                 # first row 0, column argmax |b| = last


def test_aca_interpolation_and_full_rank(O):
    rng = np.random.default_rng(5)
    X = rng.uniform(size=(30, 3)); Y = rng.uniform(size=(25, 3)) + np.array([3.0, 0, 0])
    A = 1.0 / np.linalg.norm(X[:, None] - Y[None], axis=2)
    U, V, piv = O.aca_matrix(A, 1e-8, 64)
    R = U @ V.T
    for i, j in piv:                               # pivot rows/cols reproduced
        assert np.abs(R[i] - A[i]).max() <= 1e-12 * np.abs(A).max()
        assert np.abs(R[:, j] - A[:, j]).max() <= 1e-12 * np.abs(A).max()
    assert np.linalg.norm(A - R) <= 1e-7 * np.linalg.norm(A)
    # k_cap >= min(m, n), eps -> 0: exact reconstruction of a nonsingular block
    B = rng.standard_normal((12, 12)) + 12 * np.eye(12)
    U, V, _ = O.aca_matrix(B, 1e-300, 64)
    assert U.shape[1] == 12 and np.linalg.norm(B - U @ V.T) <= 1e-12 * np.linalg.norm(B)


def test_fixed_rank_aca(O):
    """eps_aca = 0 is the paper's fixed-rank mode: exactly K = min(m, n, kcap) terms on a
    matrix of full numerical rank; the residual is interpolated at the K pivot rows/columns
     and shrinks with K like the smooth kernel's singular values."""
    rng = np.random.default_rng(11)
    X = rng.uniform(size=(60, 3)); Y = rng.uniform(size=(45, 3)) + np.array([2.5, 0, 0])
    A = 1.0 / np.linalg.norm(X[:, None] - Y[None], axis=2)
    s = np.linalg.svd(A, compute_uv=False)
    errs = []
    for K in (2, 4, 8, 12):
        U, V, piv = O.aca_matrix(A, 0.0, K)
        assert U.shape[1] == K
        R = A - U @ V.T
        rows, cols = piv[:, 0], piv[:, 1]
        assert np.abs(R[rows, :]).max() <= 1e-12 * np.abs(A).max()
        assert np.abs(R[:, cols]).max() <= 1e-12 * np.abs(A).max()
        errs.append(np.linalg.norm(R, 2))
        assert errs[-1] <= 1e3 * s[K]                  # quasi-optimal within a modest factor
    assert all(b < a for a, b in zip(errs, errs[1:]))
    U, V, _ = O.aca_matrix(A, 0.0, 64)                 # K >= min(m, n): exact
    assert U.shape[1] == 45
    assert np.abs(A - U @ V.T).max() <= 1e-12 * np.abs(A).max()


def test_aca_on_admissible_blocks(O):
    V, T = icosphere(3)
    P = O.Problem(V, T)
    A = P.dense()
    perm = P.perm()
    errs = []
    for q in P.leaves(0)[::17]:
        U, W, piv = P.aca_block(q, 1e-6)
        B = A[np.ix_(perm[q[0]:q[1]], perm[q[2]:q[3]])]
        errs.append(np.linalg.norm(B - U @ W.T) / np.linalg.norm(B))
        assert U.shape[1] <= min(q[1] - q[0], q[3] - q[2])
    errs = np.array(errs)
    assert np.median(errs) < 1e-6 and errs.max() < 5e-5


@pytest.fixture(scope="module")
def c1(O):
    V, T = icosphere(3)
    P = O.Problem(V, T)
    P.assemble(1e-6)
    return V, T, P, P.dense()


def test_h_equals_a_without_admissible_blocks(O):
    V, T = icosphere(2)                            # N = 320: no admissible leaf at eta = 1
    P = O.Problem(V, T)
    P.assemble(1e-6)
    A = P.dense()
    for seed in range(3):
        x = seeded_vector(320, seed)
        y = P.matvec(x)
        assert np.linalg.norm(y - A @ x) <= 1e-14 * np.linalg.norm(A @ x)


def test_h_matvec_error_bound(O, c1):
    V, T, P, A = c1
    N = T.shape[0]
    xs = [np.ones(N), P.rhs(1)] + [seeded_vector(N, s) for s in range(5)]
    for x in xs:
        y, ye = P.matvec(x), A @ x
        assert np.linalg.norm(y - ye) <= 10 * 1e-6 * np.linalg.norm(ye)   # BJ: <= 10 eps_aca
    # stored doubles: dense + k(m+n)
    adm, dense = P.leaves(0), P.leaves(1)
    s = sum(int((q[1] - q[0]) * (q[3] - q[2])) for q in dense)
    s += sum(P.rank(b) * int((q[1] - q[0]) + (q[3] - q[2])) for b, q in enumerate(adm))
    assert P.stored_doubles() == s


def test_rhs_closed_forms(O, c1):
    V, T, P, A = c1
    _, area, _ = P.geometry()
    assert np.array_equal(P.rhs(0), area)                     # f = 1 -> |T_i|
    # f = 4x^2-3y^2-z^2 is quadratic: the edge-midpoint rule is exact on flat triangles;
    # check against a 7-point degree-5 rule applied per triangle.
    f = lambda x: 4 * x[..., 0] ** 2 - 3 * x[..., 1] ** 2 - x[..., 2] ** 2
    a, b, c = V[T[:, 0]], V[T[:, 1]], V[T[:, 2]]
    bary = np.array([[1 / 3, 1 / 3, 1 / 3]] + [[0.0597158717, 0.4701420641, 0.4701420641],
                    [0.4701420641, 0.0597158717, 0.4701420641], [0.4701420641, 0.4701420641, 0.0597158717],
                    [0.7974269853, 0.1012865073, 0.1012865073], [0.1012865073, 0.7974269853, 0.1012865073],
                    [0.1012865073, 0.1012865073, 0.7974269853]])
    w = np.array([0.225] + [0.1323941527] * 3 + [0.1259391805] * 3)
    pts = bary[:, 0, None, None] * a + bary[:, 1, None, None] * b + bary[:, 2, None, None] * c
    ref = (w[:, None] * f(pts)).sum(axis=0) * area
    assert np.abs(P.rhs(1) - ref).max() <= 1e-9 * np.abs(ref).max()


def test_solvers_vs_cholesky_and_sphere_closed_forms(O, c1):
    V, T, P, A = c1
    N = T.shape[0]
    L = np.linalg.cholesky(A)
    _, area, _ = P.geometry()
    c, _, _ = P.geometry()
    for kind in (0, 1):
        b = P.rhs(kind)
        ref = np.linalg.solve(L.T, np.linalg.solve(L, b))
        x_cg, it_cg, rr_cg, st = P.cg(b, tol=1e-10)
        assert st == 0 and rr_cg <= 1e-9
        x_gm, it_gm, rr_gm, st = P.gmres(b, tol=1e-10, restart=100)
        assert st == 0 and rr_gm <= 1e-9
        for x in (x_cg, x_gm):
            assert np.linalg.norm(x - ref) <= 1e-5 * np.linalg.norm(ref)   # H vs A solve
        if kind == 0:
            # V u = 1 on the unit sphere: u = 1, capacitance sum(alpha |T|) -> 4 pi
            assert abs(x_cg.mean() - 1.0) < 1e-2
            assert abs((x_cg * area).sum() / (4 * np.pi) - 1.0) < 1e-2
        else:
            # exact density u = 5 f for the degree-2 harmonic f (eigenvalue 1/5)
            u_exact = 5 * (4 * c[:, 0] ** 2 - 3 * c[:, 1] ** 2 - c[:, 2] ** 2) / np.linalg.norm(c, axis=1) ** 2
            assert np.linalg.norm(x_cg - u_exact) / np.linalg.norm(u_exact) < 5e-2
    # restarted GMRES converges too
    b = P.rhs(1)
    x, it, rr, st = P.gmres(b, tol=1e-8, restart=5)
    assert st == 0 and rr <= 1e-7


def test_partitioned_assembly_sums_to_whole(O, c1):
    V, T, P, A = c1
    N = T.shape[0]
    x = seeded_vector(N, 11)
    y_full = P.matvec(x)
    adm, dense = P.leaves(0), P.leaves(1)
    cd = ((dense[:, 1] - dense[:, 0]) * (dense[:, 3] - dense[:, 2])).astype(np.int64)
    ca = (((adm[:, 1] - adm[:, 0]) + (adm[:, 3] - adm[:, 2])) * 10).astype(np.int64)
    for p in (2, 3):
        bd, ba = O.partition(cd, p), O.partition(ca, p)
        acc = np.zeros(N)
        for r in range(p):
            P.assemble(1e-6, dense_range=(bd[r], bd[r + 1]), adm_range=(ba[r], ba[r + 1]))
            acc += P.matvec(x)
        assert np.linalg.norm(acc - y_full) <= 1e-13 * np.linalg.norm(y_full)
    P.assemble(1e-6)
