"""GPU-vs-oracle parity on quadrilateral meshes (the paper's unit cube, reading A25;
SURVEY.md §8(f) rank 1), through the C ABI: the same bars as tests/test_gpu_parity.py.
Trees, codes, perm, leaf lists bit-exact; quad entries whose four triangle pairs are all
regular bit-exact, the rest <= 1e-14; pivots identical on >= 99.9% of blocks; matvec
<= 1e-12 vs the oracle's H and <= 10 eps_aca vs its dense rows; solutions <= 1e-5; the
interior potential against the exact U = f at the paper's rate."""
import numpy as np
import pytest

from inputs.meshes import cube, seeded_vector

pytestmark = pytest.mark.gpu

EPS = 1e-6


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    return torch


def _gpu(V, Q, leaf=32, eta=1.0):
    from paper_1806_11558_b200 import HMatrix
    H = HMatrix(device=0)
    H.build_tree(V, Q, leaf_size=leaf, eta=eta)
    return H


@pytest.mark.parametrize("L,leaf", [(1, 32), (3, 32), (5, 32), (4, 7)])
def test_cube_tree_bit_exact(O, torch_cuda, L, leaf):
    V, Q = cube(L)
    H = _gpu(V, Q, leaf)
    R = O.Problem(V, Q, leaf_size=leaf)
    assert np.array_equal(H.codes(), R.codes())
    assert np.array_equal(H.perm(), R.perm())
    for kind in (0, 1):
        assert np.array_equal(H.leaves(kind)[0], R.leaves(kind)), f"leaf list {kind}"
    cg, cr = H.clusters(), R.clusters()
    assert sorted(zip(cg["lo"], cg["hi"], map(tuple, cg["bbox"]))) == \
        sorted(zip(cr["lo"], cr["hi"], map(tuple, cr["bbox"])))


def test_cube_entries(O, torch_cuda):
    V, Q = cube(3)
    N = Q.shape[0]
    H = _gpu(V, Q)
    R = O.Problem(V, Q)
    i, j = np.meshgrid(np.arange(N), np.arange(N), indexing="ij")
    pairs = np.stack([i.ravel(), j.ravel()], axis=1).astype(np.int64)
    g = H.entries(pairs).reshape(N, N)
    o = R.entries(pairs).reshape(N, N)
    assert np.array_equal(g, g.T)
    # quads within one panel diameter may have touching triangle pairs; the rest are regular
    c, _, h = R.geometry()
    d = np.linalg.norm(c[:, None] - c[None], axis=2)
    far = d > 2.5 * h.max()
    assert far.sum() > 0.5 * N * N
    assert np.array_equal(g[far], o[far]), "all-regular quad entries bit-identical (A15, A25)"
    assert (np.abs(g - o) <= 1e-14 * np.abs(o)).all()


@pytest.fixture(scope="module")
def cube4(O, torch_cuda):
    V, Q = cube(4)                        # N = 1536, the paper's smallest cube
    H = _gpu(V, Q)
    H.set_option("record_pivots", 1)
    H.setup(EPS)
    R = O.Problem(V, Q)
    R.assemble(EPS)
    return V, Q, H, R


def test_cube_blocks_pivots_matvec(cube4, torch_cuda):
    V, Q, H, R = cube4
    dense, _ = H.leaves(1)
    for b, q in enumerate(dense):
        Bg = H.dense_block(b, (q[1] - q[0], q[3] - q[2]))
        assert (np.abs(Bg - R.dense_block(b)) <= 1e-14 * np.abs(R.dense_block(b))).all(), f"dense block {b}"
    adm, _ = H.leaves(0)
    same = 0
    for b, q in enumerate(adm):
        U, W, pv = H.lowrank(b, q[1] - q[0], q[3] - q[2], pivots=True)
        if U.shape[1] == R.rank(b) and np.array_equal(pv, R.pivots(b)):
            same += 1
    assert same >= 0.999 * len(adm), f"identical pivots on {same}/{len(adm)} blocks"
    N = Q.shape[0]
    A = R.dense()
    for x in [np.ones(N), R.rhs(1), seeded_vector(N, 0)]:
        yg = H.matvec(torch_cuda.from_numpy(x).cuda()).cpu().numpy()
        assert np.linalg.norm(yg - R.matvec(x)) <= 1e-12 * np.linalg.norm(yg)
        assert np.linalg.norm(yg - A @ x) <= 10 * EPS * np.linalg.norm(A @ x)


def test_cube_rhs_solve_and_potential(cube4, torch_cuda):
    V, Q, H, R = cube4
    f = H.assemble_rhs(1)
    assert np.array_equal(f, R.rhs(1))
    sol, it, rr = H.solve(torch_cuda.from_numpy(f).cuda(), tol=1e-10)
    xo = R.gmres(f, tol=1e-10)[0]
    sol = sol.cpu().numpy()
    assert np.linalg.norm(sol - xo) <= 1e-5 * np.linalg.norm(xo)
    X = 0.25 + 0.5 * np.random.default_rng(5).random((32, 3))
    ug = H.potential(torch_cuda.from_numpy(sol).cuda(), torch_cuda.from_numpy(X).cuda()).cpu().numpy()
    uo = R.potential(sol, X)
    assert np.abs(ug - uo).max() <= 1e-12 * np.abs(uo).max()


def test_cube_interior_error_rate_on_gpu(torch_cuda):
    # the paper's convergence study (k fixed there; eps_aca here): worst-case
    # interior error of the potential against U = f decays like N^-1.3 (N = 6144 ... 393216)
    import torch
    X = 0.25 + 0.5 * np.random.default_rng(5).random((64, 3))
    fx = 4 * X[:, 0] ** 2 - 3 * X[:, 1] ** 2 - X[:, 2] ** 2
    err = []
    for L in (5, 6, 7, 8):
        V, Q = cube(L)
        H = _gpu(V, Q)
        H.setup(EPS)
        f = H.assemble_rhs(1)
        sol, it, rr = H.solve(torch.from_numpy(f).cuda(), tol=1e-8)
        u = H.potential(sol, torch.from_numpy(X).cuda()).cpu().numpy()
        err.append(np.abs(u - fx).max())
        H.close()
    rates = [np.log(err[k] / err[k + 1]) / np.log(4.0) for k in range(3)]
    # the oracle pin's band around the paper's 1.3 (tests/golden/paper_cube_convergence_rate.txt)
    from test_oracle_quads import PAPER_RATE
    assert all(PAPER_RATE - 0.2 <= r <= PAPER_RATE + 0.3 for r in rates), (err, rates)


def test_cube_full_size_sampled_rows(O, torch_cuda):
    # the paper's largest cube, N = 1,572,864 (C6), in the bench's launch configuration
    V, Q = cube(9)
    N = Q.shape[0]
    H = _gpu(V, Q)
    H.setup(EPS)
    R = O.Problem(V, Q)
    rows = np.random.default_rng(7).permutation(N)[:128]
    Arows = R.dense_rows(rows)
    for x in [np.ones(N), seeded_vector(N, 0)]:
        yg = H.matvec(torch_cuda.from_numpy(x).cuda()).cpu().numpy()
        ye = Arows @ x
        assert np.linalg.norm(yg[rows] - ye) <= 10 * EPS * np.linalg.norm(ye)
    H.close()
