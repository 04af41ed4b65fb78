"""Pins of the oracle's tree construction (§2.3, §3.1; SPEC.md clustering/blocktree).

Each test checks the oracle against something other than itself: SPEC's worked
examples, the cluster-tree axioms
(C1)-(C4), and brute-force N x N coverage of the block partition.
"""
import numpy as np
import pytest

from inputs.meshes import icosphere


def _point_mesh(points):
    """Degenerate 'triangles' whose three vertices coincide: centroid == point exactly
    for the dyadic coordinates used below."""
    p = np.asarray(points, dtype=np.float64)
    V = np.repeat(p, 3, axis=0)
    T = np.arange(V.shape[0], dtype=np.int32).reshape(-1, 3)
    return V, T


def test_morton_spec_examples(O):
    # min corner -> 0, max corner -> all 63 bits, (0.5,0,0) in unit box -> 1<<62
    V, T = _point_mesh([[0, 0, 0], [1, 1, 1], [0.5, 0, 0]])
    P = O.Problem(V, T, leaf_size=32, eta=1.0)
    c = P.codes()
    assert int(c[0]) == 0
    assert int(c[1]) == (1 << 63) - 1
    assert int(c[2]) == 1 << 62


def test_morton_axis_order(O):
    # x most significant within each bit triple (A6): (0,0.5,0) -> 1<<61, (0,0,0.5) -> 1<<60
    V, T = _point_mesh([[0, 0, 0], [1, 1, 1], [0, 0.5, 0], [0, 0, 0.5], [0.25, 0, 0]])
    c = O.Problem(V, T).codes()
    assert int(c[2]) == 1 << 61 and int(c[3]) == 1 << 60 and int(c[4]) == 1 << 59


def test_morton_per_axis_normalisation(O):
    # A6: every axis is normalised to its OWN extent of the centroid box, here
    # [0,2] x [0,1] x [0,4]; codes computed by hand from q_a = floor(((c-lo)/(hi-lo)) 2^21) and
    # bit b of q_x, q_y, q_z at 3b+2, 3b+1, 3b.  An isotropic normalisation (by the largest
    # extent 4) would give (1,0,0) -> 1<<59 and (0,0.5,0) -> 1<<55 instead.
    V, T = _point_mesh([[0, 0, 0], [2, 1, 4], [1, 0, 0], [0, 0.5, 0], [0, 0, 1],
                        [0.5, 0.25, 3], [1.5, 0.75, 0.5]])
    c = [int(v) for v in O.Problem(V, T).codes()]
    assert c[0] == 0 and c[1] == (1 << 63) - 1
    assert c[2] == 1 << 62                                   # x: 1/2 -> q = 2^20
    assert c[3] == 1 << 61                                   # y: 1/2 -> q = 2^20
    assert c[4] == 1 << 57                                   # z: 1/4 -> q = 2^19
    assert c[5] == (1 << 59) | (1 << 58) | (1 << 60) | (1 << 57)     # x 1/4, y 1/4, z 3/4
    assert c[6] == (1 << 62) | (1 << 59) | (1 << 61) | (1 << 58) | (1 << 54)   # x 3/4, y 3/4, z 1/8


def test_cbc_spec_examples(O):
    # 5 identical points, C_leaf = 32 -> single leaf
    V, T = _point_mesh([[0.25, 0.25, 0.25]] * 5)
    cl = O.Problem(V, T, leaf_size=32).clusters()
    assert len(cl["lo"]) == 1 and cl["child0"][0] == -1
    # 5 distinct points, C_leaf = 2 -> 3|2, then 3 -> 2|1: 3 leaves
    V, T = _point_mesh([[0, 0, 0], [1, 1, 1], [0.5, 0, 0], [0, 0.5, 0], [0.25, 0.75, 0.5]])
    cl = O.Problem(V, T, leaf_size=2).clusters()
    sizes = cl["hi"] - cl["lo"]
    leaves = sizes[cl["child0"] == -1]
    assert sorted(leaves.tolist()) == [1, 2, 2]
    assert sizes[0] == 5 and sizes[1] == 3 and sizes[cl["child0"][1]] == 2


def test_icosphere_1280_leaves(O):
    # 1280 = 20*4^3 halved 6 times -> 64 leaves of exactly 20 (A8)
    V, T = icosphere(3)
    cl = O.Problem(V, T, leaf_size=32).clusters()
    sizes = cl["hi"] - cl["lo"]
    leaf = cl["child0"] == -1
    assert leaf.sum() == 64 and (sizes[leaf] == 20).all()


@pytest.mark.parametrize("level", [2, 3])
def test_cluster_axioms_and_boxes(O, level):
    V, T = icosphere(level)
    P = O.Problem(V, T, leaf_size=32)
    cl = P.clusters()
    perm = P.perm()
    cen, _, _ = P.geometry()
    N = T.shape[0]
    # permutation + stable sort of codes (A7), checked by numpy lexsort
    codes = P.codes()
    ref = np.lexsort((np.arange(N), codes))
    assert np.array_equal(perm, ref)
    lo, hi, c0 = cl["lo"], cl["hi"], cl["child0"]
    assert lo[0] == 0 and hi[0] == N                          # (C2)
    assert ((hi - lo) > 0).all()                              # (C1)
    for c in range(len(lo)):
        n = hi[c] - lo[c]
        if c0[c] == -1:
            assert n <= 32                                     # (C3)
        else:
            # children are the next two clusters in pre-order: child0 and the one after its subtree
            kids = [k for k in range(len(lo)) if lo[k] >= lo[c] and hi[k] <= hi[c] and cl["depth"][k] == cl["depth"][c] + 1]
            assert len(kids) == 2                              # (C4) binary
            k1, k2 = sorted(kids, key=lambda k: lo[k])
            assert lo[k1] == lo[c] and hi[k1] == lo[k2] and hi[k2] == hi[c]   # disjoint union
            assert (hi[k1] - lo[k1]) - (hi[k2] - lo[k2]) in (0, 1)             # CBC |t1| = ceil(|t|/2)
        pts = cen[perm[lo[c]:hi[c]]]
        assert np.array_equal(cl["bbox"][c, :3], pts.min(axis=0))            # Q_tau
        assert np.array_equal(cl["bbox"][c, 3:], pts.max(axis=0))


def test_diam_dist_admissibility_examples(O):
    unit = [0, 0, 0, 1, 1, 1]
    far = [3, 0, 0, 4, 1, 1]
    # min diam sqrt(3) <= eta * dist 2  <=>  eta >= sqrt(3)/2
    assert O.admissible(unit, far, 1.0)
    assert O.admissible(unit, far, 0.8661)
    assert not O.admissible(unit, far, 0.8660)
    # overlapping boxes with positive diameter: dist 0 -> never admissible
    assert not O.admissible(unit, [0.5, 0.5, 0.5, 2, 2, 2], 1.0)
    assert not O.admissible(unit, [0.5, 0.5, 0.5, 2, 2, 2], 100.0)
    # point cluster vs disjoint cluster: 0 <= eta * dist for any eta >= 0
    assert O.admissible([5, 5, 5, 5, 5, 5], unit, 0.0)
    # inclusive inequality (A4): diam^2 == eta^2 dist^2 is admissible
    assert O.admissible([0, 0, 0, 2, 0, 0], [4, 0, 0, 5, 0, 0], 1.0)


def _coverage(N, leaves):
    cover = np.zeros((N, N), dtype=np.int32)
    for q in leaves:
        cover[q[0]:q[1], q[2]:q[3]] += 1
    return cover


@pytest.mark.parametrize("level", [2, 3])
def test_block_tree_partition_and_kinds(O, level):
    V, T = icosphere(level)
    N = T.shape[0]
    P = O.Problem(V, T, leaf_size=32, eta=1.0)
    adm, dense = P.leaves(0), P.leaves(1)
    cover = _coverage(N, np.concatenate([adm, dense]))
    assert (cover == 1).all()                                   # exact tiling
    area = lambda q: (q[:, 1] - q[:, 0]).astype(np.int64) * (q[:, 3] - q[:, 2])
    assert area(adm).sum() + area(dense).sum() == N * N
    cl = P.clusters()
    box = {(int(l), int(h)): cl["bbox"][c] for c, (l, h) in enumerate(zip(cl["lo"], cl["hi"]))}
    for q in adm:
        assert O.admissible(box[(q[0], q[1])], box[(q[2], q[3])], 1.0)
    for q in dense:
        assert not O.admissible(box[(q[0], q[1])], box[(q[2], q[3])], 1.0)
        assert min(q[1] - q[0], q[3] - q[2]) <= 32               # Alg. 1 guard
    if level == 2:
        assert len(adm) == 0 and len(dense) == 256               # N = 320: H = A
    else:
        assert len(adm) == 1534 and len(dense) == 2502           # regression


def test_block_tree_dfs_order(O):
    # leaves in canonical DFS pre-order (A10): every leaf precedes the leaves of later
    # sibling subtrees -> re-derive the order with an explicit stack walk over the
    # cluster tree, independent of the oracle's recursion.
    V, T = icosphere(3)
    P = O.Problem(V, T, leaf_size=32, eta=1.0)
    cl = P.clusters()
    kids = {}
    for c in range(len(cl["lo"])):
        if cl["child0"][c] != -1:
            sub = [k for k in range(len(cl["lo"])) if cl["depth"][k] == cl["depth"][c] + 1
                   and cl["lo"][k] >= cl["lo"][c] and cl["hi"][k] <= cl["hi"][c]]
            kids[c] = sorted(sub, key=lambda k: cl["lo"][k])
    leafset = {tuple(q) for q in P.leaves(0)} | {tuple(q) for q in P.leaves(1)}
    order = []
    stack = [(0, 0)]
    while stack:
        t, s = stack.pop()
        key = (cl["lo"][t], cl["hi"][t], cl["lo"][s], cl["hi"][s])
        if key in leafset:
            order.append(key)
            continue
        ch = [(a, b) for a in kids[t] for b in kids[s]]
        stack.extend(reversed(ch))
    got = [tuple(q) for q in np.concatenate([P.leaves(0), P.leaves(1)])]
    pos = {k: i for i, k in enumerate(order)}
    for kind in (0, 1):
        idx = [pos[tuple(q)] for q in P.leaves(kind)]
        assert idx == sorted(idx)
    assert len(order) == len(got)


def test_small_n_and_eta_zero(O):
    V, T = icosphere(1)                    # N = 80 > 32
    P = O.Problem(V, T, leaf_size=100, eta=1.0)
    assert len(P.leaves(1)) == 1 and len(P.leaves(0)) == 0   # N <= C_leaf: one dense leaf
    V, T = icosphere(3)
    P = O.Problem(V, T, leaf_size=32, eta=0.0)
    assert len(P.leaves(0)) == 0
    q = P.leaves(1)
    assert ((q[:, 1] - q[:, 0]).astype(np.int64) * (q[:, 3] - q[:, 2])).sum() == 1280 * 1280


def test_partition_invariants(O):
    rng = np.random.default_rng(3)
    cost = rng.integers(1, 1000, size=997)
    C = cost.sum()
    for p in (1, 2, 3, 4, 8):
        b = O.partition(cost, p)
        assert b[0] == 0 and b[-1] == cost.size and (np.diff(b) >= 0).all()
        pref = np.concatenate([[0], np.cumsum(cost)])[:-1]
        for r in range(p):
            own = pref[b[r]:b[r + 1]]
            assert ((own >= (r * C) // p) & (own < ((r + 1) * C) // p)).all()
            load = cost[b[r]:b[r + 1]].sum()
            assert load <= C / p + cost.max()
    assert list(O.partition(cost, 1)) == [0, cost.size]
