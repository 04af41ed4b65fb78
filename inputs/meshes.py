"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds INPUT GENERATION ONLY: surface meshes shaped like the
workloads of BASELINE.json and seeded test vectors.  It contains none of the
method's arithmetic (no quadrature, no clustering, no ACA, no matvec), so both
`oracle/` and `paper_1806_11558_b200/` may consume what it produces.

Meshes:
  * icosphere(L)    - unit icosahedron, L times 4-split with midpoints projected
                      to the unit sphere: N = 20*4^L flat triangles
                      (configs[0..2]: L = 3, 5, 7).
  * geodesic(nu)    - class-I geodesic sphere of frequency nu: every
                      icosahedron face split into nu^2 triangles on the flat
                      face lattice, then projected to R = 1: N = 20*nu^2
                      (configs[3]: nu = 280 -> 1,568,000).
  * lobed(nu)       - geodesic(nu) pushed out radially by six Gaussian lobes
                      and stretched to the gearwheel's bounding box
                      (configs[4]: nu = 244 -> 1,190,720).
All meshes are vertex-deduplicated (the entry classification of PAPER.md
§4.1 "Duffy trick" needs shared vertex *indices*) and consistently oriented
(outward normals), vertices float64 [n_v, 3], triangles int32 [N, 3].
"""
from __future__ import annotations

import numpy as np

__all__ = ["icosahedron", "icosphere", "geodesic", "lobed", "config_mesh",
           "seeded_vector", "CONFIGS"]


def icosahedron():
    """12 unit vertices and 20 outward-oriented faces of the regular icosahedron."""
    phi = (1.0 + 5.0 ** 0.5) / 2.0
    v = []
    for a in (-1.0, 1.0):
        for b in (-phi, phi):
            v += [(0.0, a, b), (a, b, 0.0), (b, 0.0, a)]
    v = np.array(v, dtype=np.float64)
    # faces = vertex triples with pairwise distance 2 (the edge length before normalisation)
    d = np.linalg.norm(v[:, None, :] - v[None, :, :], axis=2)
    adj = np.abs(d - 2.0) < 1e-9
    faces = []
    for i in range(12):
        for j in range(i + 1, 12):
            if not adj[i, j]:
                continue
            for k in range(j + 1, 12):
                if adj[i, k] and adj[j, k]:
                    faces.append((i, j, k))
    f = np.array(faces, dtype=np.int64)
    assert f.shape == (20, 3)
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    f = _orient_outward(v, f)
    return v, f


def _orient_outward(v, f):
    a, b, c = v[f[:, 0]], v[f[:, 1]], v[f[:, 2]]
    n = np.cross(b - a, c - a)
    flip = np.einsum("ij,ij->i", n, (a + b + c)) < 0
    f = f.copy()
    f[flip, 1], f[flip, 2] = f[flip, 2].copy(), f[flip, 1].copy()
    return f


def icosphere(level: int):
    """Recursive icosahedral refinement (midpoints projected to R = 1)."""
    v, f = icosahedron()
    for _ in range(level):
        nv = v.shape[0]
        e = np.concatenate([f[:, [0, 1]], f[:, [1, 2]], f[:, [2, 0]]], axis=0)
        e.sort(axis=1)
        key = e[:, 0] * nv + e[:, 1]
        uk, inv = np.unique(key, return_inverse=True)
        a, b = uk // nv, uk % nv
        m = v[a] + v[b]
        m /= np.linalg.norm(m, axis=1, keepdims=True)
        mid = inv.reshape(3, -1).T + nv  # columns: m01, m12, m20
        v = np.concatenate([v, m], axis=0)
        m01, m12, m20 = mid[:, 0], mid[:, 1], mid[:, 2]
        f = np.concatenate([
            np.stack([f[:, 0], m01, m20], axis=1),
            np.stack([m01, f[:, 1], m12], axis=1),
            np.stack([m20, m12, f[:, 2]], axis=1),
            np.stack([m01, m12, m20], axis=1),
        ], axis=0)
    return np.ascontiguousarray(v, dtype=np.float64), np.ascontiguousarray(f, dtype=np.int32)


def geodesic(nu: int):
    """Class-I geodesic sphere of frequency nu (flat face lattice, projected to R = 1)."""
    v12, f20 = icosahedron()
    ii, jj = np.meshgrid(np.arange(nu + 1), np.arange(nu + 1), indexing="ij")
    keep = ii + jj <= nu
    bi, bj = ii[keep], jj[keep]               # barycentric weights of B and C
    ba = nu - bi - bj                          # weight of A
    lut = -np.ones((nu + 1, nu + 1), dtype=np.int64)
    lut[bi, bj] = np.arange(bi.size)
    # local triangles on the lattice (upward and downward)
    up = (ii + jj <= nu - 1)
    ui, uj = ii[up], jj[up]
    t_up = np.stack([lut[ui, uj], lut[ui + 1, uj], lut[ui, uj + 1]], axis=1)
    dn = (ii + jj <= nu - 2)
    di, dj = ii[dn], jj[dn]
    t_dn = np.stack([lut[di + 1, dj], lut[di + 1, dj + 1], lut[di, dj + 1]], axis=1)
    tloc = np.concatenate([t_up, t_dn], axis=0)
    npts = bi.size
    M = np.int64(12 * (nu + 1) + 1)
    keys = np.empty(20 * npts, dtype=np.int64)
    pos = np.empty((20 * npts, 3), dtype=np.float64)
    tris = np.empty((20 * tloc.shape[0], 3), dtype=np.int64)
    for fi in range(20):
        A, B, C = f20[fi]
        codes = np.stack([
            np.where(ba > 0, A * (nu + 1) + ba, M - 1),
            np.where(bi > 0, B * (nu + 1) + bi, M - 1),
            np.where(bj > 0, C * (nu + 1) + bj, M - 1)], axis=1).astype(np.int64)
        codes.sort(axis=1)
        keys[fi * npts:(fi + 1) * npts] = (codes[:, 0] * M + codes[:, 1]) * M + codes[:, 2]
        p = (ba[:, None] * v12[A] + bi[:, None] * v12[B] + bj[:, None] * v12[C]) / nu
        pos[fi * npts:(fi + 1) * npts] = p
        tris[fi * tloc.shape[0]:(fi + 1) * tloc.shape[0]] = tloc + fi * npts
    uk, first, inv = np.unique(keys, return_index=True, return_inverse=True)
    v = pos[first]
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    f = inv[tris]
    f = _orient_outward(v, f)
    return np.ascontiguousarray(v, dtype=np.float64), np.ascontiguousarray(f, dtype=np.int32)


def lobed(nu: int):
    """Perturbed multi-lobed closed surface (stand-in for the paper's gearwheel,
    bbox [-4,4]^2 x [-11.5,9.1], §4.3): star-shaped radial map of geodesic(nu)."""
    v, f = geodesic(nu)
    dirs = np.concatenate([np.eye(3), -np.eye(3)], axis=0)
    d2 = ((v[:, None, :] - dirs[None, :, :]) ** 2).sum(axis=2)
    r = 1.0 + 0.5 * np.exp(-d2 / 0.15).sum(axis=1)
    x = (r[:, None] * v) * (np.array([4.0, 4.0, 10.3]) / 1.5)
    return np.ascontiguousarray(x, dtype=np.float64), f


# BASELINE.json configs -> mesh recipe
CONFIGS = {
    "C1": ("icosphere", 3),      # 1,280 triangles
    "C2": ("icosphere", 5),      # 20,480
    "C3": ("icosphere", 7),      # 327,680
    "C4": ("geodesic", 280),     # 1,568,000
    "C5": ("lobed", 244),        # 1,190,720
}


def config_mesh(name: str):
    kind, p = CONFIGS[name]
    return {"icosphere": icosphere, "geodesic": geodesic, "lobed": lobed}[kind](p)


def seeded_vector(n: int, seed: int):
    """x ~ N(0,1), numpy.random.default_rng(seed), application order."""
    return np.random.default_rng(seed).standard_normal(n)
