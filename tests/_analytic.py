"""Independent analytic references used to PIN the oracle (never used by it).

* triangle_potential(x, tri): closed-form  int_T 1/|x-y| dy  for a flat triangle
  (the classical edge-sum formula of Wilton et al. 1984 / Graglia 1993: for each
  edge, P0 ln((R+ + l+)/(R- + l-)) minus the solid-angle atan terms).  Evaluated
  with numpy in float64.
* double_integral_semianalytic(tx, ty, level, order): int_Tx int_Ty 1/|x-y| with the
  inner integral exact (triangle_potential) and the outer integral by a collapsed
  Gauss rule on a uniform 4^level subdivision of Tx.  The integrand is continuous
  (bounded potential), so this converges to the exact value as level grows,
  independently of any Duffy/Sauter-Schwab transformation.
* square_pair_integral(A, B): int_A int_B 1/|x-y| for two squares (origin, e1, e2 with
  e1 _|_ e2, |e1| = |e2|): the inner integral is the closed-form potential of a uniform
  rectangle (antiderivative X asinh(Y/sqrt(X^2+z^2)) + Y asinh(X/sqrt(Y^2+z^2))
  - z atan(XY/(zR)) at the four corners, Durand 1964), the outer one a tensor Gauss rule
  graded geometrically toward all four edges of B.  Never splits a square into
  triangles, so it is independent of the quadrilateral reading A25.
* gauss_legendre_decimal(n, digits): Gauss-Legendre nodes/weights on [0,1] by
  Newton iteration in Python's decimal module, correctly rounded to binary64.
"""
from __future__ import annotations

from decimal import Decimal, getcontext

import numpy as np


def triangle_potential(x, tri):
    """int_T 1/|x - y| dy for points x [..., 3] and one flat triangle tri [3, 3]."""
    x = np.atleast_2d(np.asarray(x, dtype=np.float64))
    v = np.asarray(tri, dtype=np.float64)
    n = np.cross(v[1] - v[0], v[2] - v[0])
    n = n / np.linalg.norm(n)
    d = (x - v[0]) @ n                              # signed height
    rho = x - d[:, None] * n[None, :]                # projection to the plane
    ad = np.abs(d)
    total = np.zeros(x.shape[0])
    for i in range(3):
        a, b = v[i], v[(i + 1) % 3]
        L = b - a
        lhat = L / np.linalg.norm(L)
        uhat = np.cross(lhat, n)                     # in-plane edge normal (outward for CCW)
        P0 = (a - rho) @ uhat
        lp = (b - rho) @ lhat
        lm = (a - rho) @ lhat
        Rp = np.linalg.norm(x - b, axis=1)
        Rm = np.linalg.norm(x - a, axis=1)
        R02 = P0 * P0 + d * d
        with np.errstate(divide="ignore", invalid="ignore"):
            logt = np.log((Rp + lp) / (Rm + lm))
        logt = np.where(np.abs(P0) > 0, logt, 0.0)
        at = np.arctan2(P0 * lp, R02 + ad * Rp) - np.arctan2(P0 * lm, R02 + ad * Rm)
        total += P0 * logt - ad * at
    return total


def _collapsed_gauss(order):
    g, w = np.polynomial.legendre.leggauss(order)
    g = (g + 1) / 2; w = w / 2
    xi = np.repeat(g, order); ze = np.tile(g, order)
    ww = np.repeat(w, order) * np.tile(w, order) * xi
    return xi, xi * ze, ww                            # s, t, weight (reference area 1/2)


def _subdivide(tri, level):
    tris = [np.asarray(tri, dtype=np.float64)]
    for _ in range(level):
        nxt = []
        for t in tris:
            a, b, c = t
            ab, bc, ca = (a + b) / 2, (b + c) / 2, (c + a) / 2
            nxt += [np.array([a, ab, ca]), np.array([ab, b, bc]), np.array([ca, bc, c]), np.array([ab, bc, ca])]
        tris = nxt
    return tris


def double_integral_semianalytic(tx, ty, level=4, order=8):
    tx = np.asarray(tx, dtype=np.float64).reshape(3, 3)
    ty = np.asarray(ty, dtype=np.float64).reshape(3, 3)
    s, t, w = _collapsed_gauss(order)
    pts, wts = [], []
    for sub in _subdivide(tx, level):
        v0, v1, v2 = sub
        p = v0[None] + s[:, None] * (v1 - v0)[None] + t[:, None] * (v2 - v1)[None]
        J = np.linalg.norm(np.cross(v1 - v0, v2 - v0))
        pts.append(p); wts.append(w * J)
    P = np.concatenate(pts); W = np.concatenate(wts)
    return float(np.sum(W * triangle_potential(P, ty)))


def gauss_legendre_decimal(n, digits=60):
    """Nodes ascending on [0,1] and weights (sum 1), correctly rounded to float64."""
    getcontext().prec = digits
    pi = Decimal("3.14159265358979323846264338327950288419716939937510582097494459230781640628620899")
    nodes, weights = [], []
    for k in range(n):
        import math
        t = Decimal(math.cos(math.pi * (k + 0.75) / (n + 0.5)))
        for _ in range(200):
            p0, p1 = Decimal(1), t
            for m in range(2, n + 1):
                p0, p1 = p1, ((2 * m - 1) * t * p1 - (m - 1) * p0) / m
            dp = n * (t * p1 - p0) / (t * t - 1)
            dt = p1 / dp
            t -= dt
            if abs(dt) < Decimal(10) ** (-(digits - 5)):
                break
        p0, p1 = Decimal(1), t
        for m in range(2, n + 1):
            p0, p1 = p1, ((2 * m - 1) * t * p1 - (m - 1) * p0) / m
        dp = n * (t * p1 - p0) / (t * t - 1)
        nodes.append(float((1 - t) / 2))             # Decimal -> float rounds correctly
        weights.append(float(1 / ((1 - t * t) * dp * dp)))
    del pi
    return np.array(nodes), np.array(weights)


def _rect_antiderivative(X, Y, z):
    R = np.sqrt(X * X + Y * Y + z * z)
    with np.errstate(divide="ignore", invalid="ignore"):
        t1 = np.where(X == 0, 0.0, X * np.arcsinh(Y / np.sqrt(X * X + z * z)))
        t2 = np.where(Y == 0, 0.0, Y * np.arcsinh(X / np.sqrt(Y * Y + z * z)))
        t3 = np.where(z == 0, 0.0, z * np.arctan2(X * Y, z * R))
    return t1 + t2 - t3


def square_potential(P, o, e1, e2):
    """int over the square {o + a e1 + b e2 : a, b in [0,1]} of 1/|p - y| for points P [M, 3]."""
    P = np.atleast_2d(np.asarray(P, dtype=np.float64))
    s = np.linalg.norm(e1)
    u1, u2 = e1 / s, e2 / s
    n = np.cross(u1, u2)
    d = P - o
    px, py, pz = d @ u1, d @ u2, np.abs(d @ n)
    F = _rect_antiderivative
    return F(s - px, s - py, pz) - F(-px, s - py, pz) - F(s - px, -py, pz) + F(-px, -py, pz)


def _graded01(levels, pts):
    g, w = np.polynomial.legendre.leggauss(pts)
    g, w = (g + 1) / 2, w / 2
    edges = [0.0] + [0.5 * 2.0 ** (-k) for k in range(levels, 0, -1)] + [0.5]
    a, b = np.array(edges[:-1]), np.array(edges[1:])
    x = (a[:, None] + (b - a)[:, None] * g[None, :]).ravel()
    ww = ((b - a)[:, None] * w[None, :]).ravel()
    return np.concatenate([x, 1 - x[::-1]]), np.concatenate([ww, ww[::-1]])


def square_pair_integral(A, B, levels=22, pts=10):
    """int_A int_B 1/|x - y| dy dx, A and B = (origin, e1, e2) squares."""
    oA, e1A, e2A = (np.asarray(v, dtype=np.float64) for v in A)
    oB, e1B, e2B = (np.asarray(v, dtype=np.float64) for v in B)
    x, w = _graded01(levels, pts)
    S, T = np.meshgrid(x, x, indexing="ij")
    P = (oB[None, None, :] + S[..., None] * e1B + T[..., None] * e2B).reshape(-1, 3)
    val = square_potential(P, oA, e1A, e2A)
    return float((val * np.outer(w, w).ravel()).sum() * np.linalg.norm(np.cross(e1B, e2B)))
