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
