"""ctypes wrapper of the CPU oracle (oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs.  The product package
(paper_1806_11558_b200) never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "liboracle.so")


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", _HERE, "CC=gcc"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        P, i64, i32, d, u64 = C.c_void_p, C.c_int64, C.c_int, C.c_double, C.c_uint64
        ptr = C.c_void_p
        L.or_create.restype = P
        L.or_create.argtypes = [ptr, i64, ptr, i64, i32, d]
        L.or_create_quads.restype = P
        L.or_create_quads.argtypes = [ptr, i64, ptr, i64, i32, d]
        L.or_destroy.argtypes = [P]
        L.or_n.restype = i64; L.or_n.argtypes = [P]
        L.or_get_perm.argtypes = [P, ptr]
        L.or_get_codes.argtypes = [P, ptr]
        L.or_get_geometry.argtypes = [P, ptr, ptr, ptr]
        L.or_num_clusters.restype = i64; L.or_num_clusters.argtypes = [P]
        L.or_get_clusters.argtypes = [P, ptr, ptr, ptr, ptr, ptr]
        L.or_num_leaves.restype = i64; L.or_num_leaves.argtypes = [P, i32]
        L.or_get_leaves.argtypes = [P, i32, ptr]
        L.or_admissible.restype = i32; L.or_admissible.argtypes = [ptr, ptr, d]
        L.or_gauss_legendre01.argtypes = [i32, ptr, ptr]
        L.or_entries.argtypes = [P, i64, ptr, ptr]
        L.or_entry_class.restype = i32; L.or_entry_class.argtypes = [P, i64, i64]
        L.or_selfterm_closed.restype = d; L.or_selfterm_closed.argtypes = [ptr, ptr, ptr]
        L.or_sauter_schwab.restype = d; L.or_sauter_schwab.argtypes = [i32, ptr, ptr, i32]
        L.or_potential.argtypes = [P, ptr, i64, ptr, ptr]
        L.or_panel_potential.restype = d; L.or_panel_potential.argtypes = [ptr, ptr, i32]
        L.or_ss_reference_monomial.restype = d
        L.or_ss_reference_monomial.argtypes = [i32, i32, i32, i32, i32, i32]
        L.or_regular_rule.restype = d; L.or_regular_rule.argtypes = [ptr, ptr, i32]
        L.or_rule_table.restype = i32; L.or_rule_table.argtypes = [i32, ptr, ptr, ptr]
        L.or_dense_rows.argtypes = [P, i64, ptr, ptr]
        L.or_aca_block.restype = i32
        L.or_aca_block.argtypes = [P, i32, i32, i32, i32, d, i32, ptr, ptr, ptr]
        L.or_aca_matrix.restype = i32
        L.or_aca_matrix.argtypes = [ptr, i32, i32, d, i32, ptr, ptr, ptr]
        L.or_assemble.restype = i32
        L.or_assemble.argtypes = [P, d, i32, i64, i64, i64, i64]
        L.or_stored_doubles.restype = i64; L.or_stored_doubles.argtypes = [P]
        L.or_release.argtypes = [P]
        L.or_assemble_list.restype = i32
        L.or_assemble_list.argtypes = [P, d, i32, i64, ptr, i64, ptr]
        L.or_get_rank.restype = i32; L.or_get_rank.argtypes = [P, i64]
        L.or_get_factors.argtypes = [P, i64, ptr, ptr]
        L.or_get_pivots.argtypes = [P, i64, ptr]
        L.or_get_dense_block.argtypes = [P, i64, ptr]
        L.or_matvec.argtypes = [P, ptr, ptr]
        L.or_rhs.argtypes = [P, i32, ptr]
        L.or_cg.restype = i32
        L.or_cg.argtypes = [P, ptr, ptr, d, i32, C.POINTER(d), C.POINTER(i32)]
        L.or_gmres.restype = i32
        L.or_gmres.argtypes = [P, ptr, ptr, d, i32, i32, C.POINTER(d), C.POINTER(i32)]
        L.or_partition.argtypes = [ptr, i64, i32, ptr]
        L.or_counters.argtypes = [P, ptr]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def gauss_legendre01(n):
    x = np.zeros(n); w = np.zeros(n)
    lib().or_gauss_legendre01(n, _p(x), _p(w))
    return x, w


def admissible(box_t, box_s, eta):
    bt = np.ascontiguousarray(box_t, dtype=np.float64)
    bs = np.ascontiguousarray(box_s, dtype=np.float64)
    return bool(lib().or_admissible(_p(bt), _p(bs), float(eta)))


def selfterm_closed(tri):
    t = np.ascontiguousarray(tri, dtype=np.float64).reshape(3, 3)
    return lib().or_selfterm_closed(_p(t[0].copy()), _p(t[1].copy()), _p(t[2].copy()))


def sauter_schwab(kind, tx, ty, nq=6):
    a = np.ascontiguousarray(tx, dtype=np.float64).reshape(9)
    b = np.ascontiguousarray(ty, dtype=np.float64).reshape(9)
    return lib().or_sauter_schwab(kind, _p(a), _p(b), nq)


def ss_reference_monomial(kind, nq, a, b, c, d):
    return lib().or_ss_reference_monomial(kind, nq, a, b, c, d)


def regular_rule(tx, ty, n):
    a = np.ascontiguousarray(tx, dtype=np.float64).reshape(9)
    b = np.ascontiguousarray(ty, dtype=np.float64).reshape(9)
    return lib().or_regular_rule(_p(a), _p(b), n)


def rule_table(n):
    s = np.zeros(64); t = np.zeros(64); w = np.zeros(64)
    k = lib().or_rule_table(n, _p(s), _p(t), _p(w))
    return s[:k].copy(), t[:k].copy(), w[:k].copy()


def panel_potential(x, tri, n):
    """int_T 1/|x - y| dy by the collapsed Gauss n x n rule of A23."""
    a = np.ascontiguousarray(x, dtype=np.float64).reshape(3)
    t = np.ascontiguousarray(tri, dtype=np.float64).reshape(9)
    return lib().or_panel_potential(_p(a), _p(t), n)


def aca_matrix(A, eps, kcap):
    A = np.ascontiguousarray(A, dtype=np.float64)
    m, n = A.shape
    kmax = max(1, min(m, n, kcap))
    U = np.zeros((kmax, m)); V = np.zeros((kmax, n)); pv = np.zeros(2 * kmax + 2, dtype=np.int32)
    k = lib().or_aca_matrix(_p(A), m, n, eps, kcap, _p(U), _p(V), _p(pv))
    return U[:k].T.copy(), V[:k].T.copy(), pv[:2 * k].reshape(-1, 2)


def partition(cost, p):
    c = np.ascontiguousarray(cost, dtype=np.int64)
    out = np.zeros(p + 1, dtype=np.int64)
    lib().or_partition(_p(c), c.size, p, _p(out))
    return out


class Problem:
    """Oracle problem: mesh -> geometry, Morton order, trees; then assembly, matvec, solves."""

    def __init__(self, V, T, leaf_size=32, eta=1.0):
        self.V = np.ascontiguousarray(V, dtype=np.float64)
        self.T = np.ascontiguousarray(T, dtype=np.int32)
        self.N = self.T.shape[0]
        create = lib().or_create_quads if self.T.shape[1] == 4 else lib().or_create   # quads: A25
        self._h = create(_p(self.V), self.V.shape[0], _p(self.T), self.N, leaf_size, float(eta))

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.or_destroy(self._h)
            self._h = None

    # --- tree ---
    def perm(self):
        p = np.zeros(self.N, dtype=np.int32); lib().or_get_perm(self._h, _p(p)); return p

    def codes(self):
        c = np.zeros(self.N, dtype=np.uint64); lib().or_get_codes(self._h, _p(c)); return c

    def geometry(self):
        c = np.zeros((self.N, 3)); a = np.zeros(self.N); h = np.zeros(self.N)
        lib().or_get_geometry(self._h, _p(c), _p(a), _p(h)); return c, a, h

    def clusters(self):
        n = lib().or_num_clusters(self._h)
        lo = np.zeros(n, np.int32); hi = np.zeros(n, np.int32); c0 = np.zeros(n, np.int32)
        dp = np.zeros(n, np.int32); bb = np.zeros((n, 6))
        lib().or_get_clusters(self._h, _p(lo), _p(hi), _p(c0), _p(dp), _p(bb))
        return dict(lo=lo, hi=hi, child0=c0, depth=dp, bbox=bb)

    def leaves(self, kind):
        n = lib().or_num_leaves(self._h, kind)
        q = np.zeros((n, 4), dtype=np.int32)
        if n:
            lib().or_get_leaves(self._h, kind, _p(q))
        return q

    # --- entries ---
    def entries(self, pairs):
        pr = np.ascontiguousarray(pairs, dtype=np.int64).reshape(-1, 2)
        out = np.zeros(pr.shape[0])
        lib().or_entries(self._h, pr.shape[0], _p(pr), _p(out))
        return out

    def entry_class(self, i, j):
        return lib().or_entry_class(self._h, int(i), int(j))

    def dense_rows(self, rows):
        r = np.ascontiguousarray(rows, dtype=np.int64)
        out = np.zeros((r.size, self.N))
        lib().or_dense_rows(self._h, r.size, _p(r), _p(out))
        return out

    def dense(self):
        return self.dense_rows(np.arange(self.N))

    # --- ACA / assembly ---
    def aca_block(self, quad, eps, kcap=64):
        rlo, rhi, clo, chi = (int(v) for v in quad)
        m, n = rhi - rlo, chi - clo
        kmax = max(1, min(m, n, kcap))
        U = np.zeros((kmax, m)); Vv = np.zeros((kmax, n)); pv = np.zeros(2 * kmax + 2, np.int32)
        k = lib().or_aca_block(self._h, rlo, rhi, clo, chi, eps, kcap, _p(U), _p(Vv), _p(pv))
        return U[:k].T.copy(), Vv[:k].T.copy(), pv[:2 * k].reshape(-1, 2)

    def assemble(self, eps=1e-6, kcap=64, dense_range=None, adm_range=None):
        nd = lib().or_num_leaves(self._h, 1); na = lib().or_num_leaves(self._h, 0)
        d0, d1 = dense_range if dense_range is not None else (0, nd)
        a0, a1 = adm_range if adm_range is not None else (0, na)
        return lib().or_assemble(self._h, eps, kcap, d0, d1, a0, a1)

    def assemble_list(self, eps, dense_leaves, adm_leaves, kcap=64):
        """Assemble only the listed leaves (ascending indices into the canonical lists)."""
        dl = np.ascontiguousarray(dense_leaves, dtype=np.int64)
        al = np.ascontiguousarray(adm_leaves, dtype=np.int64)
        return lib().or_assemble_list(self._h, eps, kcap, dl.size, _p(dl), al.size, _p(al))

    def release(self):
        """Free the stored blocks (outside any timed region)."""
        lib().or_release(self._h)

    def stored_doubles(self):
        return lib().or_stored_doubles(self._h)

    def rank(self, b):
        return lib().or_get_rank(self._h, int(b))

    def factors(self, b):
        q = self.leaves(0)[b]
        m, n = q[1] - q[0], q[3] - q[2]
        k = self.rank(b)
        U = np.zeros((max(k, 0), m)); Vv = np.zeros((max(k, 0), n))
        if k > 0:
            lib().or_get_factors(self._h, int(b), _p(U), _p(Vv))
        return U.T.copy(), Vv.T.copy()

    def pivots(self, b):
        k = self.rank(b)
        pv = np.zeros(2 * max(k, 0), np.int32)
        if k > 0:
            lib().or_get_pivots(self._h, int(b), _p(pv))
        return pv.reshape(-1, 2)

    def dense_block(self, b):
        q = self.leaves(1)[b]
        B = np.zeros((q[1] - q[0], q[3] - q[2]))
        lib().or_get_dense_block(self._h, int(b), _p(B))
        return B

    def counters(self):
        c = np.zeros(4); lib().or_counters(self._h, _p(c)); return c

    # --- products / solves ---
    def matvec(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros(self.N)
        lib().or_matvec(self._h, _p(x), _p(y))
        return y

    def potential(self, alpha, X):
        """(1/4pi) sum_j alpha_j int_{T_j} 1/|x - y| at the rows of X (M x 3), A23."""
        a = np.ascontiguousarray(alpha, dtype=np.float64)
        X = np.ascontiguousarray(X, dtype=np.float64).reshape(-1, 3)
        out = np.zeros(X.shape[0])
        lib().or_potential(self._h, _p(a), X.shape[0], _p(X), _p(out))
        return out

    def rhs(self, kind):
        f = np.zeros(self.N); lib().or_rhs(self._h, kind, _p(f)); return f

    def cg(self, b, tol=1e-8, maxit=10000):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.zeros(self.N); rr = C.c_double(0); st = C.c_int(0)
        it = lib().or_cg(self._h, _p(b), _p(x), tol, maxit, C.byref(rr), C.byref(st))
        return x, it, rr.value, st.value

    def gmres(self, b, tol=1e-8, restart=100, maxit=10000):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.zeros(self.N); rr = C.c_double(0); st = C.c_int(0)
        it = lib().or_gmres(self._h, _p(b), _p(x), tol, restart, maxit, C.byref(rr), C.byref(st))
        return x, it, rr.value, st.value
