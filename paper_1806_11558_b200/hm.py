"""Thin ctypes binding of libhm (include/hm.h): argument marshalling only.

Every step of the path runs in libhm's CUDA kernels; this module converts numpy arrays /
torch tensors to raw pointers and status codes to exceptions.  There is no CPU fallback:
if libhm.so is missing or no CUDA device is present the import or the call fails loudly.

Function names mirror the C ABI (hm_create, hm_build_tree, hm_setup, hm_matvec, hm_solve,
...).  `HMatrix` bundles them around one context for convenience.
"""
from __future__ import annotations

import ctypes as C
import json
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhm.so")

STATUS = {0: "HM_OK", 1: "HM_ERR_ARG", 2: "HM_ERR_STATE", 3: "HM_ERR_OOM", 4: "HM_ERR_CUDA",
          5: "HM_ERR_NCCL", 6: "HM_ERR_NUMERIC", 7: "HM_ERR_BREAKDOWN"}
NCCL_ID_BYTES = 128
P2P_HANDLE_BYTES = 64


class HMError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class _Mesh(C.Structure):
    _fields_ = [("vertices", C.c_void_p), ("n_vertices", C.c_int64),
                ("triangles", C.c_void_p), ("n_triangles", C.c_int64), ("memory", C.c_int),
                ("panel_vertices", C.c_int)]


_lib = None


def lib():
    """Load libhm.so (built in-tree by __graft_entry__.build()); raise if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libhm.so not built at {LIB_PATH}: run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        vp, i64, i32, d = C.c_void_p, C.c_int64, C.c_int, C.c_double
        sig = {
            "hm_create": [C.POINTER(vp), i32, i32, i32, vp, vp],
            "hm_nccl_unique_id": [vp],
            "hm_destroy": [vp],
            "hm_set_option": [vp, C.c_char_p, d],
            "hm_get_option": [vp, C.c_char_p, C.POINTER(d)],
            "hm_build_tree": [vp, C.POINTER(_Mesh), i32, d],
            "hm_setup": [vp, d],
            "hm_matvec": [vp, vp, vp],
            "hm_solve": [vp, vp, vp, d, C.POINTER(i32), C.POINTER(d)],
            "hm_assemble_rhs": [vp, i32, vp],
            "hm_potential": [vp, vp, i64, vp, vp],
            "hm_get_perm": [vp, vp],
            "hm_get_codes": [vp, vp],
            "hm_get_leaves": [vp, i32, C.POINTER(i64), vp, C.POINTER(i64), C.POINTER(i64)],
            "hm_get_clusters": [vp, C.POINTER(i64), vp, vp, vp, vp],
            "hm_eval_entries": [vp, i64, vp, vp],
            "hm_get_dense_block": [vp, i64, vp],
            "hm_get_lowrank": [vp, i64, C.POINTER(i32), vp, vp, vp],
            "hm_quadrature_table": [i32, vp, vp],
            "hm_get_stats": [vp, C.c_char_p, i64],
            "hm_p2p_export": [vp, i64, vp],
            "hm_p2p_import": [vp, vp],
        }
        for name, args in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = C.c_int
        L.hm_last_error.argtypes = [vp]
        L.hm_last_error.restype = C.c_char_p
        _lib = L
    return _lib


def _check(ctx, st):
    if st != 0:
        msg = lib().hm_last_error(ctx).decode() if ctx else ""
        raise HMError(st, msg)


def _ptr(a):
    """Raw pointer of a contiguous numpy array or torch tensor (host or CUDA)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return C.c_void_p(a.data_ptr())
    if not a.flags["C_CONTIGUOUS"]:
        raise ValueError("array must be C-contiguous")
    return a.ctypes.data_as(C.c_void_p)


def _is_cuda(a):
    return hasattr(a, "is_cuda") and a.is_cuda


# ---- C-ABI mirrors ------------------------------------------------------------------------
def hm_nccl_unique_id() -> bytes:
    buf = (C.c_char * NCCL_ID_BYTES)()
    _check(None, lib().hm_nccl_unique_id(buf))
    return bytes(buf)


def hm_create(device=0, rank=0, world_size=1, nccl_unique_id: bytes | None = None, cuda_stream: int = 0):
    ctx = C.c_void_p()
    idbuf = None
    if nccl_unique_id is not None:
        idbuf = (C.c_char * NCCL_ID_BYTES).from_buffer_copy(nccl_unique_id)
    st = lib().hm_create(C.byref(ctx), device, rank, world_size, idbuf, C.c_void_p(cuda_stream or None))
    if st != 0:
        raise HMError(st, "hm_create failed")
    return ctx


def hm_destroy(ctx):
    lib().hm_destroy(ctx)


def hm_set_option(ctx, key: str, value: float):
    _check(ctx, lib().hm_set_option(ctx, key.encode(), float(value)))


def hm_get_option(ctx, key: str) -> float:
    v = C.c_double()
    _check(ctx, lib().hm_get_option(ctx, key.encode(), C.byref(v)))
    return v.value


def hm_build_tree(ctx, vertices, triangles, leaf_size=32, eta=1.0):
    dev = _is_cuda(vertices)
    if dev != _is_cuda(triangles):
        raise ValueError("vertices and triangles must both be host or both device")
    m = _Mesh(_ptr(vertices), int(vertices.shape[0]), _ptr(triangles), int(triangles.shape[0]), 1 if dev else 0,
              int(triangles.shape[1]))
    _check(ctx, lib().hm_build_tree(ctx, C.byref(m), int(leaf_size), float(eta)))


def hm_setup(ctx, eps_aca=1e-6):
    _check(ctx, lib().hm_setup(ctx, float(eps_aca)))


def hm_matvec(ctx, x, y):
    _check(ctx, lib().hm_matvec(ctx, _ptr(x), _ptr(y)))


def hm_solve(ctx, rhs, sol, tol=1e-8):
    it = C.c_int(); rr = C.c_double()
    _check(ctx, lib().hm_solve(ctx, _ptr(rhs), _ptr(sol), float(tol), C.byref(it), C.byref(rr)))
    return it.value, rr.value


def hm_p2p_export(ctx, n_max: int) -> bytes:
    buf = (C.c_char * P2P_HANDLE_BYTES)()
    _check(ctx, lib().hm_p2p_export(ctx, int(n_max), buf))
    return bytes(buf)


def hm_p2p_import(ctx, handles: bytes):
    buf = (C.c_char * len(handles)).from_buffer_copy(handles)
    _check(ctx, lib().hm_p2p_import(ctx, buf))


def hm_assemble_rhs(ctx, kind, f):
    _check(ctx, lib().hm_assemble_rhs(ctx, int(kind), _ptr(f)))


def hm_potential(ctx, sol, points, out):
    _check(ctx, lib().hm_potential(ctx, _ptr(sol), int(points.shape[0]), _ptr(points), _ptr(out)))


def hm_get_stats(ctx) -> dict:
    buf = C.create_string_buffer(1 << 16)
    _check(ctx, lib().hm_get_stats(ctx, buf, len(buf)))
    return json.loads(buf.value.decode())


def hm_quadrature_table(n):
    x = np.zeros(n); w = np.zeros(n)
    _check(None, lib().hm_quadrature_table(n, _ptr(x), _ptr(w)))
    return x, w


class HMatrix:
    """One libhm context: tree -> setup -> matvec / solve, vectors in application order."""

    def __init__(self, device=0, rank=0, world_size=1, nccl_unique_id=None, cuda_stream=0):
        self.ctx = hm_create(device, rank, world_size, nccl_unique_id, cuda_stream)
        self.N = 0

    def close(self):
        if getattr(self, "ctx", None):
            hm_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_option(self, key, value):
        hm_set_option(self.ctx, key, value)

    def enable_p2p(self, n_max, group=None):
        """Sharded-solve collectives over NVLink peer memory (hm_p2p_export / hm_p2p_import):
        every rank exports its exchange buffer, the IPC handles are all-gathered over the torch
        process group (plumbing only), and every rank maps its peers'.  All ranks must agree on
        the transport: if any rank cannot map its peers, every rank keeps NCCL (option
        solve_comm 0) and the error is returned (None on success)."""
        import torch
        import torch.distributed as dist
        err = None
        try:
            h = hm_p2p_export(self.ctx, n_max)
        except HMError as e:
            h, err = b"", e
        allh = [None] * dist.get_world_size(group)
        dist.all_gather_object(allh, h, group=group)
        if err is None and all(len(x) == P2P_HANDLE_BYTES for x in allh):
            try:
                hm_p2p_import(self.ctx, b"".join(allh))
            except HMError as e:
                err = e
        ok = torch.tensor([0 if err is not None or any(len(x) != P2P_HANDLE_BYTES for x in allh) else 1],
                          dtype=torch.int32, device="cuda")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
        if int(ok.item()) == 0:
            if self.get_option("solve_comm") != 0:
                self.set_option("solve_comm", 0)
            return err or RuntimeError("a peer rank could not map the P2P buffers")
        return None

    def get_option(self, key):
        return hm_get_option(self.ctx, key)

    def build_tree(self, vertices, triangles, leaf_size=32, eta=1.0):
        if not _is_cuda(vertices):
            vertices = np.ascontiguousarray(vertices, dtype=np.float64)
            triangles = np.ascontiguousarray(triangles, dtype=np.int32)
        hm_build_tree(self.ctx, vertices, triangles, leaf_size, eta)
        self.N = int(triangles.shape[0])

    def setup(self, eps_aca=1e-6):
        hm_setup(self.ctx, eps_aca)

    def matvec(self, x, y=None):
        if y is None:
            y = x.new_empty(x.shape) if hasattr(x, "new_empty") else np.empty_like(x)
        hm_matvec(self.ctx, x, y)
        return y

    def solve(self, rhs, tol=1e-8, sol=None):
        if sol is None:
            sol = rhs.new_empty(rhs.shape) if hasattr(rhs, "new_empty") else np.empty_like(rhs)
        it, rr = hm_solve(self.ctx, rhs, sol, tol)
        return sol, it, rr

    def assemble_rhs(self, kind, out=None):
        if out is None:
            out = np.empty(self.N)
        hm_assemble_rhs(self.ctx, kind, out)
        return out

    def potential(self, sol, points, out=None):
        """Single-layer potential of sol (application order) at points (m x 3)."""
        if out is None:
            out = points.new_empty(points.shape[0]) if hasattr(points, "new_empty") else np.empty(points.shape[0])
        hm_potential(self.ctx, sol, points, out)
        return out

    # ---- introspection (host arrays) ----
    def perm(self):
        p = np.empty(self.N, dtype=np.int32)
        _check(self.ctx, lib().hm_get_perm(self.ctx, _ptr(p)))
        return p

    def codes(self):
        c = np.empty(self.N, dtype=np.uint64)
        _check(self.ctx, lib().hm_get_codes(self.ctx, _ptr(c)))
        return c

    def leaves(self, kind):
        n = C.c_int64(); b = C.c_int64(); e = C.c_int64()
        _check(self.ctx, lib().hm_get_leaves(self.ctx, kind, C.byref(n), None, C.byref(b), C.byref(e)))
        q = np.empty((n.value, 4), dtype=np.int32)
        _check(self.ctx, lib().hm_get_leaves(self.ctx, kind, C.byref(n), _ptr(q), None, None))
        return q, (b.value, e.value)

    def clusters(self):
        n = C.c_int64()
        _check(self.ctx, lib().hm_get_clusters(self.ctx, C.byref(n), None, None, None, None))
        lo = np.empty(n.value, np.int32); hi = np.empty(n.value, np.int32)
        dp = np.empty(n.value, np.int32); bb = np.empty((n.value, 6))
        _check(self.ctx, lib().hm_get_clusters(self.ctx, C.byref(n), _ptr(lo), _ptr(hi), _ptr(dp), _ptr(bb)))
        return dict(lo=lo, hi=hi, depth=dp, bbox=bb)

    def entries(self, pairs):
        pr = np.ascontiguousarray(pairs, dtype=np.int64).reshape(-1, 2)
        out = np.empty(pr.shape[0])
        _check(self.ctx, lib().hm_eval_entries(self.ctx, pr.shape[0], _ptr(pr), _ptr(out)))
        return out

    def dense_block(self, leaf, shape):
        B = np.empty(shape)
        _check(self.ctx, lib().hm_get_dense_block(self.ctx, int(leaf), _ptr(B)))
        return B

    def lowrank(self, leaf, m, n, pivots=False):
        k = C.c_int32()
        _check(self.ctx, lib().hm_get_lowrank(self.ctx, int(leaf), C.byref(k), None, None, None))
        kk = k.value
        U = np.empty((kk, m)); V = np.empty((kk, n))
        pv = np.empty(2 * kk, dtype=np.int32) if pivots else None
        _check(self.ctx, lib().hm_get_lowrank(self.ctx, int(leaf), C.byref(k), _ptr(U), _ptr(V), _ptr(pv)))
        res = (U.T.copy(), V.T.copy())
        return res + ((pv.reshape(-1, 2),) if pivots else ())

    def stats(self):
        return hm_get_stats(self.ctx)
