"""Oracle -- TEST INFRASTRUCTURE ONLY.

Python (ctypes) front end of ``oracle/oracle.c``: a plain, slow, fp64 CPU
implementation of the smoothed-aggregation AMG + CG/BiCGStab method of arXiv
1811.05704 (AMGCL), written from PAPER.md (Algorithm 1, PAPER.md:95-107;
Algorithm 2; preconditioning) and the readings
in SURVEY.md §8(c) / DESIGN.md §3.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline``
leg and ``--impl reference``) may import this package.  It shares no code with
the product library ``paper_1811_05704_b200``; neither imports the other.

Parity status: every function is pinned by ``tests/test_oracle_*.py`` except the
hierarchy statistics and iteration counts at benchmark sizes, which the paper
does not print ("parity unpinned", bounds only: SPEC.md:581, 588).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_HDR = os.path.join(_HERE, "oracle.h")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

OK, NOT_CONVERGED, BREAKDOWN = 0, 1, 2

# Compiler flags: no contraction of a*b+c into FMA and no fast-math, so every
# operation is the separately rounded IEEE operation the source spells out.
CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (no GPU needed)."""
    stale = (not os.path.exists(_LIB)) or any(
        os.path.getmtime(s) > os.path.getmtime(_LIB) for s in (_SRC, _HDR))
    if force or stale:
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class Params(C.Structure):
    _fields_ = [
        ("eps_strong", C.c_double),
        ("eps_decay", C.c_double),
        ("p_omega", C.c_double),
        ("smoothed", C.c_int32),
        ("relax", C.c_int32),
        ("jacobi_omega", C.c_double),
        ("cheb_degree", C.c_int32),
        ("cheb_lower", C.c_double),
        ("cheb_scaled", C.c_int32),
        ("npre", C.c_int32),
        ("npost", C.c_int32),
        ("coarse_enough", C.c_int64),
        ("max_levels", C.c_int32),
        ("dense_max", C.c_int64),
    ]


RELAX = {"spai0": 0, "damped_jacobi": 1, "chebyshev": 2}

_P = C.c_void_p
_I64P = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_I32P = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_F64P = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_U8P = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")


def lib():
    global _lib
    with _lock:
        if _lib is None:
            L = C.CDLL(build())
            L.or_last_error.restype = C.c_char_p
            L.or_params_default.argtypes = [C.POINTER(Params)]
            L.or_spmv.argtypes = [C.c_int64, _I64P, _I32P, _F64P, _F64P, _F64P]
            L.or_strength.argtypes = [C.c_int64, _I64P, _I32P, _F64P, C.c_double, _U8P]
            L.or_aggregate.argtypes = [C.c_int64, _I64P, _I32P, _F64P, _U8P, _I32P,
                                       C.POINTER(C.c_int64)]
            L.or_tentative_p.argtypes = [C.c_int64, _I32P, C.c_int64]
            L.or_tentative_p.restype = _P
            L.or_smooth_p.argtypes = [C.c_int64, _I64P, _I32P, _F64P, _U8P, _I32P, C.c_int64,
                                      C.c_double]
            L.or_smooth_p.restype = _P
            L.or_transpose.argtypes = [_P]
            L.or_transpose.restype = _P
            L.or_spgemm.argtypes = [_P, _P]
            L.or_spgemm.restype = _P
            L.or_csr_wrap_copy.argtypes = [C.c_int64, C.c_int64, _I64P, _I32P, _F64P]
            L.or_csr_wrap_copy.restype = _P
            L.or_csr_dims.argtypes = [_P, _I64P]
            L.or_csr_copy_out.argtypes = [_P, _I64P, _I32P, _F64P]
            L.or_csr_free.argtypes = [_P]
            L.or_lu_factor.argtypes = [C.c_int64, _F64P, _I32P]
            L.or_lu_solve.argtypes = [C.c_int64, _F64P, _I32P, _F64P, _F64P]
            L.or_setup.argtypes = [C.c_int64, _I64P, _I32P, _F64P, C.POINTER(Params),
                                   C.POINTER(_P)]
            L.or_free.argtypes = [_P]
            L.or_nlevels.argtypes = [_P]
            L.or_level_info.argtypes = [_P, C.c_int, _I64P]
            L.or_level_matrix.argtypes = [_P, C.c_int, C.c_int, _I64P, _I32P, _F64P]
            L.or_level_aggregates.argtypes = [_P, C.c_int, _I32P]
            L.or_level_smoother.argtypes = [_P, C.c_int, _F64P]
            L.or_vcycle.argtypes = [_P, C.c_int, _F64P, _F64P]
            L.or_precond.argtypes = [_P, _F64P, _F64P]
            L.or_relax.argtypes = [_P, C.c_int, _F64P, _F64P]
            L.or_cheb_step.argtypes = [_P, C.c_int, C.c_int, _F64P, _F64P, _F64P, C.POINTER(C.c_double)]
            L.or_cg.argtypes = [_P, C.c_int64, _I64P, _I32P, _F64P, C.c_int, _F64P, _F64P,
                                C.c_double, C.c_int32, C.POINTER(C.c_int32),
                                C.POINTER(C.c_double), C.c_void_p]
            L.or_bicgstab.argtypes = [_P, C.c_int64, _I64P, _I32P, _F64P, C.c_int, _F64P, _F64P,
                                      C.c_double, C.c_int32, C.POINTER(C.c_int32),
                                      C.POINTER(C.c_double), C.POINTER(C.c_int32)]
            L.or_gmres.argtypes = [_P, C.c_int64, _I64P, _I32P, _F64P, C.c_int, C.c_int32, _F64P, _F64P,
                                   C.c_double, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_double),
                                   C.POINTER(C.c_int32), C.c_void_p]
            L.or_idrs_shadow.argtypes = [C.c_int64, C.c_int32, _F64P]
            L.or_idrs.argtypes = [_P, C.c_int64, _I64P, _I32P, _F64P, C.c_int, C.c_int32, C.c_double, C.c_void_p,
                                  _F64P, _F64P, C.c_double, C.c_int32, C.POINTER(C.c_int32),
                                  C.POINTER(C.c_double), C.POINTER(C.c_int32), C.c_void_p]
            _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"oracle error {code}: {msg}")
        self.code = code


def _check(rc):
    if rc < 0:
        raise OracleError(rc, lib().or_last_error().decode())
    return rc


def _csr_args(ptr, col, val):
    return (np.ascontiguousarray(ptr, np.int64), np.ascontiguousarray(col, np.int32),
            np.ascontiguousarray(val, np.float64))


def _take_csr(h):
    """Copy an or_csr* into numpy arrays and free it."""
    L = lib()
    if not h:
        raise OracleError(-6, "allocation failed")
    d = np.zeros(3, np.int64)
    L.or_csr_dims(h, d)
    nr, nc, nnz = (int(v) for v in d)
    ptr = np.zeros(nr + 1, np.int64)
    col = np.zeros(max(nnz, 1), np.int32)
    val = np.zeros(max(nnz, 1), np.float64)
    L.or_csr_copy_out(h, ptr, col, val)
    L.or_csr_free(h)
    return Csr(ptr, col[:nnz], val[:nnz], nc)


class Csr:
    """Plain CSR triple plus column count."""

    def __init__(self, ptr, col, val, ncols=None):
        self.ptr, self.col, self.val = _csr_args(ptr, col, val)
        self.nrows = len(self.ptr) - 1
        self.ncols = int(ncols) if ncols is not None else self.nrows

    @property
    def nnz(self):
        return int(self.ptr[-1])

    def _handle(self):
        return lib().or_csr_wrap_copy(self.nrows, self.ncols, self.ptr,
                                      np.ascontiguousarray(self.col) if self.nnz else np.zeros(1, np.int32),
                                      np.ascontiguousarray(self.val) if self.nnz else np.zeros(1))

    def to_dense(self):
        D = np.zeros((self.nrows, self.ncols))
        for i in range(self.nrows):
            for k in range(self.ptr[i], self.ptr[i + 1]):
                D[i, self.col[k]] = self.val[k]
        return D

    def __iter__(self):
        return iter((self.ptr, self.col, self.val))


def params(**kw) -> Params:
    p = Params()
    lib().or_params_default(C.byref(p))
    for k, v in kw.items():
        if k == "relax" and isinstance(v, str):
            v = RELAX[v]
        setattr(p, k, v)
    return p


# ---- single operations ------------------------------------------------------

def spmv(A: Csr, x):
    x = np.ascontiguousarray(x, np.float64)
    y = np.zeros(A.nrows)
    lib().or_spmv(A.nrows, A.ptr, A.col, A.val, x, y)
    return y


def strength(A: Csr, eps=0.08):
    S = np.zeros(max(A.nnz, 1), np.uint8)
    _check(lib().or_strength(A.nrows, A.ptr, A.col, A.val, eps, S))
    return S[:A.nnz]


def aggregate(A: Csr, S):
    S = np.ascontiguousarray(S, np.uint8)
    idv = np.zeros(A.nrows, np.int32)
    cnt = C.c_int64()
    _check(lib().or_aggregate(A.nrows, A.ptr, A.col, A.val, S, idv, C.byref(cnt)))
    return idv, int(cnt.value)


def tentative_p(idv, count):
    idv = np.ascontiguousarray(idv, np.int32)
    return _take_csr(lib().or_tentative_p(len(idv), idv, count))


def smooth_p(A: Csr, S, idv, count, omega=2.0 / 3.0):
    return _take_csr(lib().or_smooth_p(A.nrows, A.ptr, A.col, A.val,
                                       np.ascontiguousarray(S, np.uint8),
                                       np.ascontiguousarray(idv, np.int32), count, omega))


def transpose(A: Csr):
    h = A._handle()
    try:
        return _take_csr(lib().or_transpose(h))
    finally:
        lib().or_csr_free(h)


def spgemm(A: Csr, B: Csr):
    ha, hb = A._handle(), B._handle()
    try:
        return _take_csr(lib().or_spgemm(ha, hb))
    finally:
        lib().or_csr_free(ha)
        lib().or_csr_free(hb)


def lu_factor(a):
    a = np.array(a, np.float64, order="C", copy=True)
    n = a.shape[0]
    piv = np.zeros(max(n, 1), np.int32)
    _check(lib().or_lu_factor(n, a.reshape(-1), piv))
    return a, piv


def lu_solve(lu, piv, b):
    n = lu.shape[0]
    x = np.zeros(n)
    lib().or_lu_solve(n, np.ascontiguousarray(lu).reshape(-1), piv,
                      np.ascontiguousarray(b, np.float64), x)
    return x


# ---- hierarchy and solvers --------------------------------------------------

class Hierarchy:
    """Algorithm 1 run by the oracle."""

    def __init__(self, A: Csr, **kw):
        self.A = A
        self.prm = params(**kw)
        h = C.c_void_p()
        _check(lib().or_setup(A.nrows, A.ptr, A.col, A.val, C.byref(self.prm), C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            lib().or_free(self._h)
            self._h = None

    @property
    def nlevels(self):
        return lib().or_nlevels(self._h)

    def info(self, l):
        out = np.zeros(6, np.int64)
        _check(lib().or_level_info(self._h, l, out))
        keys = ("rows", "nnz_A", "nnz_P", "cols_P", "aggregates", "coarsest")
        return dict(zip(keys, (int(v) for v in out)))

    def matrix(self, l, which="A"):
        w = {"A": 0, "P": 1, "R": 2}[which]
        inf = self.info(l)
        if w == 0:
            nr, nc, nnz = inf["rows"], inf["rows"], inf["nnz_A"]
        elif w == 1:
            nr, nc, nnz = inf["rows"], inf["cols_P"], inf["nnz_P"]
        else:
            nr, nc, nnz = inf["cols_P"], inf["rows"], inf["nnz_P"]
        ptr = np.zeros(nr + 1, np.int64)
        col = np.zeros(max(nnz, 1), np.int32)
        val = np.zeros(max(nnz, 1))
        _check(lib().or_level_matrix(self._h, l, w, ptr, col, val))
        return Csr(ptr, col[:nnz], val[:nnz], nc)

    def aggregates(self, l):
        idv = np.zeros(self.info(l)["rows"], np.int32)
        _check(lib().or_level_aggregates(self._h, l, idv))
        return idv

    def smoother(self, l):
        n = self.info(l)["rows"]
        out = np.zeros(max(n, 4))
        _check(lib().or_level_smoother(self._h, l, out))
        return out[:4] if self.prm.relax == 2 else out[:n]

    def vcycle(self, l, f, x):
        x = np.array(x, np.float64, copy=True)
        _check(lib().or_vcycle(self._h, l, np.ascontiguousarray(f, np.float64), x))
        return x

    def precond(self, r):
        z = np.zeros(self.A.nrows)
        _check(lib().or_precond(self._h, np.ascontiguousarray(r, np.float64), z))
        return z

    def relax(self, l, f, x):
        x = np.array(x, np.float64, copy=True)
        _check(lib().or_relax(self._h, l, np.ascontiguousarray(f, np.float64), x))
        return x

    def cheb_step(self, l, k, f, x, p, alpha=0.0):
        """Step k of the Chebyshev smoother (or_cheb_step): returns (x', p',
        alpha_k) from x, p and alpha_{k-1}."""
        x = np.array(x, np.float64, copy=True)
        p = np.array(p, np.float64, copy=True)
        a = C.c_double(alpha)
        _check(lib().or_cheb_step(self._h, l, k, np.ascontiguousarray(f, np.float64), x, p, C.byref(a)))
        return x, p, a.value

    def complexities(self):
        infos = [self.info(l) for l in range(self.nlevels)]
        op = sum(i["nnz_A"] for i in infos) / infos[0]["nnz_A"]
        grid = sum(i["rows"] for i in infos) / infos[0]["rows"]
        return op, grid


def cg(A: Csr, f, x0=None, tol=1e-8, maxiter=100, hier: Hierarchy | None = None, history=False):
    """Preconditioned CG; hier=None means M = I."""
    n = A.nrows
    f = np.ascontiguousarray(f, np.float64)
    x = np.zeros(n) if x0 is None else np.array(x0, np.float64, copy=True)
    it = C.c_int32()
    rel = C.c_double()
    hist = np.zeros(maxiter + 1) if history else None
    rc = _check(lib().or_cg(hier._h if hier else None, n, A.ptr, A.col, A.val, 1 if hier else 0,
                            f, x, tol, maxiter, C.byref(it), C.byref(rel),
                            hist.ctypes.data_as(C.c_void_p) if history else None))
    out = dict(x=x, iters=it.value, rel_resid=rel.value, status=rc)
    if history:
        out["history"] = hist[:it.value + 1]
    return out


def bicgstab(A: Csr, f, x0=None, tol=1e-8, maxiter=100, hier: Hierarchy | None = None):
    """Right-preconditioned BiCGStab; hier=None means M = I."""
    n = A.nrows
    f = np.ascontiguousarray(f, np.float64)
    x = np.zeros(n) if x0 is None else np.array(x0, np.float64, copy=True)
    it = C.c_int32()
    rel = C.c_double()
    vc = C.c_int32()
    rc = _check(lib().or_bicgstab(hier._h if hier else None, n, A.ptr, A.col, A.val,
                                  1 if hier else 0, f, x, tol, maxiter, C.byref(it),
                                  C.byref(rel), C.byref(vc)))
    return dict(x=x, iters=it.value, rel_resid=rel.value, status=rc, vcycles=vc.value)


def idrs_shadow(n, s):
    """The IDR(s) shadow space P (s x n, row j = column j of the n x s matrix)."""
    P = np.zeros(n * s)
    lib().or_idrs_shadow(n, s, P)
    return P.reshape(s, n)


def idrs(A: Csr, f, x0=None, tol=1e-8, maxiter=100, s=4, kappa=0.7, P=None, hier: Hierarchy | None = None,
         history=False):
    """Right-preconditioned IDR(s) with bi-orthogonalisation;
    hier=None means M = I.  P: shadow space (s x n) or None (idrs_shadow)."""
    n = A.nrows
    f = np.ascontiguousarray(f, np.float64)
    x = np.zeros(n) if x0 is None else np.array(x0, np.float64, copy=True)
    it, rel, vc = C.c_int32(), C.c_double(), C.c_int32()
    hist = np.zeros(maxiter + 1) if history else None
    Pa = None if P is None else np.ascontiguousarray(P, np.float64).reshape(-1)
    rc = _check(lib().or_idrs(hier._h if hier else None, n, A.ptr, A.col, A.val, 1 if hier else 0, s, kappa,
                              Pa.ctypes.data_as(C.c_void_p) if Pa is not None else None, f, x, tol, maxiter,
                              C.byref(it), C.byref(rel), C.byref(vc),
                              hist.ctypes.data_as(C.c_void_p) if history else None))
    out = dict(x=x, iters=it.value, rel_resid=rel.value, status=rc, vcycles=vc.value)
    if history:
        out["history"] = hist[:it.value + 1]
    return out


def gmres(A: Csr, f, x0=None, tol=1e-8, maxiter=100, m=30, hier: Hierarchy | None = None, history=False):
    """Restarted right-preconditioned GMRES(m); hier=None means M = I."""
    n = A.nrows
    f = np.ascontiguousarray(f, np.float64)
    x = np.zeros(n) if x0 is None else np.array(x0, np.float64, copy=True)
    it, rel, vc = C.c_int32(), C.c_double(), C.c_int32()
    hist = np.zeros(maxiter + 1) if history else None
    rc = _check(lib().or_gmres(hier._h if hier else None, n, A.ptr, A.col, A.val, 1 if hier else 0, m, f, x,
                               tol, maxiter, C.byref(it), C.byref(rel), C.byref(vc),
                               hist.ctypes.data_as(C.c_void_p) if history else None))
    out = dict(x=x, iters=it.value, rel_resid=rel.value, status=rc, vcycles=vc.value)
    if history:
        out["history"] = hist[:it.value + 1]
    return out
