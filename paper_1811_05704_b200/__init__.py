"""B200-native smoothed-aggregation AMG solve phase (arXiv 1811.05704, AMGCL).

Thin Python binding of ``_lib/libamgb.so`` (C ABI: ``include/amgb.h``).  This
module only marshals arguments: the hierarchy is built inside the library
(Algorithm 1; on the GPU by default, bitwise the C++ host
build) and every step of the solve phase
(Algorithm 2, inside CG / BiCGStab) runs in
the library's sm_100a kernels.  PyTorch is used for device memory and streams
only.  There is no CPU fallback: if the shared library is missing, importing
this package raises.

Parameters use the paper's runtime key names (Listing 2)
where it has them, e.g. ``{"solver.type": "bicgstab", "precond.relax.type":
"chebyshev"}``; see ``PARAM_KEYS``.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("AMGB_LIB_PATH") or os.path.join(_HERE, "_lib", "libamgb.so")  # override: checked build

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(or `make -C paper_1811_05704_b200`). There is no CPU fallback.")

_lib = C.CDLL(LIB_PATH)

# ---- status codes (amg_status) ----
OK, NOT_CONVERGED, BREAKDOWN = 0, 1, 2
E_INVALID_ARG, E_BAD_CSR, E_ZERO_DIAG, E_SINGULAR_COARSE = -1, -2, -3, -4
E_COARSE_TOO_LARGE, E_OOM, E_NO_DEVICE, E_CUDA, E_NCCL = -5, -6, -7, -10, -11

OP_SPMV_A, OP_SPMV_P, OP_SPMV_R, OP_RESIDUAL, OP_RELAX, OP_COARSE, OP_VCYCLE = range(7)
(OP_RES0, OP_RES0_MF, OP_RESTRICT_MF, OP_PROL0, OP_PROL0_MF, OP_PROL_ADD, OP_RELAX_RHO, OP_CHEB_STEP,
 OP_CG_DIR, OP_CG_UPDATE) = range(7, 17)
FMT_CSR, FMT_SELL, FMT_TMA, FMT_TMACSR, FMT_NONE = 0, 1, 2, 3, 15
PROF_CLASSES = ("A0 pass", "A coarse", "transfer", "vector", "coarse solve")


class AmgParams(C.Structure):
    _fields_ = [
        ("struct_size", C.c_uint32),
        ("coarsening", C.c_int32),
        ("eps_strong", C.c_double),
        ("eps_decay", C.c_double),
        ("p_omega", C.c_double),
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
        ("solver", C.c_int32),
        ("device", C.c_int32),
        ("use_graph", C.c_int32),
        ("precision", C.c_int32),
        ("gmres_m", C.c_int32),
        ("setup_device", C.c_int32),
        ("idrs_s", C.c_int32),
        ("reorder", C.c_int32),
    ]


class LevelInfo(C.Structure):
    _fields_ = [
        ("rows", C.c_int64), ("nnz_A", C.c_int64), ("nnz_P", C.c_int64), ("cols_P", C.c_int64),
        ("aggregates", C.c_int64), ("is_coarsest", C.c_int32), ("dict_slices_A", C.c_int32),
        ("dev_bytes", C.c_int64), ("padded_nnz_A", C.c_int64), ("alg_bytes_vcycle", C.c_double),
        ("padded_nnz_P", C.c_int64), ("padded_nnz_R", C.c_int64), ("sigma_mask", C.c_int32),
        ("formats", C.c_int32),
    ]


class LevelOpArgs(C.Structure):
    _fields_ = [("in0", C.c_void_p), ("in1", C.c_void_p), ("out0", C.c_void_p), ("out1", C.c_void_p),
                ("out2", C.c_void_p), ("scalar", C.c_double), ("dot", C.c_double)]


class LevelExport(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in (
        "A_ptr", "A_col", "A_val", "P_ptr", "P_col", "P_val", "R_ptr", "R_col", "R_val",
        "aggregates", "smoother", "coarse_inverse")]


class AmgDist(C.Structure):
    _fields_ = [("nranks", C.c_int32), ("rank", C.c_int32), ("gather_below", C.c_int64),
                ("nccl_id", C.c_uint8 * 128)]


class DistLevelExport(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in (
        "A_ptr", "A_col", "A_val", "P_ptr", "P_col", "P_val", "R_ptr", "R_col", "R_val",
        "ghost_global", "recv_peer", "recv_off", "recv_cnt", "send_peer", "send_off", "send_cnt",
        "send_idx")]


class SolveStats(C.Structure):
    _fields_ = [
        ("iters", C.c_int32), ("vcycles", C.c_int32), ("status", C.c_int32), ("flags", C.c_int32),
        ("kernel_launches", C.c_int64), ("solve_ms", C.c_double), ("rel_resid", C.c_double),
        ("alg_bytes", C.c_double), ("prof_ms", C.c_double * 8), ("prof_bytes", C.c_double * 8),
        ("prof_launches", C.c_int64 * 8),
    ]


_V = C.c_void_p
_lib.amg_params_default.argtypes = [C.POINTER(AmgParams)]
_lib.amg_setup.argtypes = [C.c_int64, _V, _V, _V, C.POINTER(AmgParams), C.POINTER(_V)]
_lib.amg_solve.argtypes = [_V, _V, _V, C.c_double, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_double)]
_lib.amg_solve_host.argtypes = [_V, _V, _V, _V, C.c_double, C.c_int32, C.POINTER(C.c_int32),
                                C.POINTER(C.c_double)]
_lib.amg_solve_host_stream.argtypes = [_V, C.c_int32, _V, _V, C.c_double, C.c_int32, _V, _V, _V]
_lib.amg_precond_apply.argtypes = [_V, _V, _V]
_lib.amg_set_stream.argtypes = [_V, _V]
_lib.amg_set_profile.argtypes = [_V, C.c_int32]
_lib.amg_level_count.argtypes = [_V, C.POINTER(C.c_int32)]
_lib.amg_level_info_get.argtypes = [_V, C.c_int32, C.POINTER(LevelInfo)]
_lib.amg_export_level.argtypes = [_V, C.c_int32, C.POINTER(LevelExport)]
_lib.amg_solve_stats_get.argtypes = [_V, C.POINTER(SolveStats)]
_lib.amg_level_op.argtypes = [_V, C.c_int32, C.c_int32, _V, _V, _V]
_lib.amg_level_op_ex.argtypes = [_V, C.c_int32, C.c_int32, C.POINTER(LevelOpArgs)]
_lib.amg_destroy.argtypes = [_V]
_lib.amg_vector_length.argtypes = [_V, C.POINTER(C.c_int64)]
_lib.amg_nccl_unique_id.argtypes = [_V]
_lib.amg_solve_batched.argtypes = [_V, C.c_int32, _V, C.c_int64, _V, C.c_int64, C.c_double, C.c_int32, _V, _V]
_lib.amg_nccl_selftest.argtypes = [C.c_int32]
_lib.amg_shm_selftest.argtypes = [_V, C.c_int32, C.c_int32]
_lib.amg_setup_dist.argtypes = [C.c_int64, _V, _V, _V, C.POINTER(AmgParams), C.POINTER(AmgDist),
                                C.POINTER(_V)]
_lib.amg_dist_info.argtypes = [_V, C.POINTER(C.c_int32), C.POINTER(C.c_int32), _V]
_lib.amg_dist_level_info.argtypes = [_V, C.c_int32, C.c_int32, _V]
_lib.amg_dist_export.argtypes = [_V, C.c_int32, C.c_int32, C.POINTER(DistLevelExport)]
_lib.amg_last_error.restype = C.c_char_p
_lib.amg_version.restype = C.c_char_p
for _name in ("amg_setup", "amg_solve", "amg_solve_host", "amg_solve_host_stream", "amg_precond_apply", "amg_set_stream",
              "amg_set_profile", "amg_level_count", "amg_level_info_get", "amg_export_level",
              "amg_solve_stats_get", "amg_level_op", "amg_level_op_ex", "amg_vector_length", "amg_nccl_unique_id", "amg_setup_dist",
              "amg_dist_info", "amg_dist_level_info", "amg_dist_export", "amg_nccl_selftest",
              "amg_solve_batched", "amg_shm_selftest", "amg_vector_length"):
    getattr(_lib, _name).restype = C.c_int

# Exported C symbols (tests check them against include/amgb.h).
SYMBOLS = ("amg_params_default", "amg_setup", "amg_solve", "amg_solve_host", "amg_solve_host_stream",
           "amg_precond_apply",
           "amg_set_stream", "amg_set_profile", "amg_level_count", "amg_level_info_get",
           "amg_export_level", "amg_solve_stats_get", "amg_level_op", "amg_level_op_ex", "amg_vector_length", "amg_destroy",
           "amg_last_error", "amg_version", "amg_nccl_unique_id", "amg_setup_dist", "amg_dist_info",
           "amg_dist_level_info", "amg_dist_export", "amg_nccl_selftest", "amg_solve_batched",
           "amg_shm_selftest")

RELAX = {"spai0": 0, "damped_jacobi": 1, "chebyshev": 2}
COARSENING = {"smoothed_aggregation": 0, "aggregation": 1}
SOLVER = {"cg": 0, "bicgstab": 1, "gmres": 2, "idrs": 3}

# dotted keys (Listing 2 style) -> amg_params field
PARAM_KEYS = {
    "precond.coarsening.type": "coarsening",
    "precond.coarsening.aggr.eps_strong": "eps_strong",
    "precond.coarsening.aggr.eps_decay": "eps_decay",
    "precond.coarsening.p_omega": "p_omega",
    "precond.relax.type": "relax",
    "precond.relax.damping": "jacobi_omega",
    "precond.relax.degree": "cheb_degree",
    "precond.relax.lower": "cheb_lower",
    "precond.relax.scaled": "cheb_scaled",
    "precond.npre": "npre",
    "precond.npost": "npost",
    "precond.coarse_enough": "coarse_enough",
    "precond.max_levels": "max_levels",
    "precond.dense_max": "dense_max",
    "solver.type": "solver",
    "device": "device",
    "use_graph": "use_graph",
    "precision": "precision",
    "solver.M": "gmres_m",
    "setup.device": "setup_device",
    "solver.s": "idrs_s",
}
PRECISION = {"double": 0, "mixed": 1}
SETUP_DEVICE = {"host": 0, "gpu": 1}
_ENUMS = {"relax": RELAX, "coarsening": COARSENING, "solver": SOLVER, "precision": PRECISION,
          "setup_device": SETUP_DEVICE}


class AmgError(RuntimeError):
    def __init__(self, code, where):
        msg = _lib.amg_last_error().decode()
        super().__init__(f"{where} failed ({code}): {msg}")
        self.code = code


def _check(rc, where):
    if rc < 0:
        raise AmgError(rc, where)
    return rc


def make_params(params: dict | None = None, **kw) -> AmgParams:
    p = AmgParams()
    _lib.amg_params_default(C.byref(p))
    items = dict(params or {})
    items.update(kw)
    for k, v in items.items():
        field = PARAM_KEYS.get(k, k)
        if field not in dict(AmgParams._fields_):
            raise KeyError(f"unknown parameter {k!r}")
        if field in _ENUMS and isinstance(v, str):
            v = _ENUMS[field][v]
        setattr(p, field, v)
    return p


def version() -> str:
    return _lib.amg_version().decode()


def _host_vec(a, n: int, name: str) -> np.ndarray:
    """A host vector the C ABI reads or writes n doubles of (no length argument
    crosses the ABI): exactly n C-contiguous float64 values, else ValueError."""
    if not isinstance(a, np.ndarray) or a.dtype != np.float64 or a.ndim != 1 or not a.flags.c_contiguous:
        raise ValueError(f"{name}: need a 1-D C-contiguous float64 numpy array")
    if a.shape[0] != n:
        raise ValueError(f"{name}: length {a.shape[0]} != {n} (the handle's vector length)")
    return a


def _dev_vec(t, n: int, name: str):
    """A CUDA float64 tensor of exactly n contiguous elements, else ValueError."""
    import torch
    if not isinstance(t, torch.Tensor) or t.dtype != torch.float64 or not t.is_cuda:
        raise ValueError(f"{name}: need a CUDA float64 tensor")
    if t.numel() != n or not t.is_contiguous():
        raise ValueError(f"{name}: need {n} contiguous elements (got {t.numel()})")
    return t


def _ptr(a):
    """Address of a numpy array or torch tensor (contiguous)."""
    if isinstance(a, np.ndarray):
        if not a.flags.c_contiguous:
            raise ValueError("array must be C-contiguous")
        return a.ctypes.data
    if not a.is_contiguous():
        raise ValueError("tensor must be contiguous")
    return a.data_ptr()


class Hierarchy:
    """amg_setup handle: AMG hierarchy of A, resident on the GPU (device >= 0) or
    host-only (device = -1, for setup/export only)."""

    def __init__(self, ptr, col, val, params: dict | None = None, dist: AmgDist | None = None, n: int | None = None,
                 **kw):
        self.prm = make_params(params, **kw)
        self.dist = dist
        h = C.c_void_p()
        if ptr is None:
            # scattered multi-GPU setup, rank > 0: the matrix lives on rank 0 only
            if dist is None or dist.rank <= 0 or n is None:
                raise ValueError("ptr/col/val may be omitted only on NCCL ranks > 0 (with n given)")
            self.n = int(n)
            p_ptr = p_col = p_val = None
        else:
            self._ptr = np.ascontiguousarray(ptr, np.int64)
            col = np.ascontiguousarray(col, np.int32)
            val = np.ascontiguousarray(val, np.float64)
            self.n = len(self._ptr) - 1
            p_ptr, p_col, p_val = self._ptr.ctypes.data, col.ctypes.data, val.ctypes.data
        if dist is None:
            _check(_lib.amg_setup(self.n, p_ptr, p_col, p_val, C.byref(self.prm), C.byref(h)), "amg_setup")
        else:
            _check(_lib.amg_setup_dist(self.n, p_ptr, p_col, p_val, C.byref(self.prm), C.byref(dist),
                                       C.byref(h)), "amg_setup_dist")
        self._h = h
        vl = C.c_int64()
        _check(_lib.amg_vector_length(h, C.byref(vl)), "amg_vector_length")
        self.vec_len = vl.value  # length of the f / x vectors amg_solve* take
        self.on_device = self.prm.device >= 0
        if self.on_device:
            import torch
            self.device = torch.device("cuda", self.prm.device)

    def close(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.amg_destroy(self._h)
        self._h = None

    __del__ = close

    # ---- info / export -------------------------------------------------
    @property
    def nlevels(self) -> int:
        n = C.c_int32()
        _check(_lib.amg_level_count(self._h, C.byref(n)), "amg_level_count")
        return n.value

    def level_info(self, l: int) -> dict:
        li = LevelInfo()
        _check(_lib.amg_level_info_get(self._h, l, C.byref(li)), "amg_level_info_get")
        d = {k: getattr(li, k) for k, _ in LevelInfo._fields_}
        f = d["formats"]
        d["fmt_A"], d["fmt_P"], d["fmt_R"] = f & 15, (f >> 4) & 15, (f >> 8) & 15
        d["vidx_A"], d["vidx_P"], d["vidx_R"] = (f >> 12) & 3, (f >> 14) & 3, (f >> 16) & 3
        return d

    def complexities(self):
        inf = [self.level_info(l) for l in range(self.nlevels)]
        return (sum(i["nnz_A"] for i in inf) / inf[0]["nnz_A"],
                sum(i["rows"] for i in inf) / inf[0]["rows"])

    def export_level(self, l: int) -> dict:
        """Host copies of level l: A, P, R (CSR triples), aggregates, smoother data
        and (coarsest level) the dense inverse."""
        inf = self.level_info(l)
        n, nnz, np_, nc = inf["rows"], inf["nnz_A"], inf["nnz_P"], inf["cols_P"]
        out = {"A": (np.zeros(n + 1, np.int64), np.zeros(nnz, np.int32), np.zeros(nnz))}
        ex = LevelExport()
        ex.A_ptr, ex.A_col, ex.A_val = (a.ctypes.data for a in out["A"])
        if not inf["is_coarsest"]:
            out["P"] = (np.zeros(n + 1, np.int64), np.zeros(np_, np.int32), np.zeros(np_))
            out["R"] = (np.zeros(nc + 1, np.int64), np.zeros(np_, np.int32), np.zeros(np_))
            out["aggregates"] = np.zeros(n, np.int32)
            out["smoother"] = np.zeros(4 if self.prm.relax == 2 else n)
            ex.P_ptr, ex.P_col, ex.P_val = (a.ctypes.data for a in out["P"])
            ex.R_ptr, ex.R_col, ex.R_val = (a.ctypes.data for a in out["R"])
            ex.aggregates = out["aggregates"].ctypes.data
            ex.smoother = out["smoother"].ctypes.data
        else:
            out["coarse_inverse"] = np.zeros((n, n))
            ex.coarse_inverse = out["coarse_inverse"].ctypes.data
        _check(_lib.amg_export_level(self._h, l, C.byref(ex)), "amg_export_level")
        return out

    # ---- partition (multi-GPU) -----------------------------------------
    def dist_info(self) -> dict:
        nr, lg = C.c_int32(), C.c_int32()
        _check(_lib.amg_dist_info(self._h, C.byref(nr), C.byref(lg), None), "amg_dist_info")
        starts = np.zeros(nr.value + 1, np.int64)
        _check(_lib.amg_dist_info(self._h, C.byref(nr), C.byref(lg), starts.ctypes.data),
               "amg_dist_info")
        return {"nranks": nr.value, "first_replicated": lg.value, "row_starts": starts}

    def dist_level_info(self, rank: int, l: int) -> dict:
        out = np.zeros(18, np.int64)
        _check(_lib.amg_dist_level_info(self._h, rank, l, out.ctypes.data), "amg_dist_level_info")
        keys = ("row0", "row1", "ghosts", "nnz_A", "nnz_P", "nnz_R", "crow0", "crow1", "replicated",
                "send_total", "recv_peers", "send_peers", "A_ib0", "A_ib1", "P_ib0", "P_ib1", "R_ib0", "R_ib1")
        return dict(zip(keys, (int(v) for v in out)))

    def dist_export(self, rank: int, l: int) -> dict:
        """Local matrices (local|ghost columns) and halo plan of (rank, level)."""
        inf = self.dist_level_info(rank, l)
        nloc = inf["row1"] - inf["row0"]
        ncr = inf["crow1"] - inf["crow0"]
        out = {"info": inf}
        ex = DistLevelExport()

        def csr(name, nr, nnz):
            a = (np.zeros(nr + 1, np.int64), np.zeros(nnz, np.int32), np.zeros(nnz))
            out[name] = a
            setattr(ex, name + "_ptr", a[0].ctypes.data)
            setattr(ex, name + "_col", a[1].ctypes.data)
            setattr(ex, name + "_val", a[2].ctypes.data)

        csr("A", nloc, inf["nnz_A"])
        if inf["nnz_P"] or inf["nnz_R"] or ncr:
            csr("P", nloc, inf["nnz_P"])
            csr("R", ncr, inf["nnz_R"])
        arrs = {"ghost_global": np.zeros(inf["ghosts"], np.int64),
                "recv_peer": np.zeros(inf["recv_peers"], np.int32),
                "recv_off": np.zeros(inf["recv_peers"], np.int64),
                "recv_cnt": np.zeros(inf["recv_peers"], np.int64),
                "send_peer": np.zeros(inf["send_peers"], np.int32),
                "send_off": np.zeros(inf["send_peers"], np.int64),
                "send_cnt": np.zeros(inf["send_peers"], np.int64),
                "send_idx": np.zeros(inf["send_total"], np.int32)}
        for k, a in arrs.items():
            setattr(ex, k, a.ctypes.data if a.size else None)
            out[k] = a
        _check(_lib.amg_dist_export(self._h, rank, l, C.byref(ex)), "amg_dist_export")
        return out

    # ---- device operations ---------------------------------------------
    def _sync_stream(self):
        if not self.on_device:
            return  # the library reports AMG_E_NO_DEVICE
        import torch
        s = torch.cuda.current_stream(self.device).cuda_stream
        _check(_lib.amg_set_stream(self._h, s), "amg_set_stream")

    def solve(self, f, x=None, tol=1e-8, maxiter=100):
        """Solve A x = f on the GPU; f, x are CUDA float64 tensors (x: initial
        guess, overwritten).  Returns (x, iters, rel_resid, status)."""
        import torch
        _dev_vec(f, self.vec_len, "f")
        if x is None:
            x = torch.zeros_like(f)
        _dev_vec(x, self.vec_len, "x")
        self._sync_stream()
        it, rel = C.c_int32(), C.c_double()
        st = _check(_lib.amg_solve(self._h, _ptr(f), _ptr(x), tol, maxiter, C.byref(it), C.byref(rel)),
                    "amg_solve")
        return x, it.value, rel.value, st

    def solve_batched(self, F, X=None, tol=1e-8, maxiter=100):
        """Solve A x_j = f_j for the k rows of the CUDA float64 tensor F (shape
        (k, n), each right-hand side contiguous).  Returns (X, iters[k],
        rel_resid[k], status)."""
        import torch
        F = F.contiguous()
        k, n = F.shape
        if X is None:
            X = torch.zeros_like(F)
        self._sync_stream()
        it = np.zeros(k, np.int32)
        rel = np.zeros(k)
        st = _check(_lib.amg_solve_batched(self._h, k, _ptr(F), n, _ptr(X), n, tol, maxiter, it.ctypes.data,
                                           rel.ctypes.data), "amg_solve_batched")
        return X, it, rel, st

    def solve_host(self, f: np.ndarray, x0: np.ndarray | None = None, tol=1e-8, maxiter=100,
                   out: np.ndarray | None = None):
        """End-to-end solve with HOST arrays (copies inside the library call).
        x0 = None: zero initial guess (not copied).  out: solution buffer."""
        n = self.vec_len
        f = _host_vec(np.ascontiguousarray(f, np.float64), n, "f")
        if out is None:
            out = np.empty_like(f)
        _host_vec(out, n, "out")
        x0 = None if x0 is None else _host_vec(np.ascontiguousarray(x0, np.float64), n, "x0")
        x0p = None if x0 is None else _ptr(x0)
        self._sync_stream()
        it, rel = C.c_int32(), C.c_double()
        st = _check(_lib.amg_solve_host(self._h, _ptr(f), x0p, _ptr(out), tol, maxiter, C.byref(it),
                                        C.byref(rel)), "amg_solve_host")
        return out, it.value, rel.value, st

    def solve_host_stream(self, fs, xs=None, tol=1e-8, maxiter=100):
        """amg_solve_host_stream: k independent solves from zero initial guesses
        with HOST arrays; the copies of system j+1's f and system j-1's x overlap
        the solve of system j (use pinned buffers for the overlap).  fs / xs:
        sequences of float64 arrays (entries may repeat).  Returns (xs, iters,
        rels, vcycles, status of the first non-OK solve)."""
        n = self.vec_len
        fs = [_host_vec(np.ascontiguousarray(f, np.float64), n, f"fs[{j}]") for j, f in enumerate(fs)]
        k = len(fs)
        if xs is None:
            xs = [np.empty_like(f) for f in fs]
        if len(xs) != k:
            raise ValueError(f"xs: {len(xs)} arrays for {k} right-hand sides")
        for j, x in enumerate(xs):
            _host_vec(x, n, f"xs[{j}]")
        fp = (C.c_void_p * max(k, 1))(*[_ptr(f) for f in fs])
        xp = (C.c_void_p * max(k, 1))(*[_ptr(x) for x in xs])
        it = (C.c_int32 * max(k, 1))()
        rel = (C.c_double * max(k, 1))()
        vc = (C.c_int32 * max(k, 1))()
        self._sync_stream()
        st = _check(_lib.amg_solve_host_stream(self._h, k, C.cast(fp, _V), C.cast(xp, _V), tol, maxiter,
                                               C.cast(it, _V), C.cast(rel, _V), C.cast(vc, _V)),
                    "amg_solve_host_stream")
        return xs, list(it)[:k], list(rel)[:k], list(vc)[:k], st

    def precond(self, r, z=None):
        """z = M r: one V-cycle from zero (asynchronous on the current stream)."""
        import torch
        _dev_vec(r, self.vec_len, "r")
        if z is None:
            z = torch.empty_like(r)
        _dev_vec(z, self.vec_len, "z")
        self._sync_stream()
        _check(_lib.amg_precond_apply(self._h, _ptr(r), _ptr(z)), "amg_precond_apply")
        return z

    def level_op(self, l: int, op: int, x=None, f=None, y=None, ny=None):
        """Test hook (amg_level_op); y is allocated if not given."""
        import torch
        if y is None:
            y = torch.empty(ny, dtype=torch.float64, device=self.device)
        self._sync_stream()
        _check(_lib.amg_level_op(self._h, l, op, _ptr(x) if x is not None else None,
                                 _ptr(f) if f is not None else None, _ptr(y)), "amg_level_op")
        return y

    def level_op_ex(self, l: int, op: int, in0=None, in1=None, out0=None, out1=None, out2=None,
                    scalar: float = 0.0) -> float:
        """Test hook (amg_level_op_ex): one fused production kernel on CUDA
        float64 tensors; returns the fused dot (0.0 if the op has none)."""
        a = LevelOpArgs()
        for k, v in (("in0", in0), ("in1", in1), ("out0", out0), ("out1", out1), ("out2", out2)):
            setattr(a, k, _ptr(v) if v is not None else None)
        a.scalar = scalar
        self._sync_stream()
        _check(_lib.amg_level_op_ex(self._h, l, op, C.byref(a)), "amg_level_op_ex")
        return a.dot

    def set_profile(self, mask: int):
        """Time kernel classes (bit c = PROF_CLASSES[c]) with CUDA events; 0 = off."""
        _check(_lib.amg_set_profile(self._h, int(mask)), "amg_set_profile")

    def stats(self) -> dict:
        s = SolveStats()
        _check(_lib.amg_solve_stats_get(self._h, C.byref(s)), "amg_solve_stats_get")
        d = {k: getattr(s, k) for k, _ in SolveStats._fields_ if k != "reserved"}
        for k in ("prof_ms", "prof_bytes", "prof_launches"):
            d[k] = list(d[k])[:len(PROF_CLASSES)]
        return d


def setup(ptr, col, val, params: dict | None = None, **kw) -> Hierarchy:
    """amg_setup: build (host) and upload (GPU) the AMG hierarchy of A."""
    return Hierarchy(ptr, col, val, params, **kw)


def nccl_unique_id() -> bytes:
    """amg_nccl_unique_id (rank 0 of a multi-GPU run)."""
    buf = (C.c_uint8 * 128)()
    _check(_lib.amg_nccl_unique_id(C.cast(buf, C.c_void_p)), "amg_nccl_unique_id")
    return bytes(buf)


def shm_selftest(tag: bytes, rank: int, nranks: int) -> None:
    """amg_shm_selftest: the host shared-memory test transport (no GPU)."""
    buf = (C.c_uint8 * 128)(*tag[:128].ljust(128, b"\0"))
    _check(_lib.amg_shm_selftest(C.cast(buf, C.c_void_p), rank, nranks), "amg_shm_selftest")


def nccl_selftest(device: int = 0) -> None:
    """amg_nccl_selftest: the NCCL calls of the multi-GPU executor on a 1-rank comm."""
    _check(_lib.amg_nccl_selftest(device), "amg_nccl_selftest")


def setup_dist(ptr, col, val, nranks: int, rank: int = -1, gather_below: int = 0,
               nccl_id: bytes | None = None, params: dict | None = None, n: int | None = None,
               **kw) -> Hierarchy:
    """amg_setup_dist: row-partitioned hierarchy (rank = -1: every rank in this
    process on one GPU; rank >= 0: one NCCL rank per process -- rank 0 builds the
    hierarchy and sends every rank its part, so ranks > 0 may pass ptr = col =
    val = None and the global row count n)."""
    d = AmgDist()
    d.nranks, d.rank, d.gather_below = nranks, rank, gather_below
    if nccl_id is not None:
        for i, b in enumerate(nccl_id[:128]):
            d.nccl_id[i] = b
    return Hierarchy(ptr, col, val, params, dist=d, n=n, **kw)
