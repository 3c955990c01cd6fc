"""ctypes binding of include/ss_b200.h (argument marshalling only).

Every step of the method runs inside libss_b200.so (CUDA kernels for sm_100a + the
host setup code of the same library).  This module only converts Python objects to
the C ABI: there is no fallback -- if the library or a CUDA device is missing, the
calls raise.
"""
from __future__ import annotations

import ctypes
import math
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libss_b200.so")

SS_OK = 0
ERR_NAMES = {1: "SS_ERR_ARG", 2: "SS_ERR_CUDA", 3: "SS_ERR_OOM", 4: "SS_ERR_BREAKDOWN", 5: "SS_ERR_STATE"}


class SSError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERR_NAMES.get(code, code)}: {msg}")
        self.code = code


class ss_params(ctypes.Structure):
    _fields_ = [("N_c", ctypes.c_int32), ("N_m", ctypes.c_int32), ("omega_m", ctypes.c_double),
                ("Delta", ctypes.c_double), ("kappa", ctypes.c_double), ("g0", ctypes.c_double),
                ("E", ctypes.c_double), ("Gamma_m", ctypes.c_double), ("n_th", ctypes.c_double),
                ("w", ctypes.c_double)]


class ss_build_info(ctypes.Structure):
    _fields_ = [("hilbert_dim", ctypes.c_int64), ("n", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("w_re", ctypes.c_double), ("w_im", ctypes.c_double), ("build_ms", ctypes.c_double)]


class ss_setup_info(ctypes.Structure):
    _fields_ = [("nnz_L", ctypes.c_int64), ("nnz_U", ctypes.c_int64), ("fill", ctypes.c_double),
                ("bandwidth_nat", ctypes.c_int64), ("bandwidth_rcm", ctypes.c_int64),
                ("levels_L", ctypes.c_int64), ("levels_U", ctypes.c_int64),
                ("pivots_repaired", ctypes.c_int32), ("pivot_swaps", ctypes.c_int32), ("pad0", ctypes.c_int32),
                ("threads", ctypes.c_int32),
                ("trsv_block", ctypes.c_int32), ("trsv_grid", ctypes.c_int32),
                ("trsv_q_L", ctypes.c_int32), ("trsv_q_U", ctypes.c_int32),
                ("rcm_ms", ctypes.c_double), ("ilut_ms", ctypes.c_double), ("upload_ms", ctypes.c_double)]


class ss_solve_info(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int32), ("cycles", ctypes.c_int32), ("converged", ctypes.c_int32),
                ("pad", ctypes.c_int32), ("rel_residual", ctypes.c_double), ("trace_re", ctypes.c_double),
                ("trace_im", ctypes.c_double), ("solve_ms", ctypes.c_double)]


def struct_dict(s) -> dict:
    return {k: getattr(s, k) for k, _ in s._fields_ if not k.startswith("pad")}


# (name, restype, argtypes) -- the exported symbols of include/ss_b200.h
P = ctypes.c_void_p
I32, I64, D = ctypes.c_int32, ctypes.c_int64, ctypes.c_double
PI64 = ctypes.POINTER(ctypes.c_int64)
PD = ctypes.POINTER(ctypes.c_double)
SIGNATURES = [
    ("ss_build", ctypes.c_int, [ctypes.POINTER(ss_params), P, ctypes.POINTER(P), ctypes.POINTER(ss_build_info)]),
    ("ss_setup", ctypes.c_int, [P, D, D, D, I32, ctypes.POINTER(ss_setup_info)]),
    ("ss_export_colperm", ctypes.c_int, [P, P]),
    ("ss_solve", ctypes.c_int, [P, I32, D, I32, ctypes.POINTER(ss_solve_info)]),
    ("ss_expect", ctypes.c_int, [P, PD, PD]),
    ("ss_get_rho", ctypes.c_int, [P, P, I32]),
    ("ss_solve_host", ctypes.c_int, [P, P, P, I32, D, I32, ctypes.POINTER(ss_solve_info)]),
    ("ss_destroy", None, [P]),
    ("ss_last_error", ctypes.c_char_p, []),
    ("ss_sizes", ctypes.c_int, [P, PI64, PI64, PI64, PI64]),
    ("ss_export_matrix", ctypes.c_int, [P, I32, P, P, P]),
    ("ss_export_perm", ctypes.c_int, [P, P]),
    ("ss_export_factors", ctypes.c_int, [P, I32, P, P, P]),
    ("ss_spmv", ctypes.c_int, [P, P, P]),
    ("ss_precond", ctypes.c_int, [P, I32, P, P]),
    ("ss_kernel_launches", ctypes.c_int64, []),
    ("ss_set_sm_budget", ctypes.c_int, [P, I32]),
    ("ss_debug_poison_smem", ctypes.c_int, [P]),
    ("ss_debug_trace_trsv", ctypes.c_int, [P, I32, P, P, P, PI64]),
    ("ss_ilutp_host", ctypes.c_int, [ctypes.c_int64, P, P, P, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                     I32, P, P, P, ctypes.c_int64, P, P, P, ctypes.c_int64, P]),
]

_lib = None


def load() -> ctypes.CDLL:
    """Load libss_b200.so (raises if it has not been built -- no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run __graft_entry__.build() "
                              "(make -C paper_1411_4356_b200/csrc); there is no CPU fallback")
        lib = ctypes.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        _lib = lib
    return _lib


def _check(rc: int):
    if rc != SS_OK:
        raise SSError(rc, load().ss_last_error().decode())


def _params(p) -> ss_params:
    w = p.w if p.w is not None else math.nan
    return ss_params(int(p.N_c), int(p.N_m), float(p.omega_m), float(p.Delta), float(p.kappa), float(p.g0),
                     float(p.E), float(p.Gamma_m), float(p.n_th), float(w))


# --------------------------------------------------------------------------- C-ABI names
def ss_build(p, stream: int = 0):
    """Returns (handle, info dict)."""
    h = P()
    info = ss_build_info()
    _check(load().ss_build(ctypes.byref(_params(p)), P(stream), ctypes.byref(h), ctypes.byref(info)))
    return h, struct_dict(info)


def ss_setup(h, drop_tol: float, fill_factor: float, permtol: float = 0.0, n_threads: int = 0) -> dict:
    info = ss_setup_info()
    _check(load().ss_setup(h, float(drop_tol), float(fill_factor), float(permtol), int(n_threads),
                           ctypes.byref(info)))
    return struct_dict(info)


def ss_export_colperm(h) -> np.ndarray:
    n = ss_sizes(h)["n"]
    perm = np.empty(n, np.int64)
    _check(load().ss_export_colperm(h, perm.ctypes.data))
    return perm


def ss_debug_poison_smem(h) -> None:
    """Fill every SM's shared memory with a NaN pattern (test hook, include/ss_b200.h)."""
    _check(load().ss_debug_poison_smem(h))


def ss_set_sm_budget(h, sms: int) -> None:
    _check(load().ss_set_sm_budget(h, int(sms)))


def ss_solve(h, restart: int, tol: float, max_iter: int) -> dict:
    info = ss_solve_info()
    _check(load().ss_solve(h, int(restart), float(tol), int(max_iter), ctypes.byref(info)))
    return struct_dict(info)


def ss_expect(h) -> tuple[float, float]:
    a, b = ctypes.c_double(), ctypes.c_double()
    _check(load().ss_expect(h, ctypes.byref(a), ctypes.byref(b)))
    return a.value, b.value


def ss_get_rho(h, dst_ptr: int, dst_is_device: bool):
    _check(load().ss_get_rho(h, P(dst_ptr), 1 if dst_is_device else 0))


def ss_solve_host(h, rhs_ptr: int | None, x_ptr: int, restart: int, tol: float, max_iter: int) -> dict:
    info = ss_solve_info()
    _check(load().ss_solve_host(h, P(rhs_ptr) if rhs_ptr else None, P(x_ptr), int(restart), float(tol),
                                int(max_iter), ctypes.byref(info)))
    return struct_dict(info)


def ss_destroy(h):
    if h:
        load().ss_destroy(h)


def ss_sizes(h) -> dict:
    v = [ctypes.c_int64() for _ in range(4)]
    _check(load().ss_sizes(h, *[ctypes.byref(x) for x in v]))
    return dict(n=v[0].value, nnz=v[1].value, nnz_L=v[2].value, nnz_U=v[3].value)


def ss_export_matrix(h, which: int):
    s = ss_sizes(h)
    n, nnz = s["n"], s["nnz"]
    rp = np.empty(n + 1, np.int64)
    ci = np.empty(nnz, np.int64)
    va = np.empty(nnz, np.complex128)
    _check(load().ss_export_matrix(h, int(which), rp.ctypes.data, ci.ctypes.data, va.ctypes.data))
    return rp, ci, va


def ss_export_perm(h) -> np.ndarray:
    n = ss_sizes(h)["n"]
    perm = np.empty(n, np.int64)
    _check(load().ss_export_perm(h, perm.ctypes.data))
    return perm


def ss_export_factors(h, which: int):
    s = ss_sizes(h)
    n, nz = s["n"], (s["nnz_L"] if which == 0 else s["nnz_U"])
    rp = np.empty(n + 1, np.int64)
    ci = np.empty(max(nz, 0), np.int64)
    va = np.empty(max(nz, 0), np.complex128)
    _check(load().ss_export_factors(h, int(which), rp.ctypes.data, ci.ctypes.data, va.ctypes.data))
    return rp, ci, va


def ss_ilutp_host(rowptr, colidx, vals, drop_tol: float, fill_factor: float, permtol: float, threads: int = 0):
    """Host-only iLUTP (no GPU) of the CSR matrix (rowptr, colidx, vals): returns
    ((Lp, Lj, Lx), (Up, Uj, Ux), colperm) exactly as ss_setup computes them."""
    rp = np.ascontiguousarray(rowptr, np.int64)
    ci = np.ascontiguousarray(colidx, np.int64)
    va = np.ascontiguousarray(vals, np.complex128)
    n = rp.size - 1
    cap = int(np.sum(np.floor(fill_factor * np.diff(rp) / 2.0)))   # rule R5
    Lp, Up = np.empty(n + 1, np.int64), np.empty(n + 1, np.int64)
    Lj, Lx = np.empty(max(cap, 1), np.int64), np.empty(max(cap, 1), np.complex128)
    Uj, Ux = np.empty(cap + n, np.int64), np.empty(cap + n, np.complex128)
    cp = np.empty(n, np.int64)
    _check(load().ss_ilutp_host(n, rp.ctypes.data, ci.ctypes.data, va.ctypes.data, float(drop_tol),
                                float(fill_factor), float(permtol), int(threads), Lp.ctypes.data, Lj.ctypes.data,
                                Lx.ctypes.data, max(cap, 1), Up.ctypes.data, Uj.ctypes.data, Ux.ctypes.data,
                                cap + n, cp.ctypes.data))
    return (Lp, Lj[:Lp[n]], Lx[:Lp[n]]), (Up, Uj[:Up[n]], Ux[:Up[n]]), cp


def ss_spmv(h, x_dev_ptr: int, y_dev_ptr: int):
    _check(load().ss_spmv(h, P(x_dev_ptr), P(y_dev_ptr)))


def ss_precond(h, which: int, x_dev_ptr: int, y_dev_ptr: int):
    _check(load().ss_precond(h, int(which), P(x_dev_ptr), P(y_dev_ptr)))


TRACE_STAMPS = 16   # SS_TRACE_STAMPS


def ss_debug_trace_trsv(h, which: int, x_dev_ptr: int, y_dev_ptr: int) -> np.ndarray:
    """Per-block globaltimer stamps (ns), shape (nblk, TRACE_STAMPS); see include/ss_b200.h."""
    nb = ctypes.c_int64()
    _check(load().ss_debug_trace_trsv(h, int(which), P(x_dev_ptr), P(y_dev_ptr), None, ctypes.byref(nb)))
    tr = np.empty((nb.value, TRACE_STAMPS), np.uint64)
    _check(load().ss_debug_trace_trsv(h, int(which), P(x_dev_ptr), P(y_dev_ptr), tr.ctypes.data, ctypes.byref(nb)))
    return tr


def ss_kernel_launches() -> int:
    return int(load().ss_kernel_launches())
