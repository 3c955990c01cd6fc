"""Build/load the plain-C parts of the oracle (TEST INFRASTRUCTURE ONLY).

``build()`` compiles oracle/ilut.c + oracle/rcm_ref.c with gcc
(-O2 -ffp-contract=off: no FMA contraction, the arithmetic order is the
literal one) into oracle/liboracle.so.  Building the checker is not using it;
``__graft_entry__.build()`` calls this.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "liboracle.so")
SRCS = [os.path.join(HERE, "ilut.c"), os.path.join(HERE, "rcm_ref.c")]
_lib = None


def build(force: bool = False) -> str:
    newest = max(os.path.getmtime(s) for s in SRCS)
    if force or not os.path.exists(SO) or os.path.getmtime(SO) < newest:
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-o", SO, *SRCS, "-lm"]
        subprocess.check_call(cmd)
    return SO


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(SO)
        P64 = ctypes.POINTER(ctypes.c_int64)
        PD = ctypes.POINTER(ctypes.c_double)
        L.oracle_ilut.restype = ctypes.c_int
        L.oracle_ilut.argtypes = [ctypes.c_int64, P64, P64, PD, ctypes.c_double, ctypes.c_double,
                                  ctypes.POINTER(P64), ctypes.POINTER(P64), ctypes.POINTER(PD), P64,
                                  ctypes.POINTER(P64), ctypes.POINTER(P64), ctypes.POINTER(PD), P64]
        L.oracle_ilutp.restype = ctypes.c_int
        L.oracle_ilutp.argtypes = [ctypes.c_int64, P64, P64, PD, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                   ctypes.POINTER(P64), ctypes.POINTER(P64), ctypes.POINTER(PD), P64,
                                   ctypes.POINTER(P64), ctypes.POINTER(P64), ctypes.POINTER(PD), P64,
                                   ctypes.POINTER(P64)]
        L.oracle_rcm.restype = ctypes.c_int
        L.oracle_rcm.argtypes = [ctypes.c_int64, P64, P64, P64]
        L.oracle_free.restype = None
        L.oracle_free.argtypes = [ctypes.c_void_p]
        _lib = L
    return _lib
