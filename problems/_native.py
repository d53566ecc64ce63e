"""Build/load the generator's C helper (problems/csrc/assemble.c) via gcc + ctypes."""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(_HERE, "csrc", "assemble.c")
LIB = os.path.join(_HERE, "libmgproblems.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-shared", "-fPIC",
                               "-o", tmp, SRC])
        os.replace(tmp, LIB)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB)
        P = ctypes.c_void_p
        L.asm_condensed.restype = ctypes.c_int
        L.asm_condensed.argtypes = [ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int64, P,
                                    P, P, P, ctypes.c_int, P, P, ctypes.c_int, ctypes.c_int, P, P, P]
        L.asm_structured.restype = ctypes.c_int
        L.asm_structured.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, P, P, ctypes.c_int,
                                     ctypes.c_int64, ctypes.c_int64, ctypes.c_int, P, P, P, P]
        L.tr_structured.restype = ctypes.c_int
        L.tr_structured.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, P, ctypes.c_int64,
                                    ctypes.c_int64, ctypes.c_int, P, P, P]
        _lib = L
    return _lib


def ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None
