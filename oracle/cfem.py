"""Oracle: ctypes loader of the plain-C element-loop force (oracle/cfem.c).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  `internal_force_c` computes exactly the
definition of fem.internal_force (f = sum_e scatter(K_e u_e)) with an element loop in C
(8-coloured OpenMP, deterministic); it is pinned by the same tests as the NumPy loop
(tests/test_oracle_fem.py: brute-force assembled K, rigid modes, patch test, NumPy equality).
Built by __graft_entry__.build() (`gcc -O2 -fopenmp`) into oracle/liboracle_fem.so.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle_fem.so")
SRC_PATH = os.path.join(_HERE, "cfem.c")
_lib = None


def build(cc: str = "gcc", force: bool = False) -> str:
    """Compile cfem.c unless the library is newer than the source; the new file replaces the old one by rename,
    so a process that has the old library mapped keeps running."""
    if not force and os.path.exists(LIB_PATH) and os.path.getmtime(LIB_PATH) >= os.path.getmtime(SRC_PATH):
        return LIB_PATH
    tmp = f"{LIB_PATH}.{os.getpid()}.tmp"
    subprocess.run([cc, "-O2", "-fopenmp", "-fPIC", "-shared", "-o", tmp, SRC_PATH], check=True)
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


def available() -> bool:
    return os.path.exists(LIB_PATH)


def _load():
    global _lib
    if _lib is None:
        if not available():
            build()
        lib = ctypes.CDLL(LIB_PATH)
        lib.oracle_internal_force.argtypes = [ctypes.c_int32] * 3 + [ctypes.c_void_p] * 3
        lib.oracle_internal_force.restype = None
        lib.oracle_set_threads.argtypes = [ctypes.c_int32]
        lib.oracle_set_threads.restype = None
        lib.oracle_get_threads.restype = ctypes.c_int32
        _lib = lib
    return _lib


def set_threads(n: int) -> int:
    """Threads of the C element loop (n <= 0: all processors); returns the count now in effect."""
    lib = _load()
    lib.oracle_set_threads(int(n))
    return int(lib.oracle_get_threads())


def internal_force_c(box, Ke: np.ndarray, u: np.ndarray) -> np.ndarray:
    """f (n_nodes, 3) = sum_e scatter(K_e u_e) for the box's structured hex8 mesh (element loop in C)."""
    lib = _load()
    Ke24 = np.ascontiguousarray(Ke.reshape(24, 24), dtype=np.float64)
    u = np.ascontiguousarray(u, dtype=np.float64).reshape(box.n_nodes, 3)
    f = np.empty_like(u)
    nx, ny, nz = box.nel
    lib.oracle_internal_force(nx, ny, nz, Ke24.ctypes.data, u.ctypes.data, f.ctypes.data)
    return f
