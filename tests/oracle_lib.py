"""ctypes wrapper of oracle/_build/liboracle.so — TEST INFRASTRUCTURE ONLY
(the CPU checker; see oracle/numeric.c)."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "oracle", "_build", "liboracle.so")

_F = C.POINTER(C.c_float)


def _p(a):
    return a.ctypes.data_as(_F)


class Oracle:
    def __init__(self):
        if not os.path.exists(LIB):
            raise ImportError(f"{LIB} not built (run __graft_entry__.build())")
        self.lib = C.CDLL(LIB)
        L = self.lib
        L.oracle_input_value.restype = C.c_float
        L.oracle_input_value.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64]
        L.oracle_fill.argtypes = [_F, C.c_int64, C.c_uint64, C.c_uint32]
        L.oracle_axpy.argtypes = [_F, _F, _F, C.c_int64, C.c_float]
        L.oracle_outer.argtypes = [_F, _F, _F, C.c_int64, C.c_int64]
        L.oracle_matmul.argtypes = [_F, _F, _F, C.c_int64, C.c_int64, C.c_int64, C.c_int64]
        L.oracle_gemv.argtypes = [_F, _F, _F, C.c_int64, C.c_int64]
        L.oracle_batched.argtypes = [_F, _F, _F, C.c_int64, C.c_int64, C.c_int64, C.c_int64]
        dp = C.POINTER(C.c_double)
        L.oracle_gemv_f64.argtypes = [_F, _F, dp, dp, C.c_int64, C.c_int64]

    @staticmethod
    def tag(name: str) -> int:
        return ord(name[0])

    def fill(self, n: int, seed: int, name: str) -> np.ndarray:
        out = np.empty(n, dtype=np.float32)
        self.lib.oracle_fill(_p(out), n, seed, self.tag(name))
        return out

    def axpy(self, x, y, alpha):
        z = np.empty_like(x)
        self.lib.oracle_axpy(_p(x), _p(y), _p(z), x.size, alpha)
        return z

    def outer(self, a, b):
        c = np.empty(a.size * b.size, dtype=np.float32)
        self.lib.oracle_outer(_p(a), _p(b), _p(c), a.size, b.size)
        return c

    def matmul(self, a, b, m, n, k, s=1):
        c = np.empty(m * n, dtype=np.float32)
        self.lib.oracle_matmul(_p(a), _p(b), _p(c), m, n, k, s)
        return c

    def gemv(self, a, x, m, n):
        y = np.empty(m, dtype=np.float32)
        self.lib.oracle_gemv(_p(a), _p(x), _p(y), m, n)
        return y

    def gemv_f64(self, a, x, m, n):
        y = np.empty(m, dtype=np.float64)
        s = np.empty(m, dtype=np.float64)
        dp = C.POINTER(C.c_double)
        self.lib.oracle_gemv_f64(_p(a), _p(x), y.ctypes.data_as(dp), s.ctypes.data_as(dp), m, n)
        return y, s

    def batched(self, a, b, batch, m, n, k):
        c = np.empty(batch * m * n, dtype=np.float32)
        self.lib.oracle_batched(_p(a), _p(b), _p(c), batch, m, n, k)
        return c

    def expected(self, problem) -> dict[str, np.ndarray]:
        """Inputs and expected outputs of an ispc_problem (by region name)."""
        p = problem
        s = max(int(p.a_stride), 1)
        if p.kind == 0:
            x, y = self.fill(p.n, p.seed, "x"), self.fill(p.n, p.seed, "y")
            return {"z": self.axpy(x, y, p.alpha)}
        if p.kind == 1:
            a, b = self.fill(p.m, p.seed, "a"), self.fill(p.n, p.seed, "b")
            return {"c": self.outer(a, b)}
        if p.kind == 2:
            a, b = self.fill(p.m * p.k * s, p.seed, "a"), self.fill(p.k * p.n, p.seed, "b")
            return {"c": self.matmul(a, b, p.m, p.n, p.k, s)}
        if p.kind == 3:
            a, x = self.fill(p.m * p.n, p.seed, "a"), self.fill(p.n, p.seed, "x")
            return {"y": self.gemv(a, x, p.m, p.n)}
        if p.kind == 4:
            bt = max(int(p.batch), 1)
            a, b = self.fill(bt * p.m * p.k, p.seed, "a"), self.fill(bt * p.k * p.n, p.seed, "b")
            return {"c": self.batched(a, b, bt, p.m, p.n, p.k)}
        raise ValueError(p.kind)
