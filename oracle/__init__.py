"""CPU oracle for arXiv 1909.02871's hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` legs may import this package.  The product package
(paper_1909_02871_b200) never imports it and shares no code with it.

Thin ctypes wrapper over oracle/gf_oracle.c (plain scalar C, -O2
-fno-tree-vectorize).  See that file's header for what each function follows in
PAPER.md.  Every function here is pinned by tests/test_oracle_*.py against
values the paper / SPEC fix, closed forms, field axioms and brute force.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gf_oracle.c")
_LIB = os.path.join(_HERE, "libgforacle.so")

FIELDS = (2, 4, 16, 256)


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain scalar code)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp"
        subprocess.check_call(["gcc", "-O2", "-fno-tree-vectorize", "-Wall", "-shared",
                               "-fPIC", "-o", tmp, _SRC, "-lpthread"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        u8p = ctypes.POINTER(ctypes.c_uint8)
        sz = ctypes.c_size_t
        L.gfo_width.argtypes = [ctypes.c_int]
        L.gfo_poly.argtypes = [ctypes.c_int]
        L.gfo_poly.restype = ctypes.c_uint
        for f in (L.gfo_poly_mul, L.gfo_poly_mul_xtime, L.gfo_mulbyte):
            f.argtypes = [ctypes.c_int, ctypes.c_uint, ctypes.c_uint]
            f.restype = ctypes.c_uint
        L.gfo_inv.argtypes = [ctypes.c_int, ctypes.c_uint]
        L.gfo_inv.restype = ctypes.c_uint
        L.gfo_build_mb.argtypes = [ctypes.c_int, u8p]
        L.gfo_maddrc.argtypes = [ctypes.c_int, u8p, u8p, ctypes.c_uint, sz]
        L.gfo_mulrc.argtypes = [ctypes.c_int, u8p, ctypes.c_uint, sz]
        L.gfo_encode_gen_cols.argtypes = [ctypes.c_int, u8p, sz, u8p, u8p, ctypes.c_int,
                                          ctypes.c_int, sz, sz]
        L.gfo_encode_batch.argtypes = [ctypes.c_int, u8p, u8p, u8p, ctypes.c_int,
                                       ctypes.c_int, sz, sz]
        L.gfo_encode_batch_mt.argtypes = [ctypes.c_int, u8p, u8p, u8p, ctypes.c_int,
                                          ctypes.c_int, sz, sz, ctypes.c_int]
        L.gfo_freivalds_gen.argtypes = [ctypes.c_int, u8p, u8p, u8p, ctypes.c_int,
                                        ctypes.c_int, sz, u8p, u8p]
        L.gfo_freivalds_gen.restype = ctypes.c_long
        L.gfo_rref.argtypes = [ctypes.c_int, u8p, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.dtype == np.uint8 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))


def _check(rc):
    if rc != 0:
        raise ValueError(f"oracle call failed ({rc})")


# ---- scalar field ops ---------------------------------------------------------

def width(q: int) -> int:
    return lib().gfo_width(q)


def poly(q: int) -> int:
    return lib().gfo_poly(q)


def mul(q: int, a: int, b: int) -> int:
    """Element product, formulation 1 (shift-add then reduce)."""
    return lib().gfo_poly_mul(q, a, b)


def mul_xtime(q: int, a: int, b: int) -> int:
    """Element product, formulation 2 (reduce at every step)."""
    return lib().gfo_poly_mul_xtime(q, a, b)


def inv(q: int, a: int) -> int:
    return lib().gfo_inv(q, a)


def mulbyte(q: int, c: int, v: int) -> int:
    return lib().gfo_mulbyte(q, c, v)


def mul_table(q: int) -> np.ndarray:
    """Element product table T[a, b], a, b < q (formulation 1)."""
    L = lib()
    return np.array([[L.gfo_poly_mul(q, a, b) for b in range(q)] for a in range(q)],
                    dtype=np.uint8)


def mulbyte_table(q: int) -> np.ndarray:
    """MB[c, v] = c * v on packed bytes, shape (q, 256)."""
    MB = np.zeros(q * 256, dtype=np.uint8)
    _check(lib().gfo_build_mb(q, _p(MB)))
    return MB.reshape(q, 256)


# ---- region ops ---------------------------------------------------------------

def maddrc(q: int, dst: np.ndarray, src: np.ndarray, c: int) -> None:
    """dst ^= c * src in place."""
    assert dst.size == src.size
    _check(lib().gfo_maddrc(q, _p(dst), _p(src), c, dst.size))


def mulrc(q: int, dst: np.ndarray, c: int) -> None:
    """dst = c * dst in place."""
    _check(lib().gfo_mulrc(q, _p(dst), c, dst.size))


def encode_batch(q: int, A: np.ndarray, C: np.ndarray, threads: int = 1) -> np.ndarray:
    """B[g,k,m] = XOR_i C[g,i,k] * A[g,i,m]  (Eq. 2)."""
    A = np.ascontiguousarray(A, dtype=np.uint8)
    C = np.ascontiguousarray(C, dtype=np.uint8)
    batch, N, M = A.shape
    assert C.shape[:2] == (batch, N)
    K = C.shape[2]
    B = np.empty((batch, K, M), dtype=np.uint8)
    if batch and M:
        if threads > 1:
            _check(lib().gfo_encode_batch_mt(q, _p(A), _p(C), _p(B), N, K, M, batch, threads))
        else:
            _check(lib().gfo_encode_batch(q, _p(A), _p(C), _p(B), N, K, M, batch))
    return B


def encode_gen_cols(q: int, A_gen: np.ndarray, C_gen: np.ndarray, m0: int, m1: int) -> np.ndarray:
    """Columns [m0, m1) of one generation's coded packets; A_gen is (N, M)."""
    A_gen = np.ascontiguousarray(A_gen, dtype=np.uint8)
    C_gen = np.ascontiguousarray(C_gen, dtype=np.uint8)
    N, M = A_gen.shape
    K = C_gen.shape[1]
    out = np.empty((K, m1 - m0), dtype=np.uint8)
    if m1 > m0:
        _check(lib().gfo_encode_gen_cols(q, _p(A_gen), M, _p(C_gen), _p(out), N, K, m0, m1))
    return out


def freivalds_gen(q: int, A_gen: np.ndarray, C_gen: np.ndarray, B_gen: np.ndarray,
                  r: np.ndarray) -> int:
    """Number of byte positions where sum_i (C r)_i a_i != sum_k r_k b_k."""
    N, M = A_gen.shape
    K = C_gen.shape[1]
    scratch = np.empty(2 * M, dtype=np.uint8)
    r = np.ascontiguousarray(r, dtype=np.uint8)
    return lib().gfo_freivalds_gen(q, _p(np.ascontiguousarray(A_gen)),
                                   _p(np.ascontiguousarray(C_gen)),
                                   _p(np.ascontiguousarray(B_gen)), N, K, M, _p(r), _p(scratch))


def freivalds_trials(q: int) -> int:
    """Projections needed for an escape probability <= 2^-20 (q^-t)."""
    return {2: 20, 4: 10, 16: 5, 256: 3}[q]


def rref(q: int, Mx: np.ndarray, ecols: int | None = None) -> int:
    """In-place Gauss-Jordan; returns the rank of the first ecols columns."""
    assert Mx.dtype == np.uint8 and Mx.flags.c_contiguous and Mx.ndim == 2
    rows, cols = Mx.shape
    return lib().gfo_rref(q, _p(Mx), rows, cols, cols if ecols is None else ecols)


def rank(q: int, vectors: np.ndarray) -> int:
    Mx = np.ascontiguousarray(vectors, dtype=np.uint8).copy()
    return rref(q, Mx)


def decode(q: int, C_gen: np.ndarray, B_gen: np.ndarray):
    """Solve B = C^T A for A (K == N, C invertible): Gauss-Jordan on [C^T | B].
    Returns (rank, A or None)."""
    N, K = C_gen.shape
    M = B_gen.shape[1]
    aug = np.concatenate([np.ascontiguousarray(C_gen.T), B_gen], axis=1).astype(np.uint8)
    aug = np.ascontiguousarray(aug)
    rk = rref(q, aug, N)
    if rk < N:
        return rk, None
    return rk, aug[:N, N:].copy()
