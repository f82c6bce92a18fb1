"""Seeded, synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO finite-field arithmetic.  It defines
  * the counter-based byte generator both sides use (a splitmix64 stream,
    addressable by absolute byte index, so any shard or generation can be
    regenerated on its own), in plain numpy;
  * the coefficient draws built on it (uniform over F_q by masking -- exact
    because q divides 256 -- and rejection draws for non-zero / non-trivial
    coefficients);
  * the BASELINE.json workloads C1..C5 (shapes, seeds, fields).

The CUDA side re-implements the same generator as a device kernel
(`gf_fill_random*` in paper_1909_02871_b200/csrc); a GPU test checks the two
byte streams are identical.  The paper itself draws coding coefficients
"identically and independently distributed from F_q" (Sec. II)
and encodes random payloads (Sec. V-A); it names no dataset, so
these synthetic inputs are the workload, not a stand-in.

Generator definition (the contract the device kernel must match):
    GAMMA = 0x9E3779B97F4A7C15          (splitmix64 Weyl increment)
    key(seed, stream) = seed XOR (stream * 0xD1B54A32D192ED03)   (mod 2^64)
    word(seed, stream, w) = mix64(key + (w + 1) * GAMMA)          (mod 2^64)
    byte(seed, stream, j) = (word(seed, stream, j >> 3) >> (8 * (j & 7))) & 0xFF
with mix64 the splitmix64 finaliser.  With key == 0 this is exactly the
reference splitmix64 sequence (pinned in tests/test_inputs.py).
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
import subprocess

import numpy as np

GAMMA = 0x9E3779B97F4A7C15
STREAM_MUL = 0xD1B54A32D192ED03
_M64 = (1 << 64) - 1

SEED_BASE = 190902871          # config Cn uses SEED_BASE + n
STREAM_A = 1                   # source packets A
STREAM_C = 2                   # coefficients C
STREAM_DST = 3                 # maddrc destination region
STREAM_SRC = 4                 # maddrc source region
STREAM_FREIVALDS = 5           # Freivalds projection vectors


def config_seed(n: int) -> int:
    return SEED_BASE + n


def stream_key(seed: int, stream: int) -> int:
    return (seed ^ ((stream * STREAM_MUL) & _M64)) & _M64


def _mix64(z: np.ndarray) -> np.ndarray:
    z = z.astype(np.uint64, copy=False)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def random_words(seed: int, stream: int, w0: int, n: int) -> np.ndarray:
    """64-bit words w0 .. w0+n-1 of the (seed, stream) sequence."""
    key = np.uint64(stream_key(seed, stream))
    idx = np.arange(w0 + 1, w0 + 1 + n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = key + idx * np.uint64(GAMMA)
    return _mix64(x)


# ---- the same stream in C (seeded_inputs/fill.c), multithreaded, for
# full-size host regeneration; pinned byte-equal to the numpy definition below
_HERE = os.path.dirname(os.path.abspath(__file__))
_CLIB = None


def _clib():
    global _CLIB
    if _CLIB is None:
        src, so = os.path.join(_HERE, "fill.c"), os.path.join(_HERE, "libsifill.so")
        if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
            tmp = so + f".{os.getpid()}.tmp"
            subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-pthread", "-o", tmp, src])
            os.replace(tmp, so)
        L = ctypes.CDLL(so)
        L.si_fill_2d.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_size_t, ctypes.c_uint64,
                                 ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint8, ctypes.c_int]
        _CLIB = L
    return _CLIB


def fill_2d(out: np.ndarray, seed: int, stream: int, base: int, row_stride: int, mask: int = 0xFF,
            threads: int | None = None) -> np.ndarray:
    """out (C-contiguous uint8, viewed as [rows, cols] with cols = last dim) :=
    byte(seed, stream, base + r*row_stride + c) & mask, computed by fill.c."""
    assert out.dtype == np.uint8 and out.flags.c_contiguous
    cols = out.shape[-1] if out.ndim else 1
    rows = out.size // cols if cols else 0
    if threads is None:
        threads = len(os.sched_getaffinity(0))
    _clib().si_fill_2d(out.ctypes.data, rows, cols, seed & _M64, stream & _M64, base, row_stride, mask, threads)
    return out


def random_bytes_np(seed: int, stream: int, offset: int, n: int) -> np.ndarray:
    """The numpy definition of random_bytes (reference for fill.c)."""
    if n <= 0:
        return np.zeros(0, dtype=np.uint8)
    w0 = offset >> 3
    w1 = (offset + n + 7) >> 3
    words = random_words(seed, stream, w0, w1 - w0)
    b = words.astype("<u8").view(np.uint8)
    s = offset - (w0 << 3)
    return b[s:s + n].copy()


def random_bytes(seed: int, stream: int, offset: int, n: int) -> np.ndarray:
    """Bytes offset .. offset+n-1 of the (seed, stream) byte stream (uint8)."""
    if n <= 0:
        return np.zeros(0, dtype=np.uint8)
    if n >= 4096:
        out = np.empty(n, dtype=np.uint8)
        return fill_2d(out, seed, stream, offset, n)
    w0 = offset >> 3
    w1 = (offset + n + 7) >> 3
    words = random_words(seed, stream, w0, w1 - w0)
    b = words.astype("<u8").view(np.uint8)
    s = offset - (w0 << 3)
    return b[s:s + n].copy()


def random_bytes_2d(seed: int, stream: int, base: int, row_stride: int,
                    rows: int, cols: int) -> np.ndarray:
    """out[r, c] = byte(base + r*row_stride + c): a byte-range slice of a
    row-major stream (used for byte-range shards and sampled columns)."""
    out = np.empty((rows, cols), dtype=np.uint8)
    if rows == 0 or cols == 0:
        return out
    if row_stride == cols:
        return random_bytes(seed, stream, base, rows * cols).reshape(rows, cols)
    return fill_2d(out, seed, stream, base, row_stride)


def uniform_coeffs(q: int, seed: int, stream: int, offset: int, n: int) -> np.ndarray:
    """n i.i.d. uniform elements of F_q (one byte each): byte & (q-1)."""
    return random_bytes(seed, stream, offset, n) & np.uint8(q - 1)


def rejection_coeffs(q: int, lo: int, seed: int, stream: int, n: int) -> np.ndarray:
    """n elements uniform over [lo, q): successive stream bytes masked to
    [0, q), values below lo rejected (sequential, exact)."""
    out = []
    j = 0
    while len(out) < n:
        chunk = random_bytes(seed, stream, j, 4096) & np.uint8(q - 1)
        j += 4096
        out.extend(int(v) for v in chunk if v >= lo)
    return np.asarray(out[:n], dtype=np.uint8)


# ---- BASELINE.json workloads ------------------------------------------------

@dataclasses.dataclass(frozen=True)
class EncodeConfig:
    name: str
    fields: tuple
    N: int
    K: int
    M: int
    batch: int
    seed: int
    nonzero_coeffs: bool = False   # C1: uniform over non-zero elements
    shard: str = "generation"      # "generation" or "bytes"

    def source_bytes(self) -> int:
        return self.N * self.M * self.batch

    def hbm_bytes(self) -> int:
        # read A, write B, read C (SURVEY.md 8(d) d.3 counting rule)
        return (self.N * self.M + self.K * self.M + self.N * self.K) * self.batch

    def byte_madds(self) -> int:
        return self.N * self.K * self.M * self.batch


C1 = EncodeConfig("C1", (256,), N=16, K=1, M=1500, batch=1, seed=config_seed(1),
                  nonzero_coeffs=True)
C3 = EncodeConfig("C3", (16, 256), N=64, K=64, M=1500, batch=65536, seed=config_seed(3))
C4 = EncodeConfig("C4", (256,), N=256, K=256, M=65536, batch=2048, seed=config_seed(4),
                  shard="bytes")
C5 = EncodeConfig("C5", (2, 4), N=32, K=32, M=1 << 20, batch=4096, seed=config_seed(5))
ENCODE_CONFIGS = {c.name: c for c in (C1, C3, C4, C5)}

# C2: gf_maddrc region sweep, sizes 64 B * 4^j, j = 0..11 (64 B .. 256 MiB)
C2_SEED = config_seed(2)
C2_FIELDS = (2, 4, 16, 256)
C2_SIZES = tuple(64 * 4 ** j for j in range(12))


def c2_coeff(q: int) -> int:
    """C2's seeded coefficient: uniform over the non-trivial range [2, q) for
    q > 2, and c = 1 for GF(2) (reading X12 in DESIGN.md)."""
    if q == 2:
        return 1
    return int(rejection_coeffs(q, 2, C2_SEED, STREAM_C + 16 * q, 1)[0])


def encode_inputs(cfg: EncodeConfig, q: int, g0: int = 0, g1: int | None = None,
                  m0: int = 0, m1: int | None = None):
    """Host copies of A[g0:g1, :, m0:m1] and C[g0:g1] for workload cfg over F_q,
    addressed by absolute index so any generation / byte range regenerates
    alone.  C1 uses the sequential non-zero draw for its 16 coefficients."""
    g1 = cfg.batch if g1 is None else g1
    m1 = cfg.M if m1 is None else m1
    seed = cfg.seed + 1000 * q
    G = g1 - g0
    A = random_bytes_2d(seed, STREAM_A, (g0 * cfg.N) * cfg.M + m0, cfg.M,
                        G * cfg.N, m1 - m0).reshape(G, cfg.N, m1 - m0)
    if cfg.nonzero_coeffs:
        allc = rejection_coeffs(q, 1, seed, STREAM_C, cfg.batch * cfg.N * cfg.K)
        C = allc.reshape(cfg.batch, cfg.N, cfg.K)[g0:g1].copy()
    else:
        C = uniform_coeffs(q, seed, STREAM_C, g0 * cfg.N * cfg.K,
                           G * cfg.N * cfg.K).reshape(G, cfg.N, cfg.K)
    return A, C


def field_seed(cfg: EncodeConfig, q: int) -> int:
    """Seed of workload cfg over F_q (each field gets its own stream family)."""
    return cfg.seed + 1000 * q
