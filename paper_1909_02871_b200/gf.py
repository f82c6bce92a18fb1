"""Thin Python binding of the C ABI in include/gfrlnc.h (ctypes).

Argument marshalling only: dtype / device / contiguity checks, the current
torch stream handed to gf_set_stream, and raw pointers.  Every step of the
computation runs in the sm_100a kernels of libgfrlnc.so; there is no CPU
fallback -- if the library is missing, importing this module raises.

Names follow the C ABI: init, maddrc, mulrc, encode_batch (Eq. 2,
PAPER.md:84-88), encode_batch_host, plus the harness-only fill_random /
fill_random2d / host_tables.
"""
from __future__ import annotations

import ctypes
import os
import threading

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgfrlnc.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} not built: run `python -m paper_1909_02871_b200.build` "
        "(or __graft_entry__.build()); there is no fallback path")

_lib = ctypes.CDLL(LIB_PATH)

_u8p = ctypes.c_void_p
_sz = ctypes.c_size_t
_u64 = ctypes.c_uint64

_lib.gf_init.argtypes = [ctypes.c_int]
_lib.gf_maddrc.argtypes = [ctypes.c_int, _u8p, _u8p, ctypes.c_uint8, _sz]
_lib.gf_mulrc.argtypes = [ctypes.c_int, _u8p, ctypes.c_uint8, _sz]
_lib.gf_encode_batch.argtypes = [ctypes.c_int, _u8p, _u8p, _u8p, ctypes.c_int, ctypes.c_int, _sz, _sz]
_lib.gf_encode_batch_host.argtypes = [ctypes.c_int, _u8p, _u8p, _u8p, ctypes.c_int, ctypes.c_int,
                                      _sz, _sz, _u8p, _sz]
_lib.gf_set_stream.argtypes = [ctypes.c_void_p]
_lib.gf_strerror.argtypes = [ctypes.c_int]
_lib.gf_strerror.restype = ctypes.c_char_p
_lib.gf_fill_random.argtypes = [_u8p, _sz, _u64, _u64, _u64, ctypes.c_uint8]
_lib.gf_fill_random2d.argtypes = [_u8p, _sz, _sz, _u64, _u64, _u64, _u64, ctypes.c_uint8]
_lib.gf_host_tables.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_uint32), _sz]
_lib.gf_version.argtypes = []
_lib.gf_set_encode_path.argtypes = [ctypes.c_int]
_lib.gf_encode_path.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, _sz, _sz, _sz]
_lib.gf_verify_batch.argtypes = [ctypes.c_int, _u8p, _u8p, _u8p, _u8p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                 _sz, _sz, ctypes.c_void_p, _u8p, _sz]
_lib.gf_encode_verify_batch.argtypes = [ctypes.c_int, _u8p, _u8p, _u8p, _u8p, ctypes.c_int, ctypes.c_int,
                                        ctypes.c_int, _sz, _sz, ctypes.c_void_p, _u8p, _sz]
_lib.gf_set_verify_fault.argtypes = [ctypes.c_int, _sz, ctypes.c_int, _sz]
_lib.gf_invert_batch.argtypes = [ctypes.c_int, _u8p, _u8p, ctypes.c_void_p, ctypes.c_int, _sz]
_lib.gf_decode_batch.argtypes = [ctypes.c_int, _u8p, _u8p, _u8p, ctypes.c_void_p, ctypes.c_int, _sz, _sz,
                                 _u8p, _sz]

GF_OK, GF_EFIELD, GF_ECOEFF, GF_EARG, GF_EOVERLAP, GF_ENOINIT, GF_ECUDA = 0, -1, -2, -3, -4, -5, -6
FIELDS = (2, 4, 16, 256)
TABLE_WORDS = 16          # uint32 words per coefficient in gf_host_tables

# every symbol include/gfrlnc.h declares (tests check the library exports them)
ABI_SYMBOLS = ("gf_init", "gf_maddrc", "gf_mulrc", "gf_encode_batch", "gf_encode_batch_host",
               "gf_set_stream", "gf_strerror", "gf_fill_random", "gf_fill_random2d",
               "gf_host_tables", "gf_version", "gf_encode_path", "gf_invert_batch", "gf_decode_batch",
               "gf_verify_batch", "gf_set_encode_path", "gf_encode_verify_batch", "gf_set_verify_fault")


class GFError(RuntimeError):
    def __init__(self, status: int, what: str):
        self.status = status
        super().__init__(f"{what}: {strerror(status)} ({status})")


def lib() -> ctypes.CDLL:
    """The raw C ABI.  A caller may set the stream itself through it, so the
    binding's cached copy of this thread's stream is dropped."""
    _tls.stream = None
    return _lib


def strerror(status: int) -> str:
    return _lib.gf_strerror(status).decode()


def version() -> int:
    return _lib.gf_version()


ENCODE_PATHS = {0: "column-words", 1: "column-bytes", 2: "lanek-32", 3: "lanek-64", 6: "prow", 8: "stream",
                9: "prow-32", 10: "prow-16", 11: "gf2-split", 12: "prow-nib",
                13: "prow-32w", 14: "tmem"}


# gf_set_encode_path codes (include/gfrlnc.h GF_PATH_*)
FORCE_PATHS = {"auto": 0, "column": 1, "lanek": 2, "prow": 4, "stream": 6, "gf2": 7,
               "stream-strided4": 8, "stream-strided8": 9, "stream-strided12": 10,
               "stream-wide2": 11, "stream-wide4": 12, "tmem": 13}


def set_encode_path(name: str) -> None:
    """Harness-only: force the encode kernel of this thread's encode calls
    (thread-local; "auto" restores the router)."""
    _check(_lib.gf_set_encode_path(FORCE_PATHS[name]), "gf_set_encode_path")


def encode_path(field: int, N: int, K: int, M: int, a_align: int = 0, b_align: int = 0) -> str:
    """Name of the encode kernel gf_encode_batch picks (host-only query)."""
    rc = _lib.gf_encode_path(field, N, K, M, a_align, b_align)
    if rc < 0:
        raise GFError(rc, "gf_encode_path")
    return ENCODE_PATHS[rc]


def _check(rc: int, what: str) -> None:
    if rc != GF_OK:
        raise GFError(rc, what)


def _dev_u8(t: torch.Tensor, name: str) -> int:
    if not isinstance(t, torch.Tensor) or t.dtype != torch.uint8:
        raise TypeError(f"{name} must be a torch.uint8 tensor")
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t.data_ptr()


def _host_u8(t: torch.Tensor, name: str) -> int:
    if not isinstance(t, torch.Tensor) or t.dtype != torch.uint8:
        raise TypeError(f"{name} must be a torch.uint8 tensor")
    if t.is_cuda:
        raise ValueError(f"{name} must be a host tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t.data_ptr()


def _coeff(c: int) -> int:
    c = int(c)
    if not 0 <= c < 256:
        raise GFError(GF_ECOEFF, f"coefficient {c} does not fit a byte")
    return c


# the raw current-stream pointer without building a torch.cuda.Stream object
# (torch.cuda.current_stream costs about a microsecond per call)
_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)
_tls = threading.local()


def _use_stream(device: torch.device) -> None:
    """Hand torch's current stream of `device` to the library (gf_set_stream is
    thread-local on both sides; the call is skipped while it is unchanged)."""
    idx = device.index if device.index is not None else torch.cuda.current_device()
    s = _raw_stream(idx) if _raw_stream is not None else torch.cuda.current_stream(device).cuda_stream
    if getattr(_tls, "stream", None) != s:
        _lib.gf_set_stream(s)
        _tls.stream = s


class _on_device:
    """Make `device` current for the call (cheap no-op when it already is)."""
    __slots__ = ("idx", "prev")

    def __init__(self, device: torch.device):
        self.idx = device.index

    def __enter__(self):
        self.prev = torch.cuda.current_device()
        if self.idx is None:
            self.idx = self.prev
        elif self.prev != self.idx:
            torch.cuda.set_device(self.idx)
        return self

    def __exit__(self, *exc):
        if self.prev != self.idx:
            torch.cuda.set_device(self.prev)
        return False


def init(field: int, device=None) -> None:
    """gf_init(field) on `device` (default: current device)."""
    with torch.cuda.device(device if device is not None else torch.cuda.current_device()):
        _check(_lib.gf_init(field), f"gf_init({field})")


def maddrc(field: int, dst: torch.Tensor, src: torch.Tensor, coeff: int) -> torch.Tensor:
    """dst += coeff * src in place over F_field. Returns dst."""
    pd, ps = _dev_u8(dst, "dst"), _dev_u8(src, "src")
    if dst.numel() != src.numel():
        raise ValueError("dst and src must have the same number of bytes")
    with _on_device(dst.device):
        _use_stream(dst.device)
        _check(_lib.gf_maddrc(field, pd, ps, _coeff(coeff), dst.numel()), "gf_maddrc")
    return dst


def mulrc(field: int, dst: torch.Tensor, coeff: int) -> torch.Tensor:
    """dst = coeff * dst in place. Returns dst."""
    pd = _dev_u8(dst, "dst")
    with _on_device(dst.device):
        _use_stream(dst.device)
        _check(_lib.gf_mulrc(field, pd, _coeff(coeff), dst.numel()), "gf_mulrc")
    return dst


def encode_batch(field: int, A: torch.Tensor, C: torch.Tensor, B: torch.Tensor | None = None,
                 checked: bool = False) -> torch.Tensor:
    """B[g,k,m] = sum_i C[g,i,k] * A[g,i,m] over F_field (Eq. 2).

    A: uint8 [batch, N, M], C: uint8 [batch, N, K] on one CUDA device.
    B (optional, [batch, K, M]) is overwritten and returned.  checked=True
    verifies C < field first (one device reduction); otherwise entries of C
    are taken modulo the field size by masking, as the ABI documents."""
    if A.dim() != 3 or C.dim() != 3 or A.shape[:2] != C.shape[:2]:
        raise ValueError("expected A [batch, N, M] and C [batch, N, K]")
    batch, N, M = A.shape
    K = C.shape[2]
    if B is None:
        B = torch.empty((batch, K, M), dtype=torch.uint8, device=A.device)
    elif tuple(B.shape) != (batch, K, M):
        raise ValueError(f"B must have shape {(batch, K, M)}")
    pa, pc, pb = _dev_u8(A, "A"), _dev_u8(C, "C"), _dev_u8(B, "B")
    if checked and C.numel() and int(C.max()) >= field:
        raise GFError(GF_ECOEFF, "encode_batch(checked)")
    with _on_device(A.device):
        _use_stream(A.device)
        _check(_lib.gf_encode_batch(field, pa, pc, pb, N, K, M, batch), "gf_encode_batch")
    return B


def invert_batch(field: int, C: torch.Tensor):
    """D[g] = C[g]^{-1} over F_field for C uint8 [batch, N, N]; returns (D, rank)
    with rank an int32 tensor (D[g] unspecified where rank[g] < N)."""
    if C.dim() != 3 or C.shape[1] != C.shape[2]:
        raise ValueError("expected C [batch, N, N]")
    batch, N, _ = C.shape
    D = torch.empty_like(C)
    rank = torch.empty(batch, dtype=torch.int32, device=C.device)
    pc, pd = _dev_u8(C, "C"), _dev_u8(D, "D")
    with _on_device(C.device):
        _use_stream(C.device)
        _check(_lib.gf_invert_batch(field, pc, pd, rank.data_ptr(), N, batch), "gf_invert_batch")
    return D, rank


def decode_batch(field: int, B: torch.Tensor, C: torch.Tensor, workspace: torch.Tensor | None = None):
    """Sources A [batch, N, M] from N coded packets B [batch, N, M] and their
    coding vectors C [batch, N, N] (encode layout); returns (A, rank)."""
    if B.dim() != 3 or C.dim() != 3 or C.shape[1] != C.shape[2] or B.shape[:2] != C.shape[:2]:
        raise ValueError("expected B [batch, N, M] and C [batch, N, N]")
    batch, N, M = B.shape
    A = torch.empty_like(B)
    rank = torch.empty(batch, dtype=torch.int32, device=B.device)
    if workspace is None:
        workspace = torch.empty(batch * N * N, dtype=torch.uint8, device=B.device)
    pb, pc, pa, pw = _dev_u8(B, "B"), _dev_u8(C, "C"), _dev_u8(A, "A"), _dev_u8(workspace, "workspace")
    with _on_device(B.device):
        _use_stream(B.device)
        _check(_lib.gf_decode_batch(field, pb, pc, pa, rank.data_ptr(), N, M, batch, pw, workspace.numel()),
               "gf_decode_batch")
    return A, rank


def verify_batch(field: int, A: torch.Tensor, C: torch.Tensor, B: torch.Tensor, R: torch.Tensor,
                 workspace: torch.Tensor | None = None) -> torch.Tensor:
    """Freivalds check of B == encode(A, C) on the device with projections
    R [batch, K, t]; returns mismatching byte counts per generation (int64)."""
    batch, N, M = A.shape
    K, t = R.shape[1], R.shape[2]
    if tuple(C.shape) != (batch, N, K) or tuple(B.shape) != (batch, K, M) or R.shape[0] != batch:
        raise ValueError("shape mismatch")
    need = batch * N * t + 2 * batch * t * M + 48
    if workspace is None:
        workspace = torch.empty(need, dtype=torch.uint8, device=A.device)
    mism = torch.empty(batch, dtype=torch.int64, device=A.device)
    ptrs = [_dev_u8(x, n) for x, n in ((A, "A"), (C, "C"), (B, "B"), (R, "R"), (workspace, "workspace"))]
    with _on_device(A.device):
        _use_stream(A.device)
        _check(_lib.gf_verify_batch(field, ptrs[0], ptrs[1], ptrs[2], ptrs[3], t, N, K, M, batch,
                                    mism.data_ptr(), ptrs[4], workspace.numel()), "gf_verify_batch")
    return mism


def freivalds_trials(field: int) -> int:
    """Projections per generation for gf_verify_batch so that a wrong byte
    survives all of them with probability <= q^-t <= 2^-20."""
    return {2: 20, 4: 10, 16: 5, 256: 3}[field]


def verify_workspace_bytes(N: int, K: int, batch: int) -> int:
    """Device workspace of gf_encode_verify_batch."""
    return ((batch * -(-K // 64) * 2 * N + 15) // 16) * 16 + batch * 2 * -(-K // 32) * 4


def encode_verify_batch(field: int, A: torch.Tensor, C: torch.Tensor, R: torch.Tensor,
                        B: torch.Tensor | None = None, workspace: torch.Tensor | None = None):
    """B = A C (as encode_batch) with the Freivalds check on binary
    projections r_j = R[g, :, j] & 1 (R: uint8 [batch, K, t], t in {1, 2});
    returns (B, mismatch) with mismatch an int64 tensor [batch] of differing
    projection bytes (0 when B == A C; include/gfrlnc.h)."""
    if A.dim() != 3 or C.dim() != 3 or R.dim() != 3 or A.shape[:2] != C.shape[:2]:
        raise ValueError("expected A [batch, N, M], C [batch, N, K], R [batch, K, t]")
    batch, N, M = A.shape
    K = C.shape[2]
    if tuple(R.shape[:2]) != (batch, K):
        raise ValueError(f"R must have shape ({batch}, {K}, t)")
    t = R.shape[2]
    if B is None:
        B = torch.empty((batch, K, M), dtype=torch.uint8, device=A.device)
    elif tuple(B.shape) != (batch, K, M):
        raise ValueError(f"B must have shape {(batch, K, M)}")
    if workspace is None:
        workspace = torch.empty(verify_workspace_bytes(N, K, batch), dtype=torch.uint8, device=A.device)
    mism = torch.empty(batch, dtype=torch.int64, device=A.device)
    ptrs = [_dev_u8(x, n) for x, n in ((A, "A"), (C, "C"), (B, "B"), (R, "R"), (workspace, "workspace"))]
    with _on_device(A.device):
        _use_stream(A.device)
        _check(_lib.gf_encode_verify_batch(field, ptrs[0], ptrs[1], ptrs[2], ptrs[3], t, N, K, M, batch,
                                           mism.data_ptr(), ptrs[4], workspace.numel()), "gf_encode_verify_batch")
    return B, mism


def set_verify_fault(g: int = -1, k: int = 0, word: int = 0) -> None:
    """Harness-only: the calling thread's gf_encode_verify_batch calls corrupt
    one byte of coded packet k, word `word` of generation g (g < 0: off)."""
    if g < 0:
        _check(_lib.gf_set_verify_fault(0, 0, 0, 0), "gf_set_verify_fault")
    else:
        _check(_lib.gf_set_verify_fault(1, g, k, word), "gf_set_verify_fault")


def encode_batch_host(field: int, A: torch.Tensor, C: torch.Tensor, B: torch.Tensor,
                      workspace: torch.Tensor) -> torch.Tensor:
    """Encode from / to HOST tensors (pinned recommended) through a device
    workspace, overlapping copies and kernels; blocking.  The C entry point
    trusts the sizes it is given, so the shapes are checked here."""
    if A.dim() != 3 or C.dim() != 3 or B.dim() != 3:
        raise ValueError("expected A [batch, N, M], C [batch, N, K], B [batch, K, M]")
    batch, N, M = A.shape
    K = C.shape[2]
    if tuple(C.shape[:2]) != (batch, N) or tuple(B.shape) != (batch, K, M):
        raise ValueError(f"shape mismatch: A {tuple(A.shape)}, C {tuple(C.shape)}, B {tuple(B.shape)}")
    pa, pc, pb = _host_u8(A, "A"), _host_u8(C, "C"), _host_u8(B, "B")
    pw = _dev_u8(workspace, "workspace")
    with torch.cuda.device(workspace.device):
        _check(_lib.gf_encode_batch_host(field, pa, pc, pb, N, K, M, batch, pw, workspace.numel()),
               "gf_encode_batch_host")
    return B


def host_workspace_bytes(N: int, K: int, M: int, gens_per_chunk: int) -> int:
    """Device workspace for encode_batch_host with the given chunk size."""
    return 3 * gens_per_chunk * (N * M + N * K + K * M) + 144


# ---- harness-only --------------------------------------------------------------

def fill_random(dst: torch.Tensor, seed: int, stream: int, offset: int = 0, mask: int = 0xFF) -> torch.Tensor:
    """dst[j] = byte(seed, stream, offset + j) & mask (seeded_inputs definition)."""
    p = _dev_u8(dst, "dst")
    with _on_device(dst.device):
        _use_stream(dst.device)
        _check(_lib.gf_fill_random(p, dst.numel(), seed, stream, offset, mask), "gf_fill_random")
    return dst


def fill_random2d(dst: torch.Tensor, seed: int, stream: int, base: int, row_stride: int,
                  mask: int = 0xFF) -> torch.Tensor:
    """dst viewed as [rows, cols] (last dim = cols):
    dst[r, c] = byte(seed, stream, base + r * row_stride + c) & mask."""
    p = _dev_u8(dst, "dst")
    cols = dst.shape[-1] if dst.dim() else 1
    rows = dst.numel() // cols if cols else 0
    with _on_device(dst.device):
        _use_stream(dst.device)
        _check(_lib.gf_fill_random2d(p, rows, cols, seed, stream, base, row_stride, mask),
               "gf_fill_random2d")
    return dst


def host_tables(field: int):
    """The byte-permute tables gf_init uploads (host-only; no GPU needed):
    list of q entries, each TABLE_WORDS uint32 words (see include/gfrlnc.h)."""
    q = field
    buf = (ctypes.c_uint32 * (max(q, 1) * TABLE_WORDS))()
    _check(_lib.gf_host_tables(field, buf, len(buf)), "gf_host_tables")
    return [list(buf[TABLE_WORDS * c: TABLE_WORDS * (c + 1)]) for c in range(q)]
