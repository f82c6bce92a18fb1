"""GPU parity: the sm_100a kernels, called through the C ABI (ctypes binding),
against the CPU oracle on the same seeded inputs.  Bit-exact (integer work).

Inputs for the oracle always come from seeded_inputs on the host; the device
generator is only used where it was first shown equal to seeded_inputs
(test_device_rng_matches_host) and is then regenerated on the host for the
sampled outputs the oracle computes.
"""
import ctypes
import os

import numpy as np
import pytest
import torch

import oracle
import seeded_inputs as si

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu

FIELDS = (2, 4, 16, 256)


@pytest.fixture(scope="module")
def gfm():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1909_02871_b200 import gf
    torch.cuda.set_device(0)
    for q in FIELDS:
        gf.init(q)
    return gf


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


# ---- generator ------------------------------------------------------------------

@pytest.mark.parametrize("offset,n", [(0, 1), (0, 4096), (3, 1000), (8, 64), (13, 12345), (1 << 33, 777)])
def test_device_rng_matches_host(gfm, offset, n):
    t = torch.empty(n, dtype=torch.uint8, device="cuda")
    gfm.fill_random(t, 190902871, 1, offset)
    assert np.array_equal(t.cpu().numpy(), si.random_bytes(190902871, 1, offset, n))
    gfm.fill_random(t, 77, 2, offset, mask=15)
    assert np.array_equal(t.cpu().numpy(), si.random_bytes(77, 2, offset, n) & 15)


@pytest.mark.parametrize("rows,cols,base,stride", [(5, 64, 0, 64), (7, 24, 8, 4096), (3, 17, 5, 100),
                                                   (4, 8192, 16384, 65536)])
def test_device_rng_2d_matches_host(gfm, rows, cols, base, stride):
    t = torch.empty((rows, cols), dtype=torch.uint8, device="cuda")
    gfm.fill_random2d(t, 9, 1, base, stride)
    assert np.array_equal(t.cpu().numpy(), si.random_bytes_2d(9, 1, base, stride, rows, cols))


# ---- region ops -------------------------------------------------------------------

SIZES = (0, 1, 3, 15, 16, 17, 63, 64, 100, 1500, 4096 + 5, (1 << 20) + 7)


def coeffs_for(q):
    cs = {0, 1, q - 1, (q // 2) | 1}
    cs |= {int(c) for c in si.rejection_coeffs(q, 0, 5, 2, 3)}
    return sorted(c for c in cs if c < q)


@pytest.mark.parametrize("q", FIELDS)
def test_maddrc_parity_sizes_offsets_canaries(gfm, q):
    pad = 64
    for n in SIZES:
        for doff, soff in ((0, 0), (1, 0), (0, 3), (5, 9), (16, 4), (7, 7)):
            src_all = si.random_bytes(31, si.STREAM_SRC, 0, n + 2 * pad)
            dst_all = si.random_bytes(31, si.STREAM_DST, 0, n + 2 * pad)
            for c in coeffs_for(q):
                d = dev(dst_all)
                s = dev(src_all)
                gfm.maddrc(q, d[pad + doff: pad + doff + n], s[pad + soff: pad + soff + n], c)
                exp = dst_all.copy()
                seg = exp[pad + doff: pad + doff + n].copy()
                oracle.maddrc(q, seg, src_all[pad + soff: pad + soff + n].copy(), c)
                exp[pad + doff: pad + doff + n] = seg
                got = d.cpu().numpy()
                assert np.array_equal(got, exp), (n, doff, soff, c)   # includes canaries
                assert np.array_equal(s.cpu().numpy(), src_all)       # src untouched


@pytest.mark.parametrize("q", FIELDS)
def test_mulrc_parity(gfm, q):
    pad = 32
    for n in SIZES:
        for off in (0, 1, 6):
            base = si.random_bytes(41, si.STREAM_DST, 0, n + 2 * pad)
            for c in coeffs_for(q):
                d = dev(base)
                gfm.mulrc(q, d[pad + off: pad + off + n], c)
                exp = base.copy()
                seg = exp[pad + off: pad + off + n].copy()
                oracle.mulrc(q, seg, c)
                exp[pad + off: pad + off + n] = seg
                assert np.array_equal(d.cpu().numpy(), exp), (n, off, c)


@pytest.mark.parametrize("q", FIELDS)
def test_maddrc_exact_aliasing(gfm, q):
    a = si.random_bytes(43, 3, 0, 10007)
    for c in coeffs_for(q):
        t = dev(a)
        gfm.maddrc(q, t, t, c)                      # (1 + c) * a
        exp = a.copy()
        oracle.maddrc(q, exp, a.copy(), c)
        assert np.array_equal(t.cpu().numpy(), exp)


@pytest.mark.parametrize("q", FIELDS)
def test_c2_sweep_full_parity(gfm, q):
    """BASELINE.json configs[1]: every size 64 B .. 256 MiB, seeded c (X12)."""
    c = si.c2_coeff(q)
    for n in si.C2_SIZES:
        src = si.random_bytes(si.C2_SEED, si.STREAM_SRC, 0, n)
        dst = si.random_bytes(si.C2_SEED, si.STREAM_DST, 0, n)
        d = dev(dst)
        gfm.maddrc(q, d, dev(src), c)
        oracle.maddrc(q, dst, src, c)
        assert np.array_equal(d.cpu().numpy(), dst), n


def test_region_errors(gfm):
    L = gfm.lib()
    t = torch.zeros(256, dtype=torch.uint8, device="cuda")
    p = t.data_ptr()
    assert L.gf_maddrc(16, p, p + 128, 16, 64) == gfm.GF_ECOEFF
    assert L.gf_maddrc(4, p, p + 128, 4, 64) == gfm.GF_ECOEFF
    assert L.gf_mulrc(2, p, 2, 64) == gfm.GF_ECOEFF
    assert L.gf_maddrc(256, p, p + 8, 3, 64) == gfm.GF_EOVERLAP
    assert L.gf_maddrc(256, None, p, 3, 64) == gfm.GF_EARG
    assert L.gf_maddrc(256, None, None, 3, 0) == gfm.GF_OK
    assert L.gf_encode_batch(256, p, p, p + 64, 0, 1, 4, 1) == gfm.GF_EARG
    assert L.gf_encode_batch(256, p, p + 200, p + 8, 2, 2, 16, 1) == gfm.GF_EOVERLAP
    assert L.gf_encode_batch(256, p, p, p, 1, 1, 0, 5) == gfm.GF_OK


def test_not_initialised_in_fresh_process():
    import subprocess
    import sys
    code = ("import torch; from paper_1909_02871_b200 import gf; torch.cuda.init();"
            "t=torch.zeros(64,dtype=torch.uint8,device='cuda');"
            "L=gf.lib(); r=L.gf_maddrc(256,t.data_ptr(),t.data_ptr()+32,3,32);"
            "print(r); assert r == gf.GF_ENOINIT")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    subprocess.check_call([sys.executable, "-c", code])


# ---- encode -----------------------------------------------------------------------

def run_encode(gfm, q, A, C, **kw):
    return gfm.encode_batch(q, dev(A), dev(C), **kw).cpu().numpy()


def test_c1_full(gfm):
    """BASELINE.json configs[0]: GF(256), N=16 x 1500 B, K=1, non-zero c."""
    A, C = si.encode_inputs(si.C1, 256)
    assert np.array_equal(run_encode(gfm, 256, A, C), oracle.encode_batch(256, A, C))


@pytest.mark.parametrize("q", FIELDS)
@pytest.mark.parametrize("N,K,M,batch", [
    (1, 1, 1, 1), (1, 1, 4, 1), (3, 2, 5, 2), (16, 1, 1500, 3), (17, 33, 1500, 3),
    (64, 64, 1500, 4), (5, 7, 4096, 2), (2, 3, 130, 9), (32, 32, 4100, 2), (40, 17, 999, 2),
    (8, 5, 12, 17), (5, 24, 400, 3), (3, 40, 64, 5), (7, 65, 1540, 2), (1, 32, 8, 1),
    (33, 96, 3000, 2), (300, 260, 68, 2), (5, 520, 36, 2), (257, 3, 1500, 2), (9, 20, 1500, 3),
    (11, 12, 4096, 2)])
def test_encode_parity_shapes(gfm, q, N, K, M, batch):
    A = si.random_bytes(51 + N, si.STREAM_A, 0, batch * N * M).reshape(batch, N, M)
    C = si.uniform_coeffs(q, 52 + K, si.STREAM_C, 0, batch * N * K).reshape(batch, N, K)
    assert np.array_equal(run_encode(gfm, q, A, C), oracle.encode_batch(q, A, C))


@pytest.mark.parametrize("q", FIELDS)
def test_encode_unaligned_views(gfm, q):
    """Rows not 4-B aligned (byte path) and B at an odd address."""
    batch, N, K, M = 3, 6, 5, 64
    A = si.random_bytes(61, 1, 0, batch * N * M).reshape(batch, N, M)
    C = si.uniform_coeffs(q, 62, 2, 0, batch * N * K).reshape(batch, N, K)
    bufA = torch.zeros(A.size + 1, dtype=torch.uint8, device="cuda")
    bufA[1:] = dev(A.reshape(-1))
    bufB = torch.full((batch * K * M + 3,), 0xEE, dtype=torch.uint8, device="cuda")
    Av = bufA[1:].view(batch, N, M)
    Bv = bufB[1:-2].view(batch, K, M)
    gfm.encode_batch(q, Av, dev(C), Bv)
    got = bufB.cpu().numpy()
    assert np.array_equal(got[1:-2].reshape(batch, K, M), oracle.encode_batch(q, A, C))
    assert got[0] == 0xEE and (got[-2:] == 0xEE).all()


@pytest.mark.parametrize("q", FIELDS)
def test_encode_coefficient_edge_cases(gfm, q):
    batch, N, M = 2, 6, 1500
    A = si.random_bytes(71, 1, 0, batch * N * M).reshape(batch, N, M)
    I = np.broadcast_to(np.eye(N, dtype=np.uint8), (batch, N, N)).copy()
    assert np.array_equal(run_encode(gfm, q, A, I), A)
    Z = np.zeros((batch, N, 3), dtype=np.uint8)
    assert (run_encode(gfm, q, A, Z) == 0).all()
    F = np.full((batch, N, 4), q - 1, dtype=np.uint8)
    assert np.array_equal(run_encode(gfm, q, A, F), oracle.encode_batch(q, A, F))


def test_encode_sharding_invariance(gfm):
    """Generation shards and byte-range shards, launched separately, equal the
    unsharded launch (the multi-GPU partitioning of DESIGN.md)."""
    q, batch, N, K, M = 256, 6, 20, 9, 4096
    A = si.random_bytes(81, 1, 0, batch * N * M).reshape(batch, N, M)
    C = si.uniform_coeffs(q, 82, 2, 0, batch * N * K).reshape(batch, N, K)
    full = run_encode(gfm, q, A, C)
    parts = [run_encode(gfm, q, A[g0:g1], C[g0:g1]) for g0, g1 in ((0, 1), (1, 4), (4, 6))]
    assert np.array_equal(np.concatenate(parts), full)
    for m0, m1 in ((0, 1024), (1024, 3072), (3072, 4096)):
        assert np.array_equal(run_encode(gfm, q, A[:, :, m0:m1], C), full[:, :, m0:m1])


def test_encode_checked_mode(gfm):
    A = np.zeros((1, 2, 8), dtype=np.uint8)
    C = np.array([[[1], [16]]], dtype=np.uint8)
    with pytest.raises(gfm.GFError):
        gfm.encode_batch(16, dev(A), dev(C), checked=True)


# (full-size C3 / C4 / C5 parity: tests/test_gpu_fullsize.py)


@pytest.mark.parametrize("q", (2, 256))
@pytest.mark.parametrize("M", (1024, 1500))
def test_next2_full_size_sampled(gfm, q, M):
    """The paper's own shape (N = 16 source packets, K = 1) at
    the NEXT-2 sweep's launch size (2 GiB of source; 1 KiB packets: 16-byte
    chunks, 1500 B: the strided word kernel) through the streaming kernel:
    sampled generations recomputed by the oracle from host-regenerated inputs
    (device fill by absolute index)."""
    N, K = 16, 1
    G = (2 << 30) // (N * M)
    seed = 190902871 + 2 + 1000 * q
    assert gfm.encode_path(q, N, K, M) == "stream"
    A = torch.empty((G, N, M), dtype=torch.uint8, device="cuda")
    C = torch.empty((G, N, K), dtype=torch.uint8, device="cuda")
    gfm.fill_random(A, seed, si.STREAM_A, 0)
    gfm.fill_random(C, seed, si.STREAM_C, 0, mask=q - 1)
    B = gfm.encode_batch(q, A, C)
    rng = np.random.default_rng(q)
    for g in sorted({0, G - 1, *rng.integers(0, G, 14).tolist()}):
        Ah = si.random_bytes(seed, si.STREAM_A, g * N * M, N * M).reshape(1, N, M)
        Ch = si.uniform_coeffs(q, seed, si.STREAM_C, g * N * K, N * K).reshape(1, N, K)
        assert np.array_equal(B[g].cpu().numpy(), oracle.encode_batch(q, Ah, Ch)[0]), g
    del A, B, C
    torch.cuda.empty_cache()


@pytest.mark.parametrize("q", (4, 256))
@pytest.mark.parametrize("shape", ((37, 16, 8, 1500), (29, 64, 64, 1500), (11, 32, 32, 4096)))
def test_encode_host_path(gfm, q, shape):
    """gf_encode_batch_host (pinned host buffers, chunked pipeline) through the
    column, product-row and lane-k / product-row-32 kernels."""
    batch, N, K, M = shape
    A = si.random_bytes(91, 1, 0, batch * N * M).reshape(batch, N, M)
    C = si.uniform_coeffs(q, 92, 2, 0, batch * N * K).reshape(batch, N, K)
    Ah = torch.from_numpy(A).pin_memory()
    Ch = torch.from_numpy(C).pin_memory()
    Bh = torch.empty((batch, K, M), dtype=torch.uint8).pin_memory()
    ws = torch.empty(gfm.host_workspace_bytes(N, K, M, 5), dtype=torch.uint8, device="cuda")
    gfm.encode_batch_host(q, Ah, Ch, Bh, ws)
    assert np.array_equal(Bh.numpy(), oracle.encode_batch(q, A, C))
    L = gfm.lib()
    assert L.gf_encode_batch_host(q, Ah.data_ptr(), Ch.data_ptr(), Bh.data_ptr(), N, K, M, batch,
                                  ws.data_ptr(), 100) == gfm.GF_EARG


@pytest.mark.parametrize("q", FIELDS)
def test_encode_linear_in_coefficients_and_deterministic(gfm, q):
    """SPEC invariants on the GPU, for the shapes of
    every default kernel (streaming, column, product-row / lane-k): encode is
    linear in C (encode(A, C1 + C2) = encode(A, C1) + encode(A, C2), + = XOR in
    F_q) and repeated launches are bitwise identical."""
    for (N, K, M, batch) in ((16, 1, 1024, 40), (16, 8, 1500, 5), (64, 64, 1500, 3), (32, 32, 4096, 2)):
        A = si.random_bytes(91 + N, si.STREAM_A, 0, batch * N * M).reshape(batch, N, M)
        C1 = si.uniform_coeffs(q, 92 + K, si.STREAM_C, 0, batch * N * K).reshape(batch, N, K)
        C2 = si.uniform_coeffs(q, 93 + K, si.STREAM_C, 0, batch * N * K).reshape(batch, N, K)
        B1, B2 = run_encode(gfm, q, A, C1), run_encode(gfm, q, A, C2)
        assert np.array_equal(run_encode(gfm, q, A, C1 ^ C2), B1 ^ B2), (q, N, K, M)
        assert np.array_equal(run_encode(gfm, q, A, C1), B1), (q, N, K, M)


@pytest.mark.parametrize("q", FIELDS)
def test_encode_empty_batch_and_packets(gfm, q):
    """Degenerate sizes (batch == 0 or M == 0 returns GF_OK and
    launches nothing): empty outputs, no error; and a canary-guarded B is left
    untouched for batch == 0."""
    for batch, N, K, M in ((0, 4, 3, 64), (2, 4, 3, 0), (0, 1, 1, 0)):
        A = torch.zeros((batch, N, M), dtype=torch.uint8, device="cuda")
        C = torch.ones((batch, N, K), dtype=torch.uint8, device="cuda")
        B = gfm.encode_batch(q, A, C)
        assert tuple(B.shape) == (batch, K, M)
    L = gfm.lib()
    canary = torch.full((16,), 0xA5, dtype=torch.uint8, device="cuda")
    A = torch.zeros(16, dtype=torch.uint8, device="cuda")
    rc = L.gf_encode_batch(q, A.data_ptr(), A.data_ptr(), canary.data_ptr(), 2, 2, 4, 0)
    torch.cuda.synchronize()
    assert rc == gfm.GF_OK and (canary.cpu().numpy() == 0xA5).all()


@pytest.mark.parametrize("q", FIELDS)
def test_encode_guard_bytes_every_layout(gfm, q):
    """Out-of-bounds write check standing in for compute-sanitizer (closed on
    this pool): B is a view inside a buffer of 0xEE guard bytes (4 KiB before
    and after); every default kernel / layout on ragged shapes (partial
    product-row tiles, 2- and 4-chunk streaming blocks, strided word blocks,
    lane-k tiles) must leave the guards untouched and match the oracle."""
    shapes = [(64, 64, 1500, 3), (16, 16, 2052, 4), (16, 1, 2064, 5), (16, 1, 65552, 2),
              (16, 2, 1500, 3), (32, 32, 4100, 2), (9, 20, 1500, 3), (16, 8, 1508, 3)]
    for (N, K, M, batch) in shapes:
        A = si.random_bytes(101 + N, si.STREAM_A, 0, batch * N * M).reshape(batch, N, M)
        C = si.uniform_coeffs(q, 102 + K, si.STREAM_C, 0, batch * N * K).reshape(batch, N, K)
        guard = 4096
        nb = batch * K * M
        buf = torch.full((nb + 2 * guard,), 0xEE, dtype=torch.uint8, device="cuda")
        Bv = buf[guard:guard + nb].view(batch, K, M)
        gfm.encode_batch(q, dev(A), dev(C), Bv)
        got = buf.cpu().numpy()
        assert (got[:guard] == 0xEE).all() and (got[guard + nb:] == 0xEE).all(), (q, N, K, M)
        assert np.array_equal(got[guard:guard + nb].reshape(batch, K, M), oracle.encode_batch(q, A, C)), (q, N, K, M)


@pytest.mark.parametrize("q", FIELDS)
def test_raw_coefficient_bytes_are_masked(gfm, q):
    """include/gfrlnc.h: entries of C are not validated on the hot path, a byte
    >= q is taken modulo q by masking with q - 1.  Raw bytes through every
    default kernel equal the oracle on C & (q - 1)."""
    for (N, K, M, batch) in ((16, 1, 1024, 20), (16, 8, 1500, 3), (64, 64, 1500, 2), (32, 32, 4096, 2),
                             (9, 20, 1500, 3), (3, 5, 13, 4)):
        A = si.random_bytes(301 + N, si.STREAM_A, 0, batch * N * M).reshape(batch, N, M)
        Craw = si.random_bytes(302 + K, si.STREAM_C, 0, batch * N * K).reshape(batch, N, K)
        assert q == 256 or (Craw >= q).any()
        got = run_encode(gfm, q, A, Craw)
        assert np.array_equal(got, oracle.encode_batch(q, A, Craw & np.uint8(q - 1))), (q, N, K, M)


@pytest.mark.parametrize("q", FIELDS)
def test_mulrc_256_mib(gfm, q):
    """gf_mulrc at the top of the C2 range (256 MiB + 7 bytes: past the region
    kernel's grid-stride wrap, ragged tail), canaries on both sides."""
    n, pad = (256 << 20) + 7, 64
    base = si.random_bytes(43, si.STREAM_DST, 0, n + 2 * pad)
    c = si.c2_coeff(q) if q > 2 else 1
    for coeff in {c, q - 1}:
        d = dev(base)
        gfm.mulrc(q, d[pad:pad + n], coeff)
        exp = base.copy()
        seg = exp[pad:pad + n].copy()
        oracle.mulrc(q, seg, coeff)
        exp[pad:pad + n] = seg
        assert np.array_equal(d.cpu().numpy(), exp), (q, coeff)


GRAPH_SCRIPT = r'''
import sys, numpy as np, torch
sys.path.insert(0, %r)
import oracle, seeded_inputs as si
from paper_1909_02871_b200 import gf
for q in (2, 4, 16, 256):
    gf.init(q)
shapes = [(256, 4, 64, 64, 1500), (16, 3, 16, 8, 1500), (2, 2, 32, 32, 4096), (4, 2, 32, 32, 4096),
          (256, 20, 16, 1, 1024)]
ins, outs, exps = [], [], []
for q, batch, N, K, M in shapes:
    A = si.random_bytes(9 + N, 1, 0, batch * N * M).reshape(batch, N, M)
    C = si.uniform_coeffs(q, 10 + K, 2, 0, batch * N * K).reshape(batch, N, K)
    ins.append((q, torch.from_numpy(A).cuda(), torch.from_numpy(C).cuda()))
    outs.append(torch.zeros((batch, K, M), dtype=torch.uint8, device="cuda"))
    exps.append(oracle.encode_batch(q, A, C))
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    with torch.cuda.graph(g, stream=s):        # the FIRST encode calls of this process
        for (q, A, C), B in zip(ins, outs):
            gf.encode_batch(q, A, C, B)
for B in outs:
    B.zero_()
g.replay()
torch.cuda.synchronize()
for (q, A, C), B, e in zip(ins, outs, exps):
    assert np.array_equal(B.cpu().numpy(), e), q
print("graph ok")
''' % ROOT


def test_first_encode_captured_in_cuda_graph():
    """The hot path allocates, locks and synchronises nothing (gf_init prepared
    every kernel): the very first encode calls of a fresh process -- product-
    row, column, GF(2) split, lane-k and streaming kernels -- are captured into
    a CUDA graph and replayed bit-exactly."""
    import subprocess
    import sys
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = subprocess.run([sys.executable, "-c", GRAPH_SCRIPT], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    assert "graph ok" in out.stdout


@pytest.mark.parametrize("name", ("C3", "C4", "C5"))
def test_bench_split_shards_in_sequence_equal_unsharded(gfm, name):
    """bench.py's N-rank plan (bench.rank_shard: C3 / C5 by generation, C4 by
    byte range), every shard launched in sequence on one GPU with its inputs
    generated by absolute index, reassembles the unsharded job bit-exactly, for
    P = 2, 3, 4 and 8 (reduced generation counts / packet sizes)."""
    import dataclasses

    import bench
    from paper_1909_02871_b200 import shard
    base = si.ENCODE_CONFIGS[name]
    q = base.fields[-1]
    cfg = dataclasses.replace(base, batch={"C3": 64, "C4": 3, "C5": 8}[name],
                              M={"C3": 1500, "C4": 8192, "C5": 4096}[name])
    seed = si.field_seed(cfg, q)

    def encode(sh):
        A = torch.empty((sh.generations, cfg.N, sh.columns), dtype=torch.uint8, device="cuda")
        C = torch.empty((sh.generations, cfg.N, cfg.K), dtype=torch.uint8, device="cuda")
        gfm.fill_random2d(A.view(-1, sh.columns), seed, si.STREAM_A, sh.g0 * cfg.N * cfg.M + sh.m0, cfg.M)
        gfm.fill_random(C, seed, si.STREAM_C, sh.g0 * cfg.N * cfg.K, mask=q - 1)
        return gfm.encode_batch(q, A, C).cpu().numpy()

    full = encode(bench.rank_shard(shard, cfg, 1, 0)[0])
    Ah, Ch = si.encode_inputs(cfg, q, 0, 1)
    assert np.array_equal(full[:1], oracle.encode_batch(q, Ah, Ch))
    for P in (2, 3, 4, 8):
        B = np.zeros_like(full)
        for r in range(P):
            sh = bench.rank_shard(shard, cfg, P, r)[0]
            if sh.generations and sh.columns:
                B[sh.g0:sh.g1, :, sh.m0:sh.m1] = encode(sh)
        assert np.array_equal(B, full), (name, P)


def test_round2_kernels_edge_cases(gfm):
    """Edge cases of the round-2 kernels against the oracle: the GF(2) split
    engine over more than 65535 generations (several grid-y launches) and
    through the fused check (absolute generation index of the counts); the
    GF(16) nibble-table kernel with a misaligned coefficient pointer and
    K % 4 != 0 (scalar coefficient loads, partial 64-packet tile); the GF(256)
    768-word-tile kernel with a ragged last tile and two coded-packet tiles."""
    # GF(2), 70000 generations of N = 2, K = 24, 16-byte packets
    q, G, N, K, M = 2, 70000, 2, 24, 16
    A = si.random_bytes(61, si.STREAM_A, 0, G * N * M).reshape(G, N, M)
    C = si.uniform_coeffs(q, 62, si.STREAM_C, 0, G * N * K).reshape(G, N, K)
    assert gfm.encode_path(q, N, K, M) == "gf2-split"
    exp = oracle.encode_batch(q, A, C)
    assert np.array_equal(run_encode(gfm, q, A, C), exp)
    R = si.random_bytes(63, si.STREAM_FREIVALDS, 0, G * K).reshape(G, K, 1)
    gfm.set_verify_fault(69999, 5, 2)
    try:
        B, mism = gfm.encode_verify_batch(q, dev(A), dev(C), dev(R))
    finally:
        gfm.set_verify_fault(-1)
    m = mism.cpu().numpy()
    assert int(m.sum()) == int(m[69999]) == int(R[69999, 5, 0] & 1)
    # GF(16) nibble tables: C viewed at an odd address, K = 67
    q, G, N, K, M = 16, 3, 37, 67, 1500
    A = si.random_bytes(64, si.STREAM_A, 0, G * N * M).reshape(G, N, M)
    C = si.random_bytes(65, si.STREAM_C, 0, G * N * K).reshape(G, N, K)
    assert gfm.encode_path(q, N, K, M) == "prow-nib"
    cbuf = torch.zeros(C.size + 1, dtype=torch.uint8, device="cuda")
    cbuf[1:] = dev(C.reshape(-1))
    got = gfm.encode_batch(q, dev(A), cbuf[1:].view(G, N, K)).cpu().numpy()
    assert np.array_equal(got, oracle.encode_batch(q, A, C & 15))
    # GF(256) 768-word tiles: 6400 words (9 tiles, the last 256 words), K = 100 (four 32-packet tiles)
    q, G, N, K, M = 256, 2, 9, 100, 4 * 6400
    A = si.random_bytes(66, si.STREAM_A, 0, G * N * M).reshape(G, N, M)
    C = si.uniform_coeffs(q, 67, si.STREAM_C, 0, G * N * K).reshape(G, N, K)
    assert gfm.encode_path(q, N, K, M) == "prow-32w"
    assert np.array_equal(run_encode(gfm, q, A, C), oracle.encode_batch(q, A, C))
