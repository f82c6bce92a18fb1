"""gf_encode_verify_batch: the encode with the
Freivalds check -- B bit-exact against the oracle, per-generation mismatch
counts equal to the oracle's Freivalds projections (oracle.freivalds_gen with
the same binary r, per block of 64 coded packets), zero on a correct encode, and
a single corrupted byte (harness fault injection: inside the GF(2) split engine
before the store and the projection, else in B after the encode) caught in
exactly its generation; for the check fused into the GF(2) split engine, the
word-parallel streaming check after every other kernel (product-row, lane-k,
column, streaming) and the byte-wise check for packets that are not 4-byte
aligned."""
import numpy as np
import pytest
import torch

import oracle
import seeded_inputs as si

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gfm():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1909_02871_b200 import gf
    for q in (2, 4, 16, 256):
        gf.init(q)
    return gf


def oracle_counts(q, A, C, B, R):
    """sum over projections j and 64-coded-packet blocks of the oracle's
    Freivalds mismatch count with r restricted to the block (binary r)."""
    batch, N, M = A.shape
    K = C.shape[2]
    out = np.zeros(batch, dtype=np.int64)
    for g in range(batch):
        for j in range(R.shape[2]):
            r = (R[g, :, j] & 1).astype(np.uint8)
            for b0 in range(0, K, 64):
                rb = np.zeros(K, dtype=np.uint8)
                rb[b0:b0 + 64] = r[b0:b0 + 64]
                out[g] += oracle.freivalds_gen(q, A[g], C[g], B[g], rb)
    return out


CASES = [  # (q, N, K, M, batch, expected kernel)
    (256, 64, 64, 1500, 5, "prow"), (16, 64, 64, 1500, 4, "prow-nib"), (256, 40, 100, 2000, 3, "prow"),
    (2, 32, 32, 4096, 3, "gf2-split"), (2, 17, 40, 1040, 4, "gf2-split"), (2, 5, 24, 400, 6, "gf2-split"),
    (4, 32, 32, 4096, 2, "lanek-32"), (256, 16, 8, 1500, 3, "column-words"), (16, 16, 1, 1024, 9, "stream"),
    (2, 32, 80, 512, 2, "gf2-split"),
    # packets not a multiple of 4 bytes: the byte-wise check; long packets
    # with two coded-packet blocks and a ragged last 128-word chunk
    (256, 20, 70, 1502, 2, "column-bytes"), (256, 64, 100, 28000, 1, "prow-32w"),
    # lane-k with the check fused: 32 and 64 coded packets per CTA (GF(2) with
    # N > 32, where the split engine does not apply); 128 per CTA (K > 64) runs
    # the streaming check
    (4, 64, 64, 2048, 2, "lanek-64"), (2, 40, 48, 2048, 3, "lanek-64"), (4, 24, 70, 1024, 2, "lanek-64"),
    # the TMEM engine with the check fused: two passes of 32 coded packets,
    # a partial last group (N = 33), a ragged last span, several generations
    # per warp; K > 64 runs the streaming check after it
    (4, 33, 64, 4112, 3, "tmem"), (2, 64, 64, 8192, 2, "tmem"), (4, 32, 40, 20480, 2, "tmem"),
    (2, 7, 24, 4096, 40, "tmem"), (4, 32, 70, 4096, 2, "tmem"), (16, 32, 32, 4096, 3, "tmem"),
    (16, 20, 60, 2048, 2, "tmem")]


@pytest.mark.parametrize("q,N,K,M,batch,kern", CASES)
@pytest.mark.parametrize("t", (1, 2))
def test_fused_verify_matches_oracle(gfm, q, N, K, M, batch, kern, t):
    # the TMEM engine has no fused check: gf_encode_verify_batch runs its
    # shapes through the fused GF(2) split / lane-k kernels named here
    assert gfm.encode_path(q, N, K, M) in (kern, "tmem")
    A = si.random_bytes(500 + N, si.STREAM_A, 0, batch * N * M).reshape(batch, N, M)
    C = si.uniform_coeffs(q, 501 + K, si.STREAM_C, 0, batch * N * K).reshape(batch, N, K)
    R = si.random_bytes(502, si.STREAM_FREIVALDS, 0, batch * K * t).reshape(batch, K, t)
    B, mism = gfm.encode_verify_batch(q, *(torch.from_numpy(x).cuda() for x in (A, C, R)))
    Bh = B.cpu().numpy()
    assert np.array_equal(Bh, oracle.encode_batch(q, A, C)), (q, N, K, M)
    assert (mism.cpu().numpy() == 0).all()
    # one wrong byte, injected in the kernel before the store and the projection
    gfm.set_verify_fault(batch // 2, K - 1, (M // 4) // 3)
    try:
        B2, mism2 = gfm.encode_verify_batch(q, *(torch.from_numpy(x).cuda() for x in (A, C, R)))
    finally:
        gfm.set_verify_fault(-1)
    B2h, got = B2.cpu().numpy(), mism2.cpu().numpy()
    assert int((B2h != Bh).sum()) == 1 and B2h[batch // 2, K - 1, 4 * ((M // 4) // 3)] != Bh[batch // 2, K - 1, 4 * ((M // 4) // 3)]
    exp = oracle_counts(q, A, C, B2h, R)
    assert np.array_equal(got, exp), (got, exp)
    rsel = R[batch // 2, K - 1, :t] & 1
    assert (got[batch // 2] > 0) == bool(rsel.any())       # caught iff some r_j selects coded packet K-1
    assert got.sum() == got[batch // 2]


@pytest.mark.parametrize("q", (2, 4, 16))
def test_fused_verify_forced_tmem(gfm, q):
    """The TMEM engine's fused check on short packets (forced: the router sends
    packets below 4 KiB elsewhere), one and two projections, with and without
    an injected fault."""
    gfm.set_encode_path("tmem")
    try:
        for N, K, M, batch, t in ((5, 24, 400, 6, 2), (17, 33, 1040, 3, 1), (3, 1, 16, 9, 2), (32, 64, 272, 4, 2)):
            assert gfm.encode_path(q, N, K, M) == "tmem"
            A = si.random_bytes(700 + N, si.STREAM_A, 0, batch * N * M).reshape(batch, N, M)
            C = si.uniform_coeffs(q, 701 + K, si.STREAM_C, 0, batch * N * K).reshape(batch, N, K)
            R = si.random_bytes(702, si.STREAM_FREIVALDS, 0, batch * K * t).reshape(batch, K, t)
            B, mism = gfm.encode_verify_batch(q, *(torch.from_numpy(x).cuda() for x in (A, C, R)))
            Bh = B.cpu().numpy()
            assert np.array_equal(Bh, oracle.encode_batch(q, A, C)), (q, N, K, M)
            assert (mism.cpu().numpy() == 0).all()
            gfm.set_verify_fault(batch - 1, K - 1, (M // 4) - 1)
            try:
                B2, mism2 = gfm.encode_verify_batch(q, *(torch.from_numpy(x).cuda() for x in (A, C, R)))
            finally:
                gfm.set_verify_fault(-1)
            B2h, got = B2.cpu().numpy(), mism2.cpu().numpy()
            assert int((B2h != Bh).sum()) == 1
            assert np.array_equal(got, oracle_counts(q, A, C, B2h, R)), (got, q, N, K, M)
    finally:
        gfm.set_encode_path("auto")


@pytest.mark.parametrize("q", (2, 4, 16, 256))
def test_fused_verify_forced_lanek(gfm, q):
    """The lane-k kernel's fused check (forced: the router sends GF(16) / GF(256)
    to the product-row kernels and most GF(2) / GF(4) shapes to the TMEM
    engine), 32 and 64 coded packets per CTA, with and without an injected
    fault."""
    gfm.set_encode_path("lanek")
    try:
        for N, K, M, batch in ((20, 30, 1540, 3), (20, 40, 1540, 3)):
            assert gfm.encode_path(q, N, K, M).startswith("lanek")
            A = si.random_bytes(600 + N, si.STREAM_A, 0, batch * N * M).reshape(batch, N, M)
            C = si.uniform_coeffs(q, 601 + K, si.STREAM_C, 0, batch * N * K).reshape(batch, N, K)
            R = si.random_bytes(602, si.STREAM_FREIVALDS, 0, batch * K * 2).reshape(batch, K, 2)
            B, mism = gfm.encode_verify_batch(q, *(torch.from_numpy(x).cuda() for x in (A, C, R)))
            Bh = B.cpu().numpy()
            assert np.array_equal(Bh, oracle.encode_batch(q, A, C)) and int(mism.sum()) == 0
            gfm.set_verify_fault(1, K - 2, 100)
            try:
                B2, mism2 = gfm.encode_verify_batch(q, *(torch.from_numpy(x).cuda() for x in (A, C, R)))
            finally:
                gfm.set_verify_fault(-1)
            B2h = B2.cpu().numpy()
            assert int((B2h != Bh).sum()) == 1
            assert np.array_equal(mism2.cpu().numpy(), oracle_counts(q, A, C, B2h, R))
    finally:
        gfm.set_encode_path("auto")


def test_fused_verify_full_c3_shape_every_generation(gfm):
    """The C3 job (65536 generations, GF(256)) through the product-row encode
    and the streaming check: B identical to the plain encode, no mismatch
    anywhere."""
    cfg, q = si.C3, 256
    seed = si.field_seed(cfg, q)
    A = torch.empty((cfg.batch, cfg.N, cfg.M), dtype=torch.uint8, device="cuda")
    C = torch.empty((cfg.batch, cfg.N, cfg.K), dtype=torch.uint8, device="cuda")
    R = torch.empty((cfg.batch, cfg.K, 2), dtype=torch.uint8, device="cuda")
    gfm.fill_random(A, seed, si.STREAM_A, 0)
    gfm.fill_random(C, seed, si.STREAM_C, 0, mask=q - 1)
    gfm.fill_random(R, seed, si.STREAM_FREIVALDS, 0)
    B, mism = gfm.encode_verify_batch(q, A, C, R)
    assert int(mism.sum()) == 0
    assert torch.equal(B, gfm.encode_batch(q, A, C))


def test_encode_verify_argument_errors(gfm):
    L = gfm.lib()
    batch, N, K, M = 2, 8, 4, 64
    A = torch.zeros((batch, N, M), dtype=torch.uint8, device="cuda")
    C = torch.zeros((batch, N, K), dtype=torch.uint8, device="cuda")
    B = torch.zeros((batch, K, M), dtype=torch.uint8, device="cuda")
    R = torch.zeros((batch, K, 2), dtype=torch.uint8, device="cuda")
    mism = torch.zeros(batch, dtype=torch.int64, device="cuda")
    need = gfm.verify_workspace_bytes(N, K, batch)
    ws = torch.zeros(need + 32, dtype=torch.uint8, device="cuda")

    def call(t=2, r=R, m=mism, w=ws.data_ptr(), n=need, b=B.data_ptr()):
        return L.gf_encode_verify_batch(256, A.data_ptr(), C.data_ptr(), b, r.data_ptr() if r is not None else None,
                                        t, N, K, M, batch, m.data_ptr() if m is not None else None, w, n)
    assert call() == gfm.GF_OK
    assert call(t=0) == gfm.GF_EARG and call(t=3) == gfm.GF_EARG
    assert call(r=None) == gfm.GF_EARG and call(m=None) == gfm.GF_EARG
    assert call(n=need - 1) == gfm.GF_EARG                           # short workspace
    assert call(w=ws.data_ptr() + 4) == gfm.GF_EARG                  # not 16-byte aligned
    assert call(w=A.data_ptr()) == gfm.GF_EOVERLAP                   # workspace over A
    assert call(b=A.data_ptr()) == gfm.GF_EOVERLAP                   # B over A
    assert L.gf_encode_verify_batch(256, A.data_ptr(), C.data_ptr(), B.data_ptr(), R.data_ptr(), 2, N, K, M, 0,
                                    mism.data_ptr(), ws.data_ptr(), need) == gfm.GF_OK   # empty batch
    torch.cuda.synchronize()


@pytest.mark.parametrize("seed", range(24))
def test_verify_random_shapes(gfm, seed):
    """Seeded random shapes through gf_encode_verify_batch (whatever kernel the
    router picks: lane-k with the check fused, the GF(2) split engine, product
    rows, column, streaming, each followed by the matching check): B bit-exact
    and the per-generation counts equal to the oracle's, with and without one
    injected wrong byte."""
    rng = np.random.default_rng(9000 + seed)
    q = int(rng.choice([2, 4, 16, 256]))
    N = int(rng.integers(1, 70))
    K = int(rng.integers(1, 140))
    M = 4 * int(rng.integers(1, 700)) + (0 if seed % 6 else int(rng.integers(1, 4)))
    batch = int(rng.integers(1, 5))
    t = 1 + seed % 2
    A = si.random_bytes(9100 + seed, si.STREAM_A, 0, batch * N * M).reshape(batch, N, M)
    C = si.uniform_coeffs(q, 9200 + seed, si.STREAM_C, 0, batch * N * K).reshape(batch, N, K)
    R = si.random_bytes(9300 + seed, si.STREAM_FREIVALDS, 0, batch * K * t).reshape(batch, K, t)
    B, mism = gfm.encode_verify_batch(q, *(torch.from_numpy(x).cuda() for x in (A, C, R)))
    Bh = B.cpu().numpy()
    path = gfm.encode_path(q, N, K, M)
    assert np.array_equal(Bh, oracle.encode_batch(q, A, C)), (q, N, K, M, batch, path)
    assert int(mism.sum()) == 0, (q, N, K, M, batch, path)
    g, k, w = int(rng.integers(0, batch)), int(rng.integers(0, K)), int(rng.integers(0, M // 4)) if M >= 4 else 0
    gfm.set_verify_fault(g, k, w)
    try:
        B2, mism2 = gfm.encode_verify_batch(q, *(torch.from_numpy(x).cuda() for x in (A, C, R)))
    finally:
        gfm.set_verify_fault(-1)
    B2h = B2.cpu().numpy()
    assert int((B2h != Bh).sum()) == (1 if 4 * w < M else 0), (q, N, K, M, batch, path, g, k, w)
    assert np.array_equal(mism2.cpu().numpy(), oracle_counts(q, A, C, B2h, R)), (q, N, K, M, batch, path)
