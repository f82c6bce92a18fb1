"""Batched decode: GPU matrix inversion and decode
against the oracle's Gauss-Jordan (oracle.rank / oracle.decode)."""
import numpy as np
import pytest
import torch

import oracle
import seeded_inputs as si

pytestmark = pytest.mark.gpu

FIELDS = (2, 4, 16, 256)


@pytest.fixture(scope="module")
def gfm():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1909_02871_b200 import gf
    for q in FIELDS:
        gf.init(q)
    return gf


def mat_mul(q, X, Y):
    T = oracle.mul_table(q).astype(np.int64)
    n, m = X.shape[0], Y.shape[1]
    out = np.zeros((n, m), dtype=np.int64)
    for k in range(X.shape[1]):
        out ^= T[X[:, k][:, None], Y[k][None, :]]
    return out.astype(np.uint8)


@pytest.mark.parametrize("q", FIELDS)
@pytest.mark.parametrize("N", [1, 5, 16, 33, 64, 65, 130])
def test_invert_batch(gfm, q, N):
    batch = 24
    C = si.uniform_coeffs(q, 100 + N, 2, 0, batch * N * N).reshape(batch, N, N)
    if N > 1:
        C[3, :, 1] = C[3, :, 0]                         # rank-deficient generation
    else:
        C[3] = 0
    D, rank = gfm.invert_batch(q, torch.from_numpy(C).cuda())
    D, rank = D.cpu().numpy(), rank.cpu().numpy()
    for g in range(batch):
        assert rank[g] == oracle.rank(q, C[g]), g
        if rank[g] == N:
            assert np.array_equal(mat_mul(q, C[g], D[g]), np.eye(N, dtype=np.uint8)), g


@pytest.mark.parametrize("q", FIELDS)
def test_decode_round_trip_and_oracle(gfm, q):
    """encode (oracle) then GPU decode recovers the sources of every full-rank
    generation; equals the oracle's Gauss-Jordan decode."""
    batch, N, M = 12, 16, 1500
    A = si.random_bytes(301, 1, 0, batch * N * M).reshape(batch, N, M)
    C = si.uniform_coeffs(q, 302, 2, 0, batch * N * N).reshape(batch, N, N)
    B = oracle.encode_batch(q, A, C)
    A2, rank = gfm.decode_batch(q, torch.from_numpy(B).cuda(), torch.from_numpy(C).cuda())
    A2, rank = A2.cpu().numpy(), rank.cpu().numpy()
    for g in range(batch):
        rk, Ao = oracle.decode(q, C[g], B[g])
        assert rank[g] == rk
        if rk == N:
            assert np.array_equal(A2[g], A[g]) and np.array_equal(Ao, A[g])


def test_decode_c3_shape_gf256(gfm):
    """C3 generation shape (N = K = 64, 1500 B), GPU encode -> GPU decode."""
    q, batch, N, M = 256, 64, 64, 1500
    A = torch.empty((batch, N, M), dtype=torch.uint8, device="cuda")
    C = torch.empty((batch, N, N), dtype=torch.uint8, device="cuda")
    gfm.fill_random(A, 7, si.STREAM_A, 0)
    gfm.fill_random(C, 7, si.STREAM_C, 0)
    B = gfm.encode_batch(q, A, C)
    A2, rank = gfm.decode_batch(q, B, C)
    full = rank == N
    assert int(full.sum()) >= batch - 2                 # random GF(256) matrices are almost surely invertible
    assert torch.equal(A2[full], A[full])


def test_decode_errors(gfm):
    L = gfm.lib()
    t = torch.zeros(64, dtype=torch.uint8, device="cuda")
    p = t.data_ptr()
    assert L.gf_invert_batch(256, p, p + 32, None, 0, 1) == gfm.GF_EARG
    assert L.gf_invert_batch(256, p, p + 32, None, 300, 1) == gfm.GF_EARG
    assert L.gf_invert_batch(256, p, p + 8, None, 4, 1) == gfm.GF_EOVERLAP
    assert L.gf_decode_batch(256, p, p + 16, p + 32, None, 4, 4, 1, p + 48, 8) == gfm.GF_EARG


@pytest.mark.parametrize("q", (2, 256))
@pytest.mark.parametrize("N", (5, 33, 64, 65))
def test_invert_and_decode_guard_bytes(gfm, q, N):
    """Out-of-bounds write check (compute-sanitizer is closed on this pool):
    D, rank and the decoded A sit inside 0xEE / -7 guard regions that the warp-
    and CTA-per-matrix inversions and the decode must leave untouched."""
    batch, M = 13, 1500
    C = si.uniform_coeffs(q, 201 + N, si.STREAM_C, 0, batch * N * N).reshape(batch, N, N)
    Cd = torch.from_numpy(C).cuda()
    L = gfm.lib()
    g = 4096
    dbuf = torch.full((batch * N * N + 2 * g,), 0xEE, dtype=torch.uint8, device="cuda")
    rbuf = torch.full((batch + 64,), -7, dtype=torch.int32, device="cuda")
    rc = L.gf_invert_batch(q, Cd.data_ptr(), dbuf.data_ptr() + g, rbuf.data_ptr() + 4 * 32, N, batch)
    torch.cuda.synchronize()
    assert rc == gfm.GF_OK
    d = dbuf.cpu().numpy()
    r = rbuf.cpu().numpy()
    assert (d[:g] == 0xEE).all() and (d[g + batch * N * N:] == 0xEE).all()
    assert (r[:32] == -7).all() and (r[32 + batch:] == -7).all()
    assert (r[32:32 + batch] == [oracle.rank(q, C[i]) for i in range(batch)]).all()
    B = si.random_bytes(202 + N, si.STREAM_A, 0, batch * N * M).reshape(batch, N, M)
    abuf = torch.full((batch * N * M + 2 * g,), 0xEE, dtype=torch.uint8, device="cuda")
    ws = torch.empty(batch * N * N, dtype=torch.uint8, device="cuda")
    rc = L.gf_decode_batch(q, torch.from_numpy(B).cuda().data_ptr(), Cd.data_ptr(), abuf.data_ptr() + g,
                           rbuf.data_ptr() + 4 * 32, N, M, batch, ws.data_ptr(), ws.numel())
    torch.cuda.synchronize()
    assert rc == gfm.GF_OK
    a = abuf.cpu().numpy()
    assert (a[:g] == 0xEE).all() and (a[g + batch * N * M:] == 0xEE).all()
    # the decoded sources themselves, against the oracle's Gauss-Jordan solve of
    # B = C^T A (every full-rank generation)
    got = a[g:g + batch * N * M].reshape(batch, N, M)
    for i in range(batch):
        rk, A_ref = oracle.decode(q, C[i], B[i])
        assert rk == r[32 + i]
        if rk == N:
            assert np.array_equal(got[i], A_ref), (q, N, i)


def test_gf2_full_rank_probability_on_gpu(gfm):
    """SPEC.md:256-263 acceptance 6 on the GPU inversion: a uniform random 16 x 16
    matrix over GF(2) is invertible with probability prod_{i=1..16}(1 - 2^-i) =
    0.288788... (the oracle pins the same statistic in test_oracle_encode); over
    200,000 seeded matrices the fraction the GPU reports full rank is within 5
    standard deviations (0.0051), and the ranks of the first 2000 equal the
    oracle's Gauss-Jordan ranks."""
    n, N = 200_000, 16
    C = torch.empty((n, N, N), dtype=torch.uint8, device="cuda")
    gfm.fill_random(C, 777, si.STREAM_C, 0, mask=1)
    _, rank = gfm.invert_batch(2, C)
    r = rank.cpu().numpy()
    p = 1.0
    for i in range(1, N + 1):
        p *= 1.0 - 2.0 ** -i
    frac = float((r == N).mean())
    sd = (p * (1 - p) / n) ** 0.5
    assert abs(frac - p) < 5 * sd, (frac, p)
    Ch = si.uniform_coeffs(2, 777, si.STREAM_C, 0, 2000 * N * N).reshape(2000, N, N)
    assert all(oracle.rank(2, Ch[g]) == r[g] for g in range(2000))
