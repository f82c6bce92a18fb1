"""Pins for the oracle's region ops and batched encode (Eq. 2).

Special cases that reduce to library routines (numpy XOR, selection,
identity, permutation), invariants (linearity in c and in C, composition,
Freivalds), an independent inverse (Gauss-Jordan decode recovers A) and the
paper's GF(4) trivial-coefficient fraction.
"""
import numpy as np
import pytest

import oracle
import seeded_inputs as si

FIELDS = (2, 4, 16, 256)


def rnd(n, seed=7, stream=9, off=0):
    return si.random_bytes(seed, stream, off, n)


@pytest.mark.parametrize("q", FIELDS)
def test_maddrc_trivial_coefficients(q):
    """c = 0 leaves dst unchanged, c = 1 is a plain XOR (Alg. 1,
    PAPER.md:205-211)."""
    for n in (0, 1, 63, 64, 1500, 4097):
        a, b = rnd(n, off=1), rnd(n, off=99999)
        d = b.copy()
        oracle.maddrc(q, d, a, 0)
        assert (d == b).all()
        d = b.copy()
        oracle.maddrc(q, d, a, 1)
        assert (d == np.bitwise_xor(a, b)).all()


@pytest.mark.parametrize("q", FIELDS)
def test_maddrc_linear_in_c(q):
    """madd(c1) then madd(c2) == madd(c1 + c2) for all pairs."""
    a, b = rnd(257, off=3), rnd(257, off=5000)
    for c1 in range(q):
        for c2 in range(q):
            d1 = b.copy()
            oracle.maddrc(q, d1, a, c1)
            oracle.maddrc(q, d1, a, c2)
            d2 = b.copy()
            oracle.maddrc(q, d2, a, c1 ^ c2)
            assert (d1 == d2).all()


@pytest.mark.parametrize("q", FIELDS)
def test_mulrc_composition_and_madd_relation(q):
    """mulrc(c2) after mulrc(c1) == mulrc(c1*c2); madd into zeros == mulrc."""
    a = rnd(300, off=11)
    for c1 in range(q):
        for c2 in (0, 1, q - 1, (c1 * 7 + 3) % q):
            d = a.copy()
            oracle.mulrc(q, d, c1)
            oracle.mulrc(q, d, c2)
            e = a.copy()
            oracle.mulrc(q, e, oracle.mul(q, c1, c2))
            assert (d == e).all()
        z = np.zeros_like(a)
        oracle.maddrc(q, z, a, c1)
        m = a.copy()
        oracle.mulrc(q, m, c1)
        assert (z == m).all()


def test_mulrc_gf256_is_aes_xtime():
    """GF(256) mulrc by 2 equals the textbook xtime (FIPS-197 Sec. 4.2.1):
    shift left, XOR 0x1B when the top bit was set."""
    a = np.arange(256, dtype=np.uint8)
    d = a.copy()
    oracle.mulrc(256, d, 2)
    exp = ((a.astype(np.int32) << 1) & 0xFF) ^ np.where(a & 0x80, 0x1B, 0)
    assert (d == exp).all()


def _enc(q, A, C):
    return oracle.encode_batch(q, A, C)


@pytest.mark.parametrize("q", FIELDS)
def test_encode_special_cases(q):
    N, M = 6, 77
    A = rnd(2 * N * M, off=17).reshape(2, N, M)
    # unit vectors select packets
    for i in range(N):
        C = np.zeros((2, N, 1), dtype=np.uint8)
        C[:, i, 0] = 1
        assert (_enc(q, A, C)[:, 0] == A[:, i]).all()
    # identity -> B = A, permutation permutes, zero -> zero
    I = np.broadcast_to(np.eye(N, dtype=np.uint8), (2, N, N)).copy()
    assert (_enc(q, A, I) == A).all()
    perm = np.array([3, 0, 5, 1, 4, 2])
    P = np.zeros((2, N, N), dtype=np.uint8)
    P[:, perm, np.arange(N)] = 1            # output k takes packet perm[k]
    assert (_enc(q, A, P) == A[:, perm]).all()
    assert (_enc(q, A, np.zeros((2, N, 3), dtype=np.uint8)) == 0).all()


@pytest.mark.parametrize("q", FIELDS)
def test_encode_k1_is_n_madds(q):
    """K = 1 reduces to N maddrc calls into a zero accumulator (PAPER.md:91,
    SPEC.md:234)."""
    N, M = 16, 1500
    A = rnd(N * M, off=5).reshape(1, N, M)
    C = si.uniform_coeffs(q, 3, 2, 0, N).reshape(1, N, 1)
    b = np.zeros(M, dtype=np.uint8)
    for i in range(N):
        oracle.maddrc(q, b, A[0, i].copy(), int(C[0, i, 0]))
    assert (_enc(q, A, C)[0, 0] == b).all()


def test_encode_gf2_is_xor_of_selected():
    N, K, M = 9, 5, 333
    A = rnd(N * M, off=8).reshape(1, N, M)
    C = si.uniform_coeffs(2, 4, 2, 0, N * K).reshape(1, N, K)
    B = _enc(2, A, C)
    for k in range(K):
        exp = np.zeros(M, dtype=np.uint8)
        for i in range(N):
            if C[0, i, k]:
                exp ^= A[0, i]
        assert (B[0, k] == exp).all()


@pytest.mark.parametrize("q", FIELDS)
def test_encode_linear_in_C_and_composition(q):
    N, K, M = 5, 4, 129
    A = rnd(N * M, off=40).reshape(1, N, M)
    C1 = si.uniform_coeffs(q, 11, 2, 0, N * K).reshape(1, N, K)
    C2 = si.uniform_coeffs(q, 12, 2, 0, N * K).reshape(1, N, K)
    assert (_enc(q, A, C1) ^ _enc(q, A, C2) == _enc(q, A, C1 ^ C2)).all()
    # encode(encode(A, C1), D) == encode(A, C1 @ D), product over F_q
    D = si.uniform_coeffs(q, 13, 2, 0, K * 3).reshape(1, K, 3)
    CD = np.zeros((1, N, 3), dtype=np.uint8)
    for i in range(N):
        for j in range(3):
            acc = 0
            for k in range(K):
                acc ^= oracle.mul(q, int(C1[0, i, k]), int(D[0, k, j]))
            CD[0, i, j] = acc
    assert (_enc(q, _enc(q, A, C1), D) == _enc(q, A, CD)).all()


@pytest.mark.parametrize("q", (4, 16, 256))
def test_encode_decode_round_trip(q):
    """Independent inverse: Gauss-Jordan on [C^T | B] recovers A for a
    full-rank square C (SPEC.md:248-255 round trip, acceptance 5)."""
    N, M = 16, 8192 if q != 16 else 512
    A = rnd(N * M, off=77).reshape(1, N, M)
    off = 0
    while True:
        C = si.uniform_coeffs(q, 21, 2, off, N * N).reshape(1, N, N)
        if oracle.rank(q, C[0]) == N:
            break
        off += N * N
    B = _enc(q, A, C)
    rk, A2 = oracle.decode(q, C[0], B[0])
    assert rk == N and (A2 == A[0]).all()


def test_rank_gf2_full_rank_probability():
    """P(16 random GF(2) vectors of length 16 are independent) =
    prod_{k=1..16} (1 - 2^-k) ~= 0.2888."""
    exact = np.prod([1 - 2.0 ** -k for k in range(1, 17)])
    assert abs(exact - 0.2888) < 1e-3
    trials = 4000
    v = si.uniform_coeffs(2, 99, 2, 0, trials * 256).reshape(trials, 16, 16)
    full = sum(oracle.rank(2, v[t]) == 16 for t in range(trials))
    assert abs(full / trials - exact) < 0.025


def test_rank_small_cases():
    assert oracle.rank(256, np.eye(7, dtype=np.uint8)) == 7
    v = np.array([[3, 5, 7], [3, 5, 7]], dtype=np.uint8)
    assert oracle.rank(256, v) == 1


def test_gf4_trivial_fraction():
    """Half of uniform GF(4) coefficients are 0 or 1."""
    c = si.uniform_coeffs(4, si.config_seed(5), si.STREAM_C, 0, 10 ** 6)
    assert abs(np.isin(c, (0, 1)).mean() - 0.5) < 0.01


@pytest.mark.parametrize("q", FIELDS)
def test_freivalds_accepts_and_detects(q):
    N, K, M = 8, 6, 500
    A = rnd(N * M, off=123).reshape(N, M)
    C = si.uniform_coeffs(q, 31, 2, 0, N * K).reshape(N, K)
    B = _enc(q, A[None], C[None])[0]
    t = oracle.freivalds_trials(q)
    rs = si.uniform_coeffs(q, 32, si.STREAM_FREIVALDS, 0, t * K).reshape(t, K)
    assert all(oracle.freivalds_gen(q, A, C, B, r) == 0 for r in rs)
    Bbad = B.copy()
    Bbad[2, 77] ^= 0x10                  # one flipped bit in one coded byte
    assert sum(oracle.freivalds_gen(q, A, C, Bbad, r) for r in rs) > 0


@pytest.mark.parametrize("q", FIELDS)
def test_encode_gen_cols_matches_full(q):
    N, K, M = 7, 3, 300
    A = rnd(N * M, off=55).reshape(N, M)
    C = si.uniform_coeffs(q, 33, 2, 0, N * K).reshape(N, K)
    B = _enc(q, A[None], C[None])[0]
    assert (oracle.encode_gen_cols(q, A, C, 37, 211) == B[:, 37:211]).all()


def test_encode_mt_matches_single():
    N, K, M, G = 8, 8, 100, 13
    A = rnd(G * N * M, off=9).reshape(G, N, M)
    C = si.uniform_coeffs(256, 5, 2, 0, G * N * K).reshape(G, N, K)
    assert (oracle.encode_batch(256, A, C, threads=4) == oracle.encode_batch(256, A, C)).all()
