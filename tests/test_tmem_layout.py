"""CPU emulation of the TMEM lookup-table engine's host-checkable logic
(csrc/encode_tmem.cuh) against the oracle: the basis words x^j a_i of each
4-bit group (the packed xtime of every field, including the two-LOP3 GF(4)
form), the 16-entry XOR-subset tables in the kernel's column order, the
coefficient-bit table index idx(g, k), and the fused check's A-side index from
u = C r.  The encode rebuilt from these pieces must equal the oracle's Eq. 2
bit for bit.  No GPU needed."""
import numpy as np
import pytest

import oracle
import seeded_inputs as si

FIELDS = (2, 4, 16, 256)
GPB = 4                       # groups per step (kTmGPB)


def width(q):
    return {2: 1, 4: 2, 16: 4, 256: 8}[q]


def xtime(q, a):
    """tm_xtime<LOGW>: x * a on every packed w-bit element of 32-bit words."""
    a = a.astype(np.uint64)
    if q == 4:                                   # two LOP3 + SHF + IMAD form
        t = a >> 1
        u = (a ^ t) & 0x55555555
        r = (t & 0x55555555) | (u + u)
    elif q == 16:
        r = ((a << 1) & 0xEEEEEEEE) ^ (((a >> 3) & 0x11111111) * 3)
    else:
        r = ((a << 1) & 0xFEFEFEFE) ^ (((a >> 7) & 0x01010101) * 0x1B)
    return (r & 0xFFFFFFFF).astype(np.uint32)


def groups(q, N):
    """NG: ceil(N w / 4) rounded up to GPB (tm_groups)."""
    ng = -(-N * width(q) // 4)
    return -(-ng // GPB) * GPB


def basis(q, A32, grp):
    """The four basis words e_b = x^j a_i (t = 4 grp + b, i = t / w, j = t mod w)
    of one group for every word of every source row (rows >= N: zero -- the
    kernel reads other rows there, which only ever meet zero coefficient bits)."""
    N, Mw = A32.shape
    w = width(q)
    out = []
    for b in range(4):
        t = 4 * grp + b
        i, j = t // w, t % w
        if i >= N:
            out.append(np.zeros(Mw, dtype=np.uint32))
            continue
        v = A32[i].copy()
        for _ in range(j):
            v = xtime(q, v)
        out.append(v)
    return out


def table(e):
    """The 16 XOR-subsets in the kernel's build order: v[c] = XOR of e_b for the
    set bits b of c (v[3] = e0 ^ e1, v[4..7] = e2 ^ v[0..3], v[8..15] = e3 ^ v[0..7])."""
    v = [np.zeros_like(e[0]), e[0], e[1], e[0] ^ e[1]]
    v += [e[2] ^ v[c] for c in range(4)]
    v += [e[3] ^ v[c] for c in range(8)]
    return v


def index(q, C, grp, k):
    """idx(g, k): bit b = bit j of C[i][k] (t = 4 grp + b, i = t / w, j = t mod w)."""
    N = C.shape[0]
    w = width(q)
    idx = 0
    for b in range(4):
        t = 4 * grp + b
        i, j = t // w, t % w
        if i < N:
            idx |= ((int(C[i, k]) >> j) & 1) << b
    return idx


def tmem_encode(q, A, C):
    """One generation through the engine's arithmetic: b_k = XOR over groups of
    T_g[idx(g, k)] (the kernel's lookups and LOP3s)."""
    N, M = A.shape
    K = C.shape[1]
    A32 = A.view(np.uint32).reshape(N, M // 4)
    B32 = np.zeros((K, M // 4), dtype=np.uint32)
    for grp in range(groups(q, N)):
        T = table(basis(q, A32, grp))
        for k in range(K):
            B32[k] ^= T[index(q, C, grp, k)]
    return B32.view(np.uint8).reshape(K, M)


@pytest.mark.parametrize("q", FIELDS)
def test_table_rows_are_the_coefficient_products(q):
    """T_g[c] with c the 4 coefficient bits of a lone source i equals the
    oracle's c . a_i (GF(16): c is the whole element; GF(256): the low nibble
    of group 2i, the high nibble of group 2i + 1; GF(4): two sources per group;
    GF(2): four)."""
    w = width(q)
    A = si.random_bytes(5, si.STREAM_A, 0, 4 * 64).reshape(4, 64)
    A32 = A.view(np.uint32).reshape(4, 16)
    for grp in range(groups(q, 4)):
        T = table(basis(q, A32, grp))
        for c in range(16):
            exp = np.zeros(64, dtype=np.uint8)
            for b in range(4):
                t = 4 * grp + b
                i, j = t // w, t % w
                if c >> b & 1 and i < 4:
                    oracle.maddrc(q, exp, A[i], 1 << j)
            assert np.array_equal(T[c].view(np.uint8), exp), (q, grp, c)


@pytest.mark.parametrize("q", (4, 16, 256))
def test_xtime_equals_multiplication_by_x(q):
    a = si.random_bytes(9, si.STREAM_A, 0, 4096)
    got = xtime(q, a.view(np.uint32)).view(np.uint8)
    exp = np.zeros_like(a)
    oracle.maddrc(q, exp, a, 2)
    assert np.array_equal(got, exp)


@pytest.mark.parametrize("q", FIELDS)
@pytest.mark.parametrize("N,K,M", [(32, 32, 256), (5, 24, 64), (33, 40, 48), (1, 1, 16), (17, 3, 32)])
def test_engine_arithmetic_equals_oracle(q, N, K, M):
    A = si.random_bytes(40 + N, si.STREAM_A, 0, N * M).reshape(1, N, M)
    C = si.uniform_coeffs(q, 41 + K, si.STREAM_C, 0, N * K).reshape(1, N, K)
    assert np.array_equal(tmem_encode(q, A[0], C[0]), oracle.encode_batch(q, A, C)[0]), (q, N, K, M)


@pytest.mark.parametrize("q", FIELDS)
def test_raw_coefficient_bytes_use_only_the_field_bits(q):
    """idx reads bits j < w of each coefficient byte: raw bytes >= q act as
    byte & (q - 1) (include/gfrlnc.h masking)."""
    N, K, M = 8, 8, 32
    A = si.random_bytes(61, si.STREAM_A, 0, N * M).reshape(N, M)
    C = si.random_bytes(62, si.STREAM_C, 0, N * K).reshape(N, K)
    got = tmem_encode(q, A, C)
    exp = oracle.encode_batch(q, A[None], (C & (q - 1))[None])[0]
    assert np.array_equal(got, exp)


@pytest.mark.parametrize("q", FIELDS)
def test_check_index_gives_the_a_side_projection(q):
    """The fused check's A side: with u = C r (binary r), the lookup
    T_g[idx_u(g)] summed over groups is sum_i u_i a_i, which equals
    sum_k r_k b_k (the B side) for the correct encode."""
    N, K, M = 13, 20, 64
    A = si.random_bytes(71, si.STREAM_A, 0, N * M).reshape(N, M)
    C = si.uniform_coeffs(q, 72, si.STREAM_C, 0, N * K).reshape(N, K)
    r = si.random_bytes(73, si.STREAM_FREIVALDS, 0, K) & 1
    # u_i = sum_k r_k C[i][k] over F_q (binary r: XOR of the selected coefficients)
    u = np.zeros(N, dtype=np.uint8)
    for k in range(K):
        if r[k]:
            u ^= C[:, k]
    A32 = A.view(np.uint32).reshape(N, M // 4)
    y1 = np.zeros(M // 4, dtype=np.uint32)
    for grp in range(groups(q, N)):
        y1 ^= table(basis(q, A32, grp))[index(q, u.reshape(N, 1), grp, 0)]
    B = oracle.encode_batch(q, A[None], C[None])[0]
    y2 = np.zeros(M, dtype=np.uint8)
    for k in range(K):
        if r[k]:
            y2 ^= B[k]
    assert np.array_equal(y1.view(np.uint8), y2)
    exp = np.zeros(M, dtype=np.uint8)
    for i in range(N):
        oracle.maddrc(q, exp, A[i], int(u[i]))
    assert np.array_equal(y1.view(np.uint8), exp)
