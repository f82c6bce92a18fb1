"""CPU emulation of the product-row encode kernel's host-checkable logic
(csrc/encode_prow.cuh) against the oracle: the basis rows from the packed xtime
chain, the Gray-code table fill, the one-PRMT gather address, the bank-slot
argument behind "every LDS.128 is exactly 4 wavefronts for any data", and the
4x4 byte transpose of the write-back.  No GPU needed."""
import numpy as np
import pytest

import oracle
from test_abi_host import prmt

FIELDS = (2, 4, 16, 256)


def width(q):
    return {2: 1, 4: 2, 16: 4, 256: 8}[q]


def pr_xtime(q, a):
    """The kernel's packed x*v (every w-bit slot of every byte of a 32-bit word)."""
    if q == 256:
        return (((a << 1) & 0xFEFEFEFE) ^ (((a >> 7) & 0x01010101) * 0x1B)) & 0xFFFFFFFF
    if q == 16:
        return (((a << 1) & 0xEEEEEEEE) ^ (((a >> 3) & 0x11111111) * 3)) & 0xFFFFFFFF
    if q == 4:
        hi = (a >> 1) & 0x55555555
        return hi | ((((a & 0x55555555) ^ hi) << 1) & 0xFFFFFFFF)
    return a


def basis_words(q, cword):
    """Producer basis (per thread, per coefficient word of its 16-byte chunk):
    bit b -> slot b / w holds c * x^(b mod w) for 4 packed coefficients."""
    w = width(q)
    xt = [cword]
    for _ in range(1, w):
        xt.append(pr_xtime(q, xt[-1]))
    return [(xt[b % w] << ((b // w) * w)) & 0xFFFFFFFF for b in range(8)]


def gray_fill(basis_rows):
    """Producer table fill: rows of one 16-B chunk as XOR combinations of the 8
    basis rows, thread h writes rows 32h .. 32h+31 in Gray-code order starting
    from the XOR of basis rows 5..7 selected by h."""
    rows = [None] * 256
    for h in range(8):
        v = np.zeros(4, dtype=np.uint32)
        for j in range(3):
            if h >> j & 1:
                v ^= basis_rows[5 + j]
        rows[32 * h] = v.copy()
        for n in range(1, 32):
            flip = (n & -n).bit_length() - 1
            v ^= basis_rows[flip]
            rows[32 * h + (n ^ (n >> 1))] = v.copy()
    return rows


@pytest.mark.parametrize("q", FIELDS)
def test_basis_and_gray_table_equal_products(q):
    """Every table row P[a] built from the basis rows equals the oracle's packed
    products C[k] * a for all 256 byte values a, for random 16-coefficient chunks."""
    MB = oracle.mulbyte_table(q)
    rng = np.random.default_rng(q)
    for _ in range(6):
        coeffs = rng.integers(0, q, size=16).astype(np.uint8)
        cw = coeffs.view(np.uint32)                        # 4 little-endian words
        per_word = [basis_words(q, int(w)) for w in cw]
        basis_rows = [np.array([per_word[qq][b] for qq in range(4)], dtype=np.uint32) for b in range(8)]
        rows = gray_fill(basis_rows)
        for a in range(256):
            got = rows[a].view(np.uint8)
            want = MB[coeffs, a]
            assert np.array_equal(got, want), (q, a)


def test_basis_masks_raw_coefficients():
    """The kernel masks raw coefficient bytes with q-1 (ABI: entries taken mod q)."""
    MB = oracle.mulbyte_table(16)
    raw = np.array([0x3A, 0xF1, 0x07, 0x90], dtype=np.uint8)
    cw = int(raw.view(np.uint32)[0]) & (15 * 0x01010101)
    rows = gray_fill([np.array([basis_words(16, cw)[b], 0, 0, 0], dtype=np.uint32) for b in range(8)])
    for a in range(256):
        got = rows[a].view(np.uint8)[:4]
        assert np.array_equal(got, MB[raw & 15, a])


def test_gather_address_is_one_prmt():
    """prmt(a_word, col, 0x55j4) = byte j of a_word * 256 + col (col < 256)."""
    rng = np.random.default_rng(1)
    for _ in range(2000):
        aw = int(rng.integers(0, 2 ** 32))
        col = int(rng.integers(0, 16)) * 16
        for j in range(4):
            assert prmt(aw, col, 0x5504 | (j << 4)) == ((aw >> (8 * j)) & 0xFF) * 256 + col


@pytest.mark.parametrize("KC", (64, 32, 16))
def test_quarter_warp_bank_slots_distinct_for_any_data(KC):
    """PrCfg<KC>: S = 256/KC sources per step, NKC = KC/16 chunks, lane (jw, kc)
    = (ql / NKC, ql % NKC) of a quarter-warp reads row a (data) of the 256-B-row
    table at column ((jw + t) mod S) * KC + kc * 16 at sub-step t: the 16-B bank
    slot (address / 16 mod 8) of the 8 lanes is distinct whatever the rows are."""
    S, NKC = 256 // KC, KC // 16
    rng = np.random.default_rng(KC)
    for t in range(S):
        for _ in range(200):
            slots = set()
            for ql in range(8):
                jw, kc = ql // NKC, ql % NKC
                a = int(rng.integers(0, 256))
                addr = 0x1000 + a * 256 + ((jw + t) % S) * KC + kc * 16
                slots.add((addr // 16) % 8)
            assert len(slots) == 8


@pytest.mark.parametrize("KC", (64, 32, 16))
def test_sub_steps_cover_every_source_once(KC):
    S, NKC = 256 // KC, KC // 16
    for jw in range(8 // NKC):
        assert sorted((jw + t) % S for t in range(S)) == list(range(S))


@pytest.mark.parametrize("KC", (64, 32, 16))
def test_tile_geometry(KC):
    """Every (word, coefficient chunk) of a 384-word tile x KC coded packets is
    owned by exactly one (gatherer warp, lane, item): 12 warps, R items."""
    NKC, WQ = KC // 16, 8 // (KC // 16)
    WPW, GW, TW = 4 * WQ, 12, 384
    R = TW // (GW * WPW)
    owned = set()
    for warp in range(GW):
        for lane in range(32):
            qw, ql = lane >> 3, lane & 7
            jw, kc = ql // NKC, ql % NKC
            wbase = warp * WPW + qw * WQ + jw
            for r in range(R):
                owned.add((wbase + GW * WPW * r, kc))
    assert owned == {(w, c) for w in range(TW) for c in range(NKC)}


def test_writeback_transpose():
    """Eight PRMTs turn x_j = [B[k0+e][m_j] for e < 4] (j < 4) into
    y_e = [B[k0+e][m_0..3]]: a 4x4 byte transpose."""
    rng = np.random.default_rng(3)
    for _ in range(500):
        X = rng.integers(0, 256, size=(4, 4), dtype=np.uint8)   # X[j][e]
        x = [int(X[j].view(np.uint32)[0]) for j in range(4)]
        t0, t1 = prmt(x[0], x[1], 0x5140), prmt(x[0], x[1], 0x7362)
        t2, t3 = prmt(x[2], x[3], 0x5140), prmt(x[2], x[3], 0x7362)
        y = [prmt(t0, t2, 0x5410), prmt(t0, t2, 0x7632), prmt(t1, t3, 0x5410), prmt(t1, t3, 0x7632)]
        for e in range(4):
            assert np.array_equal(np.array([y[e]], dtype=np.uint32).view(np.uint8), X[:, e])


def test_smem_layout_fits():
    """Tables at 0x1000 + u * 0x10000 (u < 3), mbarriers at 0x400: the dynamic
    window [0x400, 0x31000) is <= 227 KiB (each producer thread derives its
    chunk's basis rows in registers: no basis buffer)."""
    end = 0x1000 + 3 * 0x10000
    assert end - 0x400 <= 227 * 1024
    assert 0x400 + 8 * 8 <= 0x1000


@pytest.mark.parametrize("TW", (512, 256))
def test_lanek_v2_gathers_conflict_free(TW):
    """encode_lanek.cuh LkGeom V2 (32 coded packets per CTA): Q row stride
    QS = TW + 2 (even, QS / 2 odd).  A half-warp's LDS.64 reads row r_k at word
    offset wg*WT + 2v: 16 lanes, rows from 16 values, land in 16 distinct 8-byte
    bank slots unless they read the same row (broadcast), for any rows; and
    rows are 8-byte aligned."""
    QS = TW + 2
    assert QS % 2 == 0 and (QS // 2) % 2 == 1
    rng = np.random.default_rng(TW)
    WT = TW // 8
    for wg in range(8):
        for v in range(0, WT // 2, 7):
            for _ in range(50):
                rows = rng.integers(0, 16, size=16)
                addr = {int(r): (int(r) * QS + wg * WT + 2 * v) * 4 for r in rows}   # distinct rows only
                assert all(a % 8 == 0 for a in addr.values())
                slots = [(a // 8) % 16 for a in addr.values()]
                assert len(set(slots)) == len(slots)
