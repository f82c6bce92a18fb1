"""CPU-side checks of the product library (no GPU compute calls):
the C ABI loads and exports every symbol include/gfrlnc.h declares, status
strings, and the host-built byte-permute tables -- emulating the kernels'
PRMT / bit-plane arithmetic in Python against the oracle's byte products
(the SURVEY.md 4 "fake backend")."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
from paper_1909_02871_b200 import gf

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gfrlnc.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gf_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported():
    syms = declared_symbols()
    assert len(syms) >= 10
    assert set(syms) == set(gf.ABI_SYMBOLS)
    L = gf.lib()
    for s in syms:
        assert hasattr(L, s), f"{s} not exported"


def test_status_strings_and_version():
    for code in range(-6, 1):
        assert gf.strerror(code) and gf.strerror(code) != "unknown status"
    assert gf.strerror(-99) == "unknown status"
    assert gf.version() >= 100


def test_host_tables_errors():
    L = gf.lib()
    buf = (ctypes.c_uint32 * (2 * gf.TABLE_WORDS))()
    assert L.gf_host_tables(3, buf, 8) == gf.GF_EFIELD
    assert L.gf_host_tables(256, buf, 8) == gf.GF_EARG        # capacity too small
    assert L.gf_host_tables(2, buf, 2 * gf.TABLE_WORDS) == gf.GF_OK


def test_abi_validation_without_gpu():
    """Argument errors are reported before any device work."""
    L = gf.lib()
    assert L.gf_init(3) == gf.GF_EFIELD
    assert L.gf_maddrc(5, None, None, 1, 16) == gf.GF_EFIELD
    assert L.gf_encode_batch(7, None, None, None, 1, 1, 1, 1) == gf.GF_EFIELD
    assert L.gf_encode_verify_batch(3, None, None, None, None, 1, 1, 1, 1, 1, None, None, 0) == gf.GF_EFIELD
    assert L.gf_set_verify_fault(1, 0, 4096, 0) == gf.GF_EARG           # k > 4095
    assert L.gf_set_verify_fault(1, 0, 3, 1 << 21) == gf.GF_EARG        # word > 2^20 - 1
    assert L.gf_set_verify_fault(0, 0, 0, 0) == gf.GF_OK
    assert gf.verify_workspace_bytes(64, 64, 65536) == 65536 * 2 * 64 + 65536 * 2 * 2 * 4
    assert gf.verify_workspace_bytes(256, 256, 3) == ((3 * 4 * 2 * 256 + 15) // 16) * 16 + 3 * 2 * 8 * 4


# ---- PRMT emulation ------------------------------------------------------------

def prmt(a, b, s):
    src = [(a >> (8 * i)) & 0xFF for i in range(4)] + [(b >> (8 * i)) & 0xFF for i in range(4)]
    out = 0
    for i in range(4):
        nib = (s >> (4 * i)) & 0xF
        v = src[nib & 7]
        if nib & 8:
            v = 0xFF if v & 0x80 else 0
        out |= v << (8 * i)
    return out


def make_sel(x):
    t0 = x & 0x07070707
    t1 = (x >> 3) & 0x07070707
    t2 = (x >> 6) & 0x03030303
    return [(t | (t >> 12)) & 0xFFFFFFFF for t in (t0, t1, t2)]


def lookup_word(T, x):
    s0, s1, s2 = make_sel(x)
    y = prmt(T[0], T[1], s0) ^ prmt(T[2], T[3], s1) ^ prmt(T[4], T[4], s2)
    return prmt(y, y, 0x3120)


@pytest.mark.parametrize("q", (2, 4, 16, 256))
def test_prmt_split_tables_match_oracle(q):
    """For every coefficient and every byte value in every byte position of a
    word, the emulated 3-PRMT lookup + un-permute equals the oracle product."""
    tabs = gf.host_tables(q)
    MB = oracle.mulbyte_table(q)
    rng = np.random.default_rng(q)
    vals = list(range(256))
    for c in range(q):
        T = tabs[c]
        for pos in range(4):
            for v in vals:
                x = (v << (8 * pos)) | (int(rng.integers(0, 2 ** 32)) & ~(0xFF << (8 * pos)) & 0xFFFFFFFF)
                y = lookup_word(T, x)
                assert (y >> (8 * pos)) & 0xFF == MB[c, v]
        # whole random words
        for _ in range(64):
            x = int(rng.integers(0, 2 ** 32))
            y = lookup_word(T, x)
            exp = sum(int(MB[c, (x >> (8 * i)) & 0xFF]) << (8 * i) for i in range(4))
            assert y == exp


def test_selectors_never_set_sign_mode():
    for x in (0, 0xFFFFFFFF, 0x80808080, 0x7F7F7F7F, 0x12345678):
        for s in make_sel(x):
            for i in range(4):
                assert not (s >> (4 * i)) & 0x8


def test_kernel_selector_packing_equals_shift_form():
    """gf_device.cuh make_sel: one AND + one IMAD.HI per group, multipliers
    c_selmul = {2^20, 2^29 + 2^17, 2^26 + 2^14} (parsed from the header), equals
    the shift-and-or selectors above in the 16 bits PRMT reads, for random and
    extreme words (the no-carry argument of the header comment)."""
    src = open(os.path.join(ROOT, "paper_1909_02871_b200", "csrc", "gf_device.cuh")).read()
    m = re.search(r"c_selmul\[3\]\s*=\s*\{([^}]*)\}", src)
    consts = [eval(e.replace("u", ""), {}) for e in m.group(1).split(",")]
    assert consts == [1 << 20, (1 << 29) | (1 << 17), (1 << 26) | (1 << 14)]
    rng = np.random.default_rng(5)
    x = np.concatenate([rng.integers(0, 2 ** 32, size=1 << 18, dtype=np.uint64),
                        np.array([0, 0xFFFFFFFF, 0x80808080, 0x7F7F7F7F, 0xC0C0C0C0, 0x38383838], dtype=np.uint64)])
    t0, t1, t2 = x & 0x07070707, x & 0x38383838, x & 0xC0C0C0C0
    got = [((t0 * consts[0]) >> 32) + t0, (t1 * consts[1]) >> 32, (t2 * consts[2]) >> 32]
    want = [((x >> s) & mk) | (((x >> s) & mk) >> 12) for s, mk in ((0, 0x07070707), (3, 0x07070707), (6, 0x03030303))]
    for g, w in zip(got, want):
        assert np.array_equal(g & 0xFFFF, w & 0xFFFF)
        assert not np.any(g & 0x8888)                     # never the sign-replicate mode


def gf4_xtime(a):
    hi = (a >> 1) & 0x55555555
    return hi | (((a & 0x55555555) ^ hi) << 1)


def test_gf4_bitplane_masks_match_oracle():
    tabs = gf.host_tables(4)
    MB = oracle.mulbyte_table(4)
    for c in range(4):
        m0, m1 = tabs[c][5], tabs[c][6]
        for v in range(256):
            x = v * 0x01010101
            y = (x & m0) ^ (gf4_xtime(x) & m1)
            assert y == int(MB[c, v]) * 0x01010101


def test_gf2_mask():
    tabs = gf.host_tables(2)
    assert tabs[0][5] == 0 and tabs[1][5] == 0xFFFFFFFF


# ---- imul (Alg. 2) emulation: the FMA-pipe half of the encode kernels --------

M32 = 0xFFFFFFFF
SLOT = {2: 0xFFFFFFFF, 4: 0x55555555, 16: 0x11111111, 256: 0x01010101}


def imul_word(q, tab, x):
    """XOR_j ((x >> j) & slot_mask) * pow[c][j], as IMAD + LOP3 do it."""
    w = oracle.width(q)
    r = 0
    for j in range(w):
        r ^= (((x >> j) & SLOT[q]) * tab[8 + j]) & M32
    return r


@pytest.mark.parametrize("q", (2, 4, 16, 256))
def test_imul_planes_match_oracle(q):
    """Carry-free plane products (reading X7: scalar constant per 32-bit lane)."""
    tabs = gf.host_tables(q)
    MB = oracle.mulbyte_table(q)
    rng = np.random.default_rng(7 + q)
    for c in range(q):
        assert tabs[c][8:8 + oracle.width(q)] == [oracle.mul(q, c, 1 << j) for j in range(oracle.width(q))]
        for _ in range(256):
            x = int(rng.integers(0, 2 ** 32))
            exp = sum(int(MB[c, (x >> (8 * i)) & 0xFF]) << (8 * i) for i in range(4))
            assert imul_word(q, tabs[c], x) == exp


def test_gf256_hybrid_prmt_imul_matches_oracle():
    """Encode engine for GF(256): bits 0-5 by PRMT (permuted byte order),
    bits 6-7 by IMAD on the byte-permuted word, one final un-permute."""
    tabs = gf.host_tables(256)
    MB = oracle.mulbyte_table(256)
    rng = np.random.default_rng(11)
    for c in range(256):
        T = tabs[c]
        for _ in range(32):
            x = int(rng.integers(0, 2 ** 32))
            s0, s1, _ = make_sel(x)
            xp = prmt(x, x, 0x3120)
            b6 = (xp >> 6) & 0x01010101
            b7 = (xp >> 7) & 0x01010101
            acc = prmt(T[0], T[1], s0) ^ prmt(T[2], T[3], s1) ^ ((b6 * T[14]) & M32) ^ ((b7 * T[15]) & M32)
            y = prmt(acc, acc, 0x3120)
            assert y == sum(int(MB[c, (x >> (8 * i)) & 0xFF]) << (8 * i) for i in range(4))


def test_gf16_permuted_imul_matches_prmt_order():
    tabs = gf.host_tables(16)
    rng = np.random.default_rng(12)
    for c in range(16):
        for _ in range(32):
            x = int(rng.integers(0, 2 ** 32))
            xp = prmt(x, x, 0x3120)
            s0, s1, s2 = make_sel(x)
            T = tabs[c]
            assert imul_word(16, T, xp) == prmt(T[0], T[1], s0) ^ prmt(T[2], T[3], s1) ^ prmt(T[4], T[4], s2)


def test_encode_path_query():
    assert gf.encode_path(256, 64, 64, 1500) == "prow"          # C3
    assert gf.encode_path(16, 64, 64, 1500) == "prow-nib"       # C3 GF(16): nibble tables
    assert gf.encode_path(256, 256, 256, 65536) == "prow-32w"   # C4: 768-word tiles
    assert gf.encode_path(256, 64, 64, 8192) == "prow"          # 2048 words: < 8 tiles of 768
    assert gf.encode_path(256, 64, 64, 4 * 6200) == "prow"      # 768-word tiles would cover 6200 words at 89.7%
    assert gf.encode_path(256, 64, 64, 4 * 7000) == "prow-32w"  # 91.1%
    assert gf.encode_path(16, 256, 256, 65536) == "prow-nib"
    assert gf.encode_path(256, 64, 32, 1500) == "prow-32"
    assert gf.encode_path(16, 32, 16, 1500) == "prow-16"
    assert gf.encode_path(256, 16, 8, 1500) == "column-words"
    assert gf.encode_path(4, 32, 32, 1500) == "lanek-32"
    # GF(4), 9 <= K < 24: product rows when tiles cover >= 85% and (K > 16 or M >= 4 KiB)
    assert gf.encode_path(4, 32, 20, 1500) == "prow-32"
    assert gf.encode_path(4, 32, 20, 2052) == "column-words"      # 2 tiles for 513 words: 67%
    assert gf.encode_path(4, 32, 12, 4100) == "prow-16"
    assert gf.encode_path(4, 32, 12, 1500) == "column-words"
    assert gf.encode_path(2, 32, 20, 4100) == "column-words"
    assert gf.encode_path(2, 32, 20, 4096) == "tmem"
    assert gf.encode_path(2, 32, 8, 4096) == "column-words"     # K = 8: the column kernel
    assert gf.encode_path(4, 64, 64, 1500) == "lanek-64"
    assert gf.encode_path(4, 64, 64, 4096) == "tmem"
    assert gf.encode_path(2, 32, 32, 1 << 20) == "tmem"         # C5 GF(2): TMEM lookup tables
    assert gf.encode_path(4, 32, 32, 1 << 20) == "tmem"         # C5 GF(4)
    assert gf.encode_path(2, 33, 32, 1 << 20) == "tmem"         # GF(2), N > 32
    assert gf.encode_path(4, 32, 32, 1 << 20, a_align=8) == "lanek-32"   # TMEM engine: 16-byte aligned
    assert gf.encode_path(4, 32, 32, 4096 + 8) == "lanek-32"    # ... and M % 16 == 0
    assert gf.encode_path(2, 32, 32, 240) == "gf2-split"        # M < 256: the split engine
    assert gf.encode_path(2, 33, 32, 240) == "lanek-32"         # GF(2), N > 32, short packets
    assert gf.encode_path(4, 32, 16, 1 << 20) == "tmem"
    assert gf.encode_path(16, 32, 32, 1 << 20) == "tmem"        # GF(16), 24 <= K <= 32
    assert gf.encode_path(16, 32, 16, 1 << 20) == "prow-16"    # 13 <= K <= 16, >= 8 KiB
    assert gf.encode_path(16, 32, 16, 1024) == "tmem"
    assert gf.encode_path(16, 16, 8, 65536) == "tmem"
    assert gf.encode_path(16, 16, 8, 1500) == "column-words"
    assert gf.encode_path(16, 32, 64, 1 << 20) == "tmem"        # K > 32, N <= 32
    assert gf.encode_path(16, 64, 64, 1 << 20) == "prow-nib"
    assert gf.encode_path(256, 32, 32, 1 << 20) == "prow-32"    # GF(256) keeps the product rows
    assert gf.encode_path(2, 32, 32, 1500) == "lanek-32"        # GF(2), M % 16 != 0
    assert gf.encode_path(2, 32, 32, 4096, a_align=4) == "lanek-32"
    assert gf.encode_path(2, 16, 24, 128) == "gf2-split"
    assert gf.encode_path(2, 16, 24, 4096) == "tmem"
    assert gf.encode_path(256, 16, 1, 1024) == "stream"         # NEXT-2 (paper: N = 16, K = 1)
    assert gf.encode_path(2, 16, 4, 65536) == "stream"
    assert gf.encode_path(256, 16, 1, 1024, a_align=4) == "stream"    # 4-byte chunks
    assert gf.encode_path(256, 16, 1, 1500) == "stream"                # C1 (M % 16 != 0)
    assert gf.encode_path(256, 16, 1, 1500, a_align=2) == "column-bytes"
    assert gf.encode_path(256, 16, 5, 1024) == "column-words"
    assert gf.encode_path(256, 16, 8, 1500) == "column-words"
    assert gf.encode_path(4, 3, 5, 13) == "column-bytes"
    assert gf.encode_path(256, 64, 64, 1500, a_align=1) == "column-bytes"
    with pytest.raises(gf.GFError):
        gf.encode_path(3, 1, 1, 4)


@pytest.mark.parametrize("q", (4, 16, 256))
def test_corrupted_table_is_caught(q):
    """SURVEY 4 negative test: one flipped bit in one coefficient's
    split table makes the table-identity check (the emulated 3-PRMT lookup
    against the oracle's products) fail."""
    tabs = [list(t) for t in gf.host_tables(q)]
    MB = oracle.mulbyte_table(q)
    c = q - 1
    tabs[c][1] ^= 1 << 9                        # T0[5] (byte 1 of word 1), bit 1
    bad = 0
    for v in range(256):
        x = v * 0x01010101
        y = lookup_word(tabs[c], x)
        bad += y != int(MB[c, v]) * 0x01010101
    assert bad > 0
