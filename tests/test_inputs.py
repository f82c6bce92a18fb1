"""Pins for the seeded input generator (seeded_inputs), shared by both sides."""
import numpy as np

import seeded_inputs as si


def test_reference_splitmix64_sequence():
    """With key 0 the stream is the reference splitmix64 sequence from seed 0
    (published first outputs of Vigna's splitmix64.c)."""
    w = si.random_words(0, 0, 0, 3)
    assert [int(x) for x in w] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


def test_bytes_little_endian_and_addressable():
    b = si.random_bytes(0, 0, 0, 16)
    assert b[0] == 0xAF and b[7] == 0xE2 and b[8] == 0xF4
    full = si.random_bytes(123, 4, 0, 1000)
    for off in (0, 1, 7, 8, 13, 500):
        assert (si.random_bytes(123, 4, off, 100) == full[off:off + 100]).all()


def test_2d_slices():
    full = si.random_bytes(5, 1, 0, 40 * 30).reshape(40, 30)
    part = si.random_bytes_2d(5, 1, 3 * 30 + 7, 30, 10, 11)
    assert (part == full[3:13, 7:18]).all()


def test_streams_distinct():
    a = si.random_bytes(si.config_seed(3), si.STREAM_A, 0, 4096)
    c = si.random_bytes(si.config_seed(3), si.STREAM_C, 0, 4096)
    assert (a != c).mean() > 0.99


def test_coeff_draws():
    c = si.uniform_coeffs(16, 1, 2, 0, 100000)
    assert c.max() == 15 and abs(np.bincount(c).std() / np.bincount(c).mean()) < 0.05
    nz = si.rejection_coeffs(256, 1, si.config_seed(1), si.STREAM_C, 16)
    assert len(nz) == 16 and (nz >= 1).all()
    for q in (4, 16, 256):
        assert 2 <= si.c2_coeff(q) < q
    assert si.c2_coeff(2) == 1


def test_encode_inputs_shapes_and_slicing():
    cfg = si.C3
    A, C = si.encode_inputs(cfg, 256, 5, 7)
    assert A.shape == (2, 64, 1500) and C.shape == (2, 64, 64)
    A2, _ = si.encode_inputs(cfg, 256, 5, 7, 100, 160)
    assert (A2 == A[:, :, 100:160]).all()
    A1, C1 = si.encode_inputs(si.C1, 256)
    assert A1.shape == (1, 16, 1500) and (C1 != 0).all()


def test_c_fill_equals_numpy_definition():
    """seeded_inputs/fill.c (multithreaded, used for full-size host
    regeneration) is byte-equal to the numpy definition: 1-D ranges at every
    start alignment, lengths across the threaded split, 2-D strided slices,
    coefficient masks, and offsets past 2^32 bytes."""
    for seed, stream in ((0, 0), (190902871, 1), (2 ** 63 + 5, 7)):
        for off in (0, 1, 3, 7, 8, 9, 4095, (1 << 33) + 5):
            for n in (1, 7, 8, 4096, 4097, 70001):
                ref = si.random_bytes_np(seed, stream, off, n)
                out = np.empty(n, dtype=np.uint8)
                assert np.array_equal(si.fill_2d(out, seed, stream, off, n), ref), (seed, off, n)
                assert np.array_equal(si.random_bytes(seed, stream, off, n), ref)
    out = np.empty((37, 1500), dtype=np.uint8)
    si.fill_2d(out, 11, 1, 3 * 65536 + 13, 65536, threads=5)
    for r in (0, 17, 36):
        assert np.array_equal(out[r], si.random_bytes_np(11, 1, 3 * 65536 + 13 + r * 65536, 1500))
    m = np.empty((9, 33), dtype=np.uint8)
    si.fill_2d(m, 4, 2, 100, 33, mask=15)
    assert np.array_equal(m.reshape(-1), si.random_bytes_np(4, 2, 100, 9 * 33) & 15)
