"""Full-size parity at SURVEY.md 8(c) c.4's pins, in the launch configuration
bench.py times, against the CPU oracle on host-regenerated inputs:

  * C3 (65536 generations, GF(16) and GF(256)): EVERY byte of every
    generation, oracle.encode_batch on all host cores;
  * C4 (2048 generations, 64 KiB packets) and the whole C5 job (4096
    generations of 32 x 1 MiB, GF(2) and GF(4), in the bench's 256-generation
    chunks): >= 1% of the generations compared byte for byte with the oracle,
    plus the oracle's Freivalds projection check (oracle.freivalds_gen, Eq. 2
    PAPER.md:84-88 projected on random r) over EVERY generation.

Inputs are generated on the device by absolute index (gf_fill_random, shown
byte-equal to seeded_inputs in test_gpu_parity) and regenerated on the host by
seeded_inputs' C fill (pinned to the numpy definition in test_inputs).  No
expected value comes from the CUDA path.  Host projections per generation:
t = 2 (a systematic error confined to one coded packet escapes with
probability q^-2 per generation, over thousands of generations).
"""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
import torch

import oracle
import seeded_inputs as si

pytestmark = pytest.mark.gpu

CORES = len(os.sched_getaffinity(0))
T_HOST = 2


@pytest.fixture(scope="module")
def gfm():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1909_02871_b200 import gf
    for q in (2, 4, 16, 256):
        gf.init(q)
    return gf


@pytest.fixture(scope="module")
def pool():
    with ThreadPoolExecutor(max_workers=CORES) as ex:     # ctypes releases the GIL
        yield ex


def device_job(gfm, cfg, q, g0, G):
    seed = si.field_seed(cfg, q)
    A = torch.empty((G, cfg.N, cfg.M), dtype=torch.uint8, device="cuda")
    C = torch.empty((G, cfg.N, cfg.K), dtype=torch.uint8, device="cuda")
    gfm.fill_random(A, seed, si.STREAM_A, g0 * cfg.N * cfg.M)
    gfm.fill_random(C, seed, si.STREAM_C, g0 * cfg.N * cfg.K, mask=q - 1)
    return A, C, gfm.encode_batch(q, A, C)


def host_exact(pool, q, Ah_g, Ch_g, Bh_g, block):
    """Every byte of one generation against the oracle, computed as parallel
    column blocks (oracle.encode_gen_cols; a block's rows stay in cache).
    Returns the number of mismatching bytes."""
    M = Ah_g.shape[1]

    def one(m0):
        m1 = min(M, m0 + block)
        return int(np.count_nonzero(oracle.encode_gen_cols(q, Ah_g, Ch_g, m0, m1) != Bh_g[:, m0:m1]))
    return sum(pool.map(one, range(0, M, block)))


def to_host(B, g0, g1, pinned):
    """B[g0:g1] through a pinned staging buffer (pageable D2H is several times slower)."""
    n = g1 - g0
    pinned[:n].copy_(B[g0:g1])
    return pinned[:n].numpy()


def host_freivalds(pool, cfg, q, g0, Ah, Ch, Bh):
    """oracle.freivalds_gen over every generation of a host chunk, T_HOST
    projections each (r from the seeded Freivalds stream by absolute index);
    returns the total number of mismatching byte positions."""
    seed = si.field_seed(cfg, q)
    G = Ah.shape[0]
    R = si.uniform_coeffs(q, seed, si.STREAM_FREIVALDS, g0 * T_HOST * cfg.K, G * T_HOST * cfg.K)
    R = R.reshape(G, T_HOST, cfg.K)

    def one(g):
        return sum(oracle.freivalds_gen(q, Ah[g], Ch[g], Bh[g], R[g, j].copy()) for j in range(T_HOST))
    return sum(pool.map(one, range(G)))


@pytest.mark.parametrize("q", (16, 256))
def test_c3_every_generation_vs_oracle(gfm, q):
    cfg = si.C3
    A, C, B = device_job(gfm, cfg, q, 0, cfg.batch)
    del A, C
    step = 4096
    for g0 in range(0, cfg.batch, step):
        Ah, Ch = si.encode_inputs(cfg, q, g0, g0 + step)
        exp = oracle.encode_batch(q, Ah, Ch, threads=CORES)
        got = B[g0:g0 + step].cpu().numpy()
        bad = int(np.count_nonzero(got != exp))
        assert bad == 0, (q, g0, bad)
    del B
    torch.cuda.empty_cache()


def test_c4_one_percent_exact_and_freivalds_every_generation(gfm, pool):
    cfg, q = si.C4, 256
    free, _ = torch.cuda.mem_get_info()
    need = cfg.batch * (cfg.N + cfg.K) * cfg.M + cfg.batch * cfg.N * cfg.K
    if free < need * 1.05:
        pytest.skip(f"needs {need / 2**30:.1f} GiB")
    A, C, B = device_job(gfm, cfg, q, 0, cfg.batch)
    del A, C
    exact = sorted({0, cfg.batch - 1, *range(7, cfg.batch, 107)})         # 21 of 2048 = 1.03%
    assert len(exact) / cfg.batch >= 0.01
    step = 32
    pinned = torch.empty((step, cfg.K, cfg.M), dtype=torch.uint8).pin_memory()
    checked = bad_exact = bad_proj = 0
    for g0 in range(0, cfg.batch, step):
        Ah, Ch = si.encode_inputs(cfg, q, g0, g0 + step)
        Bh = to_host(B, g0, g0 + step, pinned)
        bad_proj += host_freivalds(pool, cfg, q, g0, Ah, Ch, Bh)
        for g in (g for g in exact if g0 <= g < g0 + step):
            bad_exact += host_exact(pool, q, Ah[g - g0], Ch[g - g0], Bh[g - g0], 4096)
            checked += 1
    assert checked == len(exact) and bad_exact == 0 and bad_proj == 0
    del B
    torch.cuda.empty_cache()


@pytest.mark.parametrize("q", (2, 4))
def test_c5_whole_job_one_percent_exact_and_freivalds_every_generation(gfm, pool, q):
    """The whole 4096-generation C5 job in the bench's 256-generation launches
    (the GF(2) split engine / the GF(4) lane-k kernel)."""
    cfg = si.C5
    chunk, step = 256, 16
    exact = set(range(5, cfg.batch, 103)) | {0, cfg.batch - 1}              # 42 of 4096 = 1.03%
    assert len(exact) / cfg.batch >= 0.01
    pinned = torch.empty((step, cfg.K, cfg.M), dtype=torch.uint8).pin_memory()
    checked = bad_exact = bad_proj = 0
    for c0 in range(0, cfg.batch, chunk):
        A, C, B = device_job(gfm, cfg, q, c0, chunk)
        del A, C
        for g0 in range(c0, c0 + chunk, step):
            Ah, Ch = si.encode_inputs(cfg, q, g0, g0 + step)
            Bh = to_host(B, g0 - c0, g0 - c0 + step, pinned)
            bad_proj += host_freivalds(pool, cfg, q, g0, Ah, Ch, Bh)
            for g in (g for g in exact if g0 <= g < g0 + step):
                bad_exact += host_exact(pool, q, Ah[g - g0], Ch[g - g0], Bh[g - g0], 16384)
                checked += 1
        del B
        torch.cuda.empty_cache()
    assert checked == len(exact) and bad_exact == 0 and bad_proj == 0


def test_host_freivalds_catches_a_single_wrong_byte(gfm, pool):
    """The host projection pass above detects one flipped byte in one coded
    packet of one generation (its escape probability is q^-T_HOST)."""
    cfg = si.C5
    q = 4
    A, C, B = device_job(gfm, cfg, q, 100, 4)
    Bh = B.cpu().numpy()
    Ah, Ch = si.encode_inputs(cfg, q, 100, 104)
    assert host_freivalds(pool, cfg, q, 100, Ah, Ch, Bh) == 0
    Bh[2, 31, 777777] ^= 0x40
    assert host_freivalds(pool, cfg, q, 100, Ah, Ch, Bh) > 0
