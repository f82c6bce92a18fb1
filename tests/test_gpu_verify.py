"""On-device Freivalds check: agrees with the oracle's
projection counts, and verifies EVERY generation of the full-size C3/C4 and a
C5 chunk (the lane-k results, checked through the column kernels)."""
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


@pytest.mark.parametrize("q", FIELDS)
def test_verify_counts_match_oracle(gfm, q):
    batch, N, K, M = 6, 9, 7, 333
    t = oracle.freivalds_trials(q)
    A = si.random_bytes(11, 1, 0, batch * N * M).reshape(batch, N, M)
    C = si.uniform_coeffs(q, 12, 2, 0, batch * N * K).reshape(batch, N, K)
    R = si.uniform_coeffs(q, 13, si.STREAM_FREIVALDS, 0, batch * K * t).reshape(batch, K, t)
    B = oracle.encode_batch(q, A, C)
    B[2, 3, 17] ^= 0x41
    B[4, 0, 0] ^= 0x01
    got = gfm.verify_batch(q, *(torch.from_numpy(x).cuda() for x in (A, C, B, R))).cpu().numpy()
    for g in range(batch):
        exp = sum(oracle.freivalds_gen(q, A[g], C[g], B[g], R[g][:, j].copy()) for j in range(t))
        assert got[g] == exp, g
    assert got[0] == 0 and got[2] > 0 and got[4] > 0


def _device_inputs(gfm, cfg, q, G, g0=0):
    seed = si.field_seed(cfg, q)
    A = torch.empty((G, cfg.N, cfg.M), dtype=torch.uint8, device="cuda")
    C = torch.empty((G, cfg.N, cfg.K), dtype=torch.uint8, device="cuda")
    gfm.fill_random(A, seed, si.STREAM_A, g0 * cfg.N * cfg.M)
    gfm.fill_random(C, seed, si.STREAM_C, g0 * cfg.N * cfg.K, mask=q - 1)
    return A, C


@pytest.mark.parametrize("name,q,G", [("C3", 256, 65536), ("C3", 16, 65536), ("C4", 256, 2048),
                                      ("C5", 2, 256), ("C5", 4, 256)])
def test_full_size_freivalds_every_generation(gfm, name, q, G):
    cfg = si.ENCODE_CONFIGS[name]
    t = oracle.freivalds_trials(q)
    free, _ = torch.cuda.mem_get_info()
    need = G * ((cfg.N + cfg.K) * cfg.M + cfg.N * cfg.K) + G * (cfg.N * t + 2 * t * cfg.M)
    if free < 1.1 * need:
        pytest.skip("not enough device memory")
    A, C = _device_inputs(gfm, cfg, q, G)
    B = gfm.encode_batch(q, A, C)
    R = torch.from_numpy(si.uniform_coeffs(q, cfg.seed, si.STREAM_FREIVALDS, 0, G * cfg.K * t)
                         .reshape(G, cfg.K, t)).cuda()
    mism = gfm.verify_batch(q, A, C, B, R)
    assert int(mism.sum()) == 0
    B[G // 2, cfg.K - 1, cfg.M // 3] ^= 0x80          # one corrupted byte is caught
    mism = gfm.verify_batch(q, A, C, B, R).cpu().numpy()
    assert mism[G // 2] > 0 and mism.sum() == mism[G // 2]
    del A, B, C, R
    torch.cuda.empty_cache()
