"""Every encode kernel and streaming layout the router can pick, forced through
the thread-local harness setter gf_set_encode_path (nothing is read from the
environment), against the oracle, with B inside guard bytes."""
import numpy as np
import pytest
import torch

import oracle
import seeded_inputs as si

pytestmark = pytest.mark.gpu

ALL = (2, 4, 16, 256)
GENERIC = ((17, 33, 1500, 3), (64, 64, 1500, 2), (32, 32, 4100, 2), (5, 24, 400, 3), (33, 96, 3000, 2),
           (7, 65, 1540, 2))
STREAM = ((16, 1, 1024, 50), (16, 1, 128, 300), (5, 2, 4096, 3), (17, 3, 2064, 4), (64, 4, 16, 100),
          (1, 1, 16, 10), (16, 1, 1500, 7), (9, 3, 1028, 5), (3, 4, 4, 33), (16, 1, 1500, 700),
          (7, 2, 516, 40), (16, 4, 2052, 9))
CASES = {
    "column": [(q, s) for q in ALL for s in GENERIC],
    "lanek": [(q, s) for q in ALL for s in GENERIC],
    "prow": [(q, s) for q in ALL for s in GENERIC] +
            [(q, s) for q in (16, 256) for s in ((1, 64, 1500, 5), (3, 1, 1536, 9), (4, 70, 4, 400),
                                                 (19, 12, 1500, 3), (16, 16, 16384, 2), (40, 9, 388, 7),
                                                 (33, 65, 28000, 2), (5, 40, 24576, 2))],
    # GF(2) split engine: N <= 32, 16-byte multiple packets (ragged last span,
    # N < 16 and 16 < N < 32 instances, K from 1 to 96)
    "gf2": [(2, s) for s in ((32, 32, 4096, 3), (17, 33, 1504, 3), (5, 24, 400, 3), (32, 1, 512, 4),
                             (1, 9, 16, 5), (16, 16, 2064, 2), (31, 96, 1040, 2), (32, 32, 65536, 2),
                             (12, 40, 528, 6))],
    # TMEM lookup-table engine (any field; M % 16 == 0): ragged last span
    # (M % 256 != 0), partial last 4-bit group (N w % 16 != 0), one to three
    # passes of 32 coded packets, K % 32 != 0, four-word packets
    "tmem": [(q, s) for q in ALL for s in ((32, 32, 4096, 3), (17, 33, 1504, 3), (5, 24, 400, 3), (1, 1, 16, 5),
                                           (3, 70, 2064, 2), (33, 64, 65552, 1), (8, 40, 272, 7),
                                           (32, 96, 1008, 2), (2, 5, 16, 9))] +
            [(q, s) for q in (2, 4, 16) for s in ((64, 96, 1008, 2), (64, 64, 1504, 4))],
}
for name in ("stream", "stream-strided4", "stream-strided8", "stream-strided12", "stream-wide2",
             "stream-wide4"):
    CASES[name] = [(q, s) for q in ALL for s in STREAM]
PREFIX = {"column": "column", "lanek": "lanek", "prow": "prow", "gf2": "gf2", "tmem": "tmem"}


@pytest.fixture(scope="module")
def gfm():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1909_02871_b200 import gf
    for q in ALL:
        gf.init(q)
    return gf


@pytest.mark.parametrize("path", sorted(CASES))
def test_forced_encode_path(gfm, path):
    want = PREFIX.get(path, "stream")
    try:
        gfm.set_encode_path(path)
        for q, (N, K, M, batch) in CASES[path]:
            A = si.random_bytes(7 + N, 1, 0, batch * N * M).reshape(batch, N, M)
            C = si.uniform_coeffs(q, 8 + K, 2, 0, batch * N * K).reshape(batch, N, K)
            got_path = gfm.encode_path(q, N, K, M)
            assert got_path.startswith(want), (got_path, path, q, N, K, M)
            nb = batch * K * M
            buf = torch.full((nb + 8192,), 0xEE, dtype=torch.uint8, device="cuda")
            gfm.encode_batch(q, torch.from_numpy(A).cuda(), torch.from_numpy(C).cuda(),
                             buf[4096:4096 + nb].view(batch, K, M))
            allb = buf.cpu().numpy()
            assert (allb[:4096] == 0xEE).all() and (allb[4096 + nb:] == 0xEE).all(), ("guard", q, N, K, M)
            got = allb[4096:4096 + nb].reshape(batch, K, M)
            assert np.array_equal(got, oracle.encode_batch(q, A, C)), (path, q, N, K, M)
    finally:
        gfm.set_encode_path("auto")


def test_forced_path_is_thread_local(gfm):
    """A forced path set on one thread does not leak into another."""
    import threading
    seen = {}
    gfm.set_encode_path("column")
    try:
        def other():
            seen["other"] = gfm.encode_path(256, 64, 64, 1500)
        t = threading.Thread(target=other)
        t.start()
        t.join()
        assert gfm.encode_path(256, 64, 64, 1500) == "column-words"
        assert seen["other"] == "prow"
    finally:
        gfm.set_encode_path("auto")
