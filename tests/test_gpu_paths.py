"""Every encode kernel, forced through GFRLNC_ENCODE_PATH in a fresh process
(the library reads the override once), against the oracle."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import sys, numpy as np, torch
sys.path.insert(0, %r)
import oracle, seeded_inputs as si
from paper_1909_02871_b200 import gf
want = sys.argv[1]
if want == "lanek2":       # persistent lane-k: GF(2)/GF(4), K <= 32
    cases = [(q, s) for q in (2, 4) for s in ((17, 32, 1500, 3), (32, 32, 4100, 2), (5, 24, 400, 3),
                                              (7, 9, 1540, 2), (33, 32, 2052, 2), (32, 32, 65536, 2), (4, 1, 2048, 300))]
elif want == "stream":    # few coded packets, 16-byte aligned packets (the paper's N = 16, K = 1)
    cases = [(q, s) for q in (2, 4, 16, 256) for s in ((16, 1, 1024, 50), (16, 1, 128, 300), (5, 2, 4096, 3),
                                                       (17, 3, 2064, 4), (64, 4, 16, 100), (1, 1, 16, 10),
                                                       (16, 1, 1500, 7), (9, 3, 1028, 5), (3, 4, 4, 33),
                                                       (16, 1, 1500, 700), (7, 2, 516, 40), (16, 4, 2052, 9))]
else:
    cases = [(q, s) for q in (2, 4, 16, 256) for s in ((17, 33, 1500, 3), (64, 64, 1500, 2), (32, 32, 4100, 2),
                                                       (5, 24, 400, 3), (33, 96, 3000, 2), (7, 65, 1540, 2))]
    if want == "prow":     # one-step tiles (N <= 4), a single coded packet, many small tiles
        cases += [(q, s) for q in (16, 256) for s in ((1, 64, 1500, 5), (3, 1, 1536, 9), (4, 70, 4, 400),
                                                     (19, 12, 1500, 3), (16, 16, 16384, 2), (40, 9, 388, 7))]
for q, (N, K, M, batch) in cases:
    gf.init(q)
    A = si.random_bytes(7 + N, 1, 0, batch * N * M).reshape(batch, N, M)
    C = si.uniform_coeffs(q, 8 + K, 2, 0, batch * N * K).reshape(batch, N, K)
    path = gf.encode_path(q, N, K, M)
    assert path.startswith(want), (path, want)
    # B inside 0xEE guard bytes: no kernel may write outside its output
    nb = batch * K * M
    buf = torch.full((nb + 8192,), 0xEE, dtype=torch.uint8, device="cuda")
    gf.encode_batch(q, torch.from_numpy(A).cuda(), torch.from_numpy(C).cuda(), buf[4096:4096 + nb].view(batch, K, M))
    allb = buf.cpu().numpy()
    assert (allb[:4096] == 0xEE).all() and (allb[4096 + nb:] == 0xEE).all(), ("guard", q, N, K, M, path)
    got = allb[4096:4096 + nb].reshape(batch, K, M)
    assert np.array_equal(got, oracle.encode_batch(q, A, C)), (q, N, K, M, path)
print("ok", want)
''' % ROOT


@pytest.mark.parametrize("path", ["column", "lanek", "fused", "prow", "lanek2", "stream", "stream-strided",
                                  "stream-strided8", "stream-strided12", "stream-wide2", "stream-wide4"])
def test_forced_encode_path(path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, GFRLNC_ENCODE_PATH=path)
    if path.startswith("stream-strided"):   # word-aligned packets through the strided kernel at any size
        wmax = path[len("stream-strided"):] or "4"
        path = "stream"
        env.update(GFRLNC_ENCODE_PATH=path, GFRLNC_STREAM_STRIDED_MIN_WORDS="1", GFRLNC_STREAM_STRIDED_W=wmax)
    if path in ("stream-wide2", "stream-wide4"):   # 16-byte-aligned packets, 2 / 4 chunks per thread, any size
        w4 = "1" if path == "stream-wide4" else "0"
        path = "stream"
        env.update(GFRLNC_ENCODE_PATH=path, GFRLNC_STREAM_WIDE2_MIN_CHUNKS="1", GFRLNC_STREAM_WIDE4=w4)
    out = subprocess.run([sys.executable, "-c", SCRIPT, path], env=env, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    assert ("ok " + path) in out.stdout
