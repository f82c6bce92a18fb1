#!/usr/bin/env python
"""Tiny launches of every encode kernel, each checked against the oracle, sized
for compute-sanitizer (memcheck / racecheck / synccheck) where the pool allows it
(it does not on the current one): python tools/sanitize_small.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import seeded_inputs as si  # noqa: E402
from paper_1909_02871_b200 import gf  # noqa: E402

cases = [("prow", 256, (9, 40, 1500, 2)), ("prow", 16, (5, 20, 1028, 2)), ("prow", 256, (33, 12, 400, 3)),
         ("lanek", 2, (9, 32, 2048, 2)), ("lanek", 4, (6, 30, 1024, 2)), ("stream", 256, (16, 1, 1024, 3)),
         ("stream", 16, (5, 3, 1500, 2)), ("column", 256, (16, 8, 1500, 2)), ("gf2", 2, (32, 32, 2048, 2)),
         ("gf2", 2, (9, 24, 528, 2))]
for path, q, (N, K, M, batch) in cases:
    gf.init(q)
    gf.set_encode_path(path)
    A = si.random_bytes(3, 1, 0, batch * N * M).reshape(batch, N, M)
    C = si.uniform_coeffs(q, 4, 2, 0, batch * N * K).reshape(batch, N, K)
    got = gf.encode_batch(q, torch.from_numpy(A).cuda(), torch.from_numpy(C).cuda()).cpu().numpy()
    ok = np.array_equal(got, oracle.encode_batch(q, A, C))
    print(path, gf.encode_path(q, N, K, M), q, (N, K, M, batch), "ok" if ok else "MISMATCH", flush=True)
gf.set_encode_path("auto")
gf.init(256)
Cm = torch.from_numpy(si.uniform_coeffs(256, 5, 2, 0, 9 * 64 * 64).reshape(9, 64, 64)).cuda()
D, rank = gf.invert_batch(256, Cm)
print("invert ok", int(rank.sum()))
Cm = torch.from_numpy(si.uniform_coeffs(256, 6, 2, 0, 3 * 80 * 80).reshape(3, 80, 80)).cuda()
D, rank = gf.invert_batch(256, Cm)                     # CTA-per-matrix inversion (N > 64)
print("invert cta ok", int(rank.sum()))
for q, (N, K, M, batch) in ((256, (64, 64, 1500, 2)), (2, (32, 32, 2048, 2))):
    A = si.random_bytes(7, 1, 0, batch * N * M).reshape(batch, N, M)
    C = si.uniform_coeffs(q, 8, 2, 0, batch * N * K).reshape(batch, N, K)
    R = si.random_bytes(9, 5, 0, batch * K * 2).reshape(batch, K, 2)
    B, mism = gf.encode_verify_batch(q, *(torch.from_numpy(x).cuda() for x in (A, C, R)))
    print("fused verify", q, "ok" if np.array_equal(B.cpu().numpy(), oracle.encode_batch(q, A, C)) else "MISMATCH",
          int(mism.sum()), flush=True)
