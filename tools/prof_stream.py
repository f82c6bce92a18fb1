#!/usr/bin/env python
"""One NEXT-2 shaped encode (N=16, K=1, M bytes, ~2 GiB of source) for ncu:
    python tools/prof_stream.py [field] [M] [launches]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1909_02871_b200 import gf  # noqa: E402

q = int(sys.argv[1]) if len(sys.argv) > 1 else 256
M = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
launches = int(sys.argv[3]) if len(sys.argv) > 3 else 2
N, K = 16, 1
G = (2 << 30) // (N * M)
gf.init(q)
A = torch.empty((G, N, M), dtype=torch.uint8, device="cuda")
C = torch.empty((G, N, K), dtype=torch.uint8, device="cuda")
gf.fill_random(A, 7, 1, 0)
gf.fill_random(C, 7, 2, 0, mask=q - 1)
for _ in range(launches):
    B = gf.encode_batch(q, A, C)
torch.cuda.synchronize()
print("ok", q, M, G, gf.encode_path(q, N, K, M), int(B[0, 0, 0]))
