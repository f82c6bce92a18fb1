#!/usr/bin/env python
"""One batched inversion (decode NEXT-3, C3 shape) for ncu: python tools/prof_invert.py [field] [gens]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1909_02871_b200 import gf  # noqa: E402

q = int(sys.argv[1]) if len(sys.argv) > 1 else 256
G = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
N = 64
gf.init(q)
C = torch.empty((G, N, N), dtype=torch.uint8, device="cuda")
gf.fill_random(C, 5, 2, 0, mask=q - 1)
for _ in range(2):
    D, rank = gf.invert_batch(q, C)
torch.cuda.synchronize()
print("ok", q, G, int(rank.sum()))
