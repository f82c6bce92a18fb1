#!/usr/bin/env python
"""One encode launch of a BASELINE workload (for ncu captures):
    python tools/prof_encode.py C3 256 [gens] [launches]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import seeded_inputs as si  # noqa: E402
from paper_1909_02871_b200 import gf  # noqa: E402

name, q = sys.argv[1], int(sys.argv[2])
cfg = si.ENCODE_CONFIGS[name]
G = int(sys.argv[3]) if len(sys.argv) > 3 else cfg.batch
launches = int(sys.argv[4]) if len(sys.argv) > 4 else 2
gf.init(q)
A = torch.empty((G, cfg.N, cfg.M), dtype=torch.uint8, device="cuda")
C = torch.empty((G, cfg.N, cfg.K), dtype=torch.uint8, device="cuda")
seed = si.field_seed(cfg, q)
gf.fill_random(A, seed, si.STREAM_A, 0)
gf.fill_random(C, seed, si.STREAM_C, 0, mask=q - 1)
for _ in range(launches):
    B = gf.encode_batch(q, A, C)
torch.cuda.synchronize()
print("ok", name, q, G, int(B[0, 0, 0]))
