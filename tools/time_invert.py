#!/usr/bin/env python
"""Device time of gf_invert_batch and gf_decode_batch at the C3 decode shape
(N = 64, 1500-byte packets):  python tools/time_invert.py [q] [gens] [N]"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1909_02871_b200 import gf  # noqa: E402

q = int(sys.argv[1]) if len(sys.argv) > 1 else 256
G = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
N = int(sys.argv[3]) if len(sys.argv) > 3 else 64
M = 1500
gf.init(q)
C = torch.empty((G, N, N), dtype=torch.uint8, device="cuda")
gf.fill_random(C, 5, 2, 0, mask=q - 1)
B = torch.empty((G, N, M), dtype=torch.uint8, device="cuda")
gf.fill_random(B, 5, 1, 0)


def med(fn, reps=10):
    for _ in range(2):
        fn()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


ti = med(lambda: gf.invert_batch(q, C))
td = med(lambda: gf.decode_batch(q, B, C))
D, rank = gf.invert_batch(q, C)
print(f"GF({q}) N={N} G={G}: invert {ti:.3f} ms, decode {td:.3f} ms ({G * N * M / td / 1e6:.1f} GB/s of coded "
      f"input), full rank {int((rank == N).sum())}/{G}")
