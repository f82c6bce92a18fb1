#!/usr/bin/env python
"""Median device time (CUDA events) of gf_encode_batch for one shape:
    python tools/time_encode.py q N K M G [reps]"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1909_02871_b200 import gf  # noqa: E402

q, N, K, M, G = (int(x) for x in sys.argv[1:6])
reps = int(sys.argv[6]) if len(sys.argv) > 6 else 20
gf.init(q)
A = torch.empty((G, N, M), dtype=torch.uint8, device="cuda")
C = torch.empty((G, N, K), dtype=torch.uint8, device="cuda")
B = torch.empty((G, K, M), dtype=torch.uint8, device="cuda")
gf.fill_random(A, 5, 1, 0)
gf.fill_random(C, 5, 2, 0, mask=q - 1)
for _ in range(3):
    gf.encode_batch(q, A, C, B)
ts = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    gf.encode_batch(q, A, C, B)
    e1.record()
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = statistics.median(ts)
print(f"GF({q}) N={N} K={K} M={M} G={G} path={gf.encode_path(q, N, K, M)} {ms * 1e3:.1f} us "
      f"{G * N * M / ms / 1e6:.1f} GB/s")
