#!/usr/bin/env python
"""Source GB/s of gf_encode_batch for assorted (N, K, M) shapes and every
applicable forced kernel (CUDA events, median of 10): python tools/exp_shapes.py"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1909_02871_b200 import gf  # noqa: E402

SHAPES = [(16, 8, 1500), (16, 12, 1500), (16, 16, 1500), (32, 16, 1500), (32, 32, 1500), (64, 32, 1500),
          (16, 16, 16384), (64, 64, 1500)]
FIELDS = [int(x) for x in sys.argv[1].split(',')] if len(sys.argv) > 1 else [16, 256]
for q in FIELDS:
    gf.init(q)
    for (N, K, M) in SHAPES:
        G = max(1, int(4e9 // (N * M)))
        A = torch.empty((G, N, M), dtype=torch.uint8, device="cuda")
        C = torch.empty((G, N, K), dtype=torch.uint8, device="cuda")
        B = torch.empty((G, K, M), dtype=torch.uint8, device="cuda")
        gf.fill_random(A, 3, 1, 0)
        gf.fill_random(C, 3, 2, 0, mask=q - 1)
        res = {}
        for path in ("auto", "column", "lanek", "prow"):
            gf.set_encode_path(path)
            for _ in range(2):
                gf.encode_batch(q, A, C, B)
            ts = []
            for _ in range(10):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                gf.encode_batch(q, A, C, B)
                e1.record()
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            res[path] = round(G * N * M / statistics.median(ts) / 1e6, 1)
        gf.set_encode_path("auto")
        print(f"GF({q}) N={N} K={K} M={M} auto={gf.encode_path(q, N, K, M)}: {res}", flush=True)
        del A, B, C
        torch.cuda.empty_cache()
