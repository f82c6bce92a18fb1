#!/usr/bin/env python
"""Routing evidence for the TMEM lookup-table engine: source GB/s of
gf_encode_batch with the automatic kernel and with the TMEM engine forced, on
assorted (N, K, M) shapes of every field (CUDA events, median of 7; ~4 GB of
sources per shape):  python tools/exp_tmem_route.py [fields]"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1909_02871_b200 import gf  # noqa: E402

SHAPES = [(32, 32, 1 << 20), (32, 32, 4096), (32, 32, 1024), (32, 32, 512), (32, 32, 256),
          (16, 16, 65536), (16, 24, 65536), (32, 16, 65536), (8, 32, 1 << 20), (64, 64, 65536),
          (64, 32, 16384), (32, 64, 262144), (16, 8, 65536), (16, 12, 65536), (32, 8, 65536), (16, 5, 65536),
          (16, 16, 1024), (16, 8, 1024), (32, 20, 16384), (128, 128, 65536)]
FIELDS = [int(x) for x in sys.argv[1].split(',')] if len(sys.argv) > 1 else [2, 4, 16]


def timed(q, A, C, B):
    for _ in range(2):
        gf.encode_batch(q, A, C, B)
    ts = []
    for _ in range(7):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        gf.encode_batch(q, A, C, B)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


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
        for path in ("auto", "tmem"):
            gf.set_encode_path(path)
            name = gf.encode_path(q, N, K, M)
            if path == "tmem" and name != "tmem":
                continue
            res[f"{path}:{name}"] = round(G * N * M / timed(q, A, C, B) / 1e6, 1)
        gf.set_encode_path("auto")
        print(f"GF({q}) N={N} K={K} M={M} G={G}: {res}", flush=True)
        del A, B, C
        torch.cuda.empty_cache()
