#!/usr/bin/env python
"""Experiment: C5 encode with the generations split between two kernels on two
streams (lane-k on the shared-memory pipe, column on the ALU pipe), to see
whether co-resident CTAs of both kernels add up.
    python tools/exp_concurrent.py [field] [gens]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import seeded_inputs as si  # noqa: E402
from paper_1909_02871_b200 import gf  # noqa: E402

q = int(sys.argv[1]) if len(sys.argv) > 1 else 2
G = int(sys.argv[2]) if len(sys.argv) > 2 else 512
cfg = si.ENCODE_CONFIGS["C5"]
gf.init(q)
A = torch.empty((G, cfg.N, cfg.M), dtype=torch.uint8, device="cuda")
C = torch.empty((G, cfg.N, cfg.K), dtype=torch.uint8, device="cuda")
B = torch.empty((G, cfg.K, cfg.M), dtype=torch.uint8, device="cuda")
seed = si.field_seed(cfg, q)
gf.fill_random(A, seed, si.STREAM_A, 0)
gf.fill_random(C, seed, si.STREAM_C, 0, mask=q - 1)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
ref = torch.empty_like(B)


def run(split, p1="lanek", p2="column", reps=5):
    g1 = int(round(G * split))
    times = []
    for it in range(reps + 2):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        s1.wait_stream(torch.cuda.current_stream())
        s2.wait_stream(torch.cuda.current_stream())
        if g1 > 0:
            with torch.cuda.stream(s1):
                gf.set_encode_path(p1)
                gf.encode_batch(q, A[:g1], C[:g1], B=B[:g1])
        if g1 < G:
            with torch.cuda.stream(s2):
                gf.set_encode_path(p2)
                gf.encode_batch(q, A[g1:], C[g1:], B=B[g1:])
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
        e1.record()
        e1.synchronize()
        if it >= 2:
            times.append(e0.elapsed_time(e1))
    gf.set_encode_path("auto")
    t = sorted(times)[len(times) // 2]
    return t, G * cfg.N * cfg.M / t / 1e6


gf.set_encode_path("lanek")
gf.encode_batch(q, A, C, B=ref)
for split in (1.0, 0.0, 0.8, 0.7, 0.6, 0.5):
    t, gbs = run(split)
    ok = bool(torch.equal(B, ref))
    print(f"GF({q}) gens={G} lanek share={split:.2f}: {t:8.3f} ms  {gbs:8.1f} GB/s  equal={ok}", flush=True)
