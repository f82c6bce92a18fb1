"""GF(2) C5 encode (default kernel: the TMEM engine since 0.2.01): per-launch time of 256-generation launches over a
long back-to-back run (does the board's 1 kW power cap slow it down?), with
nvidia-smi clocks / power sampled alongside."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import seeded_inputs as si  # noqa: E402
from bench import ClockSampler  # noqa: E402
from paper_1909_02871_b200 import gf  # noqa: E402

cfg, q, G = si.C5, 2, 256
gf.init(q)
A = torch.empty((G, cfg.N, cfg.M), dtype=torch.uint8, device="cuda")
C = torch.empty((G, cfg.N, cfg.K), dtype=torch.uint8, device="cuda")
B = torch.empty((G, cfg.K, cfg.M), dtype=torch.uint8, device="cuda")
gf.fill_random(A, 1, 1, 0)
gf.fill_random(C, 1, 2, 0, mask=1)
torch.cuda.synchronize()
smp = ClockSampler(0)
smp.start()
n = 400
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
for a, b in ev:
    a.record()
    gf.encode_batch(q, A, C, B)
    b.record()
torch.cuda.synchronize()
clk = smp.stop()
ms = [a.elapsed_time(b) for a, b in ev]
src = G * cfg.N * cfg.M
for lo in range(0, n, 50):
    m = sum(ms[lo:lo + 50]) / 50
    print(f"launches {lo:3d}-{lo + 49:3d}: {m:.3f} ms  {src / m / 1e6:.1f} GB/s")
print("clocks", clk)
