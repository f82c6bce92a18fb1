"""Time gf_encode_batch on C5-shaped chunks (N = K = 32, 1 MiB packets) for
GF(2) / GF(4): CUDA events around back-to-back launches on device-resident
inputs.  Usage: python tools/time_c5.py [gens ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import seeded_inputs as si  # noqa: E402
from paper_1909_02871_b200 import gf  # noqa: E402


def main():
    gens = [int(x) for x in sys.argv[1:]] or [256, 512]
    cfg = si.C5
    for q in (2, 4):
        gf.init(q)
        for G in gens:
            A = torch.empty((G, cfg.N, cfg.M), dtype=torch.uint8, device="cuda")
            C = torch.empty((G, cfg.N, cfg.K), dtype=torch.uint8, device="cuda")
            B = torch.empty((G, cfg.K, cfg.M), dtype=torch.uint8, device="cuda")
            gf.fill_random(A, 1, 1, 0)
            gf.fill_random(C, 1, 2, 0, mask=q - 1)
            for _ in range(3):
                gf.encode_batch(q, A, C, B)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 10
            e0.record()
            for _ in range(reps):
                gf.encode_batch(q, A, C, B)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            src = G * cfg.N * cfg.M
            print(f"GF({q}) {gf.encode_path(q, cfg.N, cfg.K, cfg.M)} G={G}: {ms:.3f} ms  "
                  f"{src / ms / 1e6:.1f} GB/s source ({src / ms / 1e6 / 3273 * 100:.1f}% of 3273)", flush=True)
            del A, B, C
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
