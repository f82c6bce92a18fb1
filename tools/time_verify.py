"""Cost of the Freivalds check (gf_encode_verify_batch, t = 2 and t = 1) against
the plain encode on the bench shapes: C3 GF(256) / GF(16) (65536 generations),
a C5 GF(2) and GF(4) launch (256 generations) and a C4 launch (16 generations).
    python tools/time_verify.py [C3 | C4 | C5 | C5-4 ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import seeded_inputs as si  # noqa: E402
from paper_1909_02871_b200 import gf  # noqa: E402


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    only = sys.argv[1:]                                        # optional config names, e.g. C4 C5-4
    for cfg, q, G in ((si.C3, 256, 65536), (si.C3, 16, 65536), (si.C5, 2, 256), (si.C5, 4, 256), (si.C4, 256, 16)):
        if only and f"{cfg.name}-{q}" not in only and cfg.name not in only:
            continue
        gf.init(q)
        A = torch.empty((G, cfg.N, cfg.M), dtype=torch.uint8, device="cuda")
        C = torch.empty((G, cfg.N, cfg.K), dtype=torch.uint8, device="cuda")
        B = torch.empty((G, cfg.K, cfg.M), dtype=torch.uint8, device="cuda")
        R = torch.empty((G, cfg.K, 2), dtype=torch.uint8, device="cuda")
        R1 = torch.empty((G, cfg.K, 1), dtype=torch.uint8, device="cuda")
        gf.fill_random(R1, 1, 5, 0)
        gf.fill_random(A, 1, 1, 0)
        gf.fill_random(C, 1, 2, 0, mask=q - 1)
        gf.fill_random(R, 1, 5, 0)
        ws = torch.empty(gf.verify_workspace_bytes(cfg.N, cfg.K, G), dtype=torch.uint8, device="cuda")
        t_enc = timeit(lambda: gf.encode_batch(q, A, C, B))
        t_ver = timeit(lambda: gf.encode_verify_batch(q, A, C, R, B, ws))
        t_ver1 = timeit(lambda: gf.encode_verify_batch(q, A, C, R1, B, ws))
        _, mism = gf.encode_verify_batch(q, A, C, R, B, ws)
        src = G * cfg.N * cfg.M
        print(f"{cfg.name} GF({q}) {gf.encode_path(q, cfg.N, cfg.K, cfg.M)}: encode {t_enc:.3f} ms "
              f"({src / t_enc / 1e6:.1f} GB/s), encode+verify {t_ver:.3f} ms ({src / t_ver / 1e6:.1f} GB/s), "
              f"+{(t_ver / t_enc - 1) * 100:.1f}% (t = 2), +{(t_ver1 / t_enc - 1) * 100:.1f}% (t = 1), "
              f"mismatches {int(mism.sum())}", flush=True)
        del A, B, C, R, R1, ws
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
