"""Host cost per call of the C1 encode (GF(256), N = 16 x 1500 B, K = 1, one
generation; device time ~3.8 us): the Python binding, a raw ctypes call of
gf_encode_batch, and a CUDA-graph replay, each over many back-to-back calls."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import seeded_inputs as si  # noqa: E402
from paper_1909_02871_b200 import gf  # noqa: E402


def main():
    gf.init(256)
    A0, C0 = si.encode_inputs(si.C1, 256)
    A, C = torch.from_numpy(A0).cuda(), torch.from_numpy(C0).cuda()
    B = torch.empty((1, 1, 1500), dtype=torch.uint8, device="cuda")
    n = 20000
    for _ in range(100):
        gf.encode_batch(256, A, C, B)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        gf.encode_batch(256, A, C, B)
    torch.cuda.synchronize()
    t_bind = (time.perf_counter() - t0) / n
    L = gf.lib()
    pa, pc, pb = A.data_ptr(), C.data_ptr(), B.data_ptr()
    L.gf_set_stream(torch.cuda.current_stream().cuda_stream)
    t0 = time.perf_counter()
    for _ in range(n):
        L.gf_encode_batch(256, pa, pc, pb, 16, 1, 1500, 1)
    torch.cuda.synchronize()
    t_raw = (time.perf_counter() - t0) / n
    t0 = time.perf_counter()
    for _ in range(n):
        L.gf_fill_random(pb, 8, 1, 1, 0, 255)            # the launch floor: a trivial kernel, same ABI
    torch.cuda.synchronize()
    t_fill = (time.perf_counter() - t0) / n
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    reps = 100
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                gf.encode_batch(256, A, C, B)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    t_graph = e0.elapsed_time(e1) / 1e3 / (20 * reps)
    print(f"C1 per call: python binding {t_bind * 1e6:.2f} us, raw ctypes {t_raw * 1e6:.2f} us, "
          f"raw ctypes 8-byte fill kernel {t_fill * 1e6:.2f} us, "
          f"CUDA graph replay {t_graph * 1e6:.2f} us (device)")


if __name__ == "__main__":
    main()
