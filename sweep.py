#!/usr/bin/env python
"""sweep.py -- every BASELINE.json workload on one GPU, one JSON line each.

    python sweep.py [--configs C1,C2,C3,C4,C5] [--out gpurun_out/sweep.jsonl]

C1: single-generation latency (us per gf_encode_batch call).
C2: gf_maddrc / gf_mulrc region sweep, 64 B .. 256 MiB per field; points whose
    3 x size working set fits twice in L2 are timed both with an L2 flush
    between reps (HBM numbers) and L2-resident (labelled).
C3, C4, C5: batched encode, source GB/s, % of HBM and of the ALU-pipe peak.
Timing: CUDA events on the launching stream, >= 3 warm-ups, >= 10 reps and
>= 0.5 s per point; median reported.  Inputs come from the device generator.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import seeded_inputs as si  # noqa: E402
from bench import ClockSampler, dominant_roofline, load_peaks  # noqa: E402


def bound_of(q, N, K, M, gens, path, kernel_s, peaks):
    """The kernel's binding resource and its fraction on the method's
    algorithmic work (bench.dominant_roofline)."""
    r, _ = dominant_roofline(q, N, K, M, gens, path, kernel_s, peaks)
    return {"kernel": path, "bound": r["bound"], "bound_frac": r["frac"]}


def timed(torch, fn, stream, min_reps=10, min_s=0.5, warmup=3, flush=None):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    times = []
    total = 0.0
    while len(times) < min_reps or total < min_s * 1e3:
        if flush is not None:
            flush()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        e1.synchronize()
        t = e0.elapsed_time(e1)
        times.append(t)
        total += t
        if len(times) > 20000:
            break
    return statistics.median(times), min(times), len(times)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C1,C2,C3,C4,C5")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "sweep.jsonl"))
    args = ap.parse_args()
    import torch

    from paper_1909_02871_b200 import gf

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    for q in (2, 4, 16, 256):
        gf.init(q)
    st = torch.cuda.current_stream(dev)
    peaks = load_peaks()

    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush_buf = torch.empty(2 * l2 + (64 << 20), dtype=torch.uint8, device=dev)

    def flush():
        flush_buf.fill_(1)

    out = open(args.out, "a")
    sampler = ClockSampler(0)
    sampler.start()

    def emit(rec):
        rec["gpu"] = torch.cuda.get_device_name(dev)
        print(json.dumps(rec), flush=True)
        out.write(json.dumps(rec) + "\n")
        out.flush()

    todo = args.configs.split(",")
    if "C1" in todo:
        cfg = si.C1
        A = torch.empty((1, cfg.N, cfg.M), dtype=torch.uint8, device=dev)
        Ah, Chh = si.encode_inputs(cfg, 256)
        A.copy_(torch.from_numpy(Ah))
        C = torch.from_numpy(Chh).to(dev)
        B = torch.empty((1, cfg.K, cfg.M), dtype=torch.uint8, device=dev)
        med, best, n = timed(torch, lambda: gf.encode_batch(256, A, C, B), st, min_reps=1000)
        # device time per call without the Python/ctypes submission cost:
        # capture 100 calls in a CUDA graph and replay it
        reps = 100
        g = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream()
        cap.wait_stream(st)
        with torch.cuda.stream(cap):
            gf.encode_batch(256, A, C, B)
            with torch.cuda.graph(g, stream=cap):
                for _ in range(reps):
                    gf.encode_batch(256, A, C, B)
        st.wait_stream(cap)
        gmed, gbest, gn = timed(torch, g.replay, st, min_reps=50)
        emit({"config": "C1", "field": 256, "us_per_call_median": round(med * 1e3, 3),
              "us_per_call_best": round(best * 1e3, 3), "reps": n,
              "us_per_call_graph": round(gmed * 1e3 / reps, 3),
              "source_GBps": round(cfg.source_bytes() / (med / 1e3) / 1e9, 3),
              "source_GBps_graph": round(cfg.source_bytes() / (gmed / reps / 1e3) / 1e9, 3),
              "path": gf.encode_path(256, cfg.N, cfg.K, cfg.M),
              "note": "launch-latency bound (25.5 KB per call), L2-resident; per-call = one "
                      "gf_encode_batch through ctypes incl. submission; graph = 100 calls "
                      "captured in a CUDA graph, device time per call"})

    if "C2" in todo:
        nmax = si.C2_SIZES[-1]
        src = torch.empty(nmax, dtype=torch.uint8, device=dev)
        dst = torch.empty(nmax, dtype=torch.uint8, device=dev)
        gf.fill_random(src, si.C2_SEED, si.STREAM_SRC, 0)
        gf.fill_random(dst, si.C2_SEED, si.STREAM_DST, 0)
        for q in (2, 4, 16, 256):
            c = si.c2_coeff(q)
            for n in si.C2_SIZES:
                s, d = src[:n], dst[:n]
                for op in ("maddrc", "mulrc"):
                    # GF(2) mulrc by c = 1 is a no-op (nothing launched): time c = 0
                    # (the zeroing kernel, write-only) instead
                    cm = 0 if (op == "mulrc" and q == 2) else c
                    fn = (lambda: gf.maddrc(q, d, s, c)) if op == "maddrc" else (lambda: gf.mulrc(q, d, cm))
                    traffic = 3 * n if op == "maddrc" else (n if cm == 0 else 2 * n)
                    resident = traffic < 2 * l2
                    modes = [("hbm", flush)] + ([("l2", None)] if resident else [])
                    for mode, fl in modes:
                        med, best, reps = timed(torch, fn, st, flush=fl,
                                                min_s=0.2 if n < (1 << 20) else 0.5)
                        rec = {"config": "C2", "op": op, "field": q, "coeff": c if op == "maddrc" else cm,
                               "bytes": n,
                               "mode": mode, "us_median": round(med * 1e3, 3), "reps": reps,
                               "source_GBps": round(n / (med / 1e3) / 1e9, 3),
                               "hbm_GBps": round(traffic / (med / 1e3) / 1e9, 2)}
                        if mode == "hbm":
                            rec["hbm_frac"] = round(traffic / (med / 1e3) / 1e9 / peaks["hbm_gbs"], 4)
                        emit(rec)
        del src, dst

    for name in ("C3", "C4", "C5"):
        if name not in todo:
            continue
        cfg = si.ENCODE_CONFIGS[name]
        free, _ = torch.cuda.mem_get_info(dev)
        per_gen = (cfg.N + cfg.K) * cfg.M + cfg.N * cfg.K
        chunk = min(cfg.batch, int(0.7 * (free - flush_buf.numel()) // per_gen))
        A = torch.empty((chunk, cfg.N, cfg.M), dtype=torch.uint8, device=dev)
        C = torch.empty((chunk, cfg.N, cfg.K), dtype=torch.uint8, device=dev)
        B = torch.empty((chunk, cfg.K, cfg.M), dtype=torch.uint8, device=dev)
        for q in cfg.fields:
            seed = si.field_seed(cfg, q)
            gf.fill_random(A, seed, si.STREAM_A, 0)
            gf.fill_random(C, seed, si.STREAM_C, 0, mask=q - 1)
            med, best, reps = timed(torch, lambda: gf.encode_batch(q, A, C, B), st, min_reps=5,
                                    min_s=1.0)
            src_b = chunk * cfg.N * cfg.M
            bm = chunk * cfg.N * cfg.K * cfg.M
            emit({"config": name, "field": q, "gens_per_launch": chunk, "of_batch": cfg.batch,
                  "ms_median": round(med, 3), "ms_best": round(best, 3), "reps": reps,
                  "source_GBps": round(src_b / (med / 1e3) / 1e9, 2),
                  "byte_madds_per_s_T": round(bm / (med / 1e3) / 1e12, 3),
                  "hbm_frac": round(per_gen * chunk / (med / 1e3) / 1e9 / peaks["hbm_gbs"], 4),
                  **bound_of(q, cfg.N, cfg.K, cfg.M, chunk, gf.encode_path(q, cfg.N, cfg.K, cfg.M),
                             med / 1e3, peaks)})
        del A, B, C
        torch.cuda.empty_cache()

    if "DEC" in todo:
        # NEXT-3: batched decode of C3-shaped generations (N = K = 64, 1500 B):
        # invert 64 x 64 coefficient matrices, then encode with the inverses
        cfg = si.C3
        G = 16384
        for q in (16, 256):
            A = torch.empty((G, cfg.N, cfg.M), dtype=torch.uint8, device=dev)
            C = torch.empty((G, cfg.N, cfg.N), dtype=torch.uint8, device=dev)
            gf.fill_random(A, 5, si.STREAM_A, 0)
            gf.fill_random(C, 5, si.STREAM_C, 0, mask=q - 1)
            B = gf.encode_batch(q, A, C)
            ws = torch.empty(G * cfg.N * cfg.N, dtype=torch.uint8, device=dev)
            inv_med, _, _ = timed(torch, lambda: gf.invert_batch(q, C), st, min_reps=5, min_s=0.5)
            dec_med, _, _ = timed(torch, lambda: gf.decode_batch(q, B, C, ws), st, min_reps=5, min_s=0.5)
            A2, rank = gf.decode_batch(q, B, C, ws)
            ok = bool(torch.equal(A2[rank == cfg.N], A[rank == cfg.N]))
            emit({"config": "DEC", "field": q, "N": cfg.N, "M": cfg.M, "gens": G,
                  "invert_ms": round(inv_med, 3), "decode_ms": round(dec_med, 3),
                  "decoded_GBps": round(G * cfg.N * cfg.M / (dec_med / 1e3) / 1e9, 2),
                  "matrices_per_s_M": round(G / (inv_med / 1e3) / 1e6, 3),
                  "full_rank": int((rank == cfg.N).sum()), "round_trip_ok": ok})
            del A, B, C, ws, A2
        torch.cuda.empty_cache()

    if "NEXT2" in todo:
        # paper-shaped sweep (Fig. 2): random linear
        # combinations of N=16 packets, K=1 coded packet, packet sizes 128 B ..
        # 64 KiB, all fields, plus the 1500-byte packets of C1/C3 (word- but not
        # 16-byte-aligned rows); enough generations per launch for ~2 GiB of
        # source. Coded throughput in Gbit/s is the paper's unit (X13).
        for q in (2, 4, 16, 256):
            for size in [128 << j for j in range(10)] + [1500]:
                N, K = 16, 1
                gens = max(1, (2 << 30) // (N * size))
                A = torch.empty((gens, N, size), dtype=torch.uint8, device=dev)
                C = torch.empty((gens, N, K), dtype=torch.uint8, device=dev)
                B = torch.empty((gens, K, size), dtype=torch.uint8, device=dev)
                gf.fill_random(A, 77, si.STREAM_A, 0)
                gf.fill_random(C, 77, si.STREAM_C, 0, mask=q - 1)
                med, best, reps = timed(torch, lambda: gf.encode_batch(q, A, C, B), st, min_reps=10,
                                        min_s=0.3)
                src_b = gens * N * size
                hbm = gens * ((N + K) * size + N * K)
                emit({"config": "NEXT2", "field": q, "packet_bytes": size, "N": N, "K": K,
                      "gens_per_launch": gens, "ms_median": round(med, 4),
                      "source_GBps": round(src_b / (med / 1e3) / 1e9, 2),
                      "coded_Gbitps": round(gens * K * size * 8 / (med / 1e3) / 1e9, 2),
                      "hbm_frac": round(hbm / (med / 1e3) / 1e9 / peaks["hbm_gbs"], 4),
                      "path": gf.encode_path(q, N, K, size)})
                del A, B, C
        torch.cuda.empty_cache()
        # the paper's "L2-bounded average" (Fig. 3: mean
        # throughput over the packet sizes whose working set stays in the cache):
        # GPU analog -- 64 MiB of source per launch (A + B stay in the 126 MB
        # L2), ten launches back to back per timed span without a flush,
        # averaged over 128 B .. 8 KiB
        for q in (2, 4, 16, 256):
            vals = []
            for size in [128 << j for j in range(7)]:
                N, K = 16, 1
                gens = max(1, (64 << 20) // (N * size))
                A = torch.empty((gens, N, size), dtype=torch.uint8, device=dev)
                C = torch.empty((gens, N, K), dtype=torch.uint8, device=dev)
                B = torch.empty((gens, K, size), dtype=torch.uint8, device=dev)
                gf.fill_random(A, 78, si.STREAM_A, 0)
                gf.fill_random(C, 78, si.STREAM_C, 0, mask=q - 1)
                def ten():
                    for _ in range(10):
                        gf.encode_batch(q, A, C, B)
                med, _, _ = timed(torch, ten, st, min_reps=10, min_s=0.2)
                med /= 10
                gbps = gens * N * size / (med / 1e3) / 1e9
                vals.append(gbps)
                emit({"config": "NEXT2-L2", "field": q, "packet_bytes": size, "N": N, "K": K,
                      "gens_per_launch": gens, "ms_median": round(med, 4), "source_GBps": round(gbps, 2),
                      "coded_Gbitps": round(gbps * 8 / N, 2), "mode": "L2-resident (no flush, 10 launches per timed span)",
                      "path": gf.encode_path(q, N, K, size)})
                del A, B, C
            emit({"config": "NEXT2-L2-average", "field": q, "source_GBps": round(sum(vals) / len(vals), 2),
                  "coded_Gbitps": round(sum(vals) / len(vals) * 8 / 16, 2),
                  "sizes": "128 B .. 8 KiB", "note": "mean over sizes, the paper's Fig. 3 summary"})
        torch.cuda.empty_cache()

    emit({"clocks": sampler.stop()})


if __name__ == "__main__":
    main()
