#!/usr/bin/env python
"""bench.py -- RLNC encode throughput on B200 (source GB/s), driver contract.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--field 256]
    python bench.py --impl reference ...        (the CPU oracle, rank 0 only)

A step is one gf_encode_batch launch over the whole workload batch (the full
hot path: per-coefficient tables, trivial-coefficient handling and the
N x K x M multiply-add of Eq. 2).  Default workload: C3 =
BASELINE.json configs[2] over GF(256) (N=64, M=1500, K=64, 65536 generations),
the largest RLNC-encode config that fits one GPU unchunked; the same run also
times GF(16) (C3's other field) under "per_field".

Multi-GPU (torchrun, one process per GPU): every rank encodes its own 65536
generations (generation-sharded, no collective on the data path), so
"scaling" is "weak"; value = all ranks' source bytes / max-over-ranks time.

The oracle is used only by the cpu_baseline leg and by --impl reference.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import seeded_inputs as si  # noqa: E402

METRIC = "source GB/s per field for RLNC encode at 1/2/4/8 B200; % of HBM roofline"
ALU_LANES_PER_SM_CLK = 64     # B300_MICROARCH.md: alu pipe rt_SMSP = 2 -> 16 lanes/clk/SMSP x 4
N_SM = 148
# algorithmic ALU ops per byte-madd of the inner loop:
# GF(256)/GF(16) 3 PRMT + 2 LOP3 per 4 byte-madds; GF(4) 2 LOP3; GF(2) 1 LOP3
OPS_PER_BYTE_MADD = {256: 5 / 4, 16: 5 / 4, 4: 2 / 4, 2: 1 / 4}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return {"hbm_gbs": float(d["hbm_gbs"]), "sm_max_mhz": float(d.get("sm_max_mhz", 1965.0)),
                "source": "MEASURED_PEAKS.json"}
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "source": "fallback (B200_PROFILING.md)"}


# ---------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.path = os.path.join("/tmp", f"bench_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-i", str(self.idx), "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 9:
                rows.append(f)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        smax = max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[j] for r in rows for j in range(4) if r[5 + j].lower() == "active"})
        busy = [s for s in sm if s > 0.5 * smax] or sm
        return {"sm_mhz": statistics.median(busy), "sm_max_mhz": smax, "reasons": reasons,
                "samples": len(rows), "power_w_max": max(float(r[3]) for r in rows
                                                         if r[3].replace(".", "").isdigit())}


# ---------------------------------------------------------------- oracle baseline

def cpu_baseline(cfg, q, seconds_target=12.0):
    """The oracle (scalar C, plain loops), as it stands, on a bounded sample
    of the same workload, on this host's cores."""
    import oracle
    cores = len(os.sched_getaffinity(0))
    per_gen = cfg.N * cfg.K * cfg.M
    # calibrate on up to 2 generations single-threaded (C1 has one)
    g_cal = min(2, cfg.batch)
    A, C = si.encode_inputs(cfg, q, 0, g_cal)
    t0 = time.perf_counter()
    oracle.encode_batch(q, A, C)
    t1 = time.perf_counter() - t0
    rate_1t = g_cal * per_gen / t1
    gens = int(max(cores, min(cfg.batch, seconds_target * rate_1t * cores / per_gen)))
    gens = max(1, min(gens, cfg.batch))
    A, C = si.encode_inputs(cfg, q, 0, gens)
    t0 = time.perf_counter()
    oracle.encode_batch(q, A, C, threads=cores)
    dt = time.perf_counter() - t0
    src = gens * cfg.N * cfg.M
    return {"value": round(src / dt / 1e9, 4), "unit": "GB/s", "cores": cores, "kind": "oracle",
            "sample": f"{gens} of {cfg.batch} generations of {cfg.name} GF({q}), threads={cores}; "
                      f"1-thread rate {g_cal * cfg.N * cfg.M / t1 / 1e9:.4f} GB/s",
            "seconds": round(dt, 2)}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ---------------------------------------------------------------- helpers

def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3", choices=sorted(si.ENCODE_CONFIGS))
    ap.add_argument("--field", type=int, default=None)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extra-fields", action="store_true")
    ap.add_argument("--e2e-chunk-bytes", type=float, default=0.2e9,
                    help="host bytes per pipeline chunk of the e2e (host-buffer) path")
    ap.add_argument("--chunk-gens", type=int, default=0,
                    help="generations per launch for configs that do not fit one GPU")
    return ap.parse_args()


def workload_name(cfg, q, batch_per_rank):
    return (f"{cfg.name} RLNC encode GF({q}): N={cfg.N} source packets x M={cfg.M} B, "
            f"K={cfg.K} coded, {batch_per_rank} generations per GPU")


# ---------------------------------------------------------------- reference arm

def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    cfg = si.ENCODE_CONFIGS[args.config]
    q = args.field or cfg.fields[-1]
    cores = len(os.sched_getaffinity(0))
    import oracle
    per_gen = cfg.N * cfg.K * cfg.M
    A, C = si.encode_inputs(cfg, q, 0, 1)
    t0 = time.perf_counter()
    oracle.encode_batch(q, A, C)
    t1 = time.perf_counter() - t0
    # each step: a bounded sample sized so that warmup + steps take ~2 minutes
    budget = 120.0 / max(1, args.steps + args.warmup)
    gens = int(max(1, min(cfg.batch, budget * cores / t1)))
    A, C = si.encode_inputs(cfg, q, 0, gens)
    for _ in range(args.warmup):
        oracle.encode_batch(q, A, C, threads=cores)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.encode_batch(q, A, C, threads=cores)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = args.steps * gens * cfg.N * cfg.M / tot / 1e9
    out = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GB/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * tot / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (seeded splitmix64 byte stream, seeded_inputs)",
        "config": {"workload": workload_name(cfg, q, cfg.batch), "N": cfg.N, "K": cfg.K, "M": cfg.M,
                   "batch": cfg.batch, "field": q},
        "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": cores, "kind": "oracle",
                         "sample": f"{gens} generations per step of {cfg.name} GF({q}) "
                                   f"(scalar C oracle, {cores} threads, {cpu_model()})"},
        "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "byte_madds_per_step": gens * per_gen,
    }
    print(json.dumps(out), flush=True)


# ---------------------------------------------------------------- our arm

def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    from paper_1909_02871_b200 import gf, shard

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=device)

    cfg = si.ENCODE_CONFIGS[args.config]
    q = args.field or cfg.fields[-1]
    fields = [q] + ([f for f in cfg.fields if f != q] if not args.no_extra_fields else [])
    for f in fields:
        gf.init(f)
    peaks = load_peaks()

    # ---- this rank's shard: weak scaling by generation (C1, C3, C5) or
    # strong scaling by packet byte range (C4), SURVEY.md 8(e)
    by_bytes = cfg.shard == "bytes"
    sh = shard.plan(cfg.batch, cfg.M, ws, rank, by="bytes" if by_bytes else "generation",
                    weak=not by_bytes)
    G, Ms, N, K, M = sh.generations, sh.columns, cfg.N, cfg.K, cfg.M
    free, _ = torch.cuda.mem_get_info(device)
    per_gen = (N + K) * Ms + N * K
    chunk = min(G, args.chunk_gens or G)
    if per_gen * chunk > 0.8 * free:
        chunk = max(1, int(0.8 * free // per_gen))
    nchunks = -(-G // chunk)
    stream = torch.cuda.current_stream(device)

    A = torch.empty((chunk, N, Ms), dtype=torch.uint8, device=device)
    Cm = torch.empty((chunk, N, K), dtype=torch.uint8, device=device)
    B = torch.empty((chunk, K, Ms), dtype=torch.uint8, device=device)

    def fill(f, j):
        """Inputs of chunk j, generated on device by absolute index."""
        seed = si.field_seed(cfg, f)
        g = sh.g0 + j * chunk
        n = min(chunk, G - j * chunk)
        gf.fill_random2d(A[:n].view(n * N, Ms), seed, si.STREAM_A, g * N * M + sh.m0, M)
        gf.fill_random(Cm[:n], seed, si.STREAM_C, g * N * K, mask=f - 1)
        return n

    def time_field(f, steps, warmup, sampler=None):
        """Device-resident throughput: inputs in HBM before the timed region.
        One chunk: CUDA-event span over all steps.  Several chunks (C5 does not
        fit): inputs of each chunk are regenerated between launches and only
        the encode launches are timed (sum of their event durations)."""
        n0 = fill(f, 0)
        torch.cuda.synchronize()
        for _ in range(warmup):
            gf.encode_batch(f, A[:n0], Cm[:n0], B[:n0])
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        if sampler:
            sampler.start()
            time.sleep(0.3)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(steps * nchunks)]
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        launches = 0
        t_start.record(stream)
        for s in range(steps):
            for j in range(nchunks):
                n = fill(f, j) if nchunks > 1 else n0
                e0, e1 = ev[s * nchunks + j]
                e0.record(stream)
                gf.encode_batch(f, A[:n], Cm[:n], B[:n])
                e1.record(stream)
                launches += 1
        t_end.record(stream)
        torch.cuda.synchronize()
        clocks = sampler.stop() if sampler else None
        kern_ms = [a.elapsed_time(b) for a, b in ev]
        total_ms = t_start.elapsed_time(t_end) if nchunks == 1 else sum(kern_ms)
        if ws > 1:
            t = torch.tensor([total_ms], device=device)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            total_ms = float(t.item())
            dist.barrier()
        return total_ms, kern_ms, launches, clocks

    job_src_per_step = (cfg.batch * N * M) if by_bytes else ws * G * N * M
    sampler = ClockSampler(local)
    total_ms, kern_ms, launches, clocks = time_field(q, args.steps, args.warmup, sampler)
    value = job_src_per_step * args.steps / (total_ms / 1e3) / 1e9
    ms_per_step = total_ms / args.steps

    per_field = {str(q): round(value, 3)}
    for f in fields[1:]:
        st = max(3, args.steps // 2)
        tms, _, _, _ = time_field(f, st, args.warmup)
        per_field[str(f)] = round(job_src_per_step * st / (tms / 1e3) / 1e9, 3)

    # ---- roofline of the dominant kernel: the encode launch (every launch of
    # the timed region is one); algorithmic work per launch / mean duration
    avg_kernel_s = statistics.mean(kern_ms) / 1e3
    gens_per_launch = chunk
    path = gf.encode_path(q, N, K, Ms)
    roof, hbm = dominant_roofline(q, N, K, Ms, gens_per_launch, path, avg_kernel_s, peaks)
    roof["traffic"] = lookup_traffic(q, cfg, gens_per_launch, Ms, path)
    roof["kernel_ms"] = round(statistics.mean(kern_ms), 4)
    del A, Cm, B
    torch.cuda.empty_cache()

    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(gf, torch, dist, cfg, q, sh, device, ws, args)

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        cpu = cpu_baseline(cfg, q)
        cpu["cpu_model"] = cpu_model()

    if rank == 0:
        out = {
            "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
            "higher_is_better": True, "scaling": "strong" if by_bytes else "weak",
            "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (seeded splitmix64 byte stream: uniform payload bytes, "
                    "i.i.d. uniform coefficients over F_q; generated on device)",
            "config": {"workload": workload_name(cfg, q, G), "field": q, "N": N, "K": K, "M": M,
                       "gens_per_gpu": G, "bytes_per_packet_per_gpu": Ms,
                       "global_batch": cfg.batch if by_bytes else ws * G,
                       "gens_per_launch": gens_per_launch, "launches_per_step": nchunks,
                       "parallelism": (f"byte-range sharded x{ws}" if by_bytes else
                                       f"generation-sharded x{ws}") + ", no collective",
                       "l2": (f"inputs {G * N * Ms / 1e9:.2f} GB per GPU >> 126 MB L2 (no flush)"
                              if G * N * Ms > 2 * 126e6 else "L2-resident working set")},
            "per_field": per_field,
            "roofline": roof,
            "hbm": hbm,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clocks,
            "gpu_launches": launches,
            "kernel_ms_per_launch": round(statistics.mean(kern_ms), 4),
        }
        print(json.dumps(out), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()


SMEM_BYTES_PER_SM_CLK = 128   # shared-memory crossbar (B300_MICROARCH.md; tools/ubench_smem.cu)
LANEK = {2: (4, 1, 15), 4: (2, 1, 15), 16: (1, 1, 15), 256: (1, 2, 30)}   # SG, gathers/unit, build rows


def dominant_roofline(q, N, K, Ms, gens, path, kernel_s, peaks):
    """Roofline of the encode launch.

    The product-row kernel is bound by the shared-memory pipe: algorithmic
    smem bytes = one gathered byte per byte-madd + the product tables written
    (256 x 64 B per source, coded-packet tile and 384-word tile).
    lane-k kernels are bound by the shared-memory pipe: algorithmic smem bytes
    = gathers (4 B per gathered word, G per (step, k, word)) + table build
    (R rows x 4 B per (step, word), once per CTA k-tile); peak = 148 SMs x
    128 B/clk x max SM clock.  Column kernels are bound by the ALU pipe:
    byte-madds x ops per byte-madd of the method; peak = 148 x 64 lanes/clk x
    clock.  Both carry the HBM view (read A, write B, read C)."""
    clk = peaks["sm_max_mhz"] * 1e6
    bm = N * K * Ms * gens
    hbm_bytes = ((N + K) * Ms + N * K) * gens
    hbm_ach = hbm_bytes / kernel_s / 1e9
    hbm = {"achieved": round(hbm_ach, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
           "frac": round(hbm_ach / peaks["hbm_gbs"], 4), "peak_source": peaks["source"]}
    if path == "prow":
        # product-row kernel: every byte-madd is one gathered product byte;
        # tables: 256 rows x 64 B per (source, 64-coded-packet tile, word tile)
        tw = 384
        m_tiles = -(-(Ms // 4) // tw)
        k_tiles = -(-K // 64)
        n_pad = -(-N // 4) * 4
        smem_bytes = bm + gens * n_pad * k_tiles * m_tiles * 256 * 64
        peak = N_SM * SMEM_BYTES_PER_SM_CLK * clk
        ach = smem_bytes / kernel_s
        roof = {"bound": "smem", "achieved": round(ach / 1e12, 3), "peak": round(peak / 1e12, 3),
                "unit": "TB/s", "frac": round(ach / peak, 4),
                "peak_source": f"{N_SM} SMs x {SMEM_BYTES_PER_SM_CLK} B/clk shared-memory pipe x "
                               f"{peaks['sm_max_mhz']:.0f} MHz (DESIGN.md 'roofline')",
                "smem_bytes_per_launch": smem_bytes}
    elif path.startswith("lanek"):
        SG, G, R = LANEK[q]
        ktl = 64 if path == "lanek-64" else 32
        steps = -(-N // SG)
        k_tiles = -(-K // ktl)
        smem_bytes = gens * steps * (Ms // 4) * 4 * (K * G + R * k_tiles)
        peak = N_SM * SMEM_BYTES_PER_SM_CLK * clk
        ach = smem_bytes / kernel_s
        roof = {"bound": "smem", "achieved": round(ach / 1e12, 3), "peak": round(peak / 1e12, 3),
                "unit": "TB/s", "frac": round(ach / peak, 4),
                "peak_source": f"{N_SM} SMs x {SMEM_BYTES_PER_SM_CLK} B/clk shared-memory pipe x "
                               f"{peaks['sm_max_mhz']:.0f} MHz (DESIGN.md 'roofline')",
                "smem_bytes_per_launch": smem_bytes}
    else:
        ops = bm * OPS_PER_BYTE_MADD[q]
        peak = N_SM * ALU_LANES_PER_SM_CLK * clk
        ach = ops / kernel_s
        roof = {"bound": "alu", "achieved": round(ach / 1e12, 3), "peak": round(peak / 1e12, 3),
                "unit": "Tops/s", "frac": round(ach / peak, 4),
                "peak_source": f"{N_SM} SMs x {ALU_LANES_PER_SM_CLK} ALU-pipe lanes/clk x "
                               f"{peaks['sm_max_mhz']:.0f} MHz (DESIGN.md 'roofline')",
                "ops_per_byte_madd": OPS_PER_BYTE_MADD[q]}
    if hbm["frac"] > roof["frac"]:
        roof = dict(hbm, bound="hbm")
    roof["kernel"] = f"encode {path} GF({q})"
    roof["byte_madds_per_launch"] = bm
    roof["hbm_bytes_per_launch"] = hbm_bytes
    return roof, hbm


KERNEL_SOURCES = {"prow": "encode_prow.cuh", "prow-32": "encode_prow.cuh", "prow-16": "encode_prow.cuh",
                  "lanek-32": "encode_lanek.cuh", "lanek-64": "encode_lanek.cuh", "stream": "encode_stream.cuh",
                  "column-words": "encode_kernels.cuh"}


def kernel_sha(path):
    """sha256 of the CUDA source of the kernel an encode path launches (ties a
    committed ncu capture to the kernel code it measured)."""
    import hashlib
    f = KERNEL_SOURCES.get(path)
    if not f:
        return None
    return hashlib.sha256(open(os.path.join(ROOT, "paper_1909_02871_b200", "csrc", f), "rb").read()).hexdigest()[:16]


def lookup_traffic(q, cfg, gens, Ms, path):
    """dram__bytes_read + dram__bytes_write per launch of the encode kernel from
    the committed ncu --set full capture of the same launch (profiles/), or None
    when the kernel source changed since that capture."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        d = json.load(open(p))
        e = d.get(f"{cfg.name}/GF{q}/{gens}/{Ms}")
        if e and e.get("kernel_sha") == kernel_sha(path):
            return e["bytes"]
    except Exception:
        pass
    return None


def run_e2e(gf, torch, dist, cfg, q, sh, device, ws, args):
    """Same metric through gf_encode_batch_host: pinned host A/C in, host B
    out, host<->device copies inside the timed region every step."""
    N, K, M, Ms = cfg.N, cfg.K, cfg.M, sh.columns
    per_gen_host = N * Ms + N * K + K * Ms
    # pinned host buffers: <= 14 GB per rank and <= 48 GB per node in total
    G = min(sh.generations, max(1, int(min(14e9, 48e9 / ws) // per_gen_host)))
    err = None
    try:
        Ah = torch.empty((G, N, Ms), dtype=torch.uint8).pin_memory()
        Ch = torch.empty((G, N, K), dtype=torch.uint8).pin_memory()
        Bh = torch.empty((G, K, Ms), dtype=torch.uint8).pin_memory()
    except Exception as e:  # pinned host memory exhausted
        err = f"pinned alloc failed: {e}"
    if ws > 1:                       # every rank skips together (no rank left in a barrier)
        ok = torch.tensor([0 if err else 1], device=device)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if int(ok.item()) == 0 and err is None:
            err = "pinned alloc failed on another rank"
    if err:
        return {"value": None, "unit": "GB/s", "error": err}
    seed = si.field_seed(cfg, q)
    step = max(1, min(G, int(2e9 // (N * Ms + N * K))))
    tmpA = torch.empty((step, N, Ms), dtype=torch.uint8, device=device)
    tmpC = torch.empty((step, N, K), dtype=torch.uint8, device=device)
    for j in range(0, G, step):
        n = min(step, G - j)
        g = sh.g0 + j
        gf.fill_random2d(tmpA[:n].view(n * N, Ms), seed, si.STREAM_A, g * N * M + sh.m0, M)
        gf.fill_random(tmpC[:n], seed, si.STREAM_C, g * N * K, mask=q - 1)
        Ah[j:j + n].copy_(tmpA[:n])
        Ch[j:j + n].copy_(tmpC[:n])
    del tmpA, tmpC
    chunk = max(1, min(G, int(args.e2e_chunk_bytes // per_gen_host)))
    ws_t = torch.empty(gf.host_workspace_bytes(N, K, Ms, chunk), dtype=torch.uint8, device=device)
    torch.cuda.synchronize()
    gf.encode_batch_host(q, Ah, Ch, Bh, ws_t)
    steps = max(1, min(args.steps, 5))
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        gf.encode_batch_host(q, Ah, Ch, Bh, ws_t)   # blocking: returns with B on the host
    dt = time.perf_counter() - t0
    if ws > 1:
        t = torch.tensor([dt], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    src = (G * N * Ms) * ws
    value = steps * src / dt / 1e9
    # the PCIe roofline of this path: plain pinned copies of the same sizes,
    # concurrently in both directions (the e2e pipeline overlaps them)
    h2d_b, d2h_b = G * (N * Ms + N * K), G * K * Ms
    pcie = {}
    try:
        nb = min(h2d_b, 2 << 30)
        dbuf = torch.empty(nb, dtype=torch.uint8, device=device)
        hsrc = Ah.view(-1)[:nb]
        hdst = Bh.view(-1)[:min(nb, Bh.numel())]
        s1, s2 = torch.cuda.Stream(device), torch.cuda.Stream(device)
        t_h2d = t_d2h = t_both = float("inf")        # best of 4 (the first warms the path)
        for _ in range(4):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            with torch.cuda.stream(s1):
                dbuf.copy_(hsrc, non_blocking=True)
            torch.cuda.synchronize()
            t_h2d = min(t_h2d, time.perf_counter() - t0)
            t0 = time.perf_counter()
            with torch.cuda.stream(s2):
                hdst.copy_(dbuf[:hdst.numel()], non_blocking=True)
            torch.cuda.synchronize()
            t_d2h = min(t_d2h, time.perf_counter() - t0)
        # both directions at once, as the e2e pipeline runs them (full duplex)
        dbuf2 = torch.empty(hdst.numel(), dtype=torch.uint8, device=device)
        for _ in range(4):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            with torch.cuda.stream(s1):
                dbuf.copy_(hsrc, non_blocking=True)
            with torch.cuda.stream(s2):
                hdst.copy_(dbuf2, non_blocking=True)
            torch.cuda.synchronize()
            t_both = min(t_both, time.perf_counter() - t0)
        del dbuf2
        pcie = {"h2d_GBps": round(nb / t_h2d / 1e9, 1), "d2h_GBps": round(hdst.numel() / t_d2h / 1e9, 1),
                "concurrent_h2d_plus_d2h_s": round(t_both, 4), "concurrent_bytes_each_way": [nb, hdst.numel()]}
        # e2e bound: the step's H2D and D2H bytes at the concurrent (duplex) rates
        rate_h2d, rate_d2h = nb / t_both, hdst.numel() / t_both
        bound_s = max(h2d_b / rate_h2d, d2h_b / rate_d2h)
        pcie["e2e_bound_GBps"] = round(G * N * Ms / bound_s / 1e9, 2)
        pcie["e2e_frac_of_bound"] = round(value / ws / pcie["e2e_bound_GBps"], 3)
        del dbuf
    except Exception as e:  # diagnostics only
        pcie = {"error": str(e)[:200]}
    del ws_t
    torch.cuda.empty_cache()
    return {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": h2d_b,
            "d2h_bytes_per_step": d2h_b, "steps": steps, "gens_per_step": G, "pcie": pcie,
            "path": f"gf_encode_batch_host: pinned host buffers, {chunk}-generation chunks, "
                    "3-stream copy/compute overlap",
            "timing": "host wall clock around blocking calls, max over ranks"}


if __name__ == "__main__":
    main()
