#!/usr/bin/env python
"""bench.py -- RLNC encode throughput on B200 (source GB/s per field), driver contract.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--field 256]
    python bench.py --impl reference ...        (the CPU oracle, rank 0 only)

A step is one gf_encode_batch launch over this rank's share of the workload
(the whole hot path: per-coefficient tables, the N x K x M multiply-add of
Eq. 2, output written).  Headline workload: C3 =
BASELINE.json configs[2] over GF(256) (N=64, M=1500, K=64, 65536
generations); "per_field" adds GF(16) on the same C3 job and GF(2) / GF(4)
on the whole C5 job (configs[4]: N=K=32, 1 MiB packets, 4096 generations,
launched in chunks of generations because it does not fit one GPU).

Multi-GPU: `--gpus N` without torchrun re-launches itself under
torch.distributed.run with N ranks (one process per GPU); under torchrun the
world size must equal --gpus.  The BASELINE job is SPLIT across ranks
(SURVEY.md 8(e)): C3 / C5 by generation (65536 / N, 4096 / N), C4 by packet
byte range; no collective on the data path, NCCL only for the barrier, the
max-over-ranks time and the parity gate.  "scaling" is "strong".

Verification gate: after the timed loop every rank
checks its timed output on the device (gf_verify_batch, Freivalds projections
over sampled generations); rank 0's cpu_baseline leg also compares the
oracle's result on its sample with the GPU's bytes.  Any mismatch prints
"parity": "FAIL" and exits 2.

The oracle is used only by the cpu_baseline leg and by --impl reference.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import seeded_inputs as si  # noqa: E402

METRIC = "source GB/s per field for RLNC encode at 1/2/4/8 B200; % of HBM roofline"
ALU_LANES_PER_SM_CLK = 64     # B300_MICROARCH.md: alu pipe rt_SMSP = 2 -> 16 lanes/clk/SMSP x 4
ISSUE_LANES_PER_SM_CLK = 128  # 4 SMSPs x 1 warp-instruction / clk x 32 lanes
N_SM = 148
SMEM_BYTES_PER_SM_CLK = 128   # shared-memory pipe (tools/ubench_smem.cu, profiles/r01_ubench_smem.txt)
TMEM_X2_BYTES_PER_SM_CLK = 132.8   # tcgen05.ld.32x32b.x2 from 32 warps (tools/ubench_tmem2.cu, profiles/r02_ubench_tmem2.txt)
# algorithmic ALU ops per byte-madd of the column kernel's inner loop:
# GF(256)/GF(16) 3 PRMT + 2 LOP3 per 4 byte-madds; GF(4) 2 LOP3; GF(2) 1 LOP3
OPS_PER_BYTE_MADD = {256: 5 / 4, 16: 5 / 4, 4: 2 / 4, 2: 1 / 4}
# GF(2) split engine (encode_gf2.cuh): per (source word, coded packet) 21 LOP3 +
# 22 IMAD per 32 terms -> issue slots per byte-madd (a 4-byte word = 4 byte-madds)
GF2_SPLIT_ISSUE_PER_BYTE_MADD = 43 / 32 / 4
LANEK = {2: (4, 1, 15), 4: (2, 1, 15), 16: (1, 1, 15), 256: (1, 2, 30)}   # SG, gathers/unit, build rows


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

def cpu_baseline(cfg, q, seconds_target=12.0, gpu_B=None):
    """The oracle (scalar C, plain loops), as it stands, on a bounded sample of
    the same workload (the first generations of the job), on this host's cores.
    gpu_B(g0, g1) -> host uint8 [g1-g0, K, M]: when given, the oracle's bytes
    are also compared with the GPU's for the sample (the bench's parity gate)."""
    import numpy as np

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
    Bo = oracle.encode_batch(q, A, C, threads=cores)
    dt = time.perf_counter() - t0
    src = gens * cfg.N * cfg.M
    out = {"value": round(src / dt / 1e9, 4), "unit": "GB/s", "cores": cores, "kind": "oracle",
           "sample": f"{gens} of {cfg.batch} generations of {cfg.name} GF({q}), threads={cores}; "
                     f"1-thread rate {g_cal * cfg.N * cfg.M / t1 / 1e9:.4f} GB/s",
           "seconds": round(dt, 2), "cpu_model": cpu_model()}
    if gpu_B is not None:
        bad = 0
        for g0 in range(0, gens, 1024):                # chunked: no second full-size copy
            g1 = min(gens, g0 + 1024)
            bad += int(np.count_nonzero(gpu_B(g0, g1) != Bo[g0:g1]))
        out["parity_vs_gpu"] = {"generations": gens, "mismatched_bytes": bad}
    return out


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


def parse(argv=None):
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
                    help="generations per launch for jobs that do not fit one GPU")
    ap.add_argument("--verify-gens", type=int, default=256,
                    help="generations per launch checked on the device after the timed loop")
    return ap.parse_args(argv)


def relaunch_under_torchrun(args) -> int:
    """--gpus N > 1 without a torchrun environment: start N ranks (one process
    per GPU) through torch.distributed.run on this node and return its code."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def workload_name(cfg, q, gens, ws, by_bytes):
    split = (f"byte-range sharded over {ws} GPU(s)" if by_bytes else
             f"{cfg.batch} generations split over {ws} GPU(s), {gens} per GPU")
    return (f"{cfg.name} RLNC encode GF({q}): N={cfg.N} source packets x M={cfg.M} B, "
            f"K={cfg.K} coded, {split}")


def rank_shard(shard, cfg, ws, rank):
    """This rank's part of the BASELINE job: by generation for
    C1 / C3 / C5, by packet byte range for C4 (cfg.shard)."""
    by_bytes = cfg.shard == "bytes"
    return shard.plan(cfg.batch, cfg.M, ws, rank, by="bytes" if by_bytes else "generation"), by_bytes


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
        "scaling": "strong", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (seeded splitmix64 byte stream, seeded_inputs)",
        "config": {"workload": workload_name(cfg, q, cfg.batch, 1, cfg.shard == "bytes"), "N": cfg.N,
                   "K": cfg.K, "M": cfg.M, "batch": cfg.batch, "field": q},
        "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": cores, "kind": "oracle",
                         "sample": f"{gens} generations per step of {cfg.name} GF({q}) "
                                   f"(scalar C oracle, {cores} threads, {cpu_model()})"},
        "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "byte_madds_per_step": gens * per_gen,
    }
    print(json.dumps(out), flush=True)


# ---------------------------------------------------------------- one workload on this rank

class Job:
    """This rank's share of one BASELINE workload over one field, resident in
    HBM in chunks of generations (one chunk when it fits)."""

    def __init__(self, gf, torch, cfg, q, sh, device, chunk_gens=0, mem_frac=0.8):
        self.gf, self.torch, self.cfg, self.q, self.sh, self.device = gf, torch, cfg, q, sh, device
        G, Ms, N, K = sh.generations, sh.columns, cfg.N, cfg.K
        self.G, self.Ms = G, Ms
        free, _ = torch.cuda.mem_get_info(device)
        per_gen = (N + K) * Ms + N * K
        chunk = min(G, chunk_gens or G)
        if per_gen * chunk > mem_frac * free:
            chunk = max(1, int(mem_frac * free // per_gen))
        self.chunk = chunk
        self.nchunks = -(-G // chunk) if G else 0
        self.A = torch.empty((chunk, N, Ms), dtype=torch.uint8, device=device)
        self.C = torch.empty((chunk, N, K), dtype=torch.uint8, device=device)
        self.B = torch.empty((chunk, K, Ms), dtype=torch.uint8, device=device)
        self.filled = -1

    def fill(self, j):
        """Inputs of chunk j, generated on the device by absolute index."""
        cfg, q, sh = self.cfg, self.q, self.sh
        seed = si.field_seed(cfg, q)
        g = sh.g0 + j * self.chunk
        n = min(self.chunk, self.G - j * self.chunk)
        self.gf.fill_random2d(self.A[:n].view(n * cfg.N, self.Ms), seed, si.STREAM_A,
                              g * cfg.N * cfg.M + sh.m0, cfg.M)
        self.gf.fill_random(self.C[:n], seed, si.STREAM_C, g * cfg.N * cfg.K, mask=q - 1)
        self.filled = j
        return n

    def encode(self, n):
        self.gf.encode_batch(self.q, self.A[:n], self.C[:n], self.B[:n])

    def verify(self, n, max_gens):
        """Freivalds check of the chunk's B on the device (gf_verify_batch) for
        up to max_gens generations spread over the chunk; returns the number of
        mismatching bytes."""
        torch, gf, q = self.torch, self.gf, self.q
        if n <= 0:
            return 0, 0
        step = max(1, n // max(1, max_gens))
        idx = torch.arange(0, n, step, device=self.device)[:max_gens]
        t = gf.freivalds_trials(q)
        A, C, B = self.A[idx].contiguous(), self.C[idx].contiguous(), self.B[idx].contiguous()
        R = torch.empty((idx.numel(), self.cfg.K, t), dtype=torch.uint8, device=self.device)
        gf.fill_random(R, si.field_seed(self.cfg, q), si.STREAM_FREIVALDS, 0, mask=q - 1)
        mism = gf.verify_batch(q, A, C, B, R)
        return int(mism.sum().item()), int(idx.numel())

    def free(self):
        del self.A, self.C, self.B


def time_job(job, steps, warmup, ws, dist, sampler=None):
    """Device-resident throughput.  One chunk: CUDA-event span over all steps.
    Several chunks (C5 does not fit one GPU): each chunk's inputs are generated
    before its launch and only the encode launches are timed (the sum of their
    event durations).  Returns (ms, per-launch ms list, launches, clocks)."""
    torch = job.torch
    stream = torch.cuda.current_stream(job.device)
    n0 = job.fill(0)
    torch.cuda.synchronize()
    for _ in range(warmup):
        job.encode(n0)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    if sampler:
        sampler.start()
        time.sleep(0.3)
    nl = steps * job.nchunks
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(nl)]
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    launches = 0
    t_start.record(stream)
    for s in range(steps):
        for j in range(job.nchunks):
            n = job.fill(j) if job.nchunks > 1 else n0
            e0, e1 = ev[s * job.nchunks + j]
            e0.record(stream)
            job.encode(n)
            e1.record(stream)
            launches += 1
    t_end.record(stream)
    torch.cuda.synchronize()
    clocks = sampler.stop() if sampler else None
    kern_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = t_start.elapsed_time(t_end) if job.nchunks == 1 else sum(kern_ms)
    if ws > 1:
        t = torch.tensor([total_ms], device=job.device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    return total_ms, kern_ms, launches, clocks


# ---------------------------------------------------------------- our arm

def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(args))
    ws, rank, local = dist_env()
    if ws != args.gpus:
        print(json.dumps({"error": f"WORLD_SIZE={ws} but --gpus {args.gpus}"}), flush=True)
        sys.exit(1)

    import torch
    import torch.distributed as dist

    from paper_1909_02871_b200 import gf, shard

    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=device)

    cfg = si.ENCODE_CONFIGS[args.config]
    q = args.field or cfg.fields[-1]
    for f in (2, 4, 16, 256):
        gf.init(f)
    peaks = load_peaks()
    sh, by_bytes = rank_shard(shard, cfg, ws, rank)
    N, K, M = cfg.N, cfg.K, cfg.M
    parity = {}

    # ---- headline: the configured workload over field q
    job = Job(gf, torch, cfg, q, sh, device, args.chunk_gens)
    sampler = ClockSampler(local)
    total_ms, kern_ms, launches, clocks = time_job(job, args.steps, args.warmup, ws, dist, sampler)
    job_src = cfg.batch * N * M                        # the whole job, all ranks
    value = job_src * args.steps / (total_ms / 1e3) / 1e9
    ms_per_step = total_ms / args.steps
    # gate: the last timed chunk's output, on the device
    bad, nver = job.verify(min(job.chunk, job.G - (job.nchunks - 1) * job.chunk), args.verify_gens)
    parity[f"GF({q})"] = {"device_freivalds_gens": nver, "mismatched_bytes": bad}

    # roofline of the dominant kernel: the encode launch (every launch of the
    # timed region is one); algorithmic work per launch / mean launch duration
    # (a rank without generations -- C1 at N > 1 -- launches nothing)
    avg_kernel_s = max(statistics.mean(kern_ms) if kern_ms else 0.0, 1e-6) / 1e3
    path = gf.encode_path(q, N, K, job.Ms)
    roof, hbm = dominant_roofline(q, N, K, job.Ms, job.chunk, path, avg_kernel_s, peaks)
    roof["traffic"] = lookup_traffic(q, cfg, job.chunk, job.Ms, path)
    alu = lookup_pipes(q, cfg, job.chunk, job.Ms, path)
    roof["kernel_ms"] = round(statistics.mean(kern_ms), 4) if kern_ms else None

    # the oracle's sample compared with the GPU's bytes (rank 0, N = 1): the
    # first generations of the job, still resident when the job is one chunk
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        gpu_B = None
        if job.nchunks == 1 and job.Ms == M:
            def gpu_B(g0, g1):
                return job.B[g0:g1].cpu().numpy()
        cpu = cpu_baseline(cfg, q, gpu_B=gpu_B)
        if "parity_vs_gpu" in cpu:
            parity[f"GF({q})"]["oracle_gens"] = cpu["parity_vs_gpu"]["generations"]
            parity[f"GF({q})"]["oracle_mismatched_bytes"] = cpu["parity_vs_gpu"]["mismatched_bytes"]
    job.free()
    del job
    torch.cuda.empty_cache()

    # ---- the other fields of the metric: GF(16) on C3, GF(2) / GF(4) on C5
    per_field = {str(q): field_entry(value, cfg, q, path, ms_per_step, total_ms, kern_ms, job_src, args.steps,
                                     peaks, sh, ws)}
    if not args.no_extra_fields:
        extra = [(si.C3, 16), (si.C3, 256), (si.C5, 2), (si.C5, 4)]
        for xcfg, f in extra:
            if str(f) in per_field:
                continue
            xsh, _ = rank_shard(shard, xcfg, ws, rank)
            xjob = Job(gf, torch, xcfg, f, xsh, device, 256 if xcfg is si.C5 else 0, mem_frac=0.6)
            st = max(2, args.steps // 3) if xjob.nchunks > 1 else max(3, args.steps // 2)
            xsampler = ClockSampler(local)
            tms, kms, nl, xclk = time_job(xjob, st, 1, ws, dist, xsampler)
            launches += nl
            xsrc = xcfg.batch * xcfg.N * xcfg.M
            xval = xsrc * st / (tms / 1e3) / 1e9
            bad, nver = xjob.verify(min(xjob.chunk, xjob.G - (xjob.nchunks - 1) * xjob.chunk),
                                    min(args.verify_gens, 64))
            parity[f"GF({f})"] = {"device_freivalds_gens": nver, "mismatched_bytes": bad}
            xpath = gf.encode_path(f, xcfg.N, xcfg.K, xjob.Ms)
            per_field[str(f)] = field_entry(xval, xcfg, f, xpath, tms / st, tms, kms, xsrc, st, peaks, xsh, ws,
                                            chunk=xjob.chunk, nchunks=xjob.nchunks)
            per_field[str(f)]["clocks"] = xclk
            xjob.free()
            del xjob
            torch.cuda.empty_cache()

    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(gf, torch, dist, cfg, q, sh, device, ws, args)

    # ---- parity gate over all ranks
    nbad = sum(v["mismatched_bytes"] + v.get("oracle_mismatched_bytes", 0) for v in parity.values())
    if ws > 1:
        t = torch.tensor([nbad], device=device, dtype=torch.int64)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        nbad = int(t.item())
    if rank == 0:
        out = {
            "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (seeded splitmix64 byte stream: uniform payload bytes, "
                    "i.i.d. uniform coefficients over F_q; generated on device)",
            "config": {"workload": workload_name(cfg, q, sh.generations, ws, by_bytes), "field": q,
                       "N": N, "K": K, "M": M, "batch": cfg.batch, "gens_per_gpu": sh.generations,
                       "bytes_per_packet_per_gpu": sh.columns, "global_batch": cfg.batch,
                       "launches_per_step": -(-sh.generations // max(1, roof.get("gens_per_launch", 1))),
                       "parallelism": (f"byte-range sharded x{ws}" if by_bytes else
                                       f"generation-split x{ws}") + ", no collective on the data path",
                       "l2": (f"inputs {sh.generations * N * sh.columns / 1e9:.2f} GB per GPU >> 126 MB L2 "
                              "(no flush)" if sh.generations * N * sh.columns > 2 * 126e6
                              else "L2-resident working set")},
            "per_field": per_field,
            "roofline": roof,
            "hbm": hbm,
            "alu": alu,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clocks,
            "gpu_launches": launches,
            "kernel_ms_per_launch": round(statistics.mean(kern_ms), 4) if kern_ms else None,
            "parity": "ok" if nbad == 0 else "FAIL",
            "parity_detail": parity,
        }
        print(json.dumps(out), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    if nbad:
        sys.exit(2)


def field_entry(value, cfg, q, path, ms_per_step, total_ms, kern_ms, job_src, steps, peaks, sh, ws,
                chunk=None, nchunks=1):
    """One field of the metric: source GB/s of the whole job and its fraction
    of the HBM roofline (read A, write B, read C at the measured copy peak, all
    GPUs)."""
    hbm_bytes = cfg.batch * ((cfg.N + cfg.K) * cfg.M + cfg.N * cfg.K)
    hbm_gbs = hbm_bytes * steps / (total_ms / 1e3) / 1e9
    e = {"value": round(value, 3), "unit": "GB/s", "workload": cfg.name, "N": cfg.N, "K": cfg.K, "M": cfg.M,
         "batch": cfg.batch, "kernel": path, "ms_per_step": round(ms_per_step, 4),
         "hbm_frac": round(hbm_gbs / (peaks["hbm_gbs"] * ws), 4)}
    if nchunks > 1:
        e["launches_per_step"] = nchunks
        e["gens_per_launch"] = chunk
        e["timing"] = "sum of encode-launch event durations (inputs of each chunk generated between launches)"
    alu = lookup_pipes(q, cfg, chunk if chunk else cfg.batch, sh.columns, path)
    if alu:
        e["alu"] = alu
    # the field's own encode launch against its roofline (same accounting as
    # the headline `roofline`): mean launch duration, generations per launch
    if kern_ms and sh.generations:
        gens = min(chunk, sh.generations) if chunk else sh.generations
        r, _ = dominant_roofline(q, cfg.N, cfg.K, sh.columns, gens, path, statistics.mean(kern_ms) / 1e3, peaks)
        e["roofline"] = {k: r[k] for k in ("bound", "achieved", "peak", "unit", "frac", "kernel",
                                           "tmem_read_frac", "issue_frac") if k in r}
    return e


def dominant_roofline(q, N, K, Ms, gens, path, kernel_s, peaks):
    """Roofline of the encode launch, on the METHOD'S
    algorithmic work only (no kernel-internal table builds in `achieved`).

    product-row (prow*): bound by the shared-memory pipe; algorithmic smem
    bytes = one gathered product byte per byte-madd; peak 148 SMs x 128 B/clk
    x max SM clock.  The kernel's own table stores (256 x 64 B per source,
    coded-packet tile and word tile) are reported beside it.
    lane-k: smem gathers (4 B per gathered word) + table build rows.
    gf2-split: HBM-bound design; its issue-slot use (43 per 32 terms) is
    reported beside.  column: ALU ops of the method per byte-madd.  Every entry
    carries the HBM view (read A, write B, read C)."""
    clk = peaks["sm_max_mhz"] * 1e6
    bm = N * K * Ms * gens
    hbm_bytes = ((N + K) * Ms + N * K) * gens
    hbm_ach = hbm_bytes / kernel_s / 1e9
    hbm = {"achieved": round(hbm_ach, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
           "frac": round(hbm_ach / peaks["hbm_gbs"], 4), "peak_source": peaks["source"]}
    smem_peak = N_SM * SMEM_BYTES_PER_SM_CLK * clk
    smem_src = (f"{N_SM} SMs x {SMEM_BYTES_PER_SM_CLK} B/clk shared-memory pipe x "
                f"{peaks['sm_max_mhz']:.0f} MHz (max SM clock; DESIGN.md 6)")
    if path.startswith("prow"):
        kc = {"prow": 64, "prow-32": 32, "prow-16": 16, "prow-nib": 64, "prow-32w": 32}[path]
        m_tiles = -(-(Ms // 4) // (768 if path == "prow-32w" else 384))
        k_tiles = -(-K // kc)
        s = 256 // kc                                   # sources per step (a table row is 256 B)
        n_pad = -(-N // s) * s
        builds = gens * n_pad * k_tiles * m_tiles * 256 * kc * (2 if path == "prow-32w" else 1)
        if path == "prow-nib":                          # 16 rows of 256 B per step of 4 sources
            builds = gens * (n_pad // 4) * k_tiles * m_tiles * 16 * 256
        ach = bm / kernel_s
        roof = {"bound": "smem", "achieved": round(ach / 1e12, 3), "peak": round(smem_peak / 1e12, 3),
                "unit": "TB/s", "frac": round(ach / smem_peak, 4), "peak_source": smem_src,
                "algorithmic": "1 gathered product byte per byte-madd",
                "table_build_bytes_per_launch": builds,
                "smem_frac_incl_table_builds": round((bm + builds) / kernel_s / smem_peak, 4)}
    elif path.startswith("lanek"):
        SG, G, R = LANEK[q]
        ktl = 64 if path == "lanek-64" else 32
        steps = -(-N // SG)
        k_tiles = -(-K // ktl)
        smem_bytes = gens * steps * (Ms // 4) * 4 * (K * G + R * k_tiles)
        ach = smem_bytes / kernel_s
        roof = {"bound": "smem", "achieved": round(ach / 1e12, 3), "peak": round(smem_peak / 1e12, 3),
                "unit": "TB/s", "frac": round(ach / smem_peak, 4), "peak_source": smem_src,
                "smem_bytes_per_launch": smem_bytes}
    elif path == "tmem":
        # TMEM lookup-table engine: HBM-bound design; its lookups read 8 B per
        # lane from tensor memory (tcgen05.ld.32x32b.x2), one per (4-bit group,
        # coded packet, 2-word lane slot), against the measured x2-load rate
        w = {2: 1, 4: 2, 16: 4, 256: 8}[q]
        ng = -(-(-(-N * w // 4)) // 4) * 4
        spans = -(-(Ms // 4) // 64)
        kp = -(-K // 32) * 32
        tm_bytes = gens * spans * 32 * ng * kp * 8
        tm_peak = N_SM * TMEM_X2_BYTES_PER_SM_CLK * clk
        ach = tm_bytes / kernel_s
        # the larger of the TMEM-read and HBM fractions is reported as the bound
        # (below); both stay on the line
        roof = {"bound": "tmem", "achieved": round(ach / 1e9, 1), "peak": round(tm_peak / 1e9, 1), "unit": "GB/s",
                "frac": round(ach / tm_peak, 4),
                "peak_source": (f"{N_SM} SMs x {TMEM_X2_BYTES_PER_SM_CLK} B/clk (tcgen05.ld.32x32b.x2 from plain "
                                f"warps, profiles/r02_ubench_tmem2.txt) x {peaks['sm_max_mhz']:.0f} MHz"),
                "tmem_read_bytes_per_launch": tm_bytes}
        roof["tmem_read_frac"] = roof["frac"]
    elif path == "gf2-split":
        issue_peak = N_SM * ISSUE_LANES_PER_SM_CLK * clk
        roof = dict(hbm, bound="hbm")
        roof["issue_frac"] = round(bm * GF2_SPLIT_ISSUE_PER_BYTE_MADD / kernel_s / issue_peak, 4)
        roof["issue_peak_source"] = f"{N_SM} SMs x 4 SMSPs x 32 lanes x {peaks['sm_max_mhz']:.0f} MHz"
    else:
        ops = bm * OPS_PER_BYTE_MADD[q]
        peak = N_SM * ALU_LANES_PER_SM_CLK * clk
        ach = ops / kernel_s
        roof = {"bound": "alu", "achieved": round(ach / 1e12, 3), "peak": round(peak / 1e12, 3),
                "unit": "Tops/s", "frac": round(ach / peak, 4),
                "peak_source": f"{N_SM} SMs x {ALU_LANES_PER_SM_CLK} ALU-pipe lanes/clk x "
                               f"{peaks['sm_max_mhz']:.0f} MHz (DESIGN.md 6)",
                "ops_per_byte_madd": OPS_PER_BYTE_MADD[q]}
    if hbm["frac"] > roof["frac"]:
        roof = dict(roof, **{k: v for k, v in hbm.items()}, bound="hbm")
    roof["kernel"] = f"encode {path} GF({q})"
    roof["gens_per_launch"] = gens
    roof["byte_madds_per_launch"] = bm
    roof["hbm_bytes_per_launch"] = hbm_bytes
    return roof, hbm


KERNEL_SOURCES = {"prow": "encode_prow.cuh", "prow-32": "encode_prow.cuh", "prow-16": "encode_prow.cuh",
                  "prow-nib": "encode_prow16.cuh", "prow-32w": "encode_prow.cuh",
                  "lanek-32": "encode_lanek.cuh", "lanek-64": "encode_lanek.cuh", "stream": "encode_stream.cuh",
                  "column-words": "encode_kernels.cuh", "gf2-split": "encode_gf2.cuh", "tmem": "encode_tmem.cuh"}


def kernel_sha(path):
    """sha256 of the CUDA source of the kernel an encode path launches (ties a
    committed ncu capture to the kernel code it measured)."""
    import hashlib
    f = KERNEL_SOURCES.get(path)
    if not f:
        return None
    return hashlib.sha256(open(os.path.join(ROOT, "paper_1909_02871_b200", "csrc", f), "rb").read()).hexdigest()[:16]


def lookup_pipes(q, cfg, gens, Ms, path):
    """The integer-ALU (and FMA) pipe activity of the encode launch, as fractions
    of peak, from the same committed ncu capture as `traffic` (None when the
    kernel source changed since).  The method's binding resource and its
    roofline fraction are in `roofline`; this is the integer-ALU side the
    north star asks for next to HBM."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        e = json.load(open(p)).get(f"{cfg.name}/GF{q}/{gens}/{Ms}")
        if e and e.get("kernel_sha") == kernel_sha(path) and "pipes" in e:
            return {"alu_pipe_active": e["pipes"]["alu"], "fma_pipe_active": e["pipes"]["fma"],
                    "issue_active": e["pipes"]["issue"], "unit": "fraction of peak (ncu, active cycles)",
                    "source": e["source"]}
    except Exception:
        pass
    return None


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
