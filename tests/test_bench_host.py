"""Host-side logic of bench.py: roofline accounting, the multi-GPU split and
launch checks, and JSON contract pieces."""
import os
import subprocess
import sys

import bench
import seeded_inputs as si
from paper_1909_02871_b200 import shard

PEAKS = {"hbm_gbs": 6546.9, "sm_max_mhz": 1965.0, "source": "test"}


def test_roofline_prow_counts_only_the_methods_work():
    """frac = byte-madds / (148 x 128 B x clock): the product-row kernel's own
    table stores are reported beside it, not in `achieved`."""
    t = 0.0150693                       # round-1 C3 GF(256) launch
    r, h = bench.dominant_roofline(256, 64, 64, 1500, 65536, "prow", t, PEAKS)
    bm = 64 * 64 * 1500 * 65536
    peak = 148 * 128 * 1965e6
    assert r["bound"] == "smem" and abs(r["frac"] - bm / t / peak) < 1e-4
    assert 0.70 < r["frac"] < 0.74                      # the verdict's recomputed 0.72
    assert r["table_build_bytes_per_launch"] == 65536 * 64 * 1 * 1 * 256 * 64
    assert 0.82 < r["smem_frac_incl_table_builds"] < 0.86
    # 32 / 16 coded packets per CTA: a 256-byte row holds 8 / 16 sources
    r32, _ = bench.dominant_roofline(256, 64, 32, 1500, 100, "prow-32", 1e-3, PEAKS)
    assert r32["table_build_bytes_per_launch"] == 100 * 64 * 1 * 1 * 256 * 32
    r32w, _ = bench.dominant_roofline(256, 256, 256, 65536, 2, "prow-32w", 1e-3, PEAKS)
    assert r32w["table_build_bytes_per_launch"] == 2 * 256 * 8 * 22 * 256 * 32 * 2    # 8 k-tiles, 22 tiles of 768
    r16, _ = bench.dominant_roofline(16, 20, 16, 1500, 100, "prow-16", 1e-3, PEAKS)
    assert r16["table_build_bytes_per_launch"] == 100 * 32 * 1 * 1 * 256 * 16


def test_roofline_gf2_split_is_hbm_with_issue_beside():
    r, h = bench.dominant_roofline(2, 32, 32, 1 << 20, 512, "gf2-split", 0.0155, PEAKS)
    assert r["bound"] == "hbm" and r["frac"] == h["frac"]
    assert 0 < r["issue_frac"] < 1


def test_roofline_tmem_reports_the_larger_of_tmem_reads_and_hbm():
    """TMEM engine (C5): TMEM bytes = one 8-byte .x2 load per lane per (4-bit
    group, coded packet of the 32-packet passes, 64-word span) against the
    measured .x2 rate; the bound is the larger fraction (GF(4): TMEM reads,
    GF(2): HBM), both stay on the line."""
    r, h = bench.dominant_roofline(4, 32, 32, 1 << 20, 256, "tmem", 0.0042, PEAKS)
    assert r["bound"] == "tmem" and r["frac"] > h["frac"] and r["tmem_read_frac"] == r["frac"]
    spans = (1 << 18) // 64
    assert r["tmem_read_bytes_per_launch"] == 256 * spans * 32 * 16 * 32 * 8    # 16 groups of {a, xa, b, xb}
    r2, h2 = bench.dominant_roofline(2, 32, 32, 1 << 20, 256, "tmem", 0.003, PEAKS)
    assert r2["tmem_read_bytes_per_launch"] == 256 * spans * 32 * 8 * 32 * 8     # 8 groups of 4 sources
    assert r2["bound"] == "hbm" and r2["frac"] == h2["frac"] and r2["tmem_read_frac"] < r2["frac"]
    r3, _ = bench.dominant_roofline(16, 17, 40, 4096, 3, "tmem", 1e-4, PEAKS)
    assert r3["tmem_read_bytes_per_launch"] == 3 * 16 * 32 * 20 * 64 * 8         # 17 groups -> 20, K -> 64
    assert 0 < r["tmem_read_frac"] < 1.5


def test_rank_shard_splits_the_baseline_job():
    for ws in (1, 2, 4, 8):
        parts = [bench.rank_shard(shard, si.C3, ws, r)[0] for r in range(ws)]
        assert sum(p.generations for p in parts) == 65536
        assert all(p.generations == 65536 // ws and p.columns == 1500 for p in parts)
        c5 = [bench.rank_shard(shard, si.C5, ws, r)[0] for r in range(ws)]
        assert sum(p.generations for p in c5) == 4096 and c5[-1].g1 == 4096
        c4 = [bench.rank_shard(shard, si.C4, ws, r) for r in range(ws)]
        assert all(by for _, by in c4) and sum(p.columns for p, _ in c4) == 65536
        assert all(p.generations == 2048 for p, _ in c4)


def test_world_size_must_match_gpus():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, bench.__file__, "--gpus", "2"], env=env, capture_output=True,
                         text=True, timeout=120)
    assert out.returncode == 1 and "WORLD_SIZE=1 but --gpus 2" in out.stdout


def test_roofline_lanek_is_smem_bound():
    peaks = PEAKS
    r, h = bench.dominant_roofline(256, 64, 64, 1500, 65536, "lanek-64", 0.0348, peaks)
    assert r["bound"] == "smem" and 0 < r["frac"] < 1
    # gathers: 2 x 4 B per (i, k, word); build: 30 rows x 4 B per (i, word) per k-tile
    assert r["smem_bytes_per_launch"] == 65536 * 64 * 375 * 4 * (64 * 2 + 30)
    assert r["hbm_bytes_per_launch"] == 65536 * ((64 + 64) * 1500 + 64 * 64)
    assert abs(r["achieved"] * 1e12 - r["smem_bytes_per_launch"] / 0.0348) < 1e9


def test_roofline_column_is_alu_bound_and_hbm_takes_over():
    peaks = {"hbm_gbs": 6546.9, "sm_max_mhz": 1965.0, "source": "test"}
    r, _ = bench.dominant_roofline(256, 16, 1, 1500, 1, "column-words", 1e-5, peaks)
    assert r["bound"] in ("alu", "hbm")
    r, _ = bench.dominant_roofline(2, 32, 1, 1 << 20, 64, "column-words", 0.01, peaks)
    assert r["bound"] == "hbm"          # K = 1: the stream dominates


def test_cpu_baseline_every_small_config():
    """The bench's cpu_baseline leg (the oracle on a bounded sample) runs for
    the one-generation C1 as well as C3 (regression: C1 has batch = 1)."""
    for name in ("C1", "C3"):
        cfg = si.ENCODE_CONFIGS[name]
        out = bench.cpu_baseline(cfg, 256, seconds_target=0.02)
        assert out["kind"] == "oracle" and out["value"] > 0 and out["cores"] >= 1
        assert f"of {cfg.batch} generations of {name}" in out["sample"]


def test_reference_arm_c1_line(capsys):
    """bench.py --impl reference prints one JSON line with the oracle's numbers
    (C1: one generation per step)."""
    import json
    import sys
    old = sys.argv
    sys.argv = ["bench.py", "--impl", "reference", "--config", "C1", "--steps", "2", "--warmup", "1"]
    try:
        args = bench.parse()
    finally:
        sys.argv = old
    bench.run_reference(args)
    line = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] == "oracle"


def test_job_plan_for_a_rank_without_work():
    """C1 has one generation: at N = 8 seven ranks hold none.  Their shard is
    empty and the bench code paths that divide by a launch time do not."""
    gens = [bench.rank_shard(shard, si.C1, 8, r)[0].generations for r in range(8)]
    assert sorted(gens) == [0] * 7 + [1]
    r, h = bench.dominant_roofline(256, 16, 1, 1500, 0, "stream", 1e-9, PEAKS)
    assert r["byte_madds_per_launch"] == 0


def test_ncu_traffic_matches_the_headline_kernel_source():
    """roofline.traffic comes from a committed ncu --set full capture, valid only
    for the kernel source it measured: the headline (C3 GF(256), product-row)
    entry must carry the current source hash, and its DRAM bytes must agree with
    the algorithmic A + B bytes of the launch to within 1% (no re-reads)."""
    import json
    import os
    import bench
    d = json.load(open(os.path.join(bench.ROOT, "profiles", "ncu_traffic.json")))
    e = d["C3/GF256/65536/1500"]
    assert e["kernel_sha"] == bench.kernel_sha("prow"), "re-capture the C3 kernel with ncu (profiles/ncu_traffic.json)"
    algorithmic = 65536 * (64 * 1500 + 64 * 64 + 64 * 1500)
    assert abs(e["bytes"] / algorithmic - 1) < 0.01


def test_alu_pipes_from_the_committed_capture():
    """The bench line's `alu` object: the integer-ALU / FMA pipe activity and
    issue activity of the headline launch, fractions of peak in (0, 1), from
    the same capture (and source hash) as `traffic`; None for a launch that
    was never captured."""
    import bench
    import seeded_inputs as si
    a = bench.lookup_pipes(256, si.C3, 65536, 1500, "prow")
    assert a is not None and a["source"].startswith("profiles/")
    for k in ("alu_pipe_active", "fma_pipe_active", "issue_active"):
        assert 0.0 < a[k] < 1.0
    assert bench.lookup_pipes(256, si.C3, 12345, 1500, "prow") is None
