"""Host-side logic of bench.py: roofline accounting and JSON contract pieces."""
import bench
import seeded_inputs as si


def test_roofline_lanek_is_smem_bound():
    peaks = {"hbm_gbs": 6546.9, "sm_max_mhz": 1965.0, "source": "test"}
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
