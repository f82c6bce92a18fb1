"""Host-side logic of bench.py: roofline accounting and JSON contract pieces."""
import bench


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
