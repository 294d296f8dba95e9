"""bench.py helpers that run without a GPU: the committed ncu capture feeds
roofline.traffic, and the reported library options are the non-default ones."""
import importlib.util
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    saved = sys.argv
    sys.argv = ["bench.py"]
    try:
        spec.loader.exec_module(mod)
    finally:
        sys.argv = saved
    return mod


def test_traffic_from_committed_capture():
    b = _bench()
    t = b._ncu_traffic(16384, 16)
    assert t is not None and 5e9 < t < 2e10  # DRAM bytes of one residue-GEMM launch (algorithmic 5.37e9)
    assert b._ncu_traffic(16384, 12) is None and b._ncu_traffic(1234, 16) is None


def test_option_defaults_match_library():
    import paper_2602_02549_b200 as oz
    b = _bench()
    assert set(b._OPTION_DEFAULTS) == set(oz.option_names())
    with oz.options(crt_cv=4):
        assert b.non_default_options().get("crt_cv") == 4


def test_clock_sampler_window(tmp_path):
    """The clock summary keeps only the samples inside the timed window (the
    sampler runs through the warm-up), and all of them when none fall in it."""
    import datetime
    import bench
    s = bench.ClockSampler(0)
    s.path = str(tmp_path / "clk.csv")
    t0 = datetime.datetime(2026, 10, 19, 12, 0, 0)
    lines = []
    for i, (mhz, cap) in enumerate([(1965, "Not Active"), (1965, "Not Active"), (1300, "Active"), (1310, "Active"),
                                    (1320, "Active"), (1900, "Not Active")]):
        ts = (t0 + datetime.timedelta(milliseconds=200 * i)).strftime("%Y/%m/%d %H:%M:%S.%f")[:-3]
        lines.append(f"{ts}, {mhz}, 1965, 900.0, 0x4, Not Active, Not Active, Not Active, {cap}")
    open(s.path, "w").write("\n".join(lines) + "\n")
    s.window = (t0 + datetime.timedelta(milliseconds=390), t0 + datetime.timedelta(milliseconds=810))
    out = s.summary()
    assert out["samples"] == 3 and out["sm_mhz"] == 1310.0 and out["reasons"] == ["sw_power_cap"]
    s.window = (t0 + datetime.timedelta(seconds=10), t0 + datetime.timedelta(seconds=11))
    assert s.summary()["samples"] == 6
