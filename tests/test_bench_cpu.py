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
