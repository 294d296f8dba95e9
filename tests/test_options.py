"""Tuning options (csrc/options.cpp, oz2g_set_option / oz2g_get_option): the
table of names, defaults and valid values, the environment read at first use,
and the Python wrappers.  No GPU needed (no kernel runs)."""
import json
import os
import subprocess
import sys

import pytest

import paper_2602_02549_b200 as oz

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

DEFAULTS = {"gemm": 0, "fused": 0, "fused_mc": 0, "fused_fence": 1, "spec": -1, "graph": 1, "pdl": 1, "group_m": 0,
            "group_n": 0, "l2hint": 0, "crt_overlap": 0, "crt_cv": 8, "wblock_min_mb": 2048, "gemm_fence": 0,
            "epi_warps": 0, "pair_stages": 4, "rowscan_threads": 0, "resid_stream": 0, "spec_tail": 1, "dist_pipeline": 1, "debug_sync": 0, "resid_fast": 1}


def _in_subprocess(env_extra, code):
    env = {k: v for k, v in os.environ.items() if not k.startswith("OZ2G_")}
    env.update(env_extra)
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    return json.loads(out.stdout.strip().splitlines()[-1])


def test_names_and_defaults():
    code = ("import json, paper_2602_02549_b200 as oz; "
            "print(json.dumps({n: oz.get_option(n) for n in oz.option_names()}))")
    assert _in_subprocess({}, code) == DEFAULTS


def test_environment_at_first_use():
    code = ("import json, paper_2602_02549_b200 as oz; "
            "print(json.dumps({n: oz.get_option(n) for n in ('gemm', 'spec', 'graph', 'crt_cv', 'pair_stages', 'pdl')}))")
    got = _in_subprocess({"OZ2G_GEMM": "mcast", "OZ2G_SPEC": "0", "OZ2G_GRAPH": "0", "OZ2G_CRT_CV": "4",
                          "OZ2G_PAIR_STAGES": "9", "OZ2G_PDL": "x"}, code)
    # out-of-range (pair_stages 9) and unparsable (pdl "x") values keep the default
    assert got == {"gemm": 2, "spec": 0, "graph": 0, "crt_cv": 4, "pair_stages": 4, "pdl": 1}


def test_set_get_and_validation():
    with oz.options(spec=2, gemm="pair", crt_cv=4):
        assert (oz.get_option("spec"), oz.get_option("gemm"), oz.get_option("crt_cv")) == (2, 1, 4)
    assert oz.get_option("crt_cv") in (4, 8)
    for name, bad in (("spec", 3), ("spec", -2), ("crt_cv", 6), ("epi_warps", 2), ("pdl", 3), ("graph", -1)):
        before = oz.get_option(name)
        with pytest.raises(oz.InvalidArgument, match="out of range"):
            oz.set_option(name, bad)
        assert oz.get_option(name) == before
    with pytest.raises(oz.InvalidArgument, match="unknown option"):
        oz.set_option("no_such_option", 1)
    with pytest.raises(oz.InvalidArgument, match="unknown option"):
        oz.get_option("GEMM")
    with pytest.raises(oz.InvalidArgument):
        oz.set_option("gemm", "triple")


def test_options_context_restores_on_error():
    before = oz.get_option("fused")
    with pytest.raises(RuntimeError):
        with oz.options(fused=1):
            assert oz.get_option("fused") == 1
            raise RuntimeError("boom")
    assert oz.get_option("fused") == before
