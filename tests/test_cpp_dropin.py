"""The C++ drop-in header (include/oz2g/emulate.hpp) against the C ABI:
compiles here; on a GPU box the binary runs the reference's emulate tests."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
LIBDIR = os.path.join(ROOT, "paper_2602_02549_b200")


def _build(tmp_path):
    exe = str(tmp_path / "test_dropin")
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"), SRC, "-o", exe,
                    "-L", LIBDIR, "-loz2g", f"-Wl,-rpath,{LIBDIR}"], check=True)
    return exe


def test_dropin_header_compiles_and_links(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_dropin_reference_emulate_suite(tmp_path, cuda):
    exe = _build(tmp_path)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
