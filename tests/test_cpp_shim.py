"""Builds and runs tests/cpp/shim_test.cpp: the reference's pipeline tests written
against the C++ drop-in header (include/mpole_b200.hpp) on the GPU."""
import subprocess
from pathlib import Path

import pytest

from paper_2202_02847_b200 import build
from tests import oracle_lib

ROOT = Path(__file__).resolve().parent.parent


def compile_shim_test(out: Path) -> None:
    lib_dir = build.LIB_PATH.parent
    oracle_dir = oracle_lib.build_oracle().parent
    cmd = ["g++", "-std=c++20", "-O1", f"-I{ROOT / 'include'}", "-o", str(out),
           str(ROOT / "tests" / "cpp" / "shim_test.cpp"), f"-L{lib_dir}", "-lsolidfmm_b200",
           f"-L{oracle_dir}", "-loracle", f"-Wl,-rpath,{lib_dir}", f"-Wl,-rpath,{oracle_dir}", "-pthread"]
    subprocess.run(cmd, check=True, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)


def test_shim_header_compiles(tmp_path):
    """No GPU needed: the header and the C ABI agree (compile + link only)."""
    compile_shim_test(tmp_path / "shim_test")


@pytest.mark.gpu
def test_reference_pipeline_cases_through_the_shim(tmp_path):
    exe = tmp_path / "shim_test"
    compile_shim_test(exe)
    res = subprocess.run([str(exe)], stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True, timeout=600)
    assert res.returncode == 0, res.stdout
    assert "ALL PASSED" in res.stdout


def test_text_io_matches_the_reference_tool(tmp_path):
    """SOLID / charge text format of the shim against the reference's io.cpp (CPU only; needs
    the compiled reference, which is built here and travels with the snapshot)."""
    ref = ROOT / "oracle" / "_ref" / "libmpole_ref.so"
    if not ref.exists():
        oracle_lib.Reference.try_load("fma")
    if not ref.exists():
        pytest.skip("oracle/_ref is not built")
    lib_dir = build.LIB_PATH.parent
    exe = tmp_path / "io_test"
    cmd = ["g++", "-std=c++20", "-O1", f"-I{ROOT / 'include'}", "-o", str(exe),
           str(ROOT / "tests" / "cpp" / "io_test.cpp"), f"-L{lib_dir}", "-lsolidfmm_b200",
           f"-L{ref.parent}", "-lmpole_ref", f"-Wl,-rpath,{lib_dir}", f"-Wl,-rpath,{ref.parent}", "-pthread"]
    subprocess.run(cmd, check=True, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
    res = subprocess.run([str(exe)], stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True, timeout=120)
    assert res.returncode == 0 and "ALL PASSED" in res.stdout, res.stdout
