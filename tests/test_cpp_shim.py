"""The header-only C++ drop-in (include/ihs_b200.hpp) with the reference's
hot-path unit tests re-targeted at it (tests/cpp/test_shim.cpp)."""
import pathlib
import subprocess

import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
PKG = ROOT / "paper_2006_05874_b200"


def _build(tmp_path_factory):
    out = tmp_path_factory.mktemp("shim") / "test_shim"
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", f"-I{ROOT / 'include'}", str(ROOT / "tests/cpp/test_shim.cpp"),
           f"-L{PKG}", "-lihs_b200", f"-Wl,-rpath,{PKG}", "-o", str(out)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


@pytest.fixture(scope="module")
def shim_binary(tmp_path_factory, ihs):
    return _build(tmp_path_factory)


def test_shim_compiles_against_the_c_abi(shim_binary):
    assert shim_binary.exists()


@pytest.mark.gpu
def test_reference_unit_tests_pass_on_the_shim(shim_binary, gpu):
    r = subprocess.run([str(shim_binary)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
