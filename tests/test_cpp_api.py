"""The header-only C++ mirror (include/kronprec_b200.hpp) compiles, links
against the C ABI and passes reference-style checks on the device."""
import os
import subprocess

import pytest

from paper_2311_15393_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _compile(tmp_path):
    exe = tmp_path / "test_cpp_api"
    cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
    libdir = os.path.dirname(_lib.LIB_PATH)
    subprocess.run([cxx, "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_cpp_api.cpp"), "-o", str(exe),
                    f"-L{libdir}", "-l:libkronprec_b200.so", f"-Wl,-rpath,{libdir}"], check=True)
    return exe


def test_cpp_api_compiles(tmp_path):
    assert _compile(tmp_path).exists()


@pytest.mark.gpu
def test_cpp_api_runs(tmp_path):
    exe = _compile(tmp_path)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "cpp api: ok" in out.stdout
