"""The kept C++ API (include/tiersim/*.hpp) compiles as a drop-in and passes reference-style cases."""
import subprocess
from pathlib import Path

import pytest

from conftest import has_gpu

ROOT = Path(__file__).resolve().parents[1]
SRC = ROOT / "tests" / "cpp" / "test_api.cpp"
BIN = ROOT / "tests" / "cpp" / "build" / "test_api"
LIBDIR = ROOT / "paper_2603_21257_b200"


def build():
    BIN.parent.mkdir(parents=True, exist_ok=True)
    if not BIN.exists() or BIN.stat().st_mtime < max(SRC.stat().st_mtime, (LIBDIR / "libtsb.so").stat().st_mtime,
                                                       *(p.stat().st_mtime for p in (ROOT / "include").rglob("*.h*"))):
        subprocess.run(["/usr/bin/g++", "-std=c++20", "-O1", "-Wall", "-Wextra", "-Werror", f"-I{ROOT / 'include'}",
                        str(SRC), f"-L{LIBDIR}", "-l:libtsb.so", f"-Wl,-rpath,{LIBDIR}", "-o", str(BIN)], check=True)
    return BIN


def test_cpp_api_host_cases():
    out = subprocess.run([str(build())], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "10 cases, 0 failures" in out.stdout  # every host case ran


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
def test_cpp_api_gpu_cases():
    out = subprocess.run([str(build()), "--gpu"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "17 cases, 0 failures" in out.stdout  # every host case plus every gpu case ran
