"""examples/serve_ingest.cpp: a serving engine's use of the kept C++ API + the B200 data plane
compiles as a drop-in (CPU) and runs with every page verified (GPU)."""
import subprocess
from pathlib import Path

import pytest

from conftest import has_gpu

ROOT = Path(__file__).resolve().parents[1]
SRC = ROOT / "examples" / "serve_ingest.cpp"
BIN = ROOT / "tests" / "cpp" / "build" / "serve_ingest"
LIBDIR = ROOT / "paper_2603_21257_b200"


def build():
    BIN.parent.mkdir(parents=True, exist_ok=True)
    subprocess.run(["/usr/bin/g++", "-std=c++20", "-O1", "-Wall", "-Wextra", "-Werror", f"-I{ROOT / 'include'}",
                    str(SRC), f"-L{LIBDIR}", "-l:libtsb.so", f"-Wl,-rpath,{LIBDIR}", "-o", str(BIN)], check=True)
    return BIN


def test_example_compiles():
    assert build().exists()


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
@pytest.mark.parametrize("args", [["4", "32768", "lstf", "0", "0"], ["3", "16384", "fifo", "2", "20"]])
def test_example_runs_and_verifies(args):
    out = subprocess.run([str(build()), *args], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "0 mismatching words" in out.stdout
