"""The header-only C++ drop-in (include/batchrmq_b200.hpp) compiles against the
C-ABI and, on a GPU, runs the reference-style caller tests/cpp/wrapper_demo.cpp."""
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
PKG = ROOT / "paper_1706_06940_b200"


def build_demo(tmp_path):
    if not shutil.which("g++"):
        pytest.skip("g++ missing")
    exe = tmp_path / "wrapper_demo"
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", str(ROOT / "include"),
                    str(ROOT / "tests/cpp/wrapper_demo.cpp"), "-L", str(PKG), "-lbrmq",
                    f"-Wl,-rpath,{PKG}", "-o", str(exe)], check=True)
    return exe


def test_wrapper_compiles_and_links(tmp_path):
    assert build_demo(tmp_path).exists()


@pytest.mark.gpu
def test_wrapper_runs_on_gpu(tmp_path):
    out = subprocess.run([str(build_demo(tmp_path))], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    assert "wrapper_demo OK" in out.stdout
