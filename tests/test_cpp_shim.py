"""The C++ host side (csrc/fea_gpu.hpp, mirroring the reference API) — compiled against
libfea_gpu.so on CPU, run on the GPU."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
SRC = ROOT / "tests" / "cpp" / "test_shim.cpp"
OUT = ROOT / "tests" / "cpp" / "build" / "test_shim"


def build_shim_test() -> Path:
    OUT.parent.mkdir(parents=True, exist_ok=True)
    lib_dir = ROOT / "paper_2012_00585_b200"
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", f"-I{ROOT / 'include'}",
           f"-I{lib_dir / 'csrc'}", str(SRC), f"-L{lib_dir}", "-lfea_gpu",
           f"-Wl,-rpath,{lib_dir}", "-o", str(OUT)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return OUT


def test_shim_compiles_and_links():
    assert build_shim_test().exists()


@pytest.mark.gpu
def test_shim_parity_on_gpu(gpu):
    exe = build_shim_test()
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
