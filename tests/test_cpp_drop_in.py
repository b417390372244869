"""The C++ drop-in API: a reference-style caller compiled against
csrc/include/grasp/*.hpp and linked to libgrasp_b200.so."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
SRC = ROOT / "tests" / "cpp" / "drop_in_example.cpp"


def build(tmp_path, G):
    from paper_2412_16490_b200 import _native as N
    exe = tmp_path / "drop_in_example"
    subprocess.run(["g++", "-std=c++20", "-O1", f"-I{ROOT / 'paper_2412_16490_b200/csrc/include'}", str(SRC),
                    str(N.LIB_PATH), f"-Wl,-rpath,{N.LIB_PATH.parent}", "-o", str(exe)], check=True)
    return exe


def test_cpp_example_compiles_and_links(tmp_path, G):
    assert build(tmp_path, G).exists()


@pytest.mark.gpu
def test_cpp_example_runs_on_gpu(tmp_path, G, engine):
    exe = build(tmp_path, G)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "records 6" in r.stdout
