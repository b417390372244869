"""The C++ drop-in API: reference-style callers compiled against csrc/include/grasp/*.hpp and
linked to libgrasp_b200.so. tests/cpp/hand_api_kats.cpp ports test_hand.cpp's derivative
checks onto the host hand API (runs without a GPU); tests/cpp/drop_in_example.cpp drives
synthesize (single- and multi-device), quasi_static_check, fine_contact_query,
coarse_distance_energy and fine_grasp_surrogate on the GPU."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def build(tmp_path, G, name):
    from paper_2412_16490_b200 import _native as N
    exe = tmp_path / name
    subprocess.run(["g++", "-std=c++20", "-O1", f"-I{ROOT / 'paper_2412_16490_b200/csrc/include'}",
                    str(ROOT / "tests" / "cpp" / f"{name}.cpp"), str(N.LIB_PATH), f"-Wl,-rpath,{N.LIB_PATH.parent}",
                    "-o", str(exe)], check=True)
    return exe


def test_cpp_example_compiles_and_links(tmp_path, G):
    assert build(tmp_path, G, "drop_in_example").exists()


def test_cpp_hand_api_kats(tmp_path, G):
    exe = build(tmp_path, G, "hand_api_kats")
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout


@pytest.mark.gpu
def test_cpp_example_runs_on_gpu(tmp_path, G, engine):
    exe = build(tmp_path, G, "drop_in_example")
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "records 6" in r.stdout
    assert "sharded over 2 contexts: identical" in r.stdout
    assert "drop-in checks: 0 failures" in r.stdout
