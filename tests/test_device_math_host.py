"""Device math restated on the host (same headers as the kernels, compiled by nvcc as host
code): the closed-form KKT solves and the zero-padded FullPivLU are bit-identical to the
general solve, and the correctly rounded sin/cos matches glibc on >= 99.5% of arguments."""
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.skipif(shutil.which("nvcc") is None and not Path("/usr/local/cuda/bin/nvcc").exists(),
                    reason="nvcc not available")
def test_device_math_exact_on_host(tmp_path):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    exe = tmp_path / "gjk_exact"
    subprocess.run([nvcc, "-O2", "--fmad=false", "-std=c++20", "-x", "cu", str(ROOT / "tests/cpp/gjk_exact.cu"),
                    "-o", str(exe)], check=True, capture_output=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
