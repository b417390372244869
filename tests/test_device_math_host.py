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


@pytest.mark.skipif(shutil.which("nvcc") is None and not Path("/usr/local/cuda/bin/nvcc").exists(),
                    reason="nvcc not available")
def test_support_maps_exact_on_host(tmp_path, G):
    """The GJK support maps (model.cuh) return the full scan's first maximum bit for bit on
    synthetic hulls full of exact ties and on the drill mesh's parts (tests/cpp/support_map_exact.cu)."""
    import numpy as np
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    exe = tmp_path / "support_map_exact"
    subprocess.run([nvcc, "-O2", "--fmad=false", "-std=c++20", "-x", "cu", str(ROOT / "tests/cpp/support_map_exact.cu"),
                    "-o", str(exe)], check=True, capture_output=True)
    obj = G.load_object(ROOT / "paper_2412_16490_b200/assets/objects/drill_like.obj", 0.10)
    files = []
    for p in range(obj.n_parts):
        f = tmp_path / f"part{p}.txt"
        np.savetxt(f, obj.part_vertices(p), fmt="%.17g")
        files.append(str(f))
    hand = G.HandModel.from_file(ROOT / "paper_2412_16490_b200/assets/hands/shadow_like.json")
    verts = np.ctypeslib.as_array(hand.desc.verts, shape=(3 * hand.desc.n_verts,)).reshape(-1, 3)
    for l in range(hand.n_links):
        f = tmp_path / f"link{l}.txt"
        np.savetxt(f, verts[hand.link_vert_begin[l]:hand.link_vert_begin[l + 1]], fmt="%.17g")
        files.append(str(f))
    r = subprocess.run([str(exe)] + files, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 mismatches" in r.stdout
