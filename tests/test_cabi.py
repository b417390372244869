"""The C-ABI library: it loads on a GPU-less host, exports every function
include/grasp_b200.h declares, and fails loudly (status codes) instead of
falling back to the CPU."""
import ctypes as C
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def declared_functions():
    text = (ROOT / "include" / "grasp_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(grasp_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(G):
    from paper_2412_16490_b200 import _native as N
    lib = C.CDLL(str(N.LIB_PATH))
    names = declared_functions()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(names) <= set(N.SIGNATURES), set(names) - set(N.SIGNATURES)


def test_library_is_sm100a(G):
    import subprocess
    from paper_2412_16490_b200 import _native as N
    out = subprocess.run(["cuobjdump", "--list-elf", str(N.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_gpu_means_error_not_fallback(G):
    import shutil
    import subprocess
    if shutil.which("nvidia-smi") and subprocess.run(["nvidia-smi", "-L"], capture_output=True).returncode == 0:
        pytest.skip("GPU present")
    with pytest.raises(G.CudaError):
        G.Engine(0)


def test_error_codes_map_to_reference_exceptions(G):
    with pytest.raises(G.HandError):
        G.HandModel.from_json('{"format_version": 1, "links": []}')
    with pytest.raises(G.ObjectError):
        G.make_primitive("dodecahedron", 0.1)
    with pytest.raises(G.InvalidArgument):
        G.parse_run_config('{"qp": {"alpha": 3.0}}')
    from paper_2412_16490_b200 import _native as N
    assert N.lib().grasp_last_error().decode()


def test_descriptors_round_trip(G, trident):
    d = trident.desc
    assert (d.n_links, d.dof, d.n_tips, d.n_proxies, d.n_pairs) == (7, 6, 3, 19, 15)
    assert trident.link_vert_begin[-1] == d.n_verts and trident.link_face_begin[-1] == d.n_faces
