import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C ABI")
    config.addinivalue_line("markers", "slow: longer CPU-oracle runs")


@pytest.fixture(scope="session")
def G():
    import paper_2412_16490_b200 as pkg
    from paper_2412_16490_b200 import _native
    if not _native.LIB_PATH.exists():
        import __graft_entry__
        __graft_entry__.build()
    return pkg


@pytest.fixture(scope="session")
def O():
    from oracle import oracle as orc
    orc.lib()
    return orc


@pytest.fixture(scope="session")
def trident(G):
    return G.HandModel.builtin()


def _has_gpu() -> bool:
    import shutil
    import subprocess
    if not shutil.which("nvidia-smi"):
        return False
    return subprocess.run(["nvidia-smi", "-L"], capture_output=True).returncode == 0


@pytest.fixture(scope="session")
def engine(G):
    """The CUDA engine on cuda:0. Skips only where no GPU exists; on a GPU
    box a missing/broken extension raises instead of falling back."""
    if not _has_gpu():
        pytest.skip("no CUDA device")
    return G.Engine(0)


def use(engine, hand, obj):
    if engine.hand is not hand:
        engine.set_hand(hand)
    if engine.obj is not obj:
        engine.set_object(obj)
    return engine
