import ctypes
import os
import subprocess
import sys
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
ORACLE_SO = REPO / "oracle" / "liboracle.so"
REF_SO = REPO / "oracle" / "_ref" / "libabftlp_ref.so"
LIB_SO = REPO / "paper_2103_00130_b200" / "libabftlp_b200.so"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu)")
    # The checker and the product library are build artefacts (git-ignored); build them if absent.
    if not ORACLE_SO.exists():
        subprocess.run(["make", "-s", "-C", str(REPO / "oracle")], check=True)
    if not REF_SO.exists() and Path("/root/reference/proj/src").exists():
        subprocess.run(["make", "-s", "-C", str(REPO / "oracle"), "ref"], check=False)
    if not LIB_SO.exists():
        sys.path.insert(0, str(REPO / "paper_2103_00130_b200"))
        from paper_2103_00130_b200 import build as _b  # noqa: E402
        _b.build()


def _has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container (run -m gpu on a B200)")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def oracle():
    """The C restatement (test infrastructure)."""
    return ctypes.CDLL(str(ORACLE_SO))


@pytest.fixture(scope="session")
def ref():
    """The reference's own implementation compiled from its sources (oracle/_ref), if built."""
    if not REF_SO.exists():
        pytest.skip("oracle/_ref/libabftlp_ref.so not built (needs /root/reference)")
    return ctypes.CDLL(str(REF_SO))
