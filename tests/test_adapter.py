"""The C++ operator adapter (include/abftlp_b200.hpp): builds on CPU, runs the reference-style known
answers on the GPU (tests/cpp/adapter_test.cpp)."""
import subprocess
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parents[1]
BIN = REPO / "build" / "adapter_test"


def _build():
    subprocess.run(["make", "-s", "-C", str(REPO / "tests" / "cpp")], check=True)
    assert BIN.exists()


def test_adapter_builds():
    _build()


@pytest.mark.gpu
def test_adapter_known_answers_on_gpu():
    _build()
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ALL OK" in r.stdout
