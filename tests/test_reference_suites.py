"""The reference's OWN conformance suites against the B200 library: P:tests/test_capi.cpp
(the C ABI, through a self-written doctest shim) and P:tests/acceptance.cpp (the 10 acceptance criteria, through the
API facade tests/cpp/facade) compiled unchanged from the reference's sources by `make -C oracle suites` (here,
where /root/reference exists) and linked against paper_2103_00130_b200/libabftlp_b200.so. The binaries travel to
the GPU box in oracle/_ref/; every operator they call runs on the GPU."""
import os
import subprocess
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parents[1]
REF_DIR = REPO / "oracle" / "_ref"
BINS = {"test_capi": REF_DIR / "test_capi_b200", "acceptance": REF_DIR / "acceptance_b200",
        "test_gemm_abft": REF_DIR / "test_gemm_abft_b200", "test_embedding_abft": REF_DIR / "test_embedding_abft_b200",
        "test_fault_lab": REF_DIR / "test_fault_lab_b200"}


def _ensure_built():
    if Path("/root/reference/proj/tests/acceptance.cpp").exists():
        subprocess.run(["make", "-s", "-C", str(REPO / "oracle"), "suites"], check=True)
    missing = [str(p) for p in BINS.values() if not p.exists()]
    if missing:  # the reference's sources are not on this machine and the prebuilt binaries did not travel
        pytest.skip(f"reference suites not built (run `make -C oracle suites` where /root/reference exists): {missing}")


def test_suites_built_against_b200_library():
    _ensure_built()
    for name, p in BINS.items():
        dyn = subprocess.run(["readelf", "-d", str(p)], capture_output=True, text=True, check=True).stdout
        assert "libabftlp_b200.so" in dyn, name  # the product library, not the reference's
        assert "libabftlp_ref" not in dyn, name


@pytest.mark.gpu
def test_reference_test_capi_passes_on_b200():
    _ensure_built()
    r = subprocess.run([str(BINS["test_capi"])], capture_output=True, text=True, timeout=600, cwd="/tmp")
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout + r.stderr
    assert "| 0 failed |" in r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("suite", ["test_gemm_abft", "test_embedding_abft", "test_fault_lab"])
def test_reference_operator_unit_suites_pass_on_b200(suite):
    """P:tests/test_gemm_abft.cpp (mod127 / checksum known answers, pack round trips over block layouts, 1000 random
    clean products, the aliasing sweep, the dual-encoded oracle) and P:tests/test_embedding_abft.cpp (row sums, exact
    integer path, weighted bags, the one-flagged-bag batch, ABEB file round trip) and P:tests/test_fault_lab.cpp
    (campaigns, config parsing and report serialization through the C ABI; its host-container injector cases run the
    facade's restatement), compiled unchanged."""
    _ensure_built()
    r = subprocess.run([str(BINS[suite])], capture_output=True, text=True, timeout=900, cwd="/tmp")
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout + r.stderr
    assert "| 0 failed |" in r.stdout


@pytest.mark.gpu
def test_reference_acceptance_passes_on_b200():
    _ensure_built()
    r = subprocess.run([str(BINS["acceptance"]), str(REF_DIR / "shapes.txt")], capture_output=True, text=True,
                       timeout=900, cwd="/tmp")
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all acceptance criteria passed" in r.stdout
    assert r.stdout.count("PASS criterion") == 10
