"""The C-ABI library on a CPU-only host: it loads, exports every symbol include/*.h declares, and its
host-only logic (status strings, config parsing, closed forms) behaves like the reference's
(P:tests/test_capi.cpp, P:tests/test_fault_lab.cpp:215-240). Device entry points must fail loudly
without a GPU -- there is no CPU fallback."""
import ctypes as C
import re
from pathlib import Path

import pytest

from campaign_configs import CAMPAIGNS
from paper_2103_00130_b200 import _lib as L

REPO = Path(__file__).resolve().parent.parent


def header_functions():
    names = set()
    for h in (REPO / "include").glob("*.h"):
        text = re.sub(r"/\*.*?\*/", "", h.read_text(), flags=re.S)
        names |= set(re.findall(r"\b(abftlp_[a-z0-9_]+)\s*\(", text))
    return sorted(names)


def test_every_header_symbol_is_exported_and_bound():
    names = header_functions()
    assert len(names) >= 39
    for n in names:
        assert hasattr(L.lib, n), f"{n} not exported by libabftlp_b200.so"
    assert set(names) <= set(L.EXPORTED), set(names) - set(L.EXPORTED)


def test_reference_surface_is_complete():
    # every function of the reference's include/abftlp.h (P:include/abftlp.h:25-89)
    ref_api = ["abftlp_status_str", "abftlp_last_error", "abftlp_campaign_load", "abftlp_campaign_parse",
               "abftlp_campaign_free", "abftlp_campaign_run", "abftlp_report_free", "abftlp_report_trials",
               "abftlp_report_detected", "abftlp_report_false_positives", "abftlp_report_detection_rate",
               "abftlp_report_write_csv", "abftlp_report_render", "abftlp_string_free", "abftlp_analyze",
               "abftlp_bench_gemm", "abftlp_bench_eb", "abftlp_eb_check_files"]
    for n in ref_api:
        assert hasattr(L.lib, n)


def test_status_strings():
    assert L.lib.abftlp_status_str(L.ERR_PARSE) == b"parse error"
    assert L.lib.abftlp_status_str(L.OK) == b"ok"
    assert L.lib.abftlp_status_str(7) == b"unknown status"


def test_error_paths_carry_messages():  # P:tests/test_capi.cpp:60-72
    h = C.c_void_p()
    assert L.lib.abftlp_campaign_load(b"/nonexistent/config.cfg", C.byref(h)) == L.ERR_IO
    assert "config not found" in L.last_error()
    assert L.lib.abftlp_campaign_parse(b"not a config", C.byref(h)) == L.ERR_PARSE
    assert L.lib.abftlp_campaign_parse(None, C.byref(h)) == L.ERR_INVALID_ARGUMENT
    assert L.lib.abftlp_campaign_load(b"x", None) == L.ERR_INVALID_ARGUMENT
    a = L.Analysis()
    assert L.lib.abftlp_analyze(0, 1, 1, 1, 1, C.byref(a)) == L.ERR_INVALID_ARGUMENT


def test_analyze_closed_forms():  # P:tests/test_capi.cpp:74-84
    a = L.Analysis()
    L.call("abftlp_analyze", 1, 800, 3200, 64, 100, C.byref(a))
    assert a.encode_overhead_b == pytest.approx(0.5 + 1.0 / 800 + 1.0 / 6400)
    assert a.encode_overhead_a > a.encode_overhead_b
    assert a.p_detect_b_bitflip == pytest.approx(1.0 - 3.0 / 256.0)
    assert a.p_detect_c_bitflip == 1.0
    assert a.p_detect_c_random == pytest.approx(126.0 / 127.0)
    assert a.eb_overhead == pytest.approx(1.0 / 64 + 1.0 / 300)
    assert a.eb_memory_overhead == pytest.approx(0.0625)


@pytest.mark.parametrize("text", [CAMPAIGNS[n][0] for n in CAMPAIGNS])
def test_shipped_campaign_configs_parse(text):
    h = C.c_void_p()
    L.call("abftlp_campaign_parse", text.encode(), C.byref(h))
    L.lib.abftlp_campaign_free(h)


@pytest.mark.parametrize("bad", [
    "[workload]\nkind = gemm\n",                                        # missing keys
    "[workload]\nkind = what\n",                                        # unknown kind
    CAMPAIGNS["gemm_smoke"][0] + "bogus = 1\n",                          # unknown key
    "[workload]\nkind = gemm\ntrials_per_shape = 1\nshapes = 0x4x4\n[fault]\ntarget = none\n",  # zero dim
    "[workload\nkind = gemm\n",                                         # malformed section
    "[workload]\nkind = gemm\ntrials_per_shape = 1x\nshapes = 1x4x4\n[fault]\ntarget = none\n",  # bad integer
    "[workload]\nkind = eb\ntable_rows = 10\ntable_dim = 4\npooling = 2\nbatch = 1\ntrials = 1\n"
    "[fault]\ntarget = eb_table\nbit_range = middle\n",                  # unknown bit range
])
def test_config_parse_errors(bad):  # P:tests/test_fault_lab.cpp:232-239
    h = C.c_void_p()
    assert L.lib.abftlp_campaign_parse(bad.encode(), C.byref(h)) == L.ERR_PARSE
    assert L.last_error().startswith("campaign config:")


def test_device_entry_points_fail_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = C.c_void_p()
    L.call("abftlp_campaign_parse", CAMPAIGNS["gemm_smoke"][0].encode(), C.byref(h))
    r = C.c_void_p()
    rc = L.lib.abftlp_campaign_run(h, C.byref(r))
    assert rc == L.ERR_INTERNAL and "CUDA" in L.last_error()
    L.lib.abftlp_campaign_free(h)
    w = C.c_void_p()
    assert L.lib.abftlp_gemm_encode(C.c_void_p(16), 4, 4, 4, None, C.byref(w)) == L.ERR_INTERNAL


def test_python_layer_refuses_cpu_tensors_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2103_00130_b200 import gemm
    with pytest.raises(RuntimeError, match="CUDA"):
        gemm.PackedEncodedWeight([[1, 2], [3, 4]])


def test_new_device_entry_points_reject_null_arguments():
    """The grouped-job, grouped-table and probe entry points validate their arguments before any device
    work (the reference's guarded() convention: -1 and "null argument" / the reason in last_error)."""
    vp = C.c_void_p
    assert L.lib.abftlp_eb_group_create(None, 0, None, None, None, None, None, None) == L.ERR_INVALID_ARGUMENT
    assert "null argument" in L.last_error()
    g = vp()
    tabs = (vp * 1)(None)
    assert L.lib.abftlp_eb_group_create(tabs, 1, None, None, None, None, None, C.byref(g)) == L.ERR_INVALID_ARGUMENT
    assert L.lib.abftlp_eb_group_checked_scatter(None, 1, 1, 1, 1, None, None, None) == L.ERR_INVALID_ARGUMENT
    assert L.lib.abftlp_gemm_checked_host_batched(None, 1, 1, 1, 1, None, None, 1, 1, None, 1, None, 1, None,
                                                  None) == L.ERR_INVALID_ARGUMENT
    assert L.lib.abftlp_gemm_checked_batched_faults(None, 1, 1, 1, 1, None, None, 1, 1, None, 1, 1, None, 1, None,
                                                    None, 0, None) == L.ERR_INVALID_ARGUMENT
    assert L.lib.abftlp_gemm_weight_flip_bit_batched(None, 0, 0, 0, 0, None) == L.ERR_INVALID_ARGUMENT
    assert L.lib.abftlp_gather_probe(None, 128, None, 0, None, None) == L.ERR_INVALID_ARGUMENT
    assert L.lib.abftlp_gather_probe(vp(16), 24, None, 0, vp(16), None) == L.ERR_INVALID_ARGUMENT
    assert "multiple of 16" in L.last_error()
    assert L.lib.abftlp_flip_bit(None, 4, 0, 0, None) == L.ERR_INVALID_ARGUMENT
