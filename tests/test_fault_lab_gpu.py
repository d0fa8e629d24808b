"""Fault lab on the B200: injectors, GPU campaigns against the reference's golden outcomes, reports,
eb-check over files and the overhead benches (P:tests/test_fault_lab.cpp, P:tests/test_capi.cpp,
P:tests/acceptance.cpp criteria 1-3, 7)."""
import ctypes as C
import json
import os
import tempfile
from pathlib import Path

import numpy as np
import pytest
import torch

import oracle_api as O
from campaign_configs import CAMPAIGNS

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def F():
    from paper_2103_00130_b200 import fault_lab
    return fault_lab


@pytest.mark.parametrize("name", list(CAMPAIGNS))
def test_campaign_golden_counts(F, name):
    """GPU campaigns reproduce the reference's reports exactly (2793/2800, 198/200, 7/400 ...)."""
    text, expect = CAMPAIGNS[name]
    assert json.loads((GOLD / "campaigns.json").read_text())["cases"][name] == list(expect)
    rep = F.run_campaign(text)
    assert (rep.trials, rep.detected, rep.falsePositives) == expect


def test_campaign_report_rendering(F):  # P:tests/test_capi.cpp:34-58, P:tests/test_fault_lab.cpp:242-256
    text = "[workload]\nkind = gemm\ntrials_per_shape = 25\nshapes = 2x32x32, 4x16x16\n[fault]\n" \
           "target = intermediate_c\nmodel = single_bit_flip\nseed = 3\n"
    rep = F.run_campaign(text)
    assert (rep.trials, rep.detected, rep.falsePositives) == (50, 50, 0)
    assert rep.detectionRate() == pytest.approx(1.0)
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "r.csv")
        rep.write_csv(p)
        csv = open(p).read()
    assert csv.startswith("target,model,bit_range,shape_or_dims,trials,detected,not_detected,false_positives,"
                          "detection_rate,ci_low,ci_high\n")
    assert "2x32x32" in csv and "total" in csv
    assert "intermediate_c" in rep.render()
    again = F.run_campaign(text)
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "r.csv")
        again.write_csv(p)
        assert open(p).read() == csv


def test_campaign_matches_reference_csv(F, ref):
    """Byte-identical CSV and table renderings vs the reference's own report writer."""
    R = ref
    for name in ("gemm_bitflip_b", "eb_low4"):
        text = CAMPAIGNS[name][0]
        h, r = C.c_void_p(), C.c_void_p()
        assert R.abftlp_campaign_parse(text.encode(), C.byref(h)) == 0
        assert R.abftlp_campaign_run(h, C.byref(r)) == 0
        mine = F.run_campaign(text)
        with tempfile.TemporaryDirectory() as d:
            p1, p2 = os.path.join(d, "ref.csv"), os.path.join(d, "mine.csv")
            R.abftlp_report_write_csv(r, p1.encode())
            mine.write_csv(p2)
            assert open(p1).read() == open(p2).read()
        out = C.c_char_p()
        assert R.abftlp_report_render(r, C.byref(out)) == 0
        assert out.value.decode() == mine.render()  # the aligned table, byte for byte


def test_workload_target_mismatch(F):  # P:tests/test_fault_lab.cpp:189-202
    from paper_2103_00130_b200 import _lib
    with pytest.raises(_lib.InvalidArgument):
        F.run_campaign("[workload]\nkind = gemm\ntrials_per_shape = 1\nshapes = 1x8x8\n[fault]\ntarget = eb_table\n")
    with pytest.raises(_lib.InvalidArgument):
        F.run_campaign("[workload]\nkind = eb\ntable_rows = 100\ntable_dim = 8\npooling = 4\nbatch = 2\ntrials = 1\n"
                       "[fault]\ntarget = weight_b\n")


def test_random_value_model_runs_and_detects(F):
    text = CAMPAIGNS["gemm_bitflip_c"][0].replace("single_bit_flip", "random_value").replace("= 200", "= 10")
    rep = F.run_campaign(text)
    det = O.gemm_campaign([tuple(map(int, s.split("x"))) for s in
                           text.split("shapes = ")[1].split("\n")[0].split(", ")], 10, "intermediate_c", 20260823,
                          model="random_value")
    assert rep.detected == int(det.sum())


def test_injectors_deterministic_single_mutation(F):  # P:tests/test_fault_lab.cpp:67-98
    from paper_2103_00130_b200 import gemm
    spec = F.FaultSpec(F.FaultTarget.weight_B, F.FaultModel.single_bit_flip, F.BitRange.all, 1234)
    b = np.random.default_rng(52).integers(-128, 128, (16, 24)).astype(np.int8)
    p1, p2 = gemm.PackedEncodedWeight(b), gemm.PackedEncodedWeight(b)
    r1, r2 = F.inject_weight_B(p1, spec, 5), F.inject_weight_B(p2, spec, 5)
    assert r1.injected and r1 == r2 and r1.before != r1.after
    e1 = p1.encoded().cpu().numpy()
    assert int((e1[:, :24] != b).sum()) == 1
    # same draw as the C restatement of inject_weight_B
    bb = b.copy()
    rec = np.zeros(5, np.int64)
    O.orc().orc_inject_weight_B(O.P(bb), O.sz(16), O.sz(24), 0, 0, 0, C.c_uint64(1234), C.c_uint64(5), O.P(rec))
    assert np.array_equal(e1[:, :24], bb)
    assert not F.inject_weight_B(p1, F.FaultSpec(), 0).injected


def test_inject_eb_table_high4(F):  # P:tests/test_fault_lab.cpp:100-119
    from paper_2103_00130_b200 import embedding as E
    spec = F.FaultSpec(F.FaultTarget.eb_table, F.FaultModel.single_bit_flip, F.BitRange.high4, 77)
    rng = np.random.default_rng(53)
    for trial in range(20):
        rows = rng.integers(-128, 128, (100, 8)).astype(np.int8)
        t = E.QuantEmbeddingTable(rows, np.full(100, 0.01, np.float32), np.zeros(100, np.float32))
        rec = F.inject_eb_table(t, [E.IndexBag([1, 5, 9])], spec, trial)
        delta = (rec.before ^ rec.after) & 0xFF
        assert rec.injected and delta and not (delta & 0x0F)


def test_inject_intermediate_c_matches_oracle(F):
    from paper_2103_00130_b200 import gemm
    a, b = O.gemm_inputs(20260823, 1, 64, 512, 512)
    res = gemm.abft_gemm(a, gemm.PackedEncodedWeight(b))
    spec = F.FaultSpec(F.FaultTarget.intermediate_C, F.FaultModel.single_bit_flip, F.BitRange.all, 20260823)
    rec = F.inject_intermediate_C(res, spec, 1)
    gold = [c for c in json.loads((GOLD / "gemm.json").read_text())["cases"] if c["label"] == "G1" and c["trial"] == 1][0]
    assert (rec.before, rec.after) == (gold["c_fault"]["before"], gold["c_fault"]["after"])
    assert gemm.verify_checksums(res.cTemp) == 1


def test_inject_before_encoding_is_absorbed(F):  # P:tests/test_fault_lab.cpp:121-133
    from paper_2103_00130_b200 import gemm
    rng = np.random.default_rng(54)
    a = rng.integers(0, 256, (4, 16)).astype(np.uint8)
    b = rng.integers(-128, 128, (16, 12)).astype(np.int8)
    rec = np.zeros(5, np.int64)
    O.orc().orc_inject_weight_B(O.P(b), O.sz(16), O.sz(12), 0, 0, 0, C.c_uint64(99), C.c_uint64(0), O.P(rec))
    assert gemm.abft_gemm(a, gemm.PackedEncodedWeight(b)).errCount == 0


def test_eb_check_files(F):  # P:tests/test_capi.cpp:98-138
    from paper_2103_00130_b200 import _lib
    from paper_2103_00130_b200 import embedding as E
    rng = np.random.default_rng(61)
    rows = rng.integers(-128, 128, (50, 8)).astype(np.int8)
    sums = O.row_sums(rows)
    with tempfile.TemporaryDirectory() as d:
        tp, ip = os.path.join(d, "t.abeb"), os.path.join(d, "bags.txt")
        E.save_table(E.QuantEmbeddingTable(rows, np.full(50, 0.01, np.float32), np.full(50, 0.1, np.float32)), tp)
        with open(ip, "w") as f:
            f.write("0 1 2 3\n10 10 11\n4:0.5 5:1.5\n")
        bags, flagged, text = F.eb_check_files(tp, ip)
        assert (bags, flagged) == (3, 0) and "bag 2: ok" in text
        stale = sums.copy()
        stale[1] += 100
        E.save_table(E.QuantEmbeddingTable(rows, np.full(50, 0.01, np.float32), np.full(50, 0.1, np.float32),
                                           row_sums=stale), tp)
        with pytest.raises(_lib.IoError):
            F.eb_check_files(tp, ip)
        assert F.eb_check_files(tp, ip, skip_validation=True)[1] == 1
        with pytest.raises(_lib.IoError):
            F.eb_check_files(tp, "/nonexistent/bags.txt", True)
        with open(ip, "w") as f:
            f.write("0 x1\n")
        with pytest.raises(_lib.ParseError):
            F.eb_check_files(tp, ip, True)


def test_eb_check_files_render_matches_reference(F, ref):
    """Same bag verdict lines (including the printed sums) as the reference's eb-check."""
    from paper_2103_00130_b200 import embedding as E
    rng = np.random.default_rng(62)
    rows = rng.integers(-128, 128, (300, 32)).astype(np.int8)
    with tempfile.TemporaryDirectory() as d:
        tp, ip = os.path.join(d, "t.abeb"), os.path.join(d, "bags.txt")
        E.save_table(E.QuantEmbeddingTable(rows, rng.uniform(0.005, 0.02, 300).astype(np.float32),
                                           rng.uniform(-1, 1, 300).astype(np.float32)), tp)
        with open(ip, "w") as f:
            for b in range(20):
                toks = [f"{i}" if b % 3 else f"{i}:{w:.3f}" for i, w in
                        zip(rng.integers(0, 300, 40), rng.uniform(0, 2, 40))]
                f.write(" ".join(toks) + ("  # comment\n" if b == 5 else "\n"))
            f.write("\n   \n")
        R = ref
        R.abftlp_string_free.argtypes = [C.c_void_p]
        nb, fl, out = C.c_uint64(), C.c_uint64(), C.c_void_p()
        assert R.abftlp_eb_check_files(tp.encode(), ip.encode(), 0, C.byref(nb), C.byref(fl), C.byref(out)) == 0
        ref_text = C.string_at(out).decode()
        bags, flagged, text = F.eb_check_files(tp, ip)
        assert (bags, flagged) == (nb.value, fl.value) and text == ref_text


def test_benches_validate_and_report(F):  # P:tests/test_capi.cpp:86-96
    from paper_2103_00130_b200 import _lib
    with pytest.raises(_lib.InvalidArgument):
        F.bench_gemm(2, 16, 16, 1)
    r = F.bench_gemm(2, 16, 16, 5)
    assert r["baseline_ns"] > 0 and r["abft_ns"] > 0 and np.isfinite(r["overhead_fraction"])
    r = F.bench_eb(500, 16, 20, 2, 5)
    assert r["baseline_ns"] > 0


def test_device_splitmix_against_the_reference_draws():
    """The device generator against the reference's own raw draws (tests/golden/rng.json, written from the reference
    build): kind 3 (next_below) with bound 2^64 - 1 returns the raw 64-bit draw (P:src/rng.hpp:10-43); an offset into
    the stream gives the same draws as generating from its start (counter-based)."""
    import ctypes as C
    import json

    import torch

    from paper_2103_00130_b200 import _lib as L
    from paper_2103_00130_b200 import rng as R
    cases = json.loads((GOLD / "rng.json").read_text())["cases"]
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    for c in cases:
        want = np.array([int(x) for x in c["draws"]], dtype=np.uint64)
        out = torch.empty(len(want), dtype=torch.int64, device="cuda")
        L.call("abftlp_generate", C.c_void_p(out.data_ptr()), len(want), c["seed"], c["stream"], 0, 3, 0.0, 0.0,
               (1 << 64) - 1, st)
        got = out.cpu().numpy().view(np.uint64)
        assert np.array_equal(got, want), (c["seed"], c["stream"])
        assert np.array_equal(R.draws(c["seed"], c["stream"], 0, len(want)), want)  # the host mirror too
        tail = torch.empty(3, dtype=torch.int64, device="cuda")
        L.call("abftlp_generate", C.c_void_p(tail.data_ptr()), 3, c["seed"], c["stream"], 5, 3, 0.0, 0.0, (1 << 64) - 1, st)
        assert np.array_equal(tail.cpu().numpy().view(np.uint64), want[5:8])
