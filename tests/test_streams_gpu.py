"""Concurrency: one encoded weight / table shared by calls on several streams at once (per-stream
workspaces, SURVEY 8b 'per-call scratch lives per stream'), and whole sequences captured as CUDA graphs."""
import ctypes as C

import numpy as np
import pytest
import torch

import oracle_api as O

pytestmark = pytest.mark.gpu


def test_shared_weight_across_streams():
    from paper_2103_00130_b200 import _lib
    from paper_2103_00130_b200 import gemm as G
    m, n, k = 256, 1024, 2048
    b = O.gemm_inputs(5, 0, m, n, k)[1]
    pb = G.PackedEncodedWeight(b)
    streams = [torch.cuda.Stream() for _ in range(4)]
    As = [O.gemm_inputs(5, t + 1, m, n, k)[0] for t in range(4)]
    outs = []
    for t, s in enumerate(streams):
        with torch.cuda.stream(s):
            a = torch.from_numpy(As[t]).cuda()
            c = torch.empty((m, n + 1), dtype=torch.int32, device="cuda")
            fl = torch.empty(m, dtype=torch.uint8, device="cuda")
            er = torch.empty(1, dtype=torch.int32, device="cuda")
            for _ in range(5):  # several back-to-back calls per stream, all streams in flight together
                _lib.call("abftlp_gemm_checked", C.c_void_p(a.data_ptr()), m, k, pb.handle, C.c_void_p(c.data_ptr()),
                          n + 1, C.c_void_p(c.data_ptr() + 4 * n), n + 1, C.c_void_p(fl.data_ptr()),
                          C.c_void_p(er.data_ptr()), None, C.c_void_p(s.cuda_stream))
            outs.append((a, c, fl, er))
    torch.cuda.synchronize()
    for t, (a, c, fl, er) in enumerate(outs):
        ct, _, e = O.abft_gemm(As[t], b)
        assert np.array_equal(c.cpu().numpy(), ct) and int(er.item()) == e == 0 and not fl.any()


def test_eb_graph_capture_and_streams():
    from paper_2103_00130_b200 import embedding as E
    rng = np.random.default_rng(9)
    R, d = 20000, 64
    rows = rng.integers(0, 256, (R, d // 2)).astype(np.uint8)
    sc = rng.uniform(1e-3, 1e-2, R).astype(np.float16)
    bi = rng.uniform(-1, 1, R).astype(np.float16)
    t = E.QuantEmbeddingTable(rows, sc, bi, elem="u4", dim=d)
    lens = rng.integers(0, 150, 700)
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    idx = rng.integers(0, R, off[-1]).astype(np.int64)
    w = rng.uniform(0, 1, off[-1]).astype(np.float32)
    ref = O.eb(rows, sc, bi, off, idx, w, elem="u4", dim=d)
    s = torch.cuda.Stream()
    offd, idxd, wd = (torch.from_numpy(x).cuda() for x in (off, idx, w))
    with torch.cuda.stream(s):
        res = E.eb_csr(t, offd, idxd, wd, stream=s)  # warm-up allocates the stream's workspace
    g = torch.cuda.CUDAGraph()
    out = torch.empty((700, d), dtype=torch.float32, device="cuda")
    fl = torch.empty(700, dtype=torch.uint8, device="cuda")
    from paper_2103_00130_b200 import _lib
    with torch.cuda.graph(g, stream=s):
        _lib.call("abftlp_eb_checked", t.handle, C.c_void_p(offd.data_ptr()), C.c_void_p(idxd.data_ptr()), 700,
                  C.c_void_p(wd.data_ptr()), C.c_void_p(out.data_ptr()), d, C.c_void_p(fl.data_ptr()), None, None,
                  None, None, C.c_void_p(s.cuda_stream))
    for _ in range(3):
        out.zero_()
        with torch.cuda.stream(s):
            g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().view(np.uint32), ref[0].view(np.uint32))
        assert np.array_equal(fl.cpu().numpy(), ref[3])
    del res
