// Host runtime: device buffers, TMA tensor maps, per-stream workspace, launch decisions.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <unordered_map>

#include "runtime.h"

namespace abftk {

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        cudaGetLastError();  // clear sticky-free errors
        throw CudaError(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
    }
}

static int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

int device_sm_count() {
    static int sms[kMaxDevices] = {};
    const int dev = current_device();
    if (!sms[dev]) {
        int n = 0;
        cuda_check(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev), "cudaDeviceGetAttribute");
        sms[dev] = n;
    }
    return sms[dev];
}

// ------------------------------------------------------------------ tensor maps
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        cuda_check(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q),
                   "cudaGetDriverEntryPoint(cuTensorMapEncodeTiled)");
        if (!p || q != cudaDriverEntryPointSuccess) throw CudaError("cuTensorMapEncodeTiled unavailable");
        return reinterpret_cast<EncodeTiledFn>(p);
    }();
    return fn;
}

// 2D row-major tensor: `inner` elements per row (contiguous), `outer` rows, `row_bytes` pitch.

// ------------------------------------------------------------------ per-stream workspace
// Scratch that must not live in the shared immutable weight/table handles: kernels
// leave every counter at zero on exit, so one workspace serves any number of ordered calls.
struct Workspace {
    int device = 0;
    unsigned long long* row_acc = nullptr;  // GEMM: per-row (A*cs share sum) << 32 | residue sum
    int64_t rows_cap = 0;
    int32_t* partial = nullptr;  // GEMM split-K partial tiles
    int64_t partial_cap = 0;
    uint32_t* part_flag = nullptr;  // GEMM split-K hand-over flags (self-resetting)
    int64_t part_flag_cap = 0;
    unsigned long long* err_pack = nullptr;  // GEMM per-problem (rows finished, rows flagged)
    int64_t err_pack_cap = 0;
    uint32_t* small = nullptr;  // [2] verify acc [3] verify blocks [4] eb flag acc [5] eb blocks [6..7] eb bag counter (u64) [12] eb validate count
    uint8_t* scratch = nullptr;  // A repack buffer
    size_t scratch_cap = 0;
    std::mutex mu;
};

static std::mutex g_ws_mu;
static std::unordered_map<uint64_t, Workspace*> g_ws;

static Workspace& ws_for(cudaStream_t st) {
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    const uint64_t key = (reinterpret_cast<uint64_t>(st) << 8) ^ static_cast<uint64_t>(dev);
    std::lock_guard<std::mutex> g(g_ws_mu);
    auto it = g_ws.find(key);
    if (it != g_ws.end()) return *it->second;
    auto* w = new Workspace();
    w->device = dev;
    cuda_check(cudaMalloc(&w->small, 64 * sizeof(uint32_t)), "cudaMalloc(workspace)");
    // zeroed on the stream the kernels using it run on (a legacy-stream memset is not ordered before work on
    // a non-blocking stream)
    cuda_check(cudaMemsetAsync(w->small, 0, 64 * sizeof(uint32_t), st), "cudaMemsetAsync(workspace)");
    g_ws[key] = w;
    return *w;
}

template <typename T>
static void grow(T*& ptr, int64_t& cap, int64_t need, cudaStream_t st) {
    if (need <= cap) return;
    const int64_t ncap = std::max<int64_t>(need, std::max<int64_t>(cap * 2, 256));
    if (ptr) {
        cuda_check(cudaStreamSynchronize(st), "cudaStreamSynchronize");
        cuda_check(cudaFree(ptr), "cudaFree");
    }
    cuda_check(cudaMalloc(&ptr, ncap * sizeof(T)), "cudaMalloc(workspace)");
    cuda_check(cudaMemsetAsync(ptr, 0, ncap * sizeof(T), st), "cudaMemsetAsync(workspace)");
    cap = ncap;
}

// ------------------------------------------------------------------ GEMM
static unsigned long long* g_trace = nullptr;  // debug: per-CTA phase timestamps
void set_gemm_trace(unsigned long long* d_trace) { g_trace = d_trace; }
static unsigned long long* g_eb_trace = nullptr;  // debug: per-warp EmbeddingBag timeline
void set_eb_trace(unsigned long long* d_trace) { g_eb_trace = d_trace; }

int gemm_ks(int bn);
int gemm_box_a(int bn);
int gemm_box_b(int bn);
cudaError_t launch_set_checksums(GemmWeight& w, const int8_t* src, cudaStream_t st);

// 4D view {128 bytes of a k-block, rows, k-blocks, batch} of K-contiguous byte matrices. `row_bytes` is
// the row pitch, `kb_bytes` the step between k-blocks (128 for row-major A; n_pad*128 for B'),
// `batch_bytes` the step between problems (unused when batch == 1).
static CUtensorMap make_map_kblocks(const void* base, uint64_t rows, uint64_t kblocks, uint64_t row_bytes,
                                    uint64_t kb_bytes, uint32_t box_rows, uint32_t box_kb, uint64_t batch = 1,
                                    uint64_t batch_bytes = 0) {
    CUtensorMap map;
    std::memset(&map, 0, sizeof(map));
    if (batch <= 1) batch_bytes = kb_bytes * kblocks + row_bytes * rows;  // any valid stride for a unit dim
    batch_bytes = (batch_bytes + 15) / 16 * 16;
    const cuuint64_t dims[4] = {static_cast<cuuint64_t>(kBK), rows, kblocks, batch < 1 ? 1 : batch};
    const cuuint64_t strides[3] = {row_bytes, kb_bytes, batch_bytes};
    const cuuint32_t box[4] = {static_cast<cuuint32_t>(kBK), box_rows, box_kb, 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = encode_fn()(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<void*>(base), dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled(4d) failed (code " + std::to_string(int(r)) + ")");
    return map;
}

// 3D exact-extent view {k bytes, rows, batch} of row-major A, box {128 B, 128 rows, 1}: one k-block per
// request, TMA zero-fills past k (no reads beyond a row's k bytes).
static CUtensorMap make_map_rows(const void* base, uint64_t k, uint64_t rows, uint64_t lda, uint64_t batch,
                                 uint64_t bstride) {
    CUtensorMap map;
    std::memset(&map, 0, sizeof(map));
    const uint64_t bb = batch <= 1 ? lda * rows : bstride;
    const cuuint64_t dims[3] = {k, rows, batch < 1 ? 1 : batch};
    const cuuint64_t strides[2] = {lda, (bb + 15) / 16 * 16};
    const cuuint32_t box[3] = {static_cast<cuuint32_t>(kBK), static_cast<cuuint32_t>(kBM), 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = encode_fn()(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(base), dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled(rows) failed (code " + std::to_string(int(r)) + ")");
    return map;
}

// 3D view {columns, rows, batch} of int32 C matrices, 32x32 boxes (TMA-store epilogue).
static CUtensorMap make_map_c(const void* base, uint64_t n, uint64_t m, uint64_t ldc, uint64_t batch, uint64_t bstride) {
    CUtensorMap map;
    std::memset(&map, 0, sizeof(map));
    const uint64_t bb = batch <= 1 ? ldc * 4 * m : bstride * 4;
    const cuuint64_t dims[3] = {n, m, batch < 1 ? 1 : batch};
    const cuuint64_t strides[2] = {ldc * 4, (bb + 15) / 16 * 16};
    const cuuint32_t box[3] = {32, 32, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = encode_fn()(&map, CU_TENSOR_MAP_DATA_TYPE_INT32, 3, const_cast<void*>(base), dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled(C) failed (code " + std::to_string(int(r)) + ")");
    return map;
}

static int bn_index(int bn) { return bn == 64 ? 0 : bn == 128 ? 1 : 2; }

void encode_weight_into(GemmWeight& w, const int8_t* d_b, int64_t k, int64_t n, int64_t ldb, cudaStream_t st,
                        int64_t batch, int64_t b_bstride) {
    if (k <= 0 || n <= 0) throw std::invalid_argument("compute_row_checksums: empty matrix");
    if (!d_b) throw std::invalid_argument("null argument");
    if (ldb < n) throw std::invalid_argument("abftlp_gemm_encode: ldb < n");
    if (batch < 1) throw std::invalid_argument("abftlp_gemm_encode: batch < 1");
    if (batch > 1 && b_bstride < ldb * (k - 1) + n) throw std::invalid_argument("abftlp_gemm_encode: batch stride too small");
    // B' column n holds the checksum column (PackedEncodedWeight's [B | cs], P:src/gemm_abft.hpp:30-59): n_pad leaves
    // room for it at every n, so a tile that covers it gets C'[:, n] from the tensor cores (GemmParams::cs_mma)
    const int64_t k_pad = round_up(k, kBK), n_pad = round_up(n + 1, kRowAlign);
    const size_t per_bt = static_cast<size_t>(n_pad * k_pad);
    const size_t need_bt = per_bt * static_cast<size_t>(batch), need_cs = static_cast<size_t>(k_pad * batch);
    if (!w.bt || need_bt > w.bt_cap || need_cs > w.cs_cap) {
        if (w.bt) {
            cuda_check(cudaStreamSynchronize(st), "cudaStreamSynchronize");
            cudaFree(w.bt);
            cudaFree(w.cs);
            cudaFree(w.cs_acc);
            w.bt = nullptr;
            w.cs = nullptr;
            w.cs_acc = nullptr;
        }
        cuda_check(cudaMalloc(&w.bt, need_bt), "cudaMalloc(B')");
        cuda_check(cudaMalloc(&w.cs, need_cs), "cudaMalloc(cs)");
        cuda_check(cudaMalloc(&w.cs_acc, need_cs * sizeof(int32_t)), "cudaMalloc(cs scratch)");
        cuda_check(cudaMemsetAsync(w.cs_acc, 0, need_cs * sizeof(int32_t), st), "cudaMemsetAsync(cs scratch)");
        w.bt_cap = need_bt;
        w.cs_cap = need_cs;
    }
    w.k = k;
    w.n = n;
    w.k_pad = k_pad;
    w.n_pad = n_pad;
    w.batch = batch;
    w.bt_bstride = static_cast<int64_t>(per_bt);
    w.cs_bstride = k_pad;
    for (int64_t b = 0; b < batch; ++b) {
        GemmWeight one = w;
        one.bt = w.bt + b * w.bt_bstride;
        one.cs = w.cs + b * w.cs_bstride;
        one.cs_acc = w.cs_acc + b * w.cs_bstride;
        cuda_check(launch_encode_weight(d_b + b * b_bstride, k, n, ldb, one, st), "encode_weight_kernel");
    }
    for (int bn : {64, 128, 256})
        w.map_b[bn_index(bn)] = make_map_kblocks(w.bt, static_cast<uint64_t>(n_pad), static_cast<uint64_t>(k_pad / kBK),
                                                 kBK, static_cast<uint64_t>(n_pad * kBK), bn / 2, gemm_box_b(bn),
                                                 static_cast<uint64_t>(batch), static_cast<uint64_t>(w.bt_bstride));
}

GemmWeight* encode_weight(const int8_t* d_b, int64_t k, int64_t n, int64_t ldb, cudaStream_t st, int64_t batch,
                          int64_t b_bstride) {
    if (k <= 0 || n <= 0) throw std::invalid_argument("compute_row_checksums: empty matrix");
    auto* w = new GemmWeight();
    try {
        encode_weight_into(*w, d_b, k, n, ldb, st, batch, b_bstride);
    } catch (...) {
        free_weight(w);
        throw;
    }
    return w;
}

void read_encoded(const GemmWeight& w, int8_t* d_out, cudaStream_t st) {
    cuda_check(launch_read_encoded(w, d_out, st), "read_encoded_kernel");
}

void set_checksums(GemmWeight& w, const int8_t* d_cs, cudaStream_t st) {
    cuda_check(launch_set_checksums(w, d_cs, st), "set_checksums_kernel");
}

void free_weight(GemmWeight* w) {
    if (!w) return;
    if (w->owns) {
        cudaFree(w->bt);
        cudaFree(w->cs);
        cudaFree(w->cs_acc);
    }
    delete w;
}

// Pick the pair tile (BN) and split-K. Cost model in SM cycles, from B200 measurements:
// the mainloop is bound by shared-memory bandwidth (128 B/clk/SM): every byte of a k-block's A rows
// (128 per CTA) and B' rows (BN/2) is written by TMA and read by the MMA, i.e. 2*(128 + BN/2) cycles per
// k-block, vs the MMA issue floor 4 x {46, 64, 128} cycles (N = 64, 128, 256). Split-K (single wave only)
// halves the k-blocks per unit but the partial-tile hand-over through L2 (publish, flag, poll, bulk
// pull) measured ~4 us on G2 (trace_gemm.py), more than the 2 us it saves: charged as 8000 cycles, so
// it is only picked where the mainloop saving is larger. The last tile's drain is ~BN*128*4 B at ~31 B/clk.
static int64_t gemm_kb_split(int64_t kb, int ks) { return (kb + 1) / 2 + ks - 1 - ((kb + 1) / 2 + ks - 1) % ks; }

GemmTiling choose_tiling(int64_t m, int64_t n, int64_t k_pad, bool checked, bool c_tma_ok, bool fault) {
    (void)fault;
    const int pairs = std::max(1, device_sm_count() / 2);
    const int64_t m_tiles = (m + kPairM - 1) / kPairM;
    const int64_t kb = k_pad / kBK;
    const int epi = c_tma_ok ? kEpiTmaStore : kEpiDirect;
    auto split_ok = [&](int bn, int64_t tiles) {
        const int ks = gemm_ks(bn);
        return tiles * 2 <= pairs && kb >= 4 * ks && gemm_kb_split(kb, ks) < kb;
    };
    if (const char* env = std::getenv("ABFTLP_GEMM_TILING")) {  // "bn[,epi[,split]]" tuning override
        int bn = 0, e = -1, sp = 1;
        const int got = std::sscanf(env, "%d,%d,%d", &bn, &e, &sp);
        if (got >= 1 && (bn == 64 || bn == 128 || bn == 256)) {
            GemmTiling t{bn, epi, 1};
            if (got >= 2 && (e == kEpiNone || e == kEpiDirect)) t.epi = e;
            if (got >= 2 && (e == kEpiTmaStore || e == kEpiStg) && c_tma_ok) t.epi = e;
            const int64_t tiles = m_tiles * ((n + bn - 1) / bn);
            if (got == 3 && sp == 2 && split_ok(bn, tiles)) t.split = 2;
            return t;
        }
    }
    GemmTiling best{64, epi, 1};
    double best_cost = 1e300;
    for (int bn : {256, 128, 64}) {
        const int64_t tiles = m_tiles * ((n + bn - 1) / bn);
        const double per_kb = std::max(2.0 * (kBM + bn / 2), 4.0 * (bn == 64 ? 46 : bn == 128 ? 64 : 128));
        const double drain = double(kBM) * bn * 4 / 31.0;
        for (int split : {1, 2}) {
            if (split == 2 && !split_ok(bn, tiles)) continue;
            const int64_t units = tiles * split;
            const int64_t waves = (units + pairs - 1) / pairs;
            const double kb_unit = split == 2 ? double(gemm_kb_split(kb, gemm_ks(bn))) : double(kb);
            // checked: a tile's CUDA-core GEMV share (kb / n_tiles k-blocks per row, ~1100 cycles each, run
            // alongside the mainloop) unless the checksum column rides in the MMA (last tile has room, cs_mma)
            const int64_t n_tiles = (n + bn - 1) / bn;
            const double gemv = (checked && (split == 2 || n % bn == 0)) ? 1100.0 * double(kb) / double(n_tiles) : 0.0;
            // + a fixed ~1.5 us per wave of tiles (first-stage latency and epilogue tail; measured: two half-
            // empty waves of 64-wide tiles lose to one wave of 128-wide ones on the narrow D5 shards)
            const double cost = waves * (std::max(kb_unit * per_kb, gemv) + 3000.0) +
                                (split == 2 ? 8000.0 + 8.0 * bn : 0.0) + drain;
            if (cost < best_cost * 0.97) {
                best_cost = cost;
                best = {bn, epi, split};
            }

        }
    }
    return best;
}

void gemm(const uint8_t* d_a, int64_t m, int64_t lda, const GemmWeight& w, int32_t* d_c, int64_t ldc, bool checked,
          int32_t* d_csum, int64_t csum_ld, uint8_t* d_flags, uint32_t* d_err_count, const Fault* fault,
          cudaStream_t st, const GemmTiling* force, const RequantArgs* rq, const GemmBatch* batch) {
    const GemmBatch one{};
    const GemmBatch& bt = batch ? *batch : one;
    const int64_t nb = bt.batch;
    if (nb < 1) throw std::invalid_argument("abft_gemm: batch < 1");
    if (nb > 1 && w.batch != 1 && w.batch != nb) throw std::invalid_argument("abft_gemm: weight batch mismatch");
    if (nb == 1 && w.batch != 1) throw std::invalid_argument("abft_gemm: batched weight needs a batched call");
    if (nb > 1 && (rq || (bt.a_bstride % 16) != 0 || bt.a_bstride < lda * (m - 1) + w.k))
        throw std::invalid_argument("abft_gemm: unsupported batch layout");
    if (m < 0) throw std::invalid_argument("abft_gemm: negative m");
    if (m > 0 && (!d_a || (!d_c && !rq))) throw std::invalid_argument("null argument");
    if (rq) {
        check_requant_params(rq->params);
        if (m > 0 && (!rq->row_sum_a || !rq->col_sum_b || !rq->out)) throw std::invalid_argument("null argument");
        if (rq->ld_out < w.n) throw std::invalid_argument("requantize: ld_out < n");
    }
    if (lda < w.k) throw std::invalid_argument("abft_gemm: dimension mismatch (lda < k)");
    if (ldc < w.n) throw std::invalid_argument("abft_gemm: ldc < n");
    if (checked && (!d_err_count || (m > 0 && (!d_csum || !d_flags)))) throw std::invalid_argument("null argument");
    if (m > (int64_t{1} << 31) - 1 || w.n > (int64_t{1} << 31) - 2) throw std::invalid_argument("abft_gemm: too large");
    // the call's C' faults: the single-fault form plus the batched list
    BatchFault fl[kMaxGemmFaults];
    int nf = 0;
    if (bt.nfaults < 0 || (bt.nfaults > 0 && !bt.faults)) throw std::invalid_argument("abft_gemm: bad fault list");
    if ((fault && fault->active ? 1 : 0) + bt.nfaults > kMaxGemmFaults)
        throw std::invalid_argument("abft_gemm: too many faults for one call");
    if (fault && fault->active) fl[nf++] = BatchFault{bt.fault_batch, fault->row, fault->col, fault->bit};
    for (int64_t i = 0; i < bt.nfaults; ++i) fl[nf++] = bt.faults[i];
    const bool has_fault = nf > 0;
    if (has_fault && !checked) throw std::invalid_argument("abft_gemm: fault hook needs the checked kernel");
    for (int i = 0; i < nf; ++i)
        if (fl[i].row < 0 || fl[i].row >= m || fl[i].col < 0 || fl[i].col > w.n || fl[i].bit > 31 || fl[i].batch < 0 ||
            fl[i].batch >= nb)
            throw std::out_of_range("abft_gemm: fault coordinates out of range");
    // Requests of one shape against ONE weight whose operands lie back to back are the row blocks of one tall GEMM. The
    // row checks are per row, so the stacked product is bit-identical to the separate ones, and requests of fewer than
    // 256 rows then share the 256-row tiles instead of padding one tile each (32 requests of 32 rows: 4 M tiles instead
    // of 32). The per-request flag counts are summed from the row flags afterwards. ABFTLP_GEMM_NOSTACK=1 disables.
    static const bool no_stack = std::getenv("ABFTLP_GEMM_NOSTACK") != nullptr;
    if (nb > 1 && w.batch == 1 && m > 0 && m % kPairM != 0 && nb * m > 16 && !rq && !force && !no_stack &&
        nb * m < (int64_t{1} << 31) &&
        bt.a_bstride == m * lda && (!d_c || bt.c_bstride == m * ldc) &&
        (!checked || (bt.csum_bstride == m * csum_ld && bt.flags_bstride == m))) {
        BatchFault sf[kMaxGemmFaults];
        for (int i = 0; i < nf; ++i) sf[i] = BatchFault{0, fl[i].batch * m + fl[i].row, fl[i].col, fl[i].bit};
        GemmBatch tall{};
        tall.faults = nf ? sf : nullptr;
        tall.nfaults = nf;
        tall.stack_rows = m;  // per-request flag counts, published by the kernel (GemmParams::req_rows)
        gemm(d_a, nb * m, lda, w, d_c, ldc, checked, d_csum, csum_ld, d_flags, d_err_count, nullptr, st, nullptr, nullptr,
             &tall);
        return;
    }
    auto set_faults = [&](GemmParams& p) {
        p.nfaults = nf;
        for (int i = 0; i < nf; ++i) {
            p.fault_b[i] = static_cast<int>(fl[i].batch);
            p.fault_row[i] = static_cast<int>(fl[i].row);
            p.fault_col[i] = static_cast<int>(fl[i].col);
            p.fault_bit[i] = static_cast<int>(fl[i].bit);
        }
    };
    if (m == 0) {
        if (checked) cuda_check(cudaMemsetAsync(d_err_count, 0, sizeof(uint32_t) * nb, st), "cudaMemsetAsync");
        return;
    }
    Workspace& ws = ws_for(st);
    std::lock_guard<std::mutex> g(ws.mu);

    // Small-m problems (the GEMV class of P:data/shapes.txt): stream B' once on CUDA cores (gemv.cu).
    const int64_t gemv_rows = std::getenv("ABFTLP_GEMV_MAX_ROWS") ? std::atoll(std::getenv("ABFTLP_GEMV_MAX_ROWS"))
                                                                  : kGemvMaxRows;
    const int mr = m <= 1 ? 1 : m <= 2 ? 2 : m <= 4 ? 4 : m <= 8 ? 8 : 16;
    if (nb == 1 && !rq && !force && m <= gemv_rows && m <= 16 && d_c &&
        (mr + 1) * w.k_pad + 8 * mr * 32 * 4 + 8 * mr * 32 * 4 <= 160 * 1024 && (w.n + 31) / 32 <= kMaxCheckedNTiles) {
        if (checked) {
            grow(ws.row_acc, ws.rows_cap, m, st);
            grow(ws.err_pack, ws.err_pack_cap, 1, st);
        }
        GemmParams p{};
        p.m = static_cast<int>(m);
        p.n = static_cast<int>(w.n);
        p.k = static_cast<int>(w.k);
        p.k_blocks = static_cast<int>(w.k_pad / kBK);
        p.batch = 1;
        p.c = d_c;
        p.ldc = ldc;
        p.csum = d_csum;
        p.csum_ld = csum_ld;
        p.flags = d_flags;
        p.err_count = d_err_count;
        p.a = d_a;
        p.lda = lda;
        p.cs = w.cs;
        p.row_acc = ws.row_acc;
        p.err_pack = ws.err_pack;
        set_faults(p);
        cuda_check(launch_gemv(p, w, checked, st), "gemv_checked_kernel");
        return;
    }
    // A is read through a 4D view {128 B, rows, k-blocks, batch} (several k-blocks per request) when k is a
    // multiple of 128, else through an exact-extent 3D view {k, rows, batch} (one k-block per request, the
    // tail zero-filled by TMA). Base and pitch must be 16-byte aligned; otherwise repack into scratch.
    const uint8_t* a = d_a;
    int64_t a_ld = lda, a_bstride = bt.a_bstride;
    if ((lda % 16) != 0 || (reinterpret_cast<uintptr_t>(d_a) % 16) != 0) {
        a_ld = w.k_pad;
        a_bstride = a_ld * m;
        const size_t need = static_cast<size_t>(a_ld * m * nb);
        if (need > ws.scratch_cap) {
            if (ws.scratch) {
                cuda_check(cudaStreamSynchronize(st), "cudaStreamSynchronize");
                cuda_check(cudaFree(ws.scratch), "cudaFree");
            }
            cuda_check(cudaMalloc(&ws.scratch, need), "cudaMalloc(A scratch)");
            ws.scratch_cap = need;
        }
        for (int64_t b = 0; b < nb; ++b)
            cuda_check(cudaMemcpy2DAsync(ws.scratch + b * a_bstride, a_ld, d_a + b * bt.a_bstride, lda, w.k, m,
                                         cudaMemcpyDeviceToDevice, st),
                       "cudaMemcpy2DAsync(A repack)");
        a = ws.scratch;
    }
    const bool c_tma_ok = d_c && (ldc % 4) == 0 && (reinterpret_cast<uintptr_t>(d_c) % 16) == 0 &&
                          (nb == 1 || (bt.c_bstride % 4) == 0);
    GemmTiling t = force ? *force : choose_tiling(nb * round_up(m, kPairM), w.n, w.k_pad, checked, c_tma_ok, has_fault);
    if (nb > 1) t.split = 1;
    if (!c_tma_ok && t.epi != kEpiNone) t.epi = kEpiDirect;
    if (!d_c) t.epi = kEpiNone;  // requantized output only

    const int64_t m_tiles = (m + kPairM - 1) / kPairM;
    const int64_t kb = w.k_pad / kBK;
    // The checksum column C'[:, n] comes from the tensor cores (B' column n) when the last tile has room for it
    // (no extra tile); otherwise the tiles' epilogues compute it as a GEMV share. ABFTLP_CS_MMA=0|1 overrides
    // (1 adds a tile for column n when there is no room).
    const int64_t n_tiles_plain = (w.n + t.bn - 1) / t.bn;
    bool cs_mma = checked && t.split == 1 && w.n % t.bn != 0;  // implies n < n_pad: B' column n exists
    if (const char* e = std::getenv("ABFTLP_CS_MMA"))
        cs_mma = checked && t.split == 1 && std::atoi(e) != 0 && w.n < w.n_pad && w.n / t.bn < (w.n_pad + t.bn - 1) / t.bn;
    int64_t n_tiles = cs_mma ? (w.n + 1 + t.bn - 1) / t.bn : n_tiles_plain;
    // Optional (ABFTLP_GEMM_TILEW=1): when n fills its tiles exactly, split the n + 1 columns into balanced tiles of
    // tile_w < BN columns (the MMA's N; one tile more, the checksum column on the tensor cores) instead of the
    // CUDA-core checksum share. Measured slower on the short-K DLRM shapes (serving mode 17-29 % -> 38-50 % overhead;
    // G1 20.7 -> 22.5 us), so it is off by default; grouped launches always use tile widths (runtime.cu, gemm_group).
    int64_t tile_w = t.bn;
    bool balance = false;
    if (const char* e = std::getenv("ABFTLP_GEMM_TILEW"))
        balance = checked && !cs_mma && t.split == 1 && w.n % t.bn == 0 && w.n < w.n_pad && std::atoi(e) != 0;
    if (balance) {
        cs_mma = true;
        n_tiles = (w.n + 1 + t.bn - 1) / t.bn;
        tile_w = ((w.n + 1 + n_tiles - 1) / n_tiles + 31) / 32 * 32;
    }
    if (nb * m_tiles * n_tiles * t.split > (int64_t{1} << 31) - 1) throw std::invalid_argument("abft_gemm: too many tiles");

    if (checked && n_tiles > kMaxCheckedNTiles) throw std::invalid_argument("abft_gemm: n too large for the checked kernel");
    if (checked) {
        grow(ws.row_acc, ws.rows_cap, m * nb, st);
        grow(ws.err_pack, ws.err_pack_cap, bt.stack_rows > 0 ? m / bt.stack_rows : nb, st);
    }

    GemmParams p{};
    p.m = static_cast<int>(m);
    p.n = static_cast<int>(w.n);
    p.k = static_cast<int>(w.k);
    p.k_blocks = static_cast<int>(kb);
    p.n_tiles = static_cast<int>(n_tiles);
    p.tile_w = static_cast<int>(tile_w);
    p.m_tiles = static_cast<int>(m_tiles);
    p.num_tiles = static_cast<int>(nb * m_tiles * n_tiles);
    p.batch = static_cast<int>(nb);
    p.b_shared = w.batch == 1 ? 1 : 0;
    p.a_bstride = a_bstride;
    p.cs_bstride = w.batch == 1 ? 0 : w.cs_bstride;
    p.c_bstride = bt.c_bstride;
    p.csum_bstride = bt.csum_bstride;
    p.flags_bstride = bt.flags_bstride;
    p.split = t.split;
    if (t.split == 2) {
        p.kb_half = static_cast<int>(gemm_kb_split(kb, gemm_ks(t.bn)));
        grow(ws.partial, ws.partial_cap, m_tiles * n_tiles * 2 * t.bn * kBM, st);
        grow(ws.part_flag, ws.part_flag_cap, m_tiles * n_tiles * 2, st);
        p.partial = ws.partial;
        p.part_flag = ws.part_flag;
    }
    p.c = d_c;
    p.ldc = ldc;
    p.csum = d_csum;
    p.csum_ld = csum_ld;
    p.flags = d_flags;
    p.err_count = d_err_count;
    p.a = a;
    p.lda = a_ld;
    p.cs = w.cs;
    p.row_acc = ws.row_acc;
    p.err_pack = ws.err_pack;
    p.trace = g_trace;
    p.req_rows = static_cast<int>(bt.stack_rows);
    if (rq) {
        p.rq_row_sum_a = rq->row_sum_a;
        p.rq_col_sum_b = rq->col_sum_b;
        p.rq_out = rq->out;
        p.rq_ld = rq->ld_out;
        p.rq = rq->params;
    }
    set_faults(p);
    // box = a stage's k-blocks split over the A producer warps (exact-extent view: one k-block)
    p.a_exact = (w.k % kBK) != 0 ? 1 : 0;
    const CUtensorMap map_a = p.a_exact
                                  ? make_map_rows(a, static_cast<uint64_t>(w.k), static_cast<uint64_t>(m),
                                                  static_cast<uint64_t>(a_ld), static_cast<uint64_t>(nb),
                                                  static_cast<uint64_t>(a_bstride))
                                  : make_map_kblocks(a, static_cast<uint64_t>(m), static_cast<uint64_t>(kb),
                                                     static_cast<uint64_t>(a_ld), kBK, kBM, gemm_box_a(t.bn),
                                                     static_cast<uint64_t>(nb), static_cast<uint64_t>(a_bstride));
    CUtensorMap map_c;
    std::memset(&map_c, 0, sizeof(map_c));
    if (t.epi == kEpiTmaStore)
        map_c = make_map_c(d_c, static_cast<uint64_t>(w.n), static_cast<uint64_t>(m), static_cast<uint64_t>(ldc),
                           static_cast<uint64_t>(nb), static_cast<uint64_t>(bt.c_bstride));
    const int all_pairs = std::max(1, device_sm_count() / 2);
    int pairs = static_cast<int>(std::min<int64_t>(static_cast<int64_t>(p.num_tiles) * p.split, all_pairs));
    // Tall narrow shapes leave pairs idle while one or a few N tiles would each carry a large share of the
    // checksum GEMV: the idle pairs compute it instead (gemv_helper). ABFTLP_GEMV_HELPERS=0 disables.
    const bool helpers_ok = !std::getenv("ABFTLP_GEMV_HELPERS") || std::atoi(std::getenv("ABFTLP_GEMV_HELPERS")) != 0;
    p.cs_mma = cs_mma ? 1 : 0;
    p.gemv_helpers = (checked && !cs_mma && helpers_ok && n_tiles <= 4 && all_pairs - pairs >= pairs) ? 1 : 0;
    // Epilogue warps: 8 (two groups splitting each tile's columns, one row arrival each) when a batched
    // launch's tiles have a short mainloop (k <= 1024) and the TMA-store epilogue, where the epilogue is
    // the exposed part (G1: 26 -> 21 us per 100 trials); 4 otherwise (with long mainloops the extra warps
    // slow the mainloop: grouped G2 2.9 -> 2.4 POPS). ABFTLP_GEMM_EW=4|8 overrides.
    int ew = ((nb > 1 || bt.stack_rows > 0) && kb <= 8 && t.epi == kEpiTmaStore) ? 8 : 4;  // (row-stacked requests too)
    // the fused requantization makes the epilogue the long side at any k (G2, 8 stacked runs: 67 -> 47 us with 8 warps)
    if (rq && checked && (t.epi == kEpiTmaStore || t.epi == kEpiNone)) ew = 8;
    if (const char* e = std::getenv("ABFTLP_GEMM_EW")) {
        const int f = std::atoi(e);
        if (f == 4 || (f == 8 && (t.epi == kEpiTmaStore || (rq && checked && t.epi == kEpiNone)))) ew = f;
    }
    p.row_arrivals = static_cast<int>(n_tiles) * (ew / 4) + p.gemv_helpers;
    // the arrival count is a 12-bit field of the per-row accumulator (kRowAcc*): more would carry into the
    // checksum bits. Two epilogue groups double the arrivals; fall back to one group before refusing.
    if (checked && p.row_arrivals > kMaxCheckedNTiles && ew == 8) {
        ew = 4;
        p.row_arrivals = static_cast<int>(n_tiles) + p.gemv_helpers;
    }
    if (checked && p.row_arrivals > kMaxCheckedNTiles)
        throw std::invalid_argument("abft_gemm: n too large for the checked kernel");
    if (p.gemv_helpers) pairs = all_pairs;
    cuda_check(launch_gemm_kernel(t.bn, checked, t.epi, ew, pairs, map_a, w.map_b[bn_index(t.bn)], map_c, p, st),
               "gemm_pair_kernel");
}

// ------------------------------------------------------------------ heterogeneous grouped GEMM
GemmGroup* gemm_group_create(const GemmProblem* probs, int n, bool checked) {
    if (n < 1 || n > kMaxGemmGroup) throw std::invalid_argument("gemm_group: 1 to 16 problems");
    if (!probs) throw std::invalid_argument("null argument");
    bool tma_c = true;
    for (int i = 0; i < n; ++i) {
        const GemmProblem& q = probs[i];
        if (!q.w || !q.a || !q.c) throw std::invalid_argument("null argument");
        if (checked && (!q.csum || !q.flags || !q.err_count)) throw std::invalid_argument("null argument");
        if (q.w->batch != 1) throw std::invalid_argument("gemm_group: batched weights are not supported");
        if (q.m < 1 || q.m > (int64_t{1} << 31) - 1) throw std::invalid_argument("gemm_group: m out of range");
        if (q.lda < q.w->k) throw std::invalid_argument("abft_gemm: dimension mismatch (lda < k)");
        if (q.ldc < q.w->n) throw std::invalid_argument("abft_gemm: ldc < n");
        if ((q.lda % 16) != 0 || (reinterpret_cast<uintptr_t>(q.a) % 16) != 0)
            throw std::invalid_argument("gemm_group: A needs a 16-byte aligned base and lda % 16 == 0");
        tma_c = tma_c && (q.ldc % 4) == 0 && (reinterpret_cast<uintptr_t>(q.c) % 16) == 0;
    }
    // Kernel tile width BN (each problem then takes balanced N tiles of tile_w <= BN columns, see below): these
    // launches stream A and B' through L2 (measured: the L2 -> SM path, ~6.5 TB/s, is the binding unit of the D5 MLP
    // layers), so the cost of a tile is the bytes it pulls -- its 256-row A slab plus the tile_w rows of B' -- per
    // k-block, plus a fixed ~1 us of per-tile latency (in 128-byte units at one pair's share of that path).
    const int pairs_all = std::max(1, device_sm_count() / 2);
    int best_bn = 64;
    double best = 1e300;
    for (int bn : {256, 128, 64}) {
        double sum = 0.0, longest = 0.0;
        for (int i = 0; i < n; ++i) {
            const GemmProblem& q = probs[i];
            const int64_t cols = q.w->n + (checked ? 1 : 0);
            const int64_t nt = (cols + bn - 1) / bn;
            const int64_t tw = ((cols + nt - 1) / nt + 31) / 32 * 32;
            const double tiles = double((q.m + kPairM - 1) / kPairM) * double(nt);
            const double t = double(q.w->k_pad / kBK) * double(kPairM + tw) + 700.0 + 100.0 * double(tw / 32);
            sum += tiles * t;
            longest = std::max(longest, t);
        }
        const double cost = sum / pairs_all + longest;
        if (cost < best * 0.97) {
            best = cost;
            best_bn = bn;
        }
    }
    if (const char* e = std::getenv("ABFTLP_GEMM_GROUP_BN")) {
        const int f = std::atoi(e);
        if (f == 64 || f == 128 || f == 256) best_bn = f;
    }
    auto* g = new GemmGroup();
    g->n = n;
    g->bn = best_bn;
    g->checked = checked;
    g->epi = tma_c ? kEpiTmaStore : kEpiDirect;
    if (const char* e = std::getenv("ABFTLP_GEMM_GROUP_EPI")) {  // 0 TMA store, 1 st.global after smem transpose, 2 direct
        const int f = std::atoi(e);
        if (f == kEpiDirect || (tma_c && (f == kEpiTmaStore || f == kEpiStg))) g->epi = f;
    }
    // 8 epilogue warps taking alternate tiles (TMA-store epilogue only); ABFTLP_GEMM_GROUP_EW=4|8 overrides
    g->ew = g->epi == kEpiTmaStore ? 8 : 4;
    if (const char* e = std::getenv("ABFTLP_GEMM_GROUP_EW")) {
        const int f = std::atoi(e);
        if (f == 4 || (f == 8 && g->epi == kEpiTmaStore)) g->ew = f;
    }
    // longest mainloops first (the persistent pairs take tiles round-robin, so the long tiles start early)
    g->order.resize(n);
    for (int i = 0; i < n; ++i) g->order[i] = i;
    std::stable_sort(g->order.begin(), g->order.end(),
                     [&](int x, int y) { return probs[x].w->k_pad > probs[y].w->k_pad; });
    std::vector<GemmParams> hp(n);
    std::vector<CUtensorMap> hm(4 * n);
    int64_t rows_total = 0;
    for (int i = 0; i < n; ++i) rows_total += probs[i].m;
    try {
        if (checked) {
            cuda_check(cudaMalloc(&g->row_acc, sizeof(unsigned long long) * rows_total), "cudaMalloc(group rows)");
            cuda_check(cudaMemset(g->row_acc, 0, sizeof(unsigned long long) * rows_total), "cudaMemset(group rows)");
            cuda_check(cudaMalloc(&g->err_pack, sizeof(unsigned long long) * n), "cudaMalloc(group counts)");
            cuda_check(cudaMemset(g->err_pack, 0, sizeof(unsigned long long) * n), "cudaMemset(group counts)");
        }
        int64_t row_off = 0, tiles = 0;
        GemmParams& L = g->launch;
        L.group_n = n;
        L.batch = 1;
        L.split = 1;
        for (int s = 0; s < n; ++s) {
            const GemmProblem& q = probs[g->order[s]];
            const GemmWeight& w = *q.w;
            GemmParams& P = hp[s];
            const int64_t kb = w.k_pad / kBK;
            P.m = static_cast<int>(q.m);
            P.n = static_cast<int>(w.n);
            P.k = static_cast<int>(w.k);
            P.k_blocks = static_cast<int>(kb);
            P.m_tiles = static_cast<int>((q.m + kPairM - 1) / kPairM);
            // N tiles of equal width (a multiple of 32 up to the kernel's BN): n + 1 columns just over BN split into
            // two balanced tiles instead of a full one plus a tile for the checksum column alone
            const int64_t cols = w.n + (checked ? 1 : 0);
            P.n_tiles = static_cast<int>((cols + best_bn - 1) / best_bn);
            P.tile_w = static_cast<int>(((cols + P.n_tiles - 1) / P.n_tiles + 31) / 32 * 32);
            P.num_tiles = P.m_tiles * P.n_tiles;
            P.batch = 1;
            P.b_shared = 1;
            P.split = 1;
            P.a_exact = (w.k % kBK) != 0 ? 1 : 0;
            P.cs_mma = checked ? 1 : 0;
            P.gemv_helpers = 0;
            P.row_arrivals = P.n_tiles;
            if (checked && P.row_arrivals > kMaxCheckedNTiles)
                throw std::invalid_argument("abft_gemm: n too large for the checked kernel");
            P.c = q.c;
            P.ldc = q.ldc;
            P.a = q.a;
            P.lda = q.lda;
            P.cs = w.cs;
            P.csum = q.csum;
            P.csum_ld = q.csum_ld;
            P.flags = q.flags;
            P.err_count = q.err_count;
            P.row_acc = checked ? g->row_acc + row_off : nullptr;
            P.err_pack = checked ? g->err_pack + s : nullptr;
            P.trace = g_trace;
            row_off += q.m;
            L.grp_tile_start[s] = static_cast<int>(tiles);
            tiles += P.num_tiles;
            if (tiles > (int64_t{1} << 30)) throw std::invalid_argument("abft_gemm: too many tiles");
            hm[3 * s] = P.a_exact ? make_map_rows(q.a, static_cast<uint64_t>(w.k), static_cast<uint64_t>(q.m),
                                                  static_cast<uint64_t>(q.lda), 1, 0)
                                  : make_map_kblocks(q.a, static_cast<uint64_t>(q.m), static_cast<uint64_t>(kb),
                                                     static_cast<uint64_t>(q.lda), kBK, kBM, gemm_box_a(best_bn), 1, 0);
            // B' boxed at exactly the tw / 2 rows a CTA's half tile needs
            hm[3 * s + 1] = make_map_kblocks(w.bt, static_cast<uint64_t>(w.n_pad), static_cast<uint64_t>(kb), kBK,
                                             static_cast<uint64_t>(w.n_pad * kBK), static_cast<uint32_t>(P.tile_w / 2),
                                             gemm_box_b(best_bn));
            if (g->epi == kEpiTmaStore)
                hm[3 * s + 2] = make_map_c(q.c, static_cast<uint64_t>(w.n), static_cast<uint64_t>(q.m),
                                           static_cast<uint64_t>(q.ldc), 1, 0);
            else
                std::memset(&hm[3 * s + 2], 0, sizeof(CUtensorMap));
        }
        // A prefetch views: {k/4 words, m rows}, 1 KB x 256-row boxes (SWIZZLE_NONE), for the L2 warm-up of each
        // unit's A slab (k % 4 == 0 needed; ABFTLP_GEMM_GROUP_APF=0 disables)
        bool apf = !std::getenv("ABFTLP_GEMM_GROUP_APF") || std::atoi(std::getenv("ABFTLP_GEMM_GROUP_APF")) != 0;
        for (int s = 0; s < n && apf; ++s) apf = (probs[g->order[s]].w->k % 4) == 0;
        for (int s = 0; s < n && apf; ++s) {
            const GemmProblem& q = probs[g->order[s]];
            CUtensorMap map;
            std::memset(&map, 0, sizeof(map));
            const cuuint64_t dims[2] = {static_cast<cuuint64_t>(q.w->k / 4), static_cast<cuuint64_t>(q.m)};
            const cuuint64_t strides[1] = {static_cast<cuuint64_t>(q.lda)};
            const cuuint32_t box[2] = {static_cast<cuuint32_t>(std::min<int64_t>(256, q.w->k / 4)),
                                       static_cast<cuuint32_t>(std::min<int64_t>(256, q.m))};
            const cuuint32_t estr[2] = {1, 1};
            CUresult r = encode_fn()(&map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<uint8_t*>(q.a), dims, strides, box,
                                     estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) apf = false;
            hm[3 * n + s] = map;
        }
        L.grp_apf = apf ? 1 : 0;
        L.grp_tile_start[n] = static_cast<int>(tiles);
        L.num_tiles = static_cast<int>(tiles);
        L.trace = g_trace;
        cuda_check(cudaMalloc(&g->d_params, sizeof(GemmParams) * n), "cudaMalloc(group params)");
        cuda_check(cudaMalloc(&g->d_maps, sizeof(CUtensorMap) * 4 * n), "cudaMalloc(group maps)");
        cuda_check(cudaMemcpy(g->d_params, hp.data(), sizeof(GemmParams) * n, cudaMemcpyHostToDevice), "cudaMemcpy");
        cuda_check(cudaMemcpy(g->d_maps, hm.data(), sizeof(CUtensorMap) * 4 * n, cudaMemcpyHostToDevice), "cudaMemcpy");
        L.grp_params = g->d_params;
        L.grp_maps = g->d_maps;
        g->pairs = static_cast<int>(std::min<int64_t>(tiles, pairs_all));
    } catch (...) {
        gemm_group_free(g);
        throw;
    }
    return g;
}

void gemm_group_run(const GemmGroup& g, cudaStream_t st) {
    cuda_check(launch_gemm_grouped(g.bn, g.checked, g.epi, g.ew, g.pairs, g.launch, st), "gemm_pair_kernel (grouped)");
}

void gemm_group_free(GemmGroup* g) {
    if (!g) return;
    cudaFree(g->d_params);
    cudaFree(g->d_maps);
    cudaFree(g->row_acc);
    cudaFree(g->err_pack);
    delete g;
}

// ------------------------------------------------------------------ dual-encoded locate / correct
LocateResult gemm_locate(const uint8_t* d_a, int64_t m, int64_t lda, const GemmWeight& w, int32_t* d_c, int64_t ldc,
                         int32_t* d_csum, int64_t csum_ld, uint8_t* d_flags, bool correct, cudaStream_t st) {
    if (!d_a || !d_c || !d_csum || !d_flags) throw std::invalid_argument("null argument");
    if (w.batch != 1) throw std::invalid_argument("gemm_locate: batched weights are not supported");
    if (m < 1 || lda < w.k || ldc < w.n || csum_ld < 1) throw std::invalid_argument("gemm_locate: bad dimensions");
    if (m > (int64_t{1} << 24)) throw std::invalid_argument("gemm_locate: m too large");
    LocateResult res;
    std::vector<uint8_t> flags(static_cast<size_t>(m));
    cuda_check(cudaMemcpyAsync(flags.data(), d_flags, static_cast<size_t>(m), cudaMemcpyDeviceToHost, st), "cudaMemcpyAsync");
    constexpr int kRec = 8;
    struct Scratch {
        void* p = nullptr;
        ~Scratch() { cudaFree(p); }
    } sc;
    const size_t col_bytes = sizeof(uint32_t) * static_cast<size_t>(w.k_pad);
    cuda_check(cudaMalloc(&sc.p, col_bytes + 64 + kRec * 16 + 16), "cudaMalloc(locate scratch)");
    uint32_t* colsum = static_cast<uint32_t*>(sc.p);
    uint8_t* tail = static_cast<uint8_t*>(sc.p) + col_bytes;
    uint32_t* nbad = reinterpret_cast<uint32_t*>(tail);
    int32_t* row_cs = reinterpret_cast<int32_t*>(tail + 16);
    int64_t* bad_col = reinterpret_cast<int64_t*>(tail + 64);
    long long* bad_delta = reinterpret_cast<long long*>(tail + 64 + kRec * 8);
    cuda_check(cudaMemsetAsync(nbad, 0, 4, st), "cudaMemsetAsync");
    cuda_check(launch_locate_colsum_a(d_a, m, w.k, lda, colsum, w.k_pad, st), "locate_colsum_a_kernel");
    cuda_check(launch_locate_columns(colsum, w, d_c, m, ldc, nbad, bad_col, bad_delta, kRec, st), "locate_columns_kernel");
    uint32_t hb = 0;
    int64_t hcol[kRec];
    long long hdel[kRec];
    cuda_check(cudaMemcpyAsync(&hb, nbad, 4, cudaMemcpyDeviceToHost, st), "cudaMemcpyAsync");
    cuda_check(cudaMemcpyAsync(hcol, bad_col, sizeof(hcol), cudaMemcpyDeviceToHost, st), "cudaMemcpyAsync");
    cuda_check(cudaMemcpyAsync(hdel, bad_delta, sizeof(hdel), cudaMemcpyDeviceToHost, st), "cudaMemcpyAsync");
    cuda_check(cudaStreamSynchronize(st), "cudaStreamSynchronize");
    int64_t row = -1;
    for (int64_t i = 0; i < m; ++i)
        if (flags[static_cast<size_t>(i)]) {
            ++res.rows_flagged;
            row = i;
        }
    res.cols_mismatched = hb;
    if (res.rows_flagged == 0 && hb == 0) return res;  // clean
    if (res.rows_flagged == 1 && hb == 1) {
        res.status = 1;
        res.row = row;
        res.col = hcol[0];
        res.delta = hdel[0];
        if (correct) {
            int32_t* cell = d_c + row * ldc + res.col;
            int32_t v = 0;
            cuda_check(cudaMemcpyAsync(&v, cell, 4, cudaMemcpyDeviceToHost, st), "cudaMemcpyAsync");
            cuda_check(cudaStreamSynchronize(st), "cudaStreamSynchronize");
            // the corrupted element differs from the clean one by exactly delta (both int32)
            v = static_cast<int32_t>(static_cast<int64_t>(v) - res.delta);
            cuda_check(cudaMemcpyAsync(cell, &v, 4, cudaMemcpyHostToDevice, st), "cudaMemcpyAsync");
        }
    } else if (res.rows_flagged == 1 && hb == 0) {
        res.status = 2;  // every data column checks out: C'[row][n] itself was hit
        res.row = row;
        res.col = w.n;
        if (correct) {
            cuda_check(launch_locate_row_checksum(d_a + row * lda, w.k, w.cs, row_cs, st), "locate_row_checksum_kernel");
            cuda_check(cudaMemcpyAsync(d_csum + row * csum_ld, row_cs, 4, cudaMemcpyDeviceToDevice, st), "cudaMemcpyAsync");
        }
    } else if (res.rows_flagged == 0) {
        res.status = 4;
        res.col = hcol[0];
        return res;
    } else {
        res.status = 3;
        return res;
    }
    if (correct) {  // re-check the repaired row (the reference's comparison); it must pass now
        uint32_t* cnt = reinterpret_cast<uint32_t*>(tail + 32);
        Workspace& ws = ws_for(st);
        {
            std::lock_guard<std::mutex> g(ws.mu);
            cuda_check(launch_verify(d_c + row * ldc, ldc, d_csum + row * csum_ld, csum_ld, 1, w.n, d_flags + row, cnt,
                                     ws.small + 2, ws.small + 3, st),
                       "verify_kernel");
        }
        uint32_t left = 1;
        cuda_check(cudaMemcpyAsync(&left, cnt, 4, cudaMemcpyDeviceToHost, st), "cudaMemcpyAsync");
        cuda_check(cudaStreamSynchronize(st), "cudaStreamSynchronize");
        if (left != 0) res.status = 3;  // the repair did not restore the row: more than one error
    }
    return res;
}

void check_requant_params(const RequantDev& q) {
    if (!(q.sC > 0.0)) throw std::invalid_argument("requantize: scaleC must be positive");
}

void requantize(const int32_t* d_c, int64_t ldc, int64_t m, int64_t n, const int32_t* d_row_sum_a,
                const int32_t* d_col_sum_b, const RequantDev& q, uint8_t* d_out, int64_t ld_out, cudaStream_t st) {
    check_requant_params(q);
    if (m < 0 || n < 0) throw std::invalid_argument("requantize: negative size");
    if (m == 0 || n == 0) return;
    if (!d_c || !d_row_sum_a || !d_col_sum_b || !d_out) throw std::invalid_argument("null argument");
    if (ldc < n || ld_out < n) throw std::invalid_argument("requantize: leading dimension < n");
    cuda_check(launch_requantize(d_c, ldc, m, n, d_row_sum_a, d_col_sum_b, q, d_out, ld_out, st), "requantize_kernel");
}

void row_sums_u8(const uint8_t* d_a, int64_t m, int64_t k, int64_t lda, int32_t* d_out, cudaStream_t st) {
    if (m < 0 || k < 0 || lda < k) throw std::invalid_argument("row_sums: bad dimensions");
    if (m == 0) return;
    if (!d_a || !d_out) throw std::invalid_argument("null argument");
    cuda_check(launch_row_sums_u8(d_a, m, k, lda, d_out, st), "row_sums_u8_kernel");
}

void weight_col_sums(const GemmWeight& w, int32_t* d_out, cudaStream_t st) {
    if (!d_out) throw std::invalid_argument("null argument");
    cuda_check(launch_col_sums(w, d_out, st), "col_sums_kernel");
}

void verify(const int32_t* d_c, int64_t ldc, const int32_t* d_csum, int64_t csum_ld, int64_t m, int64_t n,
            uint8_t* d_flags, uint32_t* d_err_count, cudaStream_t st) {
    if (m < 0 || n < 0) throw std::invalid_argument("verify_checksums: negative size");
    if (m > 0 && (!d_c || !d_csum)) throw std::invalid_argument("null argument");
    Workspace& ws = ws_for(st);
    std::lock_guard<std::mutex> g(ws.mu);
    cuda_check(launch_verify(d_c, ldc, d_csum, csum_ld, m, n, d_flags, d_err_count, ws.small + 2, ws.small + 3, st),
               "verify_kernel");
}

// ------------------------------------------------------------------ EmbeddingBag
int64_t eb_elem_row_bytes(int elem, int64_t dim) { return elem == kEbU4 ? (dim + 1) / 2 : dim; }

// Interleave each row with its metadata record into one 64-byte slot when both fit (e.g. int4 x 64 +
// fp16 scale/bias + row sum = 40 B): a lookup then touches one DRAM burst instead of two scattered
// ones. The copy is owned by the table; the caller's rows stay the reference copy for row sums.
void eb_pack(EbTable& t, cudaStream_t st) {
    const int64_t row_bytes = eb_elem_row_bytes(t.elem, t.dim);
    const int64_t meta_bytes = t.scale_type == kEbF32 ? sizeof(EbMetaF32) : sizeof(EbMetaF16);
    const int64_t meta_off = round_up(row_bytes, 16);
    const bool want = meta_off + meta_bytes <= 64 && std::getenv("ABFTLP_EB_NOPACK") == nullptr;
    const int64_t need = want ? 64 * t.rows : 0;
    if (t.packed && (!want || need > t.packed_cap)) {
        cuda_check(cudaStreamSynchronize(st), "cudaStreamSynchronize");
        cudaFree(t.packed);
        t.packed = nullptr;
        t.packed_cap = 0;
    }
    if (!want) {
        t.rec_stride = t.meta_off = 0;
        return;
    }
    if (!t.packed) {
        cuda_check(cudaMalloc(&t.packed, static_cast<size_t>(need)), "cudaMalloc(eb packed)");
        t.packed_cap = need;
    }
    t.rec_stride = 64;
    t.meta_off = meta_off;
    cuda_check(launch_eb_pack(t.data, t.rows, row_bytes, t.row_stride, t.meta, meta_bytes, meta_off, 64, t.packed, st),
               "eb_pack_kernel");
}

EbTable* eb_table_create(int elem, const void* d_rows, int64_t rows, int64_t dim, int64_t row_stride, int scale_type,
                         const void* d_scales, const void* d_biases, const int32_t* d_given_sums, cudaStream_t st) {
    if (elem < kEbS8 || elem > kEbU4) throw std::invalid_argument("eb_table_create: unknown element type");
    if (scale_type != kEbF32 && scale_type != kEbF16) throw std::invalid_argument("eb_table_create: unknown scale type");
    if (rows <= 0 || dim <= 0) throw std::invalid_argument("eb_table_create: empty table");
    if (!d_rows || !d_scales || !d_biases) throw std::invalid_argument("null argument");
    if (row_stride < eb_elem_row_bytes(elem, dim)) throw std::invalid_argument("eb_table_create: row stride too small");
    auto* t = new EbTable();
    t->elem = elem;
    t->scale_type = scale_type;
    t->rows = rows;
    t->dim = dim;
    t->row_stride = row_stride;
    t->data = reinterpret_cast<const uint8_t*>(d_rows);
    const size_t rec = scale_type == kEbF32 ? sizeof(EbMetaF32) : sizeof(EbMetaF16);
    try {
        cuda_check(cudaMalloc(&t->meta, rec * static_cast<size_t>(rows)), "cudaMalloc(eb meta)");
        cuda_check(launch_eb_meta(elem, scale_type, t->data, rows, dim, row_stride, d_scales, d_biases, d_given_sums,
                                  t->meta, nullptr, nullptr, st),
                   "eb_meta_kernel");
        eb_pack(*t, st);
    } catch (...) {
        eb_table_free(t);
        throw;
    }
    return t;
}

void eb_table_rebuild(EbTable& t, int elem, const void* d_rows, int64_t rows, int64_t dim, int64_t row_stride,
                      int scale_type, const void* d_scales, const void* d_biases, const int32_t* d_given_sums,
                      cudaStream_t st) {
    const size_t rec = scale_type == kEbF32 ? sizeof(EbMetaF32) : sizeof(EbMetaF16);
    const size_t old = (t.scale_type == kEbF32 ? sizeof(EbMetaF32) : sizeof(EbMetaF16)) * static_cast<size_t>(t.rows);
    if (!t.meta || rec * static_cast<size_t>(rows) > old) {
        if (t.meta) {
            cuda_check(cudaStreamSynchronize(st), "cudaStreamSynchronize");
            cudaFree(t.meta);
            t.meta = nullptr;
        }
        cuda_check(cudaMalloc(&t.meta, rec * static_cast<size_t>(rows)), "cudaMalloc(eb meta)");
    }
    t.elem = elem;
    t.scale_type = scale_type;
    t.rows = rows;
    t.dim = dim;
    t.row_stride = row_stride;
    t.data = reinterpret_cast<const uint8_t*>(d_rows);
    cuda_check(launch_eb_meta(elem, scale_type, t.data, rows, dim, row_stride, d_scales, d_biases, d_given_sums,
                              t.meta, nullptr, nullptr, st),
               "eb_meta_kernel");
    eb_pack(t, st);
}

void eb_row_sums(const EbTable& t, int32_t* d_out, cudaStream_t st) {
    cuda_check(launch_eb_meta(t.elem, t.scale_type, t.data, t.rows, t.dim, t.row_stride, nullptr, nullptr, nullptr,
                              nullptr, d_out, nullptr, st),
               "eb_meta_kernel(row sums)");
}

void eb_table_free(EbTable* t) {
    if (!t) return;
    cudaFree(t->meta);
    cudaFree(t->packed);
    delete t;
}

uint64_t eb_table_validate(const EbTable& t, const int32_t* d_given_sums, cudaStream_t st) {
    if (!d_given_sums) return 0;
    Workspace& ws = ws_for(st);
    std::lock_guard<std::mutex> g(ws.mu);
    uint32_t* cnt = ws.small + 12;  // (own slot: [8..9] is the GEMM err_pack)
    cuda_check(cudaMemsetAsync(cnt, 0, sizeof(uint32_t), st), "cudaMemsetAsync");
    cuda_check(launch_eb_meta(t.elem, t.scale_type, t.data, t.rows, t.dim, t.row_stride, nullptr, nullptr, d_given_sums,
                              nullptr, nullptr, cnt, st),
               "eb_meta_kernel(validate)");
    uint32_t h = 0;
    cuda_check(cudaMemcpyAsync(&h, cnt, sizeof(h), cudaMemcpyDeviceToHost, st), "cudaMemcpyAsync");
    cuda_check(cudaStreamSynchronize(st), "cudaStreamSynchronize");
    return h;
}

void eb_run(const EbTable& t, const int64_t* d_offsets, const int64_t* d_indices, int64_t num_bags,
            const float* d_weights, float* d_out, int64_t ld_out, bool checked, uint8_t* d_flags, double* d_rsum,
            double* d_csum, uint32_t* d_flag_count, int32_t* d_status, cudaStream_t st, const EbScatter* scatter) {
    if (num_bags < 0) throw std::invalid_argument("embedding_bag: negative bag count");
    if (num_bags == 0) {
        if (checked && d_flag_count) cuda_check(cudaMemsetAsync(d_flag_count, 0, 4, st), "cudaMemsetAsync");
        return;
    }
    if (scatter) {
        if (!scatter->out_dest || scatter->bags_per_dest <= 0 || (checked && !scatter->flag_dest))
            throw std::invalid_argument("embedding_bag: invalid scatter destinations");
    }
    if (!d_offsets || !d_indices || (!d_out && !scatter)) throw std::invalid_argument("null argument");
    if (ld_out < t.dim) throw std::invalid_argument("embedding_bag: ld_out < dim");
    Workspace& ws = ws_for(st);
    std::lock_guard<std::mutex> g(ws.mu);
    EbParams p{};
    p.data = t.packed ? t.packed : t.data;
    p.meta = t.packed ? static_cast<const void*>(t.packed + t.meta_off) : t.meta;
    p.meta_stride = t.packed ? t.rec_stride
                             : static_cast<int64_t>(t.scale_type == kEbF32 ? sizeof(EbMetaF32) : sizeof(EbMetaF16));
    p.rows = t.rows;
    p.dim = t.dim;
    p.row_stride = t.packed ? t.rec_stride : t.row_stride;
    p.offsets = d_offsets;
    p.indices = d_indices;
    p.weights = d_weights;
    p.num_bags = num_bags;
    p.out = d_out;
    p.ld_out = ld_out;
    p.flags = checked ? d_flags : nullptr;
    p.rsum = checked ? d_rsum : nullptr;
    p.csum = checked ? d_csum : nullptr;
    p.flag_count = checked ? d_flag_count : nullptr;
    p.status = d_status;
    p.ws_flag_acc = ws.small + 4;
    p.ws_block_cnt = ws.small + 5;
    p.ws_bag_ctr = reinterpret_cast<unsigned long long*>(ws.small + 6);
    p.trace = g_eb_trace;
    p.neg_zero = -0.0f;
    if (scatter) {
        p.out_dest = scatter->out_dest;
        p.flag_dest = checked ? scatter->flag_dest : nullptr;
        p.bags_per_dest = scatter->bags_per_dest;
        p.flag_ld = scatter->flag_ld;
    }
    const cudaError_t e = launch_eb_bags(t.elem, t.scale_type, p, checked, st);
    if (e == cudaErrorInvalidValue) throw std::invalid_argument("embedding_bag: unsupported dimension");
    cuda_check(e, "eb_bag_kernel");
}

static EbTableDesc eb_desc(const EbTable& t) {
    EbTableDesc d{};
    d.data = t.packed ? t.packed : t.data;
    d.meta = t.packed ? static_cast<const void*>(t.packed + t.meta_off) : t.meta;
    d.meta_stride = t.packed ? t.rec_stride
                             : static_cast<int64_t>(t.scale_type == kEbF32 ? sizeof(EbMetaF32) : sizeof(EbMetaF16));
    d.rows = t.rows;
    d.row_stride = t.packed ? t.rec_stride : t.row_stride;
    return d;
}

EbGroup* eb_group_create(const EbTable* const* tables, int64_t ntables, const int64_t* const* d_offsets,
                         const int64_t* const* d_indices, const float* const* d_weights, float* const* const* d_out_dest,
                         uint8_t* const* const* d_flag_dest) {
    if (ntables < 1 || !tables || !d_offsets || !d_indices || !d_out_dest || !d_flag_dest)
        throw std::invalid_argument("null argument");
    std::vector<EbTableDesc> h(static_cast<size_t>(ntables));
    const bool weighted = d_weights != nullptr && d_weights[0] != nullptr;
    bool fused = !std::getenv("ABFTLP_EB_GROUP_UNFUSED");
    for (int64_t i = 0; i < ntables; ++i) {
        const EbTable* t = tables[i];
        if (!t || !d_offsets[i] || !d_indices[i] || !d_out_dest[i] || !d_flag_dest[i])
            throw std::invalid_argument("null argument");
        if (t->elem != tables[0]->elem || t->scale_type != tables[0]->scale_type || t->dim != tables[0]->dim)
            throw std::invalid_argument("eb_group: tables must share element type, scale type and dim");
        if (weighted != (d_weights != nullptr && d_weights[i] != nullptr))
            throw std::invalid_argument("eb_group: either every table or none has weights");
        h[i] = eb_desc(*t);
        h[i].offsets = d_offsets[i];
        h[i].indices = d_indices[i];
        h[i].weights = weighted ? d_weights[i] : nullptr;
        h[i].out_dest = d_out_dest[i];
        h[i].flag_dest = d_flag_dest[i];
        // the fused launch runs the 16-byte cp.async gather kernel for every table with table 0's strides
        const bool al = (reinterpret_cast<uintptr_t>(h[i].data) % 16) == 0 && (h[i].row_stride % 16) == 0 &&
                        (reinterpret_cast<uintptr_t>(h[i].meta) % 16) == 0;
        fused = fused && al && t->dim % 32 == 0 && h[i].row_stride == h[0].row_stride && h[i].rows <= (int64_t{1} << 32) &&
                h[i].row_stride < (int64_t{1} << 32) &&
                h[i].meta_stride == h[0].meta_stride && (t->packed != nullptr) == (tables[0]->packed != nullptr);
    }
    auto* g = new EbGroup();
    g->tables.assign(tables, tables + ntables);
    g->host = h;
    g->weighted = weighted;
    g->fused = fused;
    cudaError_t e = cudaMalloc(&g->d_desc, sizeof(EbTableDesc) * h.size());
    if (e == cudaSuccess) e = cudaMemcpy(g->d_desc, h.data(), sizeof(EbTableDesc) * h.size(), cudaMemcpyHostToDevice);
    if (e == cudaSuccess && !fused) e = cudaMalloc(&g->d_counts, sizeof(uint32_t) * h.size());
    if (e != cudaSuccess) {
        cudaFree(g->d_desc);
        cudaFree(g->d_counts);
        delete g;
        cuda_check(e, "eb_group_create");
    }
    return g;
}

void eb_group_free(EbGroup* g) {
    if (!g) return;
    cudaFree(g->d_desc);
    cudaFree(g->d_counts);
    delete g;
}

void eb_group_set_bags(EbGroup& g, const int64_t* const* d_offsets, const int64_t* const* d_indices,
                       const float* const* d_weights, cudaStream_t st) {
    if (!d_offsets || !d_indices) throw std::invalid_argument("null argument");
    const bool weighted = d_weights != nullptr && d_weights[0] != nullptr;
    if (weighted != g.weighted) throw std::invalid_argument("eb_group: either every table or none has weights");
    for (size_t i = 0; i < g.host.size(); ++i) {
        if (!d_offsets[i] || !d_indices[i]) throw std::invalid_argument("null argument");
        if (weighted != (d_weights != nullptr && d_weights[i] != nullptr))
            throw std::invalid_argument("eb_group: either every table or none has weights");
        g.host[i].offsets = d_offsets[i];
        g.host[i].indices = d_indices[i];
        g.host[i].weights = weighted ? d_weights[i] : nullptr;
    }
    // pageable source: the call returns once the descriptors are staged, the copy itself is ordered on `st`
    cuda_check(cudaMemcpyAsync(g.d_desc, g.host.data(), sizeof(EbTableDesc) * g.host.size(), cudaMemcpyHostToDevice, st),
               "cudaMemcpyAsync(eb group descriptors)");
}

void eb_group_run(const EbGroup& g, int64_t bags_per_table, int64_t ld_out, int64_t flag_ld, int64_t bags_per_dest,
                  bool checked, uint32_t* d_flag_count, int32_t* d_status, cudaStream_t st) {
    if (bags_per_table < 0) throw std::invalid_argument("embedding_bag: negative bag count");
    const EbTable& t0 = *g.tables[0];
    if (ld_out < t0.dim || bags_per_dest <= 0) throw std::invalid_argument("embedding_bag: invalid scatter destinations");
    const int64_t total = bags_per_table * static_cast<int64_t>(g.tables.size());
    if (total == 0) {
        if (checked && d_flag_count) cuda_check(cudaMemsetAsync(d_flag_count, 0, 4, st), "cudaMemsetAsync");
        return;
    }
    if (!g.fused) {
        // one scatter launch per table (same per-bag math and destinations), flag counts summed on the device
        for (size_t i = 0; i < g.tables.size(); ++i) {
            const EbTableDesc& d = g.host[i];
            EbScatter sc;
            sc.out_dest = d.out_dest;
            sc.flag_dest = d.flag_dest;
            sc.bags_per_dest = bags_per_dest;
            sc.flag_ld = flag_ld;
            eb_run(*g.tables[i], d.offsets, d.indices, bags_per_table, d.weights, nullptr, ld_out, checked, nullptr,
                   nullptr, nullptr, checked ? g.d_counts + i : nullptr, d_status, st, &sc);
        }
        if (checked && d_flag_count)
            cuda_check(launch_sum_u32(g.d_counts, static_cast<int64_t>(g.tables.size()), d_flag_count, st), "sum_u32_kernel");
        return;
    }
    Workspace& ws = ws_for(st);
    std::lock_guard<std::mutex> lk(ws.mu);
    const EbTableDesc& d0 = g.host[0];
    EbParams p{};
    p.data = d0.data;  // table 0's layout (shared by the group) drives the kernel choice
    p.meta = d0.meta;
    p.meta_stride = d0.meta_stride;
    p.rows = d0.rows;
    p.dim = t0.dim;
    p.row_stride = d0.row_stride;
    // the weighted template variant is chosen from this pointer's presence; the kernel reads each table's own
    p.weights = g.weighted ? reinterpret_cast<const float*>(g.d_desc) : nullptr;
    p.num_bags = total;
    p.ld_out = ld_out;
    p.flag_count = checked ? d_flag_count : nullptr;
    p.status = d_status;
    p.ws_flag_acc = ws.small + 4;
    p.ws_block_cnt = ws.small + 5;
    p.ws_bag_ctr = reinterpret_cast<unsigned long long*>(ws.small + 6);
    p.trace = g_eb_trace;
    p.neg_zero = -0.0f;
    p.bags_per_dest = bags_per_dest;
    p.flag_ld = flag_ld;
    p.tables = g.d_desc;
    p.bags_per_table = bags_per_table;
    const cudaError_t e = launch_eb_bags(t0.elem, t0.scale_type, p, checked, st);
    if (e == cudaErrorNotSupported)
        throw std::invalid_argument("eb_group: needs 16-byte aligned rows / metadata and dim % 32 == 0");
    cuda_check(e, "eb_bag_async_kernel (grouped tables)");
}

void eb_flip_bit(EbTable& t, int64_t row, int64_t col, uint32_t bit, cudaStream_t st) {
    if (row < 0 || row >= t.rows || col < 0 || col >= t.dim)
        throw std::out_of_range("inject_eb_table: coordinates out of range");
    const uint32_t width = t.elem == kEbU4 ? 4u : 8u;
    if (bit >= width) throw std::out_of_range("flip_bit: bit index out of range");
    const int64_t cb = t.elem == kEbU4 ? col / 2 : col;
    const uint32_t b = bit + (t.elem == kEbU4 ? 4u * static_cast<uint32_t>(col & 1) : 0u);
    // the caller's rows are borrowed const for the lookups; injection is the one sanctioned writer
    cuda_check(launch_flip_bit(const_cast<uint8_t*>(t.data), static_cast<uint64_t>(row * t.row_stride + cb), b, st),
               "flip_bit_kernel");
    if (t.packed)
        cuda_check(launch_flip_bit(t.packed, static_cast<uint64_t>(row * t.rec_stride + cb), b, st), "flip_bit_kernel");
}

void eb_flip_bits(EbTable& t, const int64_t* d_rows, const int64_t* d_cols, const int32_t* d_bits, int64_t n,
                  int32_t* d_status, cudaStream_t st) {
    if (n < 0) throw std::invalid_argument("inject_eb_table: negative count");
    if (n > 0 && (!d_rows || !d_cols || !d_bits)) throw std::invalid_argument("null argument");
    cuda_check(launch_flip_cells(const_cast<uint8_t*>(t.data), t.row_stride, t.packed, t.rec_stride, d_rows, d_cols,
                                 d_bits, n, t.rows, t.dim, t.elem == kEbU4, d_status, st),
               "flip_cells_kernel");
}

// ------------------------------------------------------------------ fault lab
void flip_bit(void* d_base, uint64_t byte_offset, uint32_t bit, cudaStream_t st) {
    cuda_check(launch_flip_bit(d_base, byte_offset, bit, st), "flip_bit_kernel");
}
void set_random(void* d_cell, int width, uint64_t rng_state, cudaStream_t st) {
    cuda_check(launch_set_random(d_cell, width, rng_state, st), "set_random_kernel");
}
void gen(void* d_out, int64_t count, uint64_t seed, uint64_t stream, uint64_t off, int kind, double lo, double hi,
         uint64_t bound, cudaStream_t st) {
    cuda_check(launch_gen(d_out, count, seed, stream, off, kind, lo, hi, bound, st), "gen_kernel");
}
void l2_flush(void* d_buf, int64_t bytes, int salt, cudaStream_t st) {
    cuda_check(launch_flush(d_buf, bytes, salt, st), "flush_kernel");
}

}  // namespace abftk
