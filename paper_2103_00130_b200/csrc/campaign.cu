// Fault-injection campaigns, reports, benches and ABEB/bag files over the GPU operators.
//
// The campaign protocol is the reference's (P:src/fault_lab.cpp:168-285): per trial t the data
// come from SplitMix64(seed, 4t+0), fault placement from SplitMix64(seed, 4t+1) and EB bags from
// SplitMix64(seed, 4t+2). Data are generated on the device by the counter-based generator (draw e
// of a stream is mix(state0 + (e+1)*gamma)), fault coordinates on the host, and every trial's
// encode -> [inject B] -> checked GEMM -> [inject C -> verify] (or table -> row sums -> bags ->
// [inject] -> checked EB) runs as stream-ordered GPU work with one synchronisation per campaign.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <fstream>
#include <iomanip>
#include <map>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <vector>

#include "campaign.h"
#include "runtime.h"

namespace abftk {

namespace {

// draw_bit_index (P:src/fault_lab.cpp:89-96)
unsigned draw_bit(SplitMix64& rng, BitRange range, unsigned width) {
    switch (range) {
        case BitRange::high4: return width - 4 + static_cast<unsigned>(rng.next_below(4));
        case BitRange::low4: return static_cast<unsigned>(rng.next_below(4));
        case BitRange::all: break;
    }
    return static_cast<unsigned>(rng.next_below(width));
}

enum Role : uint64_t { kData = 0, kInject = 1, kBags = 2, kStride = 4 };

template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    void reserve(size_t cnt) {
        if (cnt <= n) return;
        if (p) cudaFree(p);
        p = nullptr;
        ABFT_CUDA(cudaMalloc(&p, std::max<size_t>(cnt, 1) * sizeof(T)));
        n = cnt;
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};

// The campaign report from per-trial verdicts: trials [g * per_group, (g+1) * per_group) form row g. A trial's
// verdict counts as a detection, or -- for the control campaign (target none) -- as a false positive.
template <typename Flag>
CampaignReport tally(const FaultSpec& spec, const std::vector<Flag>& verdicts, const std::vector<std::string>& labels,
                     uint64_t per_group, std::string notes) {
    CampaignReport rep;
    rep.target = fault_target_name(spec.target);
    rep.model = fault_model_name(spec.model);
    rep.bitRange = bit_range_name(spec.bitRange);
    rep.notes = std::move(notes);
    const bool control = spec.target == FaultTarget::none;
    rep.perShape.resize(labels.size());
    for (size_t g = 0; g < labels.size(); ++g) {
        ShapeStats& row = rep.perShape[g];
        row.label = labels[g];
        row.trials = per_group;
        const uint64_t hits = static_cast<uint64_t>(
            std::count_if(verdicts.begin() + g * per_group, verdicts.begin() + (g + 1) * per_group,
                          [](Flag f) { return f != 0; }));
        (control ? row.falsePositives : row.detected) = hits;
        rep.trials += row.trials;
        rep.detected += row.detected;
        rep.falsePositives += row.falsePositives;
    }
    rep.notDetected = rep.trials - rep.detected;
    return rep;
}

struct StreamGuard {
    cudaStream_t s = nullptr;
    StreamGuard() { ABFT_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); }
    ~StreamGuard() {
        if (s) {
            cudaStreamSynchronize(s);
            cudaStreamDestroy(s);
        }
    }
};

}  // namespace

// ============================================================ GEMM campaign (P:src/fault_lab.cpp:168-225)
CampaignReport run_gemm_campaign(const CampaignConfig& cfg) {
    if (!cfg.gemm) throw std::invalid_argument("run_gemm_campaign: not a gemm workload");
    const GemmWorkload& wl = *cfg.gemm;
    if (wl.shapes.empty() || wl.trialsPerShape == 0) throw std::invalid_argument("run_gemm_campaign: empty workload");
    if (cfg.fault.target == FaultTarget::eb_table)
        throw std::invalid_argument("run_gemm_campaign: eb_table target on gemm workload");
    const uint64_t total = wl.shapes.size() * wl.trialsPerShape;
    uint64_t max_mk = 0, max_kn = 0, max_mn = 0, max_m = 0;
    for (const auto& s : wl.shapes) {
        max_mk = std::max(max_mk, s.m * s.k);
        max_kn = std::max(max_kn, s.k * s.n);
        max_mn = std::max(max_mn, s.m * ((s.n + 3) / 4 * 4));
        max_m = std::max(max_m, s.m);
    }
    StreamGuard sg;
    cudaStream_t st = sg.s;
    DevBuf<uint8_t> a;
    DevBuf<int8_t> b;
    DevBuf<int32_t> c, csum;
    DevBuf<uint8_t> flags;
    DevBuf<uint32_t> errs, scratch_err;
    a.reserve(max_mk);
    b.reserve(max_kn);
    c.reserve(max_mn);
    csum.reserve(max_m);
    flags.reserve(max_m);
    errs.reserve(total);
    scratch_err.reserve(1);
    std::unique_ptr<GemmWeight, void (*)(GemmWeight*)> w(new GemmWeight(), free_weight);
    const uint64_t seed = cfg.fault.seed;
    for (uint64_t t = 0; t < total; ++t) {
        const GemmShape& sh = wl.shapes[t / wl.trialsPerShape];
        const int64_t m = sh.m, n = sh.n, k = sh.k;
        const int64_t ldc = (n + 3) / 4 * 4;
        gen(a.p, m * k, seed, t * kStride + kData, 0, 0, 0, 0, 0, st);
        gen(b.p, k * n, seed, t * kStride + kData, static_cast<uint64_t>(m * k), 1, 0, 0, 0, st);
        encode_weight_into(*w, b.p, k, n, n, st);  // checksums of the pristine B
        if (cfg.fault.target == FaultTarget::weight_B) {
            SplitMix64 rng(seed, t * kStride + kInject);
            const uint64_t i = rng.next_below(static_cast<uint64_t>(k));
            const uint64_t j = rng.next_below(static_cast<uint64_t>(n));  // checksum column excluded
            int8_t* cell = w->element(static_cast<int64_t>(i), static_cast<int64_t>(j));
            if (cfg.fault.model == FaultModel::single_bit_flip)
                flip_bit(cell, 0, draw_bit(rng, cfg.fault.bitRange, 8), st);
            else
                set_random(cell, 8, rng.state, st);
        }
        const bool c_target = cfg.fault.target == FaultTarget::intermediate_C;
        gemm(a.p, m, k, *w, c.p, ldc, true, csum.p, 1, flags.p, c_target ? scratch_err.p : errs.p + t, nullptr, st);
        if (c_target) {
            SplitMix64 rng(seed, t * kStride + kInject);
            const uint64_t i = rng.next_below(static_cast<uint64_t>(m));
            const uint64_t j = rng.next_below(static_cast<uint64_t>(n + 1));
            int32_t* cell = j < static_cast<uint64_t>(n) ? c.p + i * ldc + j : csum.p + i;
            if (cfg.fault.model == FaultModel::single_bit_flip)
                flip_bit(cell, 0, draw_bit(rng, cfg.fault.bitRange, 32), st);
            else
                set_random(cell, 32, rng.state, st);
            verify(c.p, ldc, csum.p, 1, m, n, flags.p, errs.p + t, st);
        }
    }
    std::vector<uint32_t> h(total);
    ABFT_CUDA(cudaMemcpyAsync(h.data(), errs.p, total * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    ABFT_CUDA(cudaStreamSynchronize(st));

    std::vector<std::string> labels;
    for (const GemmShape& sh : wl.shapes)
        labels.push_back(std::to_string(sh.m) + "x" + std::to_string(sh.n) + "x" + std::to_string(sh.k));
    return tally(cfg.fault, h, labels, wl.trialsPerShape, "checksum column excluded from weight_B injection");
}

// ============================================================ EB campaign (P:src/fault_lab.cpp:227-285)
CampaignReport run_eb_campaign(const CampaignConfig& cfg) {
    if (!cfg.eb) throw std::invalid_argument("run_eb_campaign: not an eb workload");
    const EbWorkload& wl = *cfg.eb;
    if (wl.trials == 0 || wl.tableRows == 0 || wl.tableDim == 0 || wl.pooling == 0 || wl.batch == 0)
        throw std::invalid_argument("run_eb_campaign: empty workload");
    if (cfg.fault.target == FaultTarget::weight_B || cfg.fault.target == FaultTarget::intermediate_C)
        throw std::invalid_argument("run_eb_campaign: gemm target on eb workload");
    const int64_t R = wl.tableRows, d = wl.tableDim, pool = wl.pooling, batch = wl.batch;
    StreamGuard sg;
    cudaStream_t st = sg.s;
    DevBuf<int8_t> rows;
    DevBuf<float> scales, biases, out;
    DevBuf<int64_t> offsets, indices;
    DevBuf<uint8_t> flags, detected;
    rows.reserve(R * d);
    scales.reserve(R);
    biases.reserve(R);
    out.reserve(batch * d);
    offsets.reserve(batch + 1);
    indices.reserve(batch * pool);
    flags.reserve(batch);
    detected.reserve(wl.trials);
    std::vector<int64_t> hoff(batch + 1);
    for (int64_t b = 0; b <= batch; ++b) hoff[b] = b * pool;
    ABFT_CUDA(cudaMemcpyAsync(offsets.p, hoff.data(), hoff.size() * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    EbTable table;
    const uint64_t seed = cfg.fault.seed;
    for (uint64_t t = 0; t < wl.trials; ++t) {
        const uint64_t data_stream = t * kStride + kData;
        gen(rows.p, R * d, seed, data_stream, 0, 1, 0, 0, 0, st);
        gen(scales.p, R, seed, data_stream, static_cast<uint64_t>(R * d), 2, 0.005, 0.02, 0, st);
        gen(biases.p, R, seed, data_stream, static_cast<uint64_t>(R * d + R), 2, -1.0, 1.0, 0, st);
        eb_table_rebuild(table, kEbS8, rows.p, R, d, d, kEbF32, scales.p, biases.p, nullptr, st);
        gen(indices.p, batch * pool, seed, t * kStride + kBags, 0, 3, 0, 0, static_cast<uint64_t>(R), st);
        if (cfg.fault.target == FaultTarget::eb_table) {
            SplitMix64 rng(seed, t * kStride + kInject);
            const uint64_t bag = rng.next_below(static_cast<uint64_t>(batch));  // every bag is non-empty
            const uint64_t pos = rng.next_below(static_cast<uint64_t>(pool));
            const uint64_t row =
                SplitMix64::draw_at(seed, t * kStride + kBags, bag * static_cast<uint64_t>(pool) + pos) %
                static_cast<uint64_t>(R);
            const uint64_t col = rng.next_below(static_cast<uint64_t>(d));
            int8_t* cell = rows.p + row * static_cast<uint64_t>(d) + col;
            if (cfg.fault.model == FaultModel::single_bit_flip)
                flip_bit(cell, 0, draw_bit(rng, cfg.fault.bitRange, 8), st);
            else
                set_random(cell, 8, rng.state, st);
            eb_pack(table, st);  // the lookups read the interleaved copy; row sums stay pristine
        }
        eb_run(table, offsets.p, indices.p, batch, nullptr, out.p, d, true, flags.p, nullptr, nullptr, nullptr,
               nullptr, st);
        ABFT_CUDA(launch_any_flag(flags.p, batch, detected.p, static_cast<int64_t>(t), st));
    }
    std::vector<uint8_t> h(wl.trials);
    ABFT_CUDA(cudaMemcpyAsync(h.data(), detected.p, wl.trials, cudaMemcpyDeviceToHost, st));
    ABFT_CUDA(cudaStreamSynchronize(st));
    if (table.meta) cudaFree(table.meta);

    const std::string label = "R" + std::to_string(wl.tableRows) + "_d" + std::to_string(wl.tableDim) + "_p" +
                              std::to_string(wl.pooling) + "_b" + std::to_string(wl.batch);
    return tally(cfg.fault, h, {label}, wl.trials, "");
}

CampaignReport run_campaign(const CampaignConfig& cfg) {
    if (cfg.gemm && cfg.eb) throw std::invalid_argument("run_campaign: config sets both gemm and eb workloads");
    if (cfg.gemm) return run_gemm_campaign(cfg);
    if (cfg.eb) return run_eb_campaign(cfg);
    throw std::invalid_argument("run_campaign: no workload configured");
}

// ============================================================ benches (P:src/bench.cpp:50-152)
namespace {
double median(std::vector<double> v) {
    std::sort(v.begin(), v.end());
    const size_t n = v.size();
    return n % 2 ? v[n / 2] : 0.5 * (v[n / 2 - 1] + v[n / 2]);
}
struct Events {
    cudaEvent_t a = nullptr, b = nullptr;
    Events() {
        ABFT_CUDA(cudaEventCreate(&a));
        ABFT_CUDA(cudaEventCreate(&b));
    }
    ~Events() {
        cudaEventDestroy(a);
        cudaEventDestroy(b);
    }
};
template <typename Fn>
double time_ns(cudaStream_t st, Events& ev, Fn&& fn) {
    ABFT_CUDA(cudaEventRecord(ev.a, st));
    fn();
    ABFT_CUDA(cudaEventRecord(ev.b, st));
    ABFT_CUDA(cudaEventSynchronize(ev.b));
    float ms = 0.f;
    ABFT_CUDA(cudaEventElapsedTime(&ms, ev.a, ev.b));
    return static_cast<double>(ms) * 1e6;
}
constexpr int64_t kFlushBytes = int64_t{256} << 20;
}  // namespace

// Baseline = encode (re-pack) + unchecked kernel, ABFT = encode + checked kernel, both timed per
// call like the reference (plain_gemm packs B inside its timing; abft_run re-encodes).
BenchTimes bench_gemm(uint64_t m, uint64_t n, uint64_t k, uint64_t reps, uint64_t seed) {
    if (reps < 5) throw std::invalid_argument("bench_gemm: need at least 5 repetitions");
    if (m == 0 || n == 0 || k == 0) throw std::invalid_argument("bench_gemm: zero dimension");
    StreamGuard sg;
    cudaStream_t st = sg.s;
    DevBuf<uint8_t> a;
    DevBuf<int8_t> b;
    DevBuf<int32_t> c1, c2, csum;
    DevBuf<uint8_t> flags;
    DevBuf<uint32_t> err;
    const int64_t ldc = (n + 3) / 4 * 4;
    a.reserve(m * k);
    b.reserve(k * n);
    c1.reserve(m * ldc);
    c2.reserve(m * ldc);
    csum.reserve(m);
    flags.reserve(m);
    err.reserve(1);
    gen(a.p, m * k, seed, 0, 0, 0, 0, 0, 0, st);
    gen(b.p, k * n, seed, 0, m * k, 1, 0, 0, 0, st);
    std::unique_ptr<GemmWeight, void (*)(GemmWeight*)> w(new GemmWeight(), free_weight);
    encode_weight_into(*w, b.p, k, n, n, st);
    gemm(a.p, m, k, *w, c1.p, ldc, false, nullptr, 0, nullptr, nullptr, nullptr, st);
    gemm(a.p, m, k, *w, c2.p, ldc, true, csum.p, 1, flags.p, err.p, nullptr, st);
    {
        std::vector<int32_t> h1(m * ldc), h2(m * ldc);
        ABFT_CUDA(cudaMemcpyAsync(h1.data(), c1.p, h1.size() * 4, cudaMemcpyDeviceToHost, st));
        ABFT_CUDA(cudaMemcpyAsync(h2.data(), c2.p, h2.size() * 4, cudaMemcpyDeviceToHost, st));
        ABFT_CUDA(cudaStreamSynchronize(st));
        for (uint64_t i = 0; i < m; ++i)
            for (uint64_t j = 0; j < n; ++j)
                if (h1[i * ldc + j] != h2[i * ldc + j])
                    throw std::runtime_error("bench_gemm: baseline and abft outputs diverge");
    }
    auto baseline_run = [&] {
        encode_weight_into(*w, b.p, k, n, n, st);
        gemm(a.p, m, k, *w, c1.p, ldc, false, nullptr, 0, nullptr, nullptr, nullptr, st);
    };
    auto abft_run = [&] {
        encode_weight_into(*w, b.p, k, n, n, st);
        gemm(a.p, m, k, *w, c2.p, ldc, true, csum.p, 1, flags.p, err.p, nullptr, st);
    };
    Events ev;
    for (int i = 0; i < 2; ++i) {
        baseline_run();
        abft_run();
    }
    std::vector<double> base, abft;
    for (uint64_t r = 0; r < reps; ++r) {
        base.push_back(time_ns(st, ev, baseline_run));
        abft.push_back(time_ns(st, ev, abft_run));
    }
    return {median(base), median(abft)};
}

BenchTimes bench_eb(uint64_t rows, uint64_t dim, uint64_t pooling, uint64_t batch, uint64_t reps, uint64_t seed) {
    if (reps < 5) throw std::invalid_argument("bench_eb: need at least 5 repetitions");
    if (rows == 0 || dim == 0 || pooling == 0 || batch == 0) throw std::invalid_argument("bench_eb: invalid dimensions");
    StreamGuard sg;
    cudaStream_t st = sg.s;
    DevBuf<int8_t> tbl;
    DevBuf<float> scales, biases, out;
    DevBuf<int64_t> offsets, indices;
    DevBuf<uint8_t> flags;
    DevBuf<char> flush;
    tbl.reserve(rows * dim);
    scales.reserve(rows);
    biases.reserve(rows);
    out.reserve(batch * dim);
    offsets.reserve(batch + 1);
    indices.reserve(batch * pooling);
    flags.reserve(batch);
    flush.reserve(kFlushBytes);
    // SplitMix64(seed, 1): rows, scales, biases, then bag indices, in that draw order.
    gen(tbl.p, rows * dim, seed, 1, 0, 1, 0, 0, 0, st);
    gen(scales.p, rows, seed, 1, rows * dim, 2, 0.005, 0.02, 0, st);
    gen(biases.p, rows, seed, 1, rows * dim + rows, 2, -1.0, 1.0, 0, st);
    gen(indices.p, batch * pooling, seed, 1, rows * dim + 2 * rows, 3, 0, 0, rows, st);
    std::vector<int64_t> hoff(batch + 1);
    for (uint64_t b = 0; b <= batch; ++b) hoff[b] = static_cast<int64_t>(b * pooling);
    ABFT_CUDA(cudaMemcpyAsync(offsets.p, hoff.data(), hoff.size() * 8, cudaMemcpyHostToDevice, st));
    std::unique_ptr<EbTable, void (*)(EbTable*)> t(
        eb_table_create(kEbS8, tbl.p, rows, dim, dim, kEbF32, scales.p, biases.p, nullptr, st), eb_table_free);
    auto baseline_run = [&] {
        eb_run(*t, offsets.p, indices.p, batch, nullptr, out.p, dim, false, nullptr, nullptr, nullptr, nullptr,
               nullptr, st);
    };
    auto abft_run = [&] {
        eb_run(*t, offsets.p, indices.p, batch, nullptr, out.p, dim, true, flags.p, nullptr, nullptr, nullptr,
               nullptr, st);
    };
    Events ev;
    for (int i = 0; i < 2; ++i) {
        baseline_run();
        abft_run();
    }
    std::vector<double> base, abft;
    for (uint64_t r = 0; r < reps; ++r) {
        l2_flush(flush.p, kFlushBytes, static_cast<int>(2 * r), st);
        base.push_back(time_ns(st, ev, baseline_run));
        l2_flush(flush.p, kFlushBytes, static_cast<int>(2 * r + 1), st);
        abft.push_back(time_ns(st, ev, abft_run));
    }
    return {median(base), median(abft)};
}

std::vector<EbResultHost> check_bags_on_device(const HostTable& t, const HostBags& bags, bool validate) {
    const int64_t nb = static_cast<int64_t>(bags.offsets.size()) - 1;
    StreamGuard sg;
    cudaStream_t st = sg.s;
    DevBuf<int8_t> rows;
    DevBuf<float> scales, biases, weights, out;
    DevBuf<int32_t> sums;
    DevBuf<int64_t> offsets, indices;
    DevBuf<uint8_t> flags;
    DevBuf<double> rsum, csum;
    DevBuf<int32_t> status;
    rows.reserve(t.data.size());
    scales.reserve(t.rows);
    biases.reserve(t.rows);
    sums.reserve(t.rows);
    ABFT_CUDA(cudaMemcpyAsync(rows.p, t.data.data(), t.data.size(), cudaMemcpyHostToDevice, st));
    ABFT_CUDA(cudaMemcpyAsync(scales.p, t.scales.data(), t.rows * 4, cudaMemcpyHostToDevice, st));
    ABFT_CUDA(cudaMemcpyAsync(biases.p, t.biases.data(), t.rows * 4, cudaMemcpyHostToDevice, st));
    ABFT_CUDA(cudaMemcpyAsync(sums.p, t.rowSums.data(), t.rows * 4, cudaMemcpyHostToDevice, st));
    std::unique_ptr<EbTable, void (*)(EbTable*)> table(
        eb_table_create(kEbS8, rows.p, t.rows, t.dim, t.dim, kEbF32, scales.p, biases.p, sums.p, st), eb_table_free);
    if (validate && eb_table_validate(*table, sums.p, st) != 0)
        throw std::runtime_error("table row-sum checksums do not match contents");
    std::vector<EbResultHost> res(static_cast<size_t>(std::max<int64_t>(nb, 0)));
    if (nb <= 0) return res;
    offsets.reserve(bags.offsets.size());
    indices.reserve(bags.indices.size());
    out.reserve(nb * t.dim);
    flags.reserve(nb);
    rsum.reserve(nb);
    csum.reserve(nb);
    status.reserve(1);
    ABFT_CUDA(cudaMemcpyAsync(offsets.p, bags.offsets.data(), bags.offsets.size() * 8, cudaMemcpyHostToDevice, st));
    if (!bags.indices.empty())
        ABFT_CUDA(cudaMemcpyAsync(indices.p, bags.indices.data(), bags.indices.size() * 8, cudaMemcpyHostToDevice, st));
    const float* wptr = nullptr;
    if (bags.weighted) {
        weights.reserve(bags.weights.size());
        ABFT_CUDA(cudaMemcpyAsync(weights.p, bags.weights.data(), bags.weights.size() * 4, cudaMemcpyHostToDevice, st));
        wptr = weights.p;
    }
    ABFT_CUDA(cudaMemsetAsync(status.p, 0, 4, st));
    eb_run(*table, offsets.p, indices.p, nb, wptr, out.p, t.dim, true, flags.p, rsum.p, csum.p, nullptr, status.p, st);
    std::vector<uint8_t> hf(nb);
    std::vector<double> hr(nb), hc(nb);
    int32_t hs = 0;
    ABFT_CUDA(cudaMemcpyAsync(hf.data(), flags.p, nb, cudaMemcpyDeviceToHost, st));
    ABFT_CUDA(cudaMemcpyAsync(hr.data(), rsum.p, nb * 8, cudaMemcpyDeviceToHost, st));
    ABFT_CUDA(cudaMemcpyAsync(hc.data(), csum.p, nb * 8, cudaMemcpyDeviceToHost, st));
    ABFT_CUDA(cudaMemcpyAsync(&hs, status.p, 4, cudaMemcpyDeviceToHost, st));
    ABFT_CUDA(cudaStreamSynchronize(st));
    if (hs & 1) throw std::out_of_range("embedding_bag: index out of range");
    for (int64_t i = 0; i < nb; ++i) res[i] = {hr[i], hc[i], hf[i] != 0};
    return res;
}

}  // namespace abftk
