// C ABI of libabftlp_b200.so: the reference-compatible surface (include/abftlp.h) and the
// device-pointer operator entry points (include/abftlp_b200.h).
//
// Error model mirrors the reference's `guarded` (P:src/capi.cpp:28-41): invalid_argument and
// out_of_range -> ABFTLP_ERR_INVALID_ARGUMENT, runtime_error -> ABFTLP_ERR_IO, anything else
// (including CUDA failures) -> ABFTLP_ERR_INTERNAL; the message goes to a thread-local string.
#include <cstdint>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iomanip>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/abftlp_b200.h"
#include "campaign.h"
#include "runtime.h"

struct abftlp_campaign_s {
    abftk::CampaignConfig cfg;
};
struct abftlp_report_s {
    abftk::CampaignReport report;
};
struct abftlp_gemm_weight_s {
    abftk::GemmWeight* w;
};
struct abftlp_eb_table_s {
    abftk::EbTable* t;
};
struct abftlp_gemm_group_s {
    abftk::GemmGroup* g;
};
struct abftlp_eb_group_s {
    abftk::EbGroup* g;
};

namespace {

thread_local std::string g_last_error;

abftlp_status fail(abftlp_status code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

template <typename Fn>
abftlp_status guarded(Fn&& fn) {
    try {
        return fn();
    } catch (const std::invalid_argument& e) {
        return fail(ABFTLP_ERR_INVALID_ARGUMENT, e.what());
    } catch (const std::out_of_range& e) {
        return fail(ABFTLP_ERR_INVALID_ARGUMENT, e.what());
    } catch (const abftk::CudaError& e) {
        return fail(ABFTLP_ERR_INTERNAL, e.what());
    } catch (const std::runtime_error& e) {
        return fail(ABFTLP_ERR_IO, e.what());
    } catch (const std::exception& e) {
        return fail(ABFTLP_ERR_INTERNAL, e.what());
    }
}

char* dup_string(const std::string& s) {
    char* out = new char[s.size() + 1];
    std::memcpy(out, s.c_str(), s.size() + 1);
    return out;
}

cudaStream_t as_stream(abftlp_stream s) { return reinterpret_cast<cudaStream_t>(s); }

// Per-stream device staging for the host-buffer entry points.
struct HostStage {
    uint8_t* a = nullptr;
    size_t a_cap = 0;
    int32_t* c = nullptr;
    size_t c_cap = 0;
    int32_t* csum = nullptr;
    size_t csum_cap = 0;
    uint8_t* flags = nullptr;
    size_t flags_cap = 0;
    uint32_t* err = nullptr;
    // pipelined host job (abftlp_gemm_checked_host_batched): copy-in / copy-out streams and per-slot events
    cudaStream_t h2d = nullptr, d2h = nullptr;
    cudaEvent_t a_ready[3] = {}, c_done[3] = {}, out_done[3] = {};
    uint8_t* ja = nullptr;
    size_t ja_cap = 0;
    int32_t* jc = nullptr;
    size_t jc_cap = 0;
    int32_t* jcs = nullptr;
    size_t jcs_cap = 0;
    uint8_t* jfl = nullptr;
    size_t jfl_cap = 0;
    uint32_t* jerr = nullptr;
    size_t jerr_cap = 0;
    // requantized job (abftlp_gemm_checked_requant_host_batched): u8 outputs, row sums of A, column sums of B
    uint8_t* jo = nullptr;
    size_t jo_cap = 0;
    int32_t* jrs = nullptr;
    size_t jrs_cap = 0;
    int32_t* jcol = nullptr;
    size_t jcol_cap = 0;
};
std::mutex g_stage_mu;
std::unordered_map<uint64_t, HostStage> g_stage;

template <typename T>
void ensure(T*& p, size_t& cap, size_t need) {
    if (need <= cap) return;
    if (p) cudaFree(p);
    p = nullptr;
    ABFT_CUDA(cudaMalloc(&p, need * sizeof(T)));
    cap = need;
}

}  // namespace

extern "C" {

// ============================================================ status
const char* abftlp_status_str(abftlp_status status) {
    switch (status) {
        case ABFTLP_OK: return "ok";
        case ABFTLP_ERR_INVALID_ARGUMENT: return "invalid argument";
        case ABFTLP_ERR_IO: return "i/o error";
        case ABFTLP_ERR_PARSE: return "parse error";
        case ABFTLP_ERR_INTERNAL: return "internal error";
    }
    return "unknown status";
}

const char* abftlp_last_error(void) { return g_last_error.c_str(); }

// ============================================================ campaigns
abftlp_status abftlp_campaign_load(const char* config_path, abftlp_campaign** out) {
    if (!config_path || !out) return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        std::ifstream in(config_path);
        if (!in) return fail(ABFTLP_ERR_IO, std::string("config not found: ") + config_path);
        std::ostringstream buf;
        buf << in.rdbuf();
        try {
            *out = new abftlp_campaign_s{abftk::parse_campaign_config(buf.str())};
        } catch (const std::invalid_argument& e) {
            return fail(ABFTLP_ERR_PARSE, e.what());
        }
        return ABFTLP_OK;
    });
}

abftlp_status abftlp_campaign_parse(const char* config_text, abftlp_campaign** out) {
    if (!config_text || !out) return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        try {
            *out = new abftlp_campaign_s{abftk::parse_campaign_config(config_text)};
        } catch (const std::invalid_argument& e) {
            return fail(ABFTLP_ERR_PARSE, e.what());
        }
        return ABFTLP_OK;
    });
}

void abftlp_campaign_free(abftlp_campaign* campaign) { delete campaign; }

abftlp_status abftlp_campaign_run(const abftlp_campaign* campaign, abftlp_report** out) {
    if (!campaign || !out) return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        *out = new abftlp_report_s{abftk::run_campaign(campaign->cfg)};
        return ABFTLP_OK;
    });
}

void abftlp_report_free(abftlp_report* report) { delete report; }
uint64_t abftlp_report_trials(const abftlp_report* report) { return report->report.trials; }
uint64_t abftlp_report_detected(const abftlp_report* report) { return report->report.detected; }
uint64_t abftlp_report_false_positives(const abftlp_report* report) { return report->report.falsePositives; }
double abftlp_report_detection_rate(const abftlp_report* report) { return report->report.detectionRate(); }

abftlp_status abftlp_report_write_csv(const abftlp_report* report, const char* path) {
    if (!report || !path) return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        std::ofstream out(path);
        if (!out) return fail(ABFTLP_ERR_IO, std::string("cannot write: ") + path);
        out << abftk::report_to_csv(report->report);
        return out ? ABFTLP_OK : fail(ABFTLP_ERR_IO, std::string("write failed: ") + path);
    });
}

abftlp_status abftlp_report_render(const abftlp_report* report, char** out) {
    if (!report || !out) return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        *out = dup_string(abftk::report_to_table(report->report));
        return ABFTLP_OK;
    });
}

void abftlp_string_free(char* s) { delete[] s; }

// ============================================================ analysis (closed forms)
abftlp_status abftlp_analyze(uint64_t m, uint64_t n, uint64_t k, uint64_t d, uint64_t pool, abftlp_analysis* out) {
    if (!out) return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        if (m < 1 || n < 1 || k < 1) throw std::invalid_argument("encode_overhead: zero dimension");
        if (pool < 1 || d < 1) throw std::invalid_argument("eb_overhead: zero argument");
        const double dm = double(m), dn = double(n), dk = double(k);
        abftlp_analysis a{};
        a.encode_overhead_a = 1.0 / (2.0 * dn) + 1.0 / dm + 1.0 / (2.0 * dk);
        a.encode_overhead_b = 1.0 / (2.0 * dm) + 1.0 / dn + 1.0 / (2.0 * dk);
        a.p_detect_b_bitflip = 1.0 - std::pow(3.0 / 256.0, dm);
        a.p_detect_b_random = 1.0 - std::pow(1018.0 / 32640.0, dm);
        a.p_detect_c_bitflip = 1.0;
        a.p_detect_c_random = 1.0 - 1.0 / 127.0;
        a.eb_overhead = 1.0 / double(d) + 1.0 / (3.0 * double(pool));
        a.eb_memory_overhead = 32.0 / (8.0 * double(d));
        *out = a;
        return ABFTLP_OK;
    });
}

// ============================================================ benches (GPU)
abftlp_status abftlp_bench_gemm(uint64_t m, uint64_t n, uint64_t k, uint32_t repetitions, uint64_t seed,
                                abftlp_bench_result* out) {
    if (!out) return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        abftk::BenchTimes r = abftk::bench_gemm(m, n, k, repetitions, seed);
        *out = {r.baseline_ns, r.abft_ns, (r.abft_ns - r.baseline_ns) / r.baseline_ns};
        return ABFTLP_OK;
    });
}

abftlp_status abftlp_bench_eb(uint64_t table_rows, uint64_t dim, uint64_t pooling, uint64_t batch,
                              uint32_t repetitions, uint64_t seed, abftlp_bench_result* out) {
    if (!out) return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        abftk::BenchTimes r = abftk::bench_eb(table_rows, dim, pooling, batch, repetitions, seed);
        *out = {r.baseline_ns, r.abft_ns, (r.abft_ns - r.baseline_ns) / r.baseline_ns};
        return ABFTLP_OK;
    });
}

// ============================================================ eb-check over files
abftlp_status abftlp_eb_check_files(const char* table_path, const char* indices_path, int skip_validation,
                                    uint64_t* bags_out, uint64_t* flagged_out, char** render_out) {
    if (!table_path || !indices_path) return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        abftk::HostTable table = abftk::load_table_file(table_path);
        std::ifstream in(indices_path);
        if (!in) return fail(ABFTLP_ERR_IO, std::string("indices file not found: ") + indices_path);
        abftk::HostBags bags;
        std::string perr;
        if (!abftk::parse_bag_lines(in, bags, perr)) return fail(ABFTLP_ERR_PARSE, perr);
        std::vector<abftk::EbResultHost> res = abftk::check_bags_on_device(table, bags, skip_validation == 0);
        uint64_t flagged = 0;
        std::ostringstream render;
        for (size_t i = 0; i < res.size(); ++i) {
            flagged += res[i].err ? 1 : 0;
            render << "bag " << i << ": " << (res[i].err ? "ERROR" : "ok") << " rsum=" << res[i].rsum
                   << " csum=" << res[i].csum << "\n";
        }
        if (bags_out) *bags_out = res.size();
        if (flagged_out) *flagged_out = flagged;
        if (render_out) *render_out = dup_string(render.str());
        return ABFTLP_OK;
    });
}

// ============================================================ device operators: GEMM
abftlp_status abftlp_gemm_encode(const int8_t* d_b, uint64_t k, uint64_t n, uint64_t ldb, abftlp_stream stream,
                                 abftlp_gemm_weight** out) {
    if (!out) return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        abftk::GemmWeight* w = abftk::encode_weight(d_b, static_cast<int64_t>(k), static_cast<int64_t>(n),
                                                    static_cast<int64_t>(ldb), as_stream(stream));
        *out = new abftlp_gemm_weight_s{w};
        return ABFTLP_OK;
    });
}

abftlp_status abftlp_gemm_reencode(abftlp_gemm_weight* w, const int8_t* d_b, uint64_t ldb, abftlp_stream stream) {
    if (!w || !d_b) return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        abftk::GemmWeight& W = *w->w;
        if (W.batch != 1) throw std::invalid_argument("batched weight: operation needs a single weight");
        abftk::encode_weight_into(W, d_b, W.k, W.n, static_cast<int64_t>(ldb), as_stream(stream));
        return ABFTLP_OK;
    });
}

abftlp_status abftlp_gemm_encode_batched(const int8_t* d_b, uint64_t batch, uint64_t k, uint64_t n, uint64_t ldb,
                                         uint64_t stride_b, abftlp_stream stream, abftlp_gemm_weight** out) {
    if (!out) return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        abftk::GemmWeight* w = abftk::encode_weight(d_b, static_cast<int64_t>(k), static_cast<int64_t>(n),
                                                    static_cast<int64_t>(ldb), as_stream(stream),
                                                    static_cast<int64_t>(batch), static_cast<int64_t>(stride_b));
        *out = new abftlp_gemm_weight_s{w};
        return ABFTLP_OK;
    });
}

void abftlp_gemm_weight_free(abftlp_gemm_weight* w) {
    if (!w) return;
    abftk::free_weight(w->w);
    delete w;
}

abftlp_status abftlp_gemm_weight_dims(const abftlp_gemm_weight* w, uint64_t* k, uint64_t* n) {
    if (!w || !k || !n) return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    *k = static_cast<uint64_t>(w->w->k);
    *n = static_cast<uint64_t>(w->w->n);
    return ABFTLP_OK;
}

abftlp_status abftlp_gemm_weight_checksums(const abftlp_gemm_weight* w, int8_t* d_cs, abftlp_stream stream) {
    if (!w || !d_cs) return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        if (w->w->batch != 1) throw std::invalid_argument("batched weight: operation needs a single weight");
        ABFT_CUDA(cudaMemcpyAsync(d_cs, w->w->cs, static_cast<size_t>(w->w->k), cudaMemcpyDeviceToDevice,
                                  as_stream(stream)));
        return ABFTLP_OK;
    });
}

abftlp_status abftlp_gemm_weight_set_checksums(abftlp_gemm_weight* w, const int8_t* d_cs, abftlp_stream stream) {
    if (!w || !d_cs) return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        if (w->w->batch != 1) throw std::invalid_argument("batched weight: operation needs a single weight");
        abftk::set_checksums(*w->w, d_cs, as_stream(stream));
        return ABFTLP_OK;
    });
}

abftlp_status abftlp_gemm_weight_read(const abftlp_gemm_weight* w, int8_t* d_out, abftlp_stream stream) {
    if (!w || !d_out) return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        if (w->w->batch != 1) throw std::invalid_argument("batched weight: operation needs a single weight");
        abftk::read_encoded(*w->w, d_out, as_stream(stream));
        return ABFTLP_OK;
    });
}

abftlp_status abftlp_gemm_checked(const uint8_t* d_a, uint64_t m, uint64_t lda, const abftlp_gemm_weight* w,
                                  int32_t* d_c, uint64_t ldc, int32_t* d_csum, uint64_t csum_ld,
                                  uint8_t* d_row_flags, uint32_t* d_err_count, const abftlp_fault* fault,
                                  abftlp_stream stream) {
    if (!w) return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        abftk::Fault f;
        if (fault && fault->active) {
            f.active = true;
            f.row = static_cast<int64_t>(fault->row);
            f.col = static_cast<int64_t>(fault->col);
            f.bit = fault->bit;
        }
        abftk::gemm(d_a, static_cast<int64_t>(m), static_cast<int64_t>(lda), *w->w, d_c, static_cast<int64_t>(ldc),
                    true, d_csum, static_cast<int64_t>(csum_ld), d_row_flags, d_err_count, &f, as_stream(stream));
        return ABFTLP_OK;
    });
}

static abftk::RequantDev to_dev(const abftlp_requant_params* p) {
    abftk::RequantDev q{};
    q.sA = p->scaleA;
    q.bA = p->biasA;
    q.sB = p->scaleB;
    q.bB = p->biasB;
    q.sC = p->scaleC;
    q.bC = p->biasC;
    q.k = static_cast<double>(p->k);
    return q;
}

abftlp_status abftlp_gemm_checked_requant(const uint8_t* d_a, uint64_t m, uint64_t lda, const abftlp_gemm_weight* w,
                                          int32_t* d_c, uint64_t ldc, int32_t* d_csum, uint64_t csum_ld,
                                          uint8_t* d_row_flags, uint32_t* d_err_count, const abftlp_fault* fault,
                                          const int32_t* d_row_sum_a, const int32_t* d_col_sum_b,
                                          const abftlp_requant_params* params, uint8_t* d_out, uint64_t ld_out,
                                          abftlp_stream stream) {
    if (!w || !params) return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        abftk::Fault f;
        if (fault && fault->active) {
            f.active = true;
            f.row = static_cast<int64_t>(fault->row);
            f.col = static_cast<int64_t>(fault->col);
            f.bit = fault->bit;
        }
        abftk::RequantArgs rq;
        rq.row_sum_a = d_row_sum_a;
        rq.col_sum_b = d_col_sum_b;
        rq.params = to_dev(params);
        rq.out = d_out;
        rq.ld_out = static_cast<int64_t>(ld_out);
        abftk::gemm(d_a, static_cast<int64_t>(m), static_cast<int64_t>(lda), *w->w, d_c, static_cast<int64_t>(ldc),
                    true, d_csum, static_cast<int64_t>(csum_ld), d_row_flags, d_err_count, &f, as_stream(stream),
                    nullptr, &rq);
        return ABFTLP_OK;
    });
}

abftlp_status abftlp_requantize(const int32_t* d_c, uint64_t ldc, uint64_t m, uint64_t n, const int32_t* d_row_sum_a,
                                const int32_t* d_col_sum_b, const abftlp_requant_params* params, uint8_t* d_out,
                                uint64_t ld_out, abftlp_stream stream) {
    if (!params) return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        abftk::requantize(d_c, static_cast<int64_t>(ldc), static_cast<int64_t>(m), static_cast<int64_t>(n), d_row_sum_a,
                          d_col_sum_b, to_dev(params), d_out, static_cast<int64_t>(ld_out), as_stream(stream));
        return ABFTLP_OK;
    });
}

abftlp_status abftlp_row_sums_u8(const uint8_t* d_a, uint64_t m, uint64_t k, uint64_t lda, int32_t* d_out,
                                 abftlp_stream stream) {
    return guarded([&] {
        abftk::row_sums_u8(d_a, static_cast<int64_t>(m), static_cast<int64_t>(k), static_cast<int64_t>(lda), d_out,
                           as_stream(stream));
        return ABFTLP_OK;
    });
}

abftlp_status abftlp_gemm_weight_col_sums(const abftlp_gemm_weight* w, int32_t* d_out, abftlp_stream stream) {
    if (!w) return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        if (w->w->batch != 1) throw std::invalid_argument("batched weight: operation needs a single weight");
        abftk::weight_col_sums(*w->w, d_out, as_stream(stream));
        return ABFTLP_OK;
    });
}

abftlp_status abftlp_gemm_checked_batched(const uint8_t* d_a, uint64_t batch, uint64_t m, uint64_t lda,
                                          uint64_t stride_a, const abftlp_gemm_weight* w, int32_t* d_c, uint64_t ldc,
                                          uint64_t stride_c, int32_t* d_csum, uint64_t csum_ld, uint64_t stride_csum,
                                          uint8_t* d_row_flags, uint64_t stride_flags, uint32_t* d_err_count,
                                          const abftlp_batch_fault* fault, abftlp_stream stream) {
    if (!w) return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        abftk::Fault f;
        abftk::GemmBatch bt;
        bt.batch = static_cast<int64_t>(batch);
        bt.a_bstride = static_cast<int64_t>(stride_a);
        bt.c_bstride = static_cast<int64_t>(stride_c);
        bt.csum_bstride = static_cast<int64_t>(stride_csum);
        bt.flags_bstride = static_cast<int64_t>(stride_flags);
        if (fault && fault->active) {
            f.active = true;
            f.row = static_cast<int64_t>(fault->row);
            f.col = static_cast<int64_t>(fault->col);
            f.bit = fault->bit;
            bt.fault_batch = static_cast<int64_t>(fault->batch);
        }
        abftk::gemm(d_a, static_cast<int64_t>(m), static_cast<int64_t>(lda), *w->w, d_c, static_cast<int64_t>(ldc),
                    true, d_csum, static_cast<int64_t>(csum_ld), d_row_flags, d_err_count, &f, as_stream(stream),
                    nullptr, nullptr, &bt);
        return ABFTLP_OK;
    });
}

abftlp_status abftlp_gemm_checked_batched_faults(const uint8_t* d_a, uint64_t batch, uint64_t m, uint64_t lda,
                                                 uint64_t stride_a, const abftlp_gemm_weight* w, int32_t* d_c,
                                                 uint64_t ldc, uint64_t stride_c, int32_t* d_csum, uint64_t csum_ld,
                                                 uint64_t stride_csum, uint8_t* d_row_flags, uint64_t stride_flags,
                                                 uint32_t* d_err_count, const abftlp_batch_fault* faults,
                                                 uint64_t nfaults, abftlp_stream stream) {
    if (!w || (nfaults && !faults)) return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        abftk::BatchFault fl[abftk::kMaxGemmFaults];
        int64_t nf = 0;
        for (uint64_t i = 0; i < nfaults; ++i) {
            if (!faults[i].active) continue;
            if (nf == abftk::kMaxGemmFaults) throw std::invalid_argument("abft_gemm: too many faults for one call");
            fl[nf++] = abftk::BatchFault{static_cast<int64_t>(faults[i].batch), static_cast<int64_t>(faults[i].row),
                                         static_cast<int64_t>(faults[i].col), faults[i].bit};
        }
        abftk::GemmBatch bt;
        bt.batch = static_cast<int64_t>(batch);
        bt.a_bstride = static_cast<int64_t>(stride_a);
        bt.c_bstride = static_cast<int64_t>(stride_c);
        bt.csum_bstride = static_cast<int64_t>(stride_csum);
        bt.flags_bstride = static_cast<int64_t>(stride_flags);
        bt.faults = fl;
        bt.nfaults = nf;
        abftk::gemm(d_a, static_cast<int64_t>(m), static_cast<int64_t>(lda), *w->w, d_c, static_cast<int64_t>(ldc),
                    true, d_csum, static_cast<int64_t>(csum_ld), d_row_flags, d_err_count, nullptr, as_stream(stream),
                    nullptr, nullptr, &bt);
        return ABFTLP_OK;
    });
}

abftlp_status abftlp_gemm_unchecked_batched(const uint8_t* d_a, uint64_t batch, uint64_t m, uint64_t lda,
                                            uint64_t stride_a, const abftlp_gemm_weight* w, int32_t* d_c, uint64_t ldc,
                                            uint64_t stride_c, abftlp_stream stream) {
    if (!w) return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        abftk::GemmBatch bt;
        bt.batch = static_cast<int64_t>(batch);
        bt.a_bstride = static_cast<int64_t>(stride_a);
        bt.c_bstride = static_cast<int64_t>(stride_c);
        abftk::gemm(d_a, static_cast<int64_t>(m), static_cast<int64_t>(lda), *w->w, d_c, static_cast<int64_t>(ldc),
                    false, nullptr, 0, nullptr, nullptr, nullptr, as_stream(stream), nullptr, nullptr, &bt);
        return ABFTLP_OK;
    });
}

abftlp_status abftlp_gemm_unchecked(const uint8_t* d_a, uint64_t m, uint64_t lda, const abftlp_gemm_weight* w,
                                    int32_t* d_c, uint64_t ldc, abftlp_stream stream) {
    if (!w) return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        abftk::gemm(d_a, static_cast<int64_t>(m), static_cast<int64_t>(lda), *w->w, d_c, static_cast<int64_t>(ldc),
                    false, nullptr, 0, nullptr, nullptr, nullptr, as_stream(stream));
        return ABFTLP_OK;
    });
}

abftlp_status abftlp_gemm_verify(const int32_t* d_c, uint64_t ldc, const int32_t* d_csum, uint64_t csum_ld, uint64_t m,
                                 uint64_t n, uint8_t* d_row_flags, uint32_t* d_err_count, abftlp_stream stream) {
    return guarded([&] {
        abftk::verify(d_c, static_cast<int64_t>(ldc), d_csum, static_cast<int64_t>(csum_ld), static_cast<int64_t>(m),
                      static_cast<int64_t>(n), d_row_flags, d_err_count, as_stream(stream));
        return ABFTLP_OK;
    });
}

abftlp_status abftlp_gemm_checked_host(const uint8_t* a, uint64_t m, uint64_t lda, const abftlp_gemm_weight* w,
                                       int32_t* c, uint64_t ldc, int32_t* csum, uint8_t* row_flags,
                                       uint32_t* err_count, abftlp_stream stream) {
    if (!w || (m && !a)) return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        const abftk::GemmWeight& W = *w->w;
        if (lda < static_cast<uint64_t>(W.k)) throw std::invalid_argument("abft_gemm: dimension mismatch (lda < k)");
        if (c && ldc < static_cast<uint64_t>(W.n)) throw std::invalid_argument("abft_gemm: ldc < n");
        cudaStream_t st = as_stream(stream);
        int dev = 0;
        ABFT_CUDA(cudaGetDevice(&dev));
        const uint64_t key = (reinterpret_cast<uint64_t>(st) << 8) ^ static_cast<uint64_t>(dev);
        std::lock_guard<std::mutex> g(g_stage_mu);
        HostStage& s = g_stage[key];
        const size_t n = static_cast<size_t>(W.n), k = static_cast<size_t>(W.k);
        const size_t dldc = (n + 3) / 4 * 4;
        ensure(s.a, s.a_cap, m * ((k + 15) / 16 * 16));
        ensure(s.c, s.c_cap, m * dldc);
        ensure(s.csum, s.csum_cap, m);
        ensure(s.flags, s.flags_cap, m);
        if (!s.err) ABFT_CUDA(cudaMalloc(&s.err, sizeof(uint32_t)));
        const size_t dlda = (k + 15) / 16 * 16;
        ABFT_CUDA(cudaMemcpy2DAsync(s.a, dlda, a, lda, k, m, cudaMemcpyHostToDevice, st));
        abftk::gemm(s.a, static_cast<int64_t>(m), static_cast<int64_t>(dlda), W, s.c, static_cast<int64_t>(dldc), true,
                    s.csum, 1, s.flags, s.err, nullptr, st);
        if (c) ABFT_CUDA(cudaMemcpy2DAsync(c, ldc * 4, s.c, dldc * 4, n * 4, m, cudaMemcpyDeviceToHost, st));
        if (csum) ABFT_CUDA(cudaMemcpyAsync(csum, s.csum, m * 4, cudaMemcpyDeviceToHost, st));
        if (row_flags) ABFT_CUDA(cudaMemcpyAsync(row_flags, s.flags, m, cudaMemcpyDeviceToHost, st));
        if (err_count) ABFT_CUDA(cudaMemcpyAsync(err_count, s.err, 4, cudaMemcpyDeviceToHost, st));
        ABFT_CUDA(cudaStreamSynchronize(st));
        return ABFTLP_OK;
    });
}

abftlp_status abftlp_gemm_checked_host_batched(const uint8_t* a, uint64_t batch, uint64_t m, uint64_t lda,
                                               uint64_t stride_a, const abftlp_gemm_weight* w, int32_t* c,
                                               uint64_t ldc, uint64_t stride_c, int32_t* csum,
                                               uint64_t stride_csum, uint8_t* row_flags, uint64_t stride_flags,
                                               uint32_t* err_count, abftlp_stream stream) {
    if (!w || (batch && m && (!a || !c || !csum || !row_flags || !err_count)))
        return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        const abftk::GemmWeight& W = *w->w;
        if (W.batch != 1) throw std::invalid_argument("batched weight: operation needs a single weight");
        const size_t n = static_cast<size_t>(W.n), k = static_cast<size_t>(W.k);
        if (lda < k) throw std::invalid_argument("abft_gemm: dimension mismatch (lda < k)");
        if (ldc < n) throw std::invalid_argument("abft_gemm: ldc < n");
        if (batch > 1 && (stride_a < lda * (m - 1) + k || stride_c < ldc * m || stride_csum < m || stride_flags < m))
            throw std::invalid_argument("abft_gemm: batch strides overlap");
        if (batch == 0 || m == 0) {
            for (uint64_t b = 0; b < batch; ++b) err_count[b] = 0;
            return ABFTLP_OK;
        }
        cudaStream_t st = as_stream(stream);
        int dev = 0;
        ABFT_CUDA(cudaGetDevice(&dev));
        const uint64_t key = (reinterpret_cast<uint64_t>(st) << 8) ^ static_cast<uint64_t>(dev);
        std::lock_guard<std::mutex> g(g_stage_mu);
        HostStage& s = g_stage[key];
        if (!s.h2d) {
            ABFT_CUDA(cudaStreamCreateWithFlags(&s.h2d, cudaStreamNonBlocking));
            ABFT_CUDA(cudaStreamCreateWithFlags(&s.d2h, cudaStreamNonBlocking));
            for (int i = 0; i < 3; ++i) {
                ABFT_CUDA(cudaEventCreateWithFlags(&s.a_ready[i], cudaEventDisableTiming));
                ABFT_CUDA(cudaEventCreateWithFlags(&s.c_done[i], cudaEventDisableTiming));
                ABFT_CUDA(cudaEventCreateWithFlags(&s.out_done[i], cudaEventDisableTiming));
            }
        }
        // chunk = runs per grouped launch: ~32 MB of C' per chunk, three slots in flight
        const size_t dlda = (k + 15) / 16 * 16, dldc = (n + 3) / 4 * 4;
        const size_t per_c = m * dldc * 4;
        const uint64_t q = std::max<uint64_t>(1, std::min<uint64_t>(batch, (32u << 20) / std::max<size_t>(per_c, 1)));
        ensure(s.ja, s.ja_cap, 3 * q * m * dlda);
        ensure(s.jc, s.jc_cap, 3 * q * m * dldc);
        ensure(s.jcs, s.jcs_cap, 3 * q * m);
        ensure(s.jfl, s.jfl_cap, 3 * q * m);
        ensure(s.jerr, s.jerr_cap, 3 * q);
        // the caller's stream may have pending work the job depends on (e.g. the weight encode)
        ABFT_CUDA(cudaEventRecord(s.c_done[0], st));
        ABFT_CUDA(cudaStreamWaitEvent(s.h2d, s.c_done[0], 0));
        const uint64_t chunks = (batch + q - 1) / q;
        // if anything below throws, copies already queued still reference the caller's host buffers: drain the
        // three streams before the error reaches the caller
        struct Drain {
            cudaStream_t a, b, c;
            bool armed = true;
            ~Drain() {
                if (!armed) return;
                cudaStreamSynchronize(a);
                cudaStreamSynchronize(b);
                cudaStreamSynchronize(c);
            }
        } drain{s.h2d, st, s.d2h};
        for (uint64_t i = 0; i < chunks; ++i) {
            const int sl = static_cast<int>(i % 3);
            const uint64_t b0 = i * q, nb = std::min<uint64_t>(q, batch - b0);
            uint8_t* da = s.ja + sl * q * m * dlda;
            int32_t* dc = s.jc + sl * q * m * dldc;
            int32_t* dcs = s.jcs + sl * q * m;
            uint8_t* dfl = s.jfl + sl * q * m;
            uint32_t* derr = s.jerr + sl * q;
            if (i >= 3) ABFT_CUDA(cudaStreamWaitEvent(s.h2d, s.c_done[sl], 0));  // slot's A no longer read
            for (uint64_t b = 0; b < nb; ++b)
                ABFT_CUDA(cudaMemcpy2DAsync(da + b * m * dlda, dlda, a + (b0 + b) * stride_a, lda, k, m,
                                            cudaMemcpyHostToDevice, s.h2d));
            ABFT_CUDA(cudaEventRecord(s.a_ready[sl], s.h2d));
            ABFT_CUDA(cudaStreamWaitEvent(st, s.a_ready[sl], 0));
            if (i >= 3) ABFT_CUDA(cudaStreamWaitEvent(st, s.out_done[sl], 0));  // slot's C' copied out
            abftk::GemmBatch bt;
            bt.batch = static_cast<int64_t>(nb);
            bt.a_bstride = static_cast<int64_t>(m * dlda);
            bt.c_bstride = static_cast<int64_t>(m * dldc);
            bt.csum_bstride = static_cast<int64_t>(m);
            bt.flags_bstride = static_cast<int64_t>(m);
            abftk::gemm(da, static_cast<int64_t>(m), static_cast<int64_t>(dlda), W, dc, static_cast<int64_t>(dldc),
                        true, dcs, 1, dfl, derr, nullptr, st, nullptr, nullptr, nb > 1 ? &bt : nullptr);
            ABFT_CUDA(cudaEventRecord(s.c_done[sl], st));
            ABFT_CUDA(cudaStreamWaitEvent(s.d2h, s.c_done[sl], 0));
            if (stride_c == ldc * m && ldc == dldc) {
                ABFT_CUDA(cudaMemcpyAsync(c + b0 * stride_c, dc, nb * m * dldc * 4, cudaMemcpyDeviceToHost, s.d2h));
            } else if (stride_c == ldc * m) {
                ABFT_CUDA(cudaMemcpy2DAsync(c + b0 * stride_c, ldc * 4, dc, dldc * 4, n * 4, nb * m,
                                            cudaMemcpyDeviceToHost, s.d2h));
            } else {
                for (uint64_t b = 0; b < nb; ++b)
                    ABFT_CUDA(cudaMemcpy2DAsync(c + (b0 + b) * stride_c, ldc * 4, dc + b * m * dldc, dldc * 4, n * 4, m,
                                                cudaMemcpyDeviceToHost, s.d2h));
            }
            if (stride_csum == m && stride_flags == m) {
                ABFT_CUDA(cudaMemcpyAsync(csum + b0 * m, dcs, nb * m * 4, cudaMemcpyDeviceToHost, s.d2h));
                ABFT_CUDA(cudaMemcpyAsync(row_flags + b0 * m, dfl, nb * m, cudaMemcpyDeviceToHost, s.d2h));
            } else {
                for (uint64_t b = 0; b < nb; ++b) {
                    ABFT_CUDA(cudaMemcpyAsync(csum + (b0 + b) * stride_csum, dcs + b * m, m * 4, cudaMemcpyDeviceToHost,
                                              s.d2h));
                    ABFT_CUDA(cudaMemcpyAsync(row_flags + (b0 + b) * stride_flags, dfl + b * m, m,
                                              cudaMemcpyDeviceToHost, s.d2h));
                }
            }
            ABFT_CUDA(cudaMemcpyAsync(err_count + b0, derr, nb * 4, cudaMemcpyDeviceToHost, s.d2h));
            ABFT_CUDA(cudaEventRecord(s.out_done[sl], s.d2h));
        }
        drain.armed = false;
        ABFT_CUDA(cudaStreamSynchronize(s.d2h));
        ABFT_CUDA(cudaStreamSynchronize(st));
        return ABFTLP_OK;
    });
}

abftlp_status abftlp_gemm_checked_requant_host_batched(const uint8_t* a, uint64_t batch, uint64_t m, uint64_t lda,
                                                       uint64_t stride_a, const abftlp_gemm_weight* w,
                                                       const abftlp_requant_params* params, uint8_t* out,
                                                       uint64_t ld_out, uint64_t stride_out, int32_t* csum,
                                                       uint64_t stride_csum, uint8_t* row_flags,
                                                       uint64_t stride_flags, uint32_t* err_count,
                                                       abftlp_stream stream) {
    if (!w || !params || (batch && m && (!a || !out || !csum || !row_flags || !err_count)))
        return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        const abftk::GemmWeight& W = *w->w;
        if (W.batch != 1) throw std::invalid_argument("batched weight: operation needs a single weight");
        const size_t n = static_cast<size_t>(W.n), k = static_cast<size_t>(W.k);
        const abftk::RequantDev rqp = to_dev(params);
        abftk::check_requant_params(rqp);
        if (lda < k) throw std::invalid_argument("abft_gemm: dimension mismatch (lda < k)");
        if (ld_out < n) throw std::invalid_argument("requantize: ld_out < n");
        if (batch > 1 && (stride_a < lda * (m - 1) + k || stride_out < ld_out * (m - 1) + n || stride_csum < m ||
                          stride_flags < m))
            throw std::invalid_argument("abft_gemm: batch strides overlap");
        if (batch == 0 || m == 0) {
            for (uint64_t b = 0; b < batch; ++b) err_count[b] = 0;
            return ABFTLP_OK;
        }
        cudaStream_t st = as_stream(stream);
        int dev = 0;
        ABFT_CUDA(cudaGetDevice(&dev));
        const uint64_t key = (reinterpret_cast<uint64_t>(st) << 8) ^ static_cast<uint64_t>(dev);
        std::lock_guard<std::mutex> g(g_stage_mu);
        HostStage& s = g_stage[key];
        if (!s.h2d) {
            ABFT_CUDA(cudaStreamCreateWithFlags(&s.h2d, cudaStreamNonBlocking));
            ABFT_CUDA(cudaStreamCreateWithFlags(&s.d2h, cudaStreamNonBlocking));
            for (int i = 0; i < 3; ++i) {
                ABFT_CUDA(cudaEventCreateWithFlags(&s.a_ready[i], cudaEventDisableTiming));
                ABFT_CUDA(cudaEventCreateWithFlags(&s.c_done[i], cudaEventDisableTiming));
                ABFT_CUDA(cudaEventCreateWithFlags(&s.out_done[i], cudaEventDisableTiming));
            }
        }
        // chunk = runs per row-stacked launch: ~16 MB of A per chunk (and as much u8 output; the copies, not the launches, bound the job), three slots in flight
        const size_t dlda = (k + 15) / 16 * 16, dldo = (n + 15) / 16 * 16;
        const size_t per_run = m * std::max(dlda, dldo);
        static const size_t chunk_bytes = [] {
            const char* e = std::getenv("ABFTLP_HOST_CHUNK_MB");  // tuning: bytes of A per chunk
            const long v = e ? std::atol(e) : 0;
            return static_cast<size_t>(v > 0 && v <= 1024 ? v : 16) << 20;  // (measured: 2 / 4 / 8 / 16 / 32 MB -> 201 / 234 / 281 / 300 / 291 TOPS on the G2 job)
        }();
        uint64_t q = std::max<uint64_t>(1, std::min<uint64_t>(batch, chunk_bytes / std::max<size_t>(per_run, 1)));
        while (q > 1 && q * m >= (uint64_t{1} << 31)) q /= 2;  // rows of one stacked launch
        ensure(s.ja, s.ja_cap, 3 * q * m * dlda);
        ensure(s.jo, s.jo_cap, 3 * q * m * dldo);
        ensure(s.jrs, s.jrs_cap, 3 * q * m);
        ensure(s.jcs, s.jcs_cap, 3 * q * m);
        ensure(s.jfl, s.jfl_cap, 3 * q * m);
        ensure(s.jerr, s.jerr_cap, 3 * q);
        ensure(s.jcol, s.jcol_cap, n);
        abftk::weight_col_sums(W, s.jcol, st);
        ABFT_CUDA(cudaEventRecord(s.c_done[0], st));
        ABFT_CUDA(cudaStreamWaitEvent(s.h2d, s.c_done[0], 0));
        const uint64_t chunks = (batch + q - 1) / q;
        struct Drain {
            cudaStream_t a, b, c;
            bool armed = true;
            ~Drain() {
                if (!armed) return;
                cudaStreamSynchronize(a);
                cudaStreamSynchronize(b);
                cudaStreamSynchronize(c);
            }
        } drain{s.h2d, st, s.d2h};
        for (uint64_t i = 0; i < chunks; ++i) {
            const int sl = static_cast<int>(i % 3);
            const uint64_t b0 = i * q, nb = std::min<uint64_t>(q, batch - b0);
            uint8_t* da = s.ja + sl * q * m * dlda;
            uint8_t* dout = s.jo + sl * q * m * dldo;
            int32_t* drs = s.jrs + sl * q * m;
            int32_t* dcs = s.jcs + sl * q * m;
            uint8_t* dfl = s.jfl + sl * q * m;
            uint32_t* derr = s.jerr + sl * q;
            if (i >= 3) ABFT_CUDA(cudaStreamWaitEvent(s.h2d, s.c_done[sl], 0));  // slot's A no longer read
            if (stride_a == lda * m && lda == dlda) {
                ABFT_CUDA(cudaMemcpyAsync(da, a + b0 * stride_a, nb * m * dlda, cudaMemcpyHostToDevice, s.h2d));
            } else {
                for (uint64_t b = 0; b < nb; ++b)
                    ABFT_CUDA(cudaMemcpy2DAsync(da + b * m * dlda, dlda, a + (b0 + b) * stride_a, lda, k, m,
                                                cudaMemcpyHostToDevice, s.h2d));
            }
            ABFT_CUDA(cudaEventRecord(s.a_ready[sl], s.h2d));
            ABFT_CUDA(cudaStreamWaitEvent(st, s.a_ready[sl], 0));
            if (i >= 3) ABFT_CUDA(cudaStreamWaitEvent(st, s.out_done[sl], 0));  // slot's outputs copied out
            // the chunk's runs as the row blocks of one tall GEMM (row checks and requantization are per row)
            const int64_t rows = static_cast<int64_t>(nb * m);
            abftk::row_sums_u8(da, rows, static_cast<int64_t>(k), static_cast<int64_t>(dlda), drs, st);
            abftk::RequantArgs rq;
            rq.row_sum_a = drs;
            rq.col_sum_b = s.jcol;
            rq.params = rqp;
            rq.out = dout;
            rq.ld_out = static_cast<int64_t>(dldo);
            abftk::GemmBatch tall;
            tall.stack_rows = static_cast<int64_t>(m);  // one flag count per run
            abftk::gemm(da, rows, static_cast<int64_t>(dlda), W, nullptr, static_cast<int64_t>(n), true, dcs, 1, dfl, derr, nullptr, st,
                        nullptr, &rq, nb > 1 ? &tall : nullptr);
            ABFT_CUDA(cudaEventRecord(s.c_done[sl], st));
            ABFT_CUDA(cudaStreamWaitEvent(s.d2h, s.c_done[sl], 0));
            if (stride_out == ld_out * m && ld_out == dldo) {
                ABFT_CUDA(cudaMemcpyAsync(out + b0 * stride_out, dout, nb * m * dldo, cudaMemcpyDeviceToHost, s.d2h));
            } else {
                for (uint64_t b = 0; b < nb; ++b)
                    ABFT_CUDA(cudaMemcpy2DAsync(out + (b0 + b) * stride_out, ld_out, dout + b * m * dldo, dldo, n, m,
                                                cudaMemcpyDeviceToHost, s.d2h));
            }
            if (stride_csum == m && stride_flags == m) {
                ABFT_CUDA(cudaMemcpyAsync(csum + b0 * m, dcs, nb * m * 4, cudaMemcpyDeviceToHost, s.d2h));
                ABFT_CUDA(cudaMemcpyAsync(row_flags + b0 * m, dfl, nb * m, cudaMemcpyDeviceToHost, s.d2h));
            } else {
                for (uint64_t b = 0; b < nb; ++b) {
                    ABFT_CUDA(cudaMemcpyAsync(csum + (b0 + b) * stride_csum, dcs + b * m, m * 4, cudaMemcpyDeviceToHost,
                                              s.d2h));
                    ABFT_CUDA(cudaMemcpyAsync(row_flags + (b0 + b) * stride_flags, dfl + b * m, m,
                                              cudaMemcpyDeviceToHost, s.d2h));
                }
            }
            ABFT_CUDA(cudaMemcpyAsync(err_count + b0, derr, nb * 4, cudaMemcpyDeviceToHost, s.d2h));
            ABFT_CUDA(cudaEventRecord(s.out_done[sl], s.d2h));
        }
        drain.armed = false;
        ABFT_CUDA(cudaStreamSynchronize(s.d2h));
        ABFT_CUDA(cudaStreamSynchronize(st));
        return ABFTLP_OK;
    });
}

// ============================================================ device operators: EmbeddingBag
abftlp_status abftlp_eb_table_create(int32_t elem_type, const void* d_rows, uint64_t rows, uint64_t dim,
                                     uint64_t row_stride_bytes, int32_t scale_type, const void* d_scales,
                                     const void* d_biases, const int32_t* d_row_sums, abftlp_stream stream,
                                     abftlp_eb_table** out) {
    if (!out) return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        abftk::EbTable* t = abftk::eb_table_create(elem_type, d_rows, static_cast<int64_t>(rows),
                                                   static_cast<int64_t>(dim), static_cast<int64_t>(row_stride_bytes),
                                                   scale_type, d_scales, d_biases, d_row_sums, as_stream(stream));
        *out = new abftlp_eb_table_s{t};
        return ABFTLP_OK;
    });
}

void abftlp_eb_table_free(abftlp_eb_table* t) {
    if (!t) return;
    abftk::eb_table_free(t->t);
    delete t;
}

abftlp_status abftlp_eb_table_validate(const abftlp_eb_table* t, const int32_t* d_row_sums, abftlp_stream stream,
                                       uint64_t* mismatched_rows) {
    if (!t || !d_row_sums || !mismatched_rows) return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        *mismatched_rows = abftk::eb_table_validate(*t->t, d_row_sums, as_stream(stream));
        return ABFTLP_OK;
    });
}

abftlp_status abftlp_eb_table_row_sums(const abftlp_eb_table* t, int32_t* d_out, abftlp_stream stream) {
    if (!t || !d_out) return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        abftk::eb_row_sums(*t->t, d_out, as_stream(stream));
        return ABFTLP_OK;
    });
}

abftlp_status abftlp_eb_checked(const abftlp_eb_table* t, const int64_t* d_offsets, const int64_t* d_indices,
                                uint64_t num_bags, const float* d_weights, float* d_out, uint64_t ld_out,
                                uint8_t* d_flags, double* d_rsum, double* d_csum, uint32_t* d_flag_count,
                                int32_t* d_status, abftlp_stream stream) {
    if (!t) return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        if (num_bags && !d_flags) throw std::invalid_argument("null argument");
        abftk::eb_run(*t->t, d_offsets, d_indices, static_cast<int64_t>(num_bags), d_weights, d_out,
                      static_cast<int64_t>(ld_out), true, d_flags, d_rsum, d_csum, d_flag_count, d_status,
                      as_stream(stream));
        return ABFTLP_OK;
    });
}

abftlp_status abftlp_eb_unchecked(const abftlp_eb_table* t, const int64_t* d_offsets, const int64_t* d_indices,
                                  uint64_t num_bags, const float* d_weights, float* d_out, uint64_t ld_out,
                                  int32_t* d_status, abftlp_stream stream) {
    if (!t) return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        abftk::eb_run(*t->t, d_offsets, d_indices, static_cast<int64_t>(num_bags), d_weights, d_out,
                      static_cast<int64_t>(ld_out), false, nullptr, nullptr, nullptr, nullptr, d_status,
                      as_stream(stream));
        return ABFTLP_OK;
    });
}

abftlp_status abftlp_eb_checked_scatter(const abftlp_eb_table* t, const int64_t* d_offsets, const int64_t* d_indices,
                                        uint64_t num_bags, const float* d_weights, float* const* d_out_dest,
                                        uint64_t ld_out, uint8_t* const* d_flag_dest, uint64_t flag_ld,
                                        uint64_t bags_per_dest, uint32_t* d_flag_count, int32_t* d_status,
                                        abftlp_stream stream) {
    if (!t || !d_out_dest || !d_flag_dest) return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        abftk::EbScatter sc;
        sc.out_dest = d_out_dest;
        sc.flag_dest = d_flag_dest;
        sc.bags_per_dest = static_cast<int64_t>(bags_per_dest);
        sc.flag_ld = static_cast<int64_t>(flag_ld);
        abftk::eb_run(*t->t, d_offsets, d_indices, static_cast<int64_t>(num_bags), d_weights, nullptr,
                      static_cast<int64_t>(ld_out), true, nullptr, nullptr, nullptr, d_flag_count, d_status,
                      as_stream(stream), &sc);
        return ABFTLP_OK;
    });
}

abftlp_status abftlp_eb_group_create(const abftlp_eb_table* const* tables, uint32_t ntables,
                                     const int64_t* const* d_offsets, const int64_t* const* d_indices,
                                     const float* const* d_weights, float* const* const* d_out_dest,
                                     uint8_t* const* const* d_flag_dest, abftlp_eb_group** out) {
    if (!out || !tables || ntables == 0) return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        std::vector<const abftk::EbTable*> ts(ntables);
        for (uint32_t i = 0; i < ntables; ++i) {
            if (!tables[i]) throw std::invalid_argument("null argument");
            ts[i] = tables[i]->t;
        }
        *out = new abftlp_eb_group_s{abftk::eb_group_create(ts.data(), ntables, d_offsets, d_indices, d_weights,
                                                            d_out_dest, d_flag_dest)};
        return ABFTLP_OK;
    });
}

void abftlp_eb_group_free(abftlp_eb_group* g) {
    if (!g) return;
    abftk::eb_group_free(g->g);
    delete g;
}

abftlp_status abftlp_eb_group_set_bags(abftlp_eb_group* g, const int64_t* const* d_offsets,
                                       const int64_t* const* d_indices, const float* const* d_weights,
                                       abftlp_stream stream) {
    if (!g || !d_offsets || !d_indices) return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        abftk::eb_group_set_bags(*g->g, d_offsets, d_indices, d_weights, as_stream(stream));
        return ABFTLP_OK;
    });
}

abftlp_status abftlp_eb_group_unchecked_scatter(const abftlp_eb_group* g, uint64_t bags_per_table, uint64_t ld_out,
                                                uint64_t bags_per_dest, int32_t* d_status, abftlp_stream stream) {
    if (!g) return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        abftk::eb_group_run(*g->g, static_cast<int64_t>(bags_per_table), static_cast<int64_t>(ld_out), 1,
                            static_cast<int64_t>(bags_per_dest), false, nullptr, d_status, as_stream(stream));
        return ABFTLP_OK;
    });
}

abftlp_status abftlp_eb_group_checked_scatter(const abftlp_eb_group* g, uint64_t bags_per_table, uint64_t ld_out,
                                              uint64_t flag_ld, uint64_t bags_per_dest, uint32_t* d_flag_count,
                                              int32_t* d_status, abftlp_stream stream) {
    if (!g) return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        abftk::eb_group_run(*g->g, static_cast<int64_t>(bags_per_table), static_cast<int64_t>(ld_out),
                            static_cast<int64_t>(flag_ld), static_cast<int64_t>(bags_per_dest), true, d_flag_count,
                            d_status, as_stream(stream));
        return ABFTLP_OK;
    });
}

// ============================================================ dual-encoded locate / correct
abftlp_status abftlp_gemm_locate(const uint8_t* d_a, uint64_t m, uint64_t lda, const abftlp_gemm_weight* w, int32_t* d_c,
                                 uint64_t ldc, int32_t* d_csum, uint64_t csum_ld, uint8_t* d_row_flags, int correct,
                                 abftlp_locate_result* out, abftlp_stream stream) {
    if (!w || !out) return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        const abftk::LocateResult r =
            abftk::gemm_locate(d_a, static_cast<int64_t>(m), static_cast<int64_t>(lda), *w->w, d_c, static_cast<int64_t>(ldc),
                               d_csum, static_cast<int64_t>(csum_ld), d_row_flags, correct != 0, as_stream(stream));
        out->status = r.status;
        out->row = r.row;
        out->col = r.col;
        out->delta = r.delta;
        out->rows_flagged = static_cast<uint64_t>(r.rows_flagged);
        out->cols_mismatched = static_cast<uint64_t>(r.cols_mismatched);
        return ABFTLP_OK;
    });
}

// ============================================================ heterogeneous grouped GEMM
abftlp_status abftlp_gemm_group_create(const abftlp_gemm_problem* problems, uint32_t count, int checked,
                                       abftlp_gemm_group** out) {
    if (!problems || !out || count == 0) return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        std::vector<abftk::GemmProblem> ps(count);
        for (uint32_t i = 0; i < count; ++i) {
            const abftlp_gemm_problem& q = problems[i];
            if (!q.w) throw std::invalid_argument("null argument");
            ps[i].a = q.d_a;
            ps[i].m = static_cast<int64_t>(q.m);
            ps[i].lda = static_cast<int64_t>(q.lda);
            ps[i].w = q.w->w;
            ps[i].c = q.d_c;
            ps[i].ldc = static_cast<int64_t>(q.ldc);
            ps[i].csum = q.d_csum;
            ps[i].csum_ld = static_cast<int64_t>(q.csum_ld);
            ps[i].flags = q.d_row_flags;
            ps[i].err_count = q.d_err_count;
        }
        *out = new abftlp_gemm_group_s{abftk::gemm_group_create(ps.data(), static_cast<int>(count), checked != 0)};
        return ABFTLP_OK;
    });
}

abftlp_status abftlp_gemm_group_run(const abftlp_gemm_group* g, abftlp_stream stream) {
    if (!g) return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        abftk::gemm_group_run(*g->g, as_stream(stream));
        return ABFTLP_OK;
    });
}

void abftlp_gemm_group_free(abftlp_gemm_group* g) {
    if (!g) return;
    abftk::gemm_group_free(g->g);
    delete g;
}

// ============================================================ fault injection
abftlp_status abftlp_flip_bit(void* d_ptr, uint32_t elem_bytes, uint64_t index, uint32_t bit, abftlp_stream stream) {
    if (!d_ptr) return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        if (elem_bytes != 1 && elem_bytes != 2 && elem_bytes != 4 && elem_bytes != 8)
            throw std::invalid_argument("flip_bit: element width must be 1, 2, 4 or 8 bytes");
        if (bit >= elem_bytes * 8) throw std::out_of_range("flip_bit: bit index out of range");
        abftk::flip_bit(d_ptr, index * elem_bytes, bit, as_stream(stream));  // little-endian element
        return ABFTLP_OK;
    });
}

abftlp_status abftlp_gemm_weight_flip_bit(abftlp_gemm_weight* w, uint64_t i, uint64_t j, uint32_t bit,
                                          abftlp_stream stream) {
    if (!w) return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        if (w->w->batch != 1) throw std::invalid_argument("batched weight: operation needs a single weight");
        const abftk::GemmWeight& W = *w->w;
        if (i >= static_cast<uint64_t>(W.k) || j > static_cast<uint64_t>(W.n))
            throw std::out_of_range("inject_weight_B: coordinates out of range");
        if (bit >= 8) throw std::out_of_range("flip_bit: bit index out of range");
        abftk::flip_bit(W.element(static_cast<int64_t>(i), static_cast<int64_t>(j)), 0, bit, as_stream(stream));
        if (j == static_cast<uint64_t>(W.n) && W.n < W.n_pad)  // the checksum column also lives in B' column n
            abftk::flip_bit(W.bt + (static_cast<int64_t>(i) / abftk::kBK) * W.n_pad * abftk::kBK + W.n * abftk::kBK +
                                static_cast<int64_t>(i) % abftk::kBK,
                            0, bit, as_stream(stream));
        return ABFTLP_OK;
    });
}

abftlp_status abftlp_gemm_weight_flip_bit_batched(abftlp_gemm_weight* w, uint64_t problem, uint64_t i, uint64_t j,
                                                  uint32_t bit, abftlp_stream stream) {
    if (!w) return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        const abftk::GemmWeight& W = *w->w;
        if (problem >= static_cast<uint64_t>(W.batch) || i >= static_cast<uint64_t>(W.k) ||
            j > static_cast<uint64_t>(W.n))
            throw std::out_of_range("inject_weight_B: coordinates out of range");
        if (bit >= 8) throw std::out_of_range("flip_bit: bit index out of range");
        const int64_t pb = static_cast<int64_t>(problem);
        int8_t* e = W.element(static_cast<int64_t>(i), static_cast<int64_t>(j)) +
                    pb * (j == static_cast<uint64_t>(W.n) ? W.cs_bstride : W.bt_bstride);
        abftk::flip_bit(e, 0, bit, as_stream(stream));
        if (j == static_cast<uint64_t>(W.n) && W.n < W.n_pad)  // the checksum column also lives in B' column n
            abftk::flip_bit(W.bt + pb * W.bt_bstride + (static_cast<int64_t>(i) / abftk::kBK) * W.n_pad * abftk::kBK +
                                W.n * abftk::kBK + static_cast<int64_t>(i) % abftk::kBK,
                            0, bit, as_stream(stream));
        return ABFTLP_OK;
    });
}

abftlp_status abftlp_eb_table_flip_bit(abftlp_eb_table* t, uint64_t row, uint64_t col, uint32_t bit,
                                       abftlp_stream stream) {
    if (!t) return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        if (row > static_cast<uint64_t>(INT64_MAX) || col > static_cast<uint64_t>(INT64_MAX))
            throw std::out_of_range("inject_eb_table: coordinates out of range");
        abftk::eb_flip_bit(*t->t, static_cast<int64_t>(row), static_cast<int64_t>(col), bit, as_stream(stream));
        return ABFTLP_OK;
    });
}

abftlp_status abftlp_eb_table_flip_bits(abftlp_eb_table* t, const int64_t* d_rows, const int64_t* d_cols,
                                        const int32_t* d_bits, uint64_t count, int32_t* d_status,
                                        abftlp_stream stream) {
    if (!t) return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        abftk::eb_flip_bits(*t->t, d_rows, d_cols, d_bits, static_cast<int64_t>(count), d_status, as_stream(stream));
        return ABFTLP_OK;
    });
}

abftlp_status abftlp_generate(void* d_out, uint64_t count, uint64_t seed, uint64_t rng_stream, uint64_t off,
                              int32_t kind, double lo, double hi, uint64_t bound, abftlp_stream stream) {
    if (!d_out && count) return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        if (kind < 0 || kind > 3) throw std::invalid_argument("generate: unknown kind");
        if (kind == 3 && bound == 0) throw std::invalid_argument("generate: bound must be > 0");
        abftk::gen(d_out, static_cast<int64_t>(count), seed, rng_stream, off, kind, lo, hi, bound, as_stream(stream));
        return ABFTLP_OK;
    });
}

// Debug: record 8 globaltimer stamps per GEMM CTA into d_trace (NULL disables). Not in the headers.
__attribute__((visibility("default"))) void abftlp_debug_gemm_trace(unsigned long long* d_trace) {
    abftk::set_gemm_trace(d_trace);
}
// Debug: 16 globaltimer stamps per EmbeddingBag warp of the async kernel (NULL disables). Not in the headers.
__attribute__((visibility("default"))) void abftlp_debug_eb_trace(unsigned long long* d_trace) {
    abftk::set_eb_trace(d_trace);
}

abftlp_status abftlp_gather_probe(const void* d_table, uint64_t rec_bytes, const int64_t* d_idx, uint64_t n,
                                  uint32_t* d_sink, abftlp_stream stream) {
    if (!d_table || !d_sink || (n && !d_idx)) return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    if (rec_bytes == 0 || rec_bytes % 16 != 0 || rec_bytes > 512)
        return fail(ABFTLP_ERR_INVALID_ARGUMENT, "gather_probe: rec_bytes must be a multiple of 16 up to 512");
    return guarded([&] {
        ABFT_CUDA(abftk::launch_gather_probe(d_table, static_cast<int64_t>(rec_bytes), d_idx, static_cast<int64_t>(n),
                                             d_sink, as_stream(stream)));
        return ABFTLP_OK;
    });
}

abftlp_status abftlp_l2_flush(void* d_buf, uint64_t bytes, int32_t salt, abftlp_stream stream) {
    if (!d_buf) return fail(ABFTLP_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        abftk::l2_flush(d_buf, static_cast<int64_t>(bytes), salt, as_stream(stream));
        return ABFTLP_OK;
    });
}

}  // extern "C"
