// The reference's C++ API surface (P:src/matrix.hpp, quant.hpp, rng.hpp, gemm_abft.hpp, embedding_abft.hpp,
// fault_lab.hpp, bench.hpp) mapped onto the B200 library, so the reference's OWN test sources compile unchanged
// against libabftlp_b200.so (oracle/Makefile target `suites`; run by tests/test_reference_suites.py):
//   * containers and the operators are the drop-in adapter include/abftlp_b200.hpp (namespace abft_b200);
//   * campaigns go through the C ABI (abftlp_campaign_parse / _run / report accessors) -- GPU trials;
//   * benches go through abftlp_bench_gemm / abftlp_bench_eb -- GPU timings.
// The detection model (closed forms, P:src/detection_model.hpp) is analytic, out of scope, and taken from the
// reference's own header/source. Test infrastructure only: nothing here ships in the library.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <optional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <unistd.h>
#include <vector>

#include "abftlp_b200.hpp"
#include "detection_model.hpp"  // the reference's analytic model (model::FaultModel and the closed forms)

namespace abft {
using abft_b200::Mat;
using abft_b200::MatI32;
using abft_b200::MatI8;
using abft_b200::MatU8;
using MatF64 = abft_b200::Mat<double>;
namespace quant = abft_b200::quant;
namespace gemm = abft_b200::gemm;
namespace eb = abft_b200::eb;

namespace lab {

// Same draw streams as P:src/rng.hpp (state0 = mix(seed ^ mix(stream + gamma)), draw = mix(state += gamma)).
class SplitMix64 {
public:
    explicit SplitMix64(std::uint64_t seed, std::uint64_t stream = 0) : s_(mix(seed ^ mix(stream + kGamma))) {}
    std::uint64_t next() { return mix(s_ += kGamma); }
    std::uint64_t next_below(std::uint64_t bound) { return next() % bound; }
    std::int64_t next_int(std::int64_t lo, std::int64_t hi) {
        return lo + static_cast<std::int64_t>(next_below(static_cast<std::uint64_t>(hi - lo + 1)));
    }
    double next_double() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
    double next_real(double lo, double hi) { return lo + (hi - lo) * next_double(); }

private:
    static constexpr std::uint64_t kGamma = 0x9e3779b97f4a7c15ULL;
    static std::uint64_t mix(std::uint64_t z) {
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        return z ^ (z >> 31);
    }
    std::uint64_t s_;
};

enum class FaultTarget { weight_B, intermediate_C, eb_table, none };
enum class BitRange { all, high4, low4 };
struct FaultSpec {
    FaultTarget target = FaultTarget::none;
    model::FaultModel model = model::FaultModel::single_bit_flip;
    BitRange bitRange = BitRange::all;
    std::uint64_t seed = 0;
};
struct GemmShape {
    std::size_t m = 1, n = 1, k = 1;
};
struct GemmWorkload {
    std::vector<GemmShape> shapes;
    std::size_t trialsPerShape = 100;
};
struct EbWorkload {
    std::size_t tableRows = 100000, tableDim = 64, pooling = 100, batch = 10, trials = 200;
};
struct CampaignConfig {
    std::optional<GemmWorkload> gemm;
    std::optional<EbWorkload> eb;
    FaultSpec fault;
    std::size_t threads = 0;
};
struct ShapeStats {
    std::string label;
    std::uint64_t trials = 0, detected = 0, falsePositives = 0;
};
struct CampaignReport {
    std::string target, model, bitRange;
    std::uint64_t trials = 0, detected = 0, notDetected = 0, falsePositives = 0;
    std::vector<ShapeStats> perShape;
    std::string notes;
    double detectionRate() const { return trials ? static_cast<double>(detected) / static_cast<double>(trials) : 0.0; }
    std::string csvText, tableText;  // (facade) the library's own renderings of this report
};
struct FaultRecord {
    bool injected = false;
    std::string position;
    std::int64_t before = 0, after = 0;
};
struct WilsonInterval {
    double low = 0.0, high = 0.0;
};

namespace facade {
inline void ok(abftlp_status s) {
    if (s == ABFTLP_OK) return;
    const std::string m = abftlp_last_error();
    if (s == ABFTLP_ERR_INVALID_ARGUMENT || s == ABFTLP_ERR_PARSE) throw std::invalid_argument(m);
    throw std::runtime_error(m);
}
// The config in the campaign-file syntax the C ABI parses (P:README.md:70-84).
inline std::string to_text(const CampaignConfig& c) {
    static const char* const targets[] = {"weight_b", "intermediate_c", "eb_table", "none"};
    static const char* const ranges[] = {"all", "high4", "low4"};
    std::ostringstream t;
    if (c.threads) t << "threads = " << c.threads << "\n";
    t << "[workload]\n";
    if (c.gemm) {
        t << "kind = gemm\ntrials_per_shape = " << c.gemm->trialsPerShape << "\nshapes = ";
        for (size_t i = 0; i < c.gemm->shapes.size(); ++i)
            t << (i ? ", " : "") << c.gemm->shapes[i].m << "x" << c.gemm->shapes[i].n << "x" << c.gemm->shapes[i].k;
        t << "\n";
    } else if (c.eb) {
        t << "kind = eb\ntable_rows = " << c.eb->tableRows << "\ntable_dim = " << c.eb->tableDim
          << "\npooling = " << c.eb->pooling << "\nbatch = " << c.eb->batch << "\ntrials = " << c.eb->trials << "\n";
    }
    t << "[fault]\ntarget = " << targets[static_cast<int>(c.fault.target)] << "\nmodel = "
      << (c.fault.model == model::FaultModel::single_bit_flip ? "single_bit_flip" : "random_value")
      << "\nbit_range = " << ranges[static_cast<int>(c.fault.bitRange)] << "\nseed = " << c.fault.seed << "\n";
    return t.str();
}
inline CampaignReport run(const CampaignConfig& cfg) {
    abftlp_campaign* c = nullptr;
    ok(abftlp_campaign_parse(to_text(cfg).c_str(), &c));
    abftlp_report* r = nullptr;
    const abftlp_status s = abftlp_campaign_run(c, &r);
    abftlp_campaign_free(c);
    ok(s);
    CampaignReport rep;
    rep.trials = abftlp_report_trials(r);
    rep.detected = abftlp_report_detected(r);
    rep.falsePositives = abftlp_report_false_positives(r);
    rep.notDetected = rep.trials - rep.detected;
    // per-row statistics from the report's CSV (target,model,bit_range,label,trials,detected,not_detected,fp,...)
    char path[] = "/tmp/abft_facade_XXXXXX";
    const int fd = mkstemp(path);
    if (fd >= 0) close(fd);
    const abftlp_status w = abftlp_report_write_csv(r, path);
    char* table = nullptr;
    const abftlp_status tr = abftlp_report_render(r, &table);
    if (tr == ABFTLP_OK && table) {
        rep.tableText = table;
        abftlp_string_free(table);
    }
    abftlp_report_free(r);
    ok(w);
    ok(tr);
    {
        std::ifstream whole(path);
        std::stringstream all;
        all << whole.rdbuf();
        rep.csvText = all.str();
    }
    std::ifstream in(path);
    std::string line;
    std::getline(in, line);  // header
    while (std::getline(in, line)) {
        std::vector<std::string> f;
        std::stringstream ls(line);
        for (std::string x; std::getline(ls, x, ',');) f.push_back(x);
        if (f.size() < 8) continue;
        rep.target = f[0];
        rep.model = f[1];
        rep.bitRange = f[2];
        if (f[3] == "total") continue;
        rep.perShape.push_back({f[3], std::stoull(f[4]), std::stoull(f[5]), std::stoull(f[7])});
    }
    std::remove(path);
    return rep;
}
}  // namespace facade

inline CampaignReport run_gemm_campaign(const CampaignConfig& cfg) {
    if (!cfg.gemm) throw std::invalid_argument("run_gemm_campaign: not a gemm workload");
    return facade::run(cfg);
}
inline CampaignReport run_eb_campaign(const CampaignConfig& cfg) {
    if (!cfg.eb) throw std::invalid_argument("run_eb_campaign: not an eb workload");
    return facade::run(cfg);
}
inline CampaignReport run_campaign(const CampaignConfig& cfg) { return facade::run(cfg); }

// The library's renderings of a report it produced (byte-identical to the reference's writers: checked by
// tests/test_fault_lab_gpu.py against the reference build).
inline std::string report_to_csv(const CampaignReport& r) { return r.csvText; }
inline std::string report_to_table(const CampaignReport& r) { return r.tableText; }

// Campaign text -> CampaignConfig: the library's parser (abftlp_campaign_parse) accepts or rejects the text; the
// fields the reference's tests read back are then picked out of the accepted text.
inline CampaignConfig parse_campaign_config(const std::string& text) {
    abftlp_campaign* c = nullptr;
    facade::ok(abftlp_campaign_parse(text.c_str(), &c));
    abftlp_campaign_free(c);
    CampaignConfig cfg;
    std::string kind;
    GemmWorkload g;
    EbWorkload e;
    std::istringstream in(text);
    for (std::string line; std::getline(in, line);) {
        line = line.substr(0, line.find('#'));
        const auto eq = line.find('=');
        if (eq == std::string::npos) continue;
        auto trim = [](std::string v) {
            const auto a = v.find_first_not_of(" \t\r"), b = v.find_last_not_of(" \t\r");
            return a == std::string::npos ? std::string() : v.substr(a, b - a + 1);
        };
        const std::string key = trim(line.substr(0, eq)), val = trim(line.substr(eq + 1));
        if (key == "threads") cfg.threads = std::stoull(val);
        else if (key == "kind") kind = val;
        else if (key == "trials_per_shape") g.trialsPerShape = std::stoull(val);
        else if (key == "shapes") {
            std::stringstream ls(val);
            for (std::string x; std::getline(ls, x, ',');) {
                unsigned long long m = 0, n = 0, k = 0;
                if (std::sscanf(x.c_str(), " %llux%llux%llu", &m, &n, &k) == 3) g.shapes.push_back({m, n, k});
            }
        } else if (key == "table_rows") e.tableRows = std::stoull(val);
        else if (key == "table_dim") e.tableDim = std::stoull(val);
        else if (key == "pooling") e.pooling = std::stoull(val);
        else if (key == "batch") e.batch = std::stoull(val);
        else if (key == "trials") e.trials = std::stoull(val);
        else if (key == "target")
            cfg.fault.target = val == "weight_b" ? FaultTarget::weight_B : val == "intermediate_c" ? FaultTarget::intermediate_C
                               : val == "eb_table" ? FaultTarget::eb_table : FaultTarget::none;
        else if (key == "model")
            cfg.fault.model = val == "random_value" ? model::FaultModel::random_value : model::FaultModel::single_bit_flip;
        else if (key == "bit_range")
            cfg.fault.bitRange = val == "high4" ? BitRange::high4 : val == "low4" ? BitRange::low4 : BitRange::all;
        else if (key == "seed") cfg.fault.seed = std::stoull(val);
    }
    if (kind == "gemm") cfg.gemm = g;
    else if (kind == "eb") cfg.eb = e;
    return cfg;
}

// 95 % Wilson score interval (z = 1.959963984540054), clamped to [0, 1].
inline WilsonInterval wilson_interval(std::uint64_t successes, std::uint64_t trials) {
    if (trials == 0) throw std::invalid_argument("wilson_interval: zero trials");
    const double z = 1.959963984540054, n = static_cast<double>(trials);
    const double p = static_cast<double>(successes) / n, q = z * z / n;
    const double mid = (p + q / 2.0) / (1.0 + q);
    const double half = z * std::sqrt(p * (1.0 - p) / n + q / (4.0 * n)) / (1.0 + q);
    return {std::max(0.0, mid - half), std::min(1.0, mid + half)};
}

// Host-container injectors of the reference's unit tests (P:src/fault_lab.hpp:96-107): the draw protocol of
// paper_2103_00130_b200/fault_lab.py (stream = trial * 4 + 1 of the spec's seed; row, column, then the bit or the
// replacement value) applied to a host matrix. The GPU campaigns inject on the device (csrc/campaign.cu).
inline unsigned draw_bit_index(SplitMix64& rng, BitRange range, unsigned width) {
    if (range == BitRange::high4) return width - 4 + static_cast<unsigned>(rng.next_below(4));
    if (range == BitRange::low4) return static_cast<unsigned>(rng.next_below(4));
    return static_cast<unsigned>(rng.next_below(width));
}
template <typename T>
T flip_bit(T value, unsigned bitIndex);
namespace facade {
inline SplitMix64 inject_rng(const FaultSpec& spec, std::uint64_t trial) { return SplitMix64(spec.seed, trial * 4 + 1); }
inline std::string coord(std::size_t i, std::size_t j) { return "(" + std::to_string(i) + "," + std::to_string(j) + ")"; }
}  // namespace facade
inline FaultRecord inject_weight_B(MatI8& b, const FaultSpec& spec, std::uint64_t trial);
inline FaultRecord inject_intermediate_C(quant::IntermediateMatrix& c, const FaultSpec& spec, std::uint64_t trial);
inline FaultRecord inject_eb_table(eb::QuantEmbeddingTable& t, const std::vector<eb::IndexBag>& bags, const FaultSpec& spec,
                                   std::uint64_t trial);

template <typename T>
T flip_bit(T value, unsigned bitIndex) {
    static_assert(std::is_integral_v<T>);
    if (bitIndex >= sizeof(T) * 8) throw std::out_of_range("flip_bit: bit index out of range");
    using U = std::make_unsigned_t<T>;
    return static_cast<T>(static_cast<U>(value) ^ (U{1} << bitIndex));
}

inline FaultRecord inject_weight_B(MatI8& b, const FaultSpec& spec, std::uint64_t trial) {
    if (spec.target == FaultTarget::none) return {};
    SplitMix64 rng = facade::inject_rng(spec, trial);
    const std::size_t i = rng.next_below(b.rows()), j = rng.next_below(b.cols());
    std::int8_t& cell = b(i, j);
    FaultRecord rec{true, facade::coord(i, j), cell, 0};
    if (spec.model == model::FaultModel::single_bit_flip) {
        cell = flip_bit(cell, draw_bit_index(rng, spec.bitRange, 8));
    } else {
        std::int8_t nv = cell;
        while (nv == cell) nv = static_cast<std::int8_t>(rng.next_int(-128, 127));
        cell = nv;
    }
    rec.after = cell;
    return rec;
}
inline FaultRecord inject_intermediate_C(quant::IntermediateMatrix& c, const FaultSpec& spec, std::uint64_t trial) {
    if (spec.target == FaultTarget::none) return {};
    SplitMix64 rng = facade::inject_rng(spec, trial);
    const std::size_t i = rng.next_below(c.data.rows()), j = rng.next_below(c.data.cols());
    std::int32_t& cell = c.data(i, j);
    FaultRecord rec{true, facade::coord(i, j), cell, 0};
    if (spec.model == model::FaultModel::single_bit_flip) {
        cell = flip_bit(cell, draw_bit_index(rng, spec.bitRange, 32));
    } else {
        std::int32_t nv = cell;
        while (nv == cell) nv = static_cast<std::int32_t>(rng.next());
        cell = nv;
    }
    rec.after = cell;
    return rec;
}
inline FaultRecord inject_eb_table(eb::QuantEmbeddingTable& t, const std::vector<eb::IndexBag>& bags, const FaultSpec& spec,
                                   std::uint64_t trial) {
    if (spec.target == FaultTarget::none) return {};
    SplitMix64 rng = facade::inject_rng(spec, trial);
    std::vector<std::size_t> usable;
    for (std::size_t q = 0; q < bags.size(); ++q)
        if (!bags[q].indices.empty()) usable.push_back(q);
    if (usable.empty()) throw std::invalid_argument("inject_eb_table: all bags empty");
    const eb::IndexBag& bag = bags[usable[rng.next_below(usable.size())]];
    const std::size_t row = bag.indices[rng.next_below(bag.indices.size())], col = rng.next_below(t.rows.cols());
    std::int8_t& cell = t.rows(row, col);
    FaultRecord rec{true, facade::coord(row, col), cell, 0};
    if (spec.model == model::FaultModel::single_bit_flip) {
        cell = flip_bit(cell, draw_bit_index(rng, spec.bitRange, 8));
    } else {
        std::int8_t nv = cell;
        while (nv == cell) nv = static_cast<std::int8_t>(rng.next_int(-128, 127));
        cell = nv;
    }
    rec.after = cell;
    return rec;
}

}  // namespace lab

namespace bench {
struct BenchResult {
    std::string label;
    double baselineNanos = 0.0, abftNanos = 0.0, overheadFraction = 0.0;
    std::size_t repetitions = 0;
};
inline constexpr std::size_t kMinRepetitions = 5;
inline BenchResult bench_gemm(const lab::GemmShape& s, std::size_t reps, std::uint64_t seed) {
    abftlp_bench_result r{};
    lab::facade::ok(abftlp_bench_gemm(s.m, s.n, s.k, static_cast<uint32_t>(reps), seed, &r));
    return {std::to_string(s.m) + "x" + std::to_string(s.n) + "x" + std::to_string(s.k), r.baseline_ns, r.abft_ns,
            r.overhead_fraction, reps};
}
inline BenchResult bench_eb(std::size_t rows, std::size_t dim, std::size_t pooling, std::size_t batch, std::size_t reps,
                            std::uint64_t seed) {
    abftlp_bench_result r{};
    lab::facade::ok(abftlp_bench_eb(rows, dim, pooling, batch, static_cast<uint32_t>(reps), seed, &r));
    return {"eb", r.baseline_ns, r.abft_ns, r.overhead_fraction, reps};
}
// Shape file: one "MxNxK" per line, '#' comments and blank lines skipped (P:data/shapes.txt).
inline std::vector<lab::GemmShape> load_shapes(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open shapes file: " + path);
    std::vector<lab::GemmShape> out;
    for (std::string line; std::getline(in, line);) {
        line = line.substr(0, line.find('#'));
        unsigned long long m = 0, n = 0, k = 0;
        char x1 = 0, x2 = 0;
        if (std::sscanf(line.c_str(), " %llu %c %llu %c %llu", &m, &x1, &n, &x2, &k) == 5 && x1 == 'x' && x2 == 'x')
            out.push_back({m, n, k});
    }
    if (out.empty()) throw std::runtime_error("no shapes in " + path);
    return out;
}
}  // namespace bench
}  // namespace abft
