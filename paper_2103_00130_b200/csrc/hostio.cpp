// Host-side text and file formats of the fault lab (no device code): campaign configuration files, the
// campaign report (CSV and the aligned table), ABEB table files and bag files.
//
// Written from the formats themselves (P:README.md:70-84 for campaign files, SPEC:356 / P:src/embedding_abft.hpp:48-50
// for ABEB, P:src/capi.cpp:195-198 for the bag-line grammar); the byte-level outputs are pinned against the
// reference's own writers by tests/test_fault_lab_gpu.py (CSV, table, eb-check rendering).
#include <algorithm>
#include <cctype>
#include <cerrno>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <functional>
#include <iterator>
#include <stdexcept>
#include <string>
#include <vector>

#include "campaign.h"

namespace abftk {

// ============================================================ campaign files
namespace {

[[noreturn]] void config_error(const std::string& what) { throw std::invalid_argument("campaign config: " + what); }

bool is_blank(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\n'; }

std::string strip(const std::string& s) {
    size_t a = 0, b = s.size();
    while (a < b && is_blank(s[a])) ++a;
    while (b > a && is_blank(s[b - 1])) --b;
    return s.substr(a, b - a);
}

// One `key = value` line, the key qualified by its section ("workload.kind"; top-level keys unqualified).
struct Setting {
    std::string key, value;
    bool used = false;
};

std::vector<Setting> read_settings(const std::string& text) {
    std::vector<Setting> out;
    std::string section;
    size_t pos = 0;
    while (pos <= text.size()) {
        size_t eol = text.find('\n', pos);
        if (eol == std::string::npos) eol = text.size();
        std::string line = text.substr(pos, eol - pos);
        pos = eol + 1;
        line = strip(line.substr(0, line.find('#')));
        if (line.empty()) continue;
        if (line[0] == '[') {
            if (line.back() != ']') config_error("malformed section '" + line + "'");
            section = strip(line.substr(1, line.size() - 2));
            continue;
        }
        const size_t eq = line.find('=');
        if (eq == std::string::npos) config_error("expected key=value, got '" + line + "'");
        const std::string key = strip(line.substr(0, eq));
        const std::string qualified = section.empty() ? key : section + "." + key;
        // a repeated key keeps its last value
        bool replaced = false;
        for (Setting& s : out)
            if (s.key == qualified) {
                s.value = strip(line.substr(eq + 1));
                replaced = true;
            }
        if (!replaced) out.push_back({qualified, strip(line.substr(eq + 1)), false});
    }
    return out;
}

uint64_t to_count(const std::string& key, const std::string& v) {
    // the whole value must be one unsigned decimal (strtoull's grammar: an optional sign, '-' wrapping)
    const char* p = v.c_str();
    char* end = nullptr;
    errno = 0;
    const unsigned long long r = std::strtoull(p, &end, 10);
    if (v.empty() || end != p + v.size() || errno == ERANGE || is_blank(v[0]))
        config_error("bad integer for '" + key + "': " + v);
    return r;
}

// "MxNxK, MxNxK, ..."
std::vector<GemmShape> to_shapes(const std::string& v) {
    std::vector<GemmShape> shapes;
    size_t pos = 0;
    while (pos <= v.size()) {
        size_t comma = v.find(',', pos);
        if (comma == std::string::npos) comma = v.size();
        const std::string item = strip(v.substr(pos, comma - pos));
        pos = comma + 1;
        if (item.empty()) continue;
        // three numbers separated by 'x' (blanks allowed around them; anything after the third is ignored)
        uint64_t dims[3] = {0, 0, 0};
        const char* p = item.c_str();
        bool ok = true;
        for (int q = 0; q < 3 && ok; ++q) {
            char* end = nullptr;
            errno = 0;
            dims[q] = std::strtoull(p, &end, 10);
            ok = end != p && errno != ERANGE;
            p = end;
            if (ok && q < 2) {
                while (is_blank(*p)) ++p;
                ok = *p++ == 'x';
            }
        }
        if (!ok || dims[0] == 0 || dims[1] == 0 || dims[2] == 0) config_error("bad shape '" + item + "' (want MxNxK)");
        shapes.push_back({dims[0], dims[1], dims[2]});
    }
    if (shapes.empty()) config_error("workload.shapes is empty");
    return shapes;
}

template <typename E>
E to_enum(const std::string& what, const std::string& v, std::initializer_list<std::pair<const char*, E>> names) {
    for (const auto& nv : names)
        if (v == nv.first) return nv.second;
    config_error("unknown " + what + " '" + v + "'");
}

}  // namespace

CampaignConfig parse_campaign_config(const std::string& text) {
    std::vector<Setting> settings = read_settings(text);
    auto find = [&](const char* key) -> Setting* {
        for (Setting& s : settings)
            if (s.key == key) return &s;
        return nullptr;
    };
    auto need = [&](const char* key) -> const std::string& {
        Setting* s = find(key);
        if (!s) config_error(std::string("missing '") + key + "'");
        s->used = true;
        return s->value;
    };
    auto maybe = [&](const char* key, const std::function<void(const std::string&)>& apply) {
        if (Setting* s = find(key)) {
            s->used = true;
            apply(s->value);
        }
    };
    CampaignConfig cfg;
    maybe("threads", [&](const std::string& v) { cfg.threads = to_count("threads", v); });
    const std::string kind = need("workload.kind");
    if (kind == "gemm") {
        GemmWorkload g;
        g.trialsPerShape = to_count("trials_per_shape", need("workload.trials_per_shape"));
        g.shapes = to_shapes(need("workload.shapes"));
        cfg.gemm = g;
    } else if (kind == "eb") {
        EbWorkload e;
        // the EB workload's five sizes, all required
        const std::pair<const char*, uint64_t EbWorkload::*> sizes[] = {
            {"table_rows", &EbWorkload::tableRows}, {"table_dim", &EbWorkload::tableDim},
            {"pooling", &EbWorkload::pooling},      {"batch", &EbWorkload::batch},
            {"trials", &EbWorkload::trials}};
        for (const auto& sz : sizes) e.*(sz.second) = to_count(sz.first, need((std::string("workload.") + sz.first).c_str()));
        cfg.eb = e;
    } else {
        config_error("unknown workload.kind '" + kind + "'");
    }
    cfg.fault.target = to_enum<FaultTarget>("fault target", need("fault.target"),
                                            {{"weight_b", FaultTarget::weight_B},
                                             {"intermediate_c", FaultTarget::intermediate_C},
                                             {"eb_table", FaultTarget::eb_table},
                                             {"none", FaultTarget::none}});
    maybe("fault.model", [&](const std::string& v) {
        cfg.fault.model = to_enum<FaultModel>(
            "fault model", v, {{"single_bit_flip", FaultModel::single_bit_flip}, {"random_value", FaultModel::random_value}});
    });
    maybe("fault.bit_range", [&](const std::string& v) {
        cfg.fault.bitRange = to_enum<BitRange>("bit_range", v,
                                               {{"all", BitRange::all}, {"high4", BitRange::high4}, {"low4", BitRange::low4}});
    });
    maybe("fault.seed", [&](const std::string& v) { cfg.fault.seed = to_count("seed", v); });
    for (const Setting& s : settings)
        if (!s.used) config_error("unknown key '" + s.key + "'");
    return cfg;
}

// ============================================================ reports
const char* fault_target_name(FaultTarget t) {
    static const char* const names[] = {"weight_b", "intermediate_c", "eb_table", "none"};
    return names[static_cast<int>(t)];
}
const char* fault_model_name(FaultModel m) {
    return m == FaultModel::single_bit_flip ? "single_bit_flip" : "random_value";
}
const char* bit_range_name(BitRange r) {
    static const char* const names[] = {"all", "high4", "low4"};
    return names[static_cast<int>(r)];
}

// 95% Wilson score interval of `successes` out of `trials` (z = 1.959963984540054), clamped to [0, 1].
WilsonInterval wilson_interval(uint64_t successes, uint64_t trials) {
    if (trials == 0) throw std::invalid_argument("wilson_interval: zero trials");
    constexpr double z = 1.959963984540054;
    const double n = static_cast<double>(trials);
    const double phat = static_cast<double>(successes) / n;
    const double zz_n = z * z / n;
    const double scale = 1.0 + zz_n;
    const double mid = (phat + zz_n / 2.0) / scale;
    const double spread = z * std::sqrt(phat * (1.0 - phat) / n + z * z / (4.0 * n * n)) / scale;
    WilsonInterval w;
    w.low = std::max(0.0, mid - spread);
    w.high = std::min(1.0, mid + spread);
    return w;
}

namespace {
// The report rows: one per shape (or EB workload), then "total" when there are several.
template <typename Fn>
void for_each_row(const CampaignReport& r, Fn&& fn) {
    for (const ShapeStats& s : r.perShape) fn(s.label, s.trials, s.detected, s.falsePositives);
    if (r.perShape.size() > 1) fn(std::string("total"), r.trials, r.detected, r.falsePositives);
}
std::string fmt(const char* f, ...) __attribute__((format(printf, 1, 2)));
std::string fmt(const char* f, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, f);
    const int n = std::vsnprintf(buf, sizeof buf, f, ap);
    va_end(ap);
    return std::string(buf, n < 0 ? 0 : std::min<size_t>(static_cast<size_t>(n), sizeof buf - 1));
}
}  // namespace

std::string report_to_csv(const CampaignReport& r) {
    std::string out =
        "target,model,bit_range,shape_or_dims,trials,detected,not_detected,false_positives,detection_rate,ci_low,"
        "ci_high\n";
    for_each_row(r, [&](const std::string& label, uint64_t n, uint64_t det, uint64_t fp) {
        const WilsonInterval ci = wilson_interval(det, n);
        out += r.target + ',' + r.model + ',' + r.bitRange + ',' + label + ',';
        out += fmt("%llu,%llu,%llu,%llu,%.10g,%.10g,%.10g\n", static_cast<unsigned long long>(n),
                   static_cast<unsigned long long>(det), static_cast<unsigned long long>(n - det),
                   static_cast<unsigned long long>(fp), n ? static_cast<double>(det) / static_cast<double>(n) : 0.0,
                   ci.low, ci.high);
    });
    return out;
}

std::string report_to_table(const CampaignReport& r) {
    std::string out = "campaign: target=" + r.target + " model=" + r.model + " bit_range=" + r.bitRange + "\n";
    if (!r.notes.empty()) out += "note: " + r.notes + "\n";
    out += fmt("%-24s%8s%10s%8s%10s%18s", "shape_or_dims", "trials", "detected", "fp", "rate", "wilson95\n");
    for_each_row(r, [&](const std::string& label, uint64_t n, uint64_t det, uint64_t fp) {
        const WilsonInterval ci = wilson_interval(det, n);
        out += fmt("%-24s%8llu%10llu%8llu%10.4f   [%.4f, %.4f]\n", label.c_str(), static_cast<unsigned long long>(n),
                   static_cast<unsigned long long>(det), static_cast<unsigned long long>(fp),
                   n ? static_cast<double>(det) / static_cast<double>(n) : 0.0, ci.low, ci.high);
    });
    return out;
}

// ============================================================ ABEB table files
// Little-endian container: "ABEB" | u16 version (1) | u64 rows | u32 dim | rows x (dim int8 values, f32 scale,
// f32 bias) | rows x i32 row sum.
namespace {
struct Cursor {
    const std::vector<char>& buf;
    size_t at = 0;
    void take(void* dst, size_t n) {
        if (buf.size() - at < n) throw std::runtime_error("table file truncated");
        std::memcpy(dst, buf.data() + at, n);
        at += n;
    }
    template <typename T>
    T pod() {
        T v;
        take(&v, sizeof v);
        return v;
    }
};
template <typename T>
void put(std::vector<char>& out, const T& v) {
    const char* p = reinterpret_cast<const char*>(&v);
    out.insert(out.end(), p, p + sizeof v);
}
}  // namespace

HostTable load_table_file(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw std::runtime_error("cannot open table file: " + path);
    const std::vector<char> buf((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
    if (buf.size() < 4 || std::memcmp(buf.data(), "ABEB", 4) != 0)
        throw std::runtime_error("not an embedding table file: " + path);
    Cursor c{buf, 4};
    if (c.pod<uint16_t>() != 1) throw std::runtime_error("unsupported table file version");
    HostTable t;
    t.rows = c.pod<uint64_t>();
    t.dim = c.pod<uint32_t>();
    if (t.rows == 0 || t.dim == 0) throw std::runtime_error("table file has empty dimensions");
    const uint64_t rec = static_cast<uint64_t>(t.dim) + 8;
    if ((buf.size() - c.at) / rec < t.rows) throw std::runtime_error("table file truncated");
    t.data.resize(t.rows * t.dim);
    t.scales.resize(t.rows);
    t.biases.resize(t.rows);
    for (uint64_t r = 0; r < t.rows; ++r) {
        c.take(t.data.data() + r * t.dim, t.dim);
        t.scales[r] = c.pod<float>();
        t.biases[r] = c.pod<float>();
    }
    t.rowSums.resize(t.rows);
    c.take(t.rowSums.data(), 4 * t.rows);
    return t;
}

void save_table_file(const HostTable& t, const std::string& path) {
    std::vector<char> out;
    out.reserve(18 + t.rows * (t.dim + 12));
    out.insert(out.end(), {'A', 'B', 'E', 'B'});
    put<uint16_t>(out, 1);
    put<uint64_t>(out, t.rows);
    put<uint32_t>(out, t.dim);
    for (uint64_t r = 0; r < t.rows; ++r) {
        const char* row = reinterpret_cast<const char*>(t.data.data() + r * t.dim);
        out.insert(out.end(), row, row + t.dim);
        put(out, t.scales[r]);
        put(out, t.biases[r]);
    }
    const char* sums = reinterpret_cast<const char*>(t.rowSums.data());
    out.insert(out.end(), sums, sums + 4 * t.rows);
    std::ofstream f(path, std::ios::binary);
    if (!f) throw std::runtime_error("cannot open table file for writing: " + path);
    f.write(out.data(), static_cast<std::streamsize>(out.size()));
    if (!f) throw std::runtime_error("failed writing table file: " + path);
}

// ============================================================ bag files
// One bag per line; whitespace-separated tokens "index" or "index:weight"; '#' starts a comment; lines with no
// token are skipped. An index is an unsigned decimal prefix of its token (what follows the digits is ignored, a
// leading '-' wraps as an unsigned value), a weight a float prefix; a token with neither is an error. A batch with
// any weighted token is weighted, its plain tokens weighing 1.0f (bit-identical to unweighted lookups).
namespace {
bool parse_index(const std::string& s, int64_t& out) {
    const char* p = s.c_str();
    char* end = nullptr;
    errno = 0;
    const unsigned long long v = std::strtoull(p, &end, 10);
    if (end == p || errno == ERANGE) return false;
    out = static_cast<int64_t>(v);
    return true;
}
bool parse_weight(const std::string& s, float& out) {
    const char* p = s.c_str();
    char* end = nullptr;
    errno = 0;
    const float v = std::strtof(p, &end);
    if (end == p || errno == ERANGE) return false;
    out = v;
    return true;
}
}  // namespace

bool parse_bag_lines(std::istream& in, HostBags& bags, std::string& error) {
    std::vector<float> w_all;
    for (std::string line; std::getline(in, line);) {
        line = line.substr(0, line.find('#'));
        size_t added = 0;
        size_t at = 0;
        while (true) {
            while (at < line.size() && std::isspace(static_cast<unsigned char>(line[at]))) ++at;
            if (at >= line.size()) break;
            size_t end = at;
            while (end < line.size() && !std::isspace(static_cast<unsigned char>(line[end]))) ++end;
            const std::string tok = line.substr(at, end - at);
            at = end;
            const size_t colon = tok.find(':');
            int64_t idx = 0;
            float w = 1.0f;
            const bool ok = colon == std::string::npos
                                ? parse_index(tok, idx)
                                : parse_index(tok.substr(0, colon), idx) && parse_weight(tok.substr(colon + 1), w);
            if (!ok) {
                error = "bad index token: " + tok;
                return false;
            }
            bags.weighted |= colon != std::string::npos;
            bags.indices.push_back(idx);
            w_all.push_back(w);
            ++added;
        }
        if (added == 0) continue;
        bags.offsets.push_back(static_cast<int64_t>(bags.indices.size()));
    }
    if (bags.weighted) bags.weights = std::move(w_all);
    return true;
}

}  // namespace abftk
