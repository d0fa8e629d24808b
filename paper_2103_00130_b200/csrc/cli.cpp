// abft_cli -- command-line front end over the C ABI (include/abftlp.h), the B200 counterpart of the reference's
// tool (P:tools/abft_cli.cpp:57-207; its CLI11 dependency is not shipped, so options are parsed here directly):
//
//   abft_cli campaign <config> [--out report.csv]             fault-injection campaign on the GPU
//   abft_cli analyze --m M --n N --k K [--d D] [--pool P]     closed-form overheads / detection probabilities
//   abft_cli bench [--shapes file] [--reps R] [--out csv] [--eb-rows N]
//                                                             ABFT overhead, checked vs unchecked kernels
//   abft_cli eb-check <table> <indices> [--skip-validation]   checked lookups over an ABEB table and a bag file
//
// Exit status: 0 ok, 1 usage or library error, 2 eb-check flagged at least one bag (P:tools/abft_cli.cpp:165).
// ABFTLP_SEED overrides the bench seed (P:tools/abft_cli.cpp:15-24).
#include <array>
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <functional>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "abftlp.h"

namespace {

// ------------------------------------------------------------------ arguments
struct Args {
    std::vector<std::string> positional;
    std::map<std::string, std::string> options;  // --name value
    std::map<std::string, bool> flags;           // --name
};

// Options named in `valued` take the next argument; any other --name is a flag.
bool parse_args(int argc, char** argv, int first, const std::vector<std::string>& valued, Args& out, std::string& err) {
    for (int i = first; i < argc; ++i) {
        const std::string a = argv[i];
        if (a.rfind("--", 0) != 0) {
            out.positional.push_back(a);
            continue;
        }
        const std::string name = a.substr(2);
        bool takes_value = false;
        for (const std::string& v : valued) takes_value = takes_value || v == name;
        if (!takes_value) {
            out.flags[name] = true;
            continue;
        }
        if (i + 1 >= argc) {
            err = "option --" + name + " needs a value";
            return false;
        }
        out.options[name] = argv[++i];
    }
    return true;
}

bool to_u64(const std::string& s, uint64_t& v) {
    if (s.empty() || s.find_first_not_of("0123456789") != std::string::npos) return false;
    errno = 0;
    v = std::strtoull(s.c_str(), nullptr, 10);
    return errno != ERANGE;
}

int report_failure(abftlp_status st, const std::string& what) {
    std::fprintf(stderr, "error (%s): %s: %s\n", abftlp_status_str(st), what.c_str(), abftlp_last_error());
    return 1;
}

int usage(const char* msg) {
    if (msg) std::fprintf(stderr, "error: %s\n", msg);
    std::fprintf(stderr,
                 "usage: abft_cli campaign <config> [--out csv]\n"
                 "       abft_cli analyze --m M --n N --k K [--d D] [--pool P]\n"
                 "       abft_cli bench [--shapes file] [--reps R] [--out csv] [--eb-rows N]\n"
                 "       abft_cli eb-check <table> <indices> [--skip-validation]\n");
    return 1;
}

// ------------------------------------------------------------------ subcommands
int run_campaign(const Args& a) {
    if (a.positional.size() != 1) return usage("campaign takes one config file");
    const std::string cfg = a.positional[0];
    const auto o = a.options.find("out");
    const std::string csv = o != a.options.end() ? o->second : cfg + ".report.csv";
    abftlp_campaign* c = nullptr;
    abftlp_status st = abftlp_campaign_load(cfg.c_str(), &c);
    if (st != ABFTLP_OK) return report_failure(st, "loading " + cfg);
    abftlp_report* r = nullptr;
    st = abftlp_campaign_run(c, &r);
    abftlp_campaign_free(c);
    if (st != ABFTLP_OK) return report_failure(st, "running campaign");
    st = abftlp_report_write_csv(r, csv.c_str());
    if (st == ABFTLP_OK) {
        char* table = nullptr;
        if (abftlp_report_render(r, &table) == ABFTLP_OK) {
            std::fputs(table, stdout);
            abftlp_string_free(table);
        }
        std::printf("report written to %s\n", csv.c_str());
    }
    abftlp_report_free(r);
    return st == ABFTLP_OK ? 0 : report_failure(st, "writing " + csv);
}

int run_analyze(const Args& a) {
    uint64_t v[5] = {0, 0, 0, 64, 100};
    const char* names[5] = {"m", "n", "k", "d", "pool"};
    for (int i = 0; i < 5; ++i) {
        const auto it = a.options.find(names[i]);
        if (it == a.options.end()) {
            if (i < 3) return usage("analyze needs --m, --n and --k");
            continue;
        }
        if (!to_u64(it->second, v[i]) || v[i] == 0) return usage("analyze options must be positive integers");
    }
    abftlp_analysis r{};
    const abftlp_status st = abftlp_analyze(v[0], v[1], v[2], v[3], v[4], &r);
    if (st != ABFTLP_OK) return report_failure(st, "analyze");
    const auto pct = [](double x) { return 100.0 * x; };
    std::printf("GEMM shape %llux%llux%llu\n", static_cast<unsigned long long>(v[0]), static_cast<unsigned long long>(v[1]),
                static_cast<unsigned long long>(v[2]));
    std::printf("  encode overhead, A side: %.4f%%\n", pct(r.encode_overhead_a));
    std::printf("  encode overhead, B side: %.4f%%\n", pct(r.encode_overhead_b));
    std::printf("  detection, error in B, bit flip:      %.4f%%\n", pct(r.p_detect_b_bitflip));
    std::printf("  detection, error in B, random value: >= %.4f%%\n", pct(r.p_detect_b_random));
    std::printf("  detection, error in C, bit flip:      %.4f%%\n", pct(r.p_detect_c_bitflip));
    std::printf("  detection, error in C, random value: >= %.4f%%\n", pct(r.p_detect_c_random));
    std::printf("EmbeddingBag d=%llu pooling=%llu\n", static_cast<unsigned long long>(v[3]),
                static_cast<unsigned long long>(v[4]));
    std::printf("  check overhead:  %.4f%%\n", pct(r.eb_overhead));
    std::printf("  memory overhead: %.4f%%\n", pct(r.eb_memory_overhead));
    return 0;
}

uint64_t bench_seed() {
    const char* env = std::getenv("ABFTLP_SEED");
    uint64_t s = 0;
    if (env && !to_u64(env, s)) {
        std::fprintf(stderr, "warning: ignoring malformed ABFTLP_SEED\n");
        s = 0;
    }
    return s;
}

int run_bench(const Args& a) {
    const auto get = [&](const char* k, const char* dflt) {
        const auto it = a.options.find(k);
        return it == a.options.end() ? std::string(dflt) : it->second;
    };
    const std::string shapes_path = get("shapes", "data/shapes.txt"), out_path = get("out", "");
    uint64_t reps = 0, eb_rows = 0;
    if (!to_u64(get("reps", "9"), reps) || !to_u64(get("eb-rows", "100000"), eb_rows))
        return usage("bench options must be integers");
    std::ifstream sf(shapes_path);
    if (!sf) {
        std::fprintf(stderr, "error: shape file not found: %s\n", shapes_path.c_str());
        return 1;
    }
    std::vector<std::array<uint64_t, 3>> shapes;
    for (std::string line; std::getline(sf, line);) {
        line = line.substr(0, line.find('#'));
        unsigned long long m = 0, n = 0, k = 0;
        char x1 = 0, x2 = 0;
        if (std::sscanf(line.c_str(), " %llu %c %llu %c %llu", &m, &x1, &n, &x2, &k) == 5) {
            if (x1 != 'x' || x2 != 'x') {
                std::fprintf(stderr, "error: bad shape line: %s\n", line.c_str());
                return 1;
            }
            shapes.push_back({m, n, k});
        }
    }
    if (shapes.empty()) {
        std::fprintf(stderr, "error: no shapes in %s\n", shapes_path.c_str());
        return 1;
    }
    const uint64_t seed = bench_seed();
    std::ostringstream csv;
    csv << "shape,baseline_ns,abft_ns,overhead_fraction,repetitions\n";
    for (const auto& s : shapes) {
        abftlp_bench_result r{};
        const abftlp_status st = abftlp_bench_gemm(s[0], s[1], s[2], static_cast<uint32_t>(reps), seed, &r);
        if (st != ABFTLP_OK) return report_failure(st, "bench gemm");
        csv << s[0] << 'x' << s[1] << 'x' << s[2] << ',' << r.baseline_ns << ',' << r.abft_ns << ',' << r.overhead_fraction
            << ',' << reps << '\n';
        std::printf("gemm %llux%llux%llu: overhead %.2f%%\n", static_cast<unsigned long long>(s[0]),
                    static_cast<unsigned long long>(s[1]), static_cast<unsigned long long>(s[2]), 100.0 * r.overhead_fraction);
    }
    for (uint64_t dim : {32ull, 64ull, 128ull, 256ull}) {
        abftlp_bench_result r{};
        const abftlp_status st = abftlp_bench_eb(eb_rows, dim, 100, 10, static_cast<uint32_t>(reps), seed, &r);
        if (st != ABFTLP_OK) return report_failure(st, "bench eb");
        csv << "eb_R" << eb_rows << "_d" << dim << "_p100_b10," << r.baseline_ns << ',' << r.abft_ns << ','
            << r.overhead_fraction << ',' << reps << '\n';
        std::printf("eb d=%llu: overhead %.2f%%\n", static_cast<unsigned long long>(dim), 100.0 * r.overhead_fraction);
    }
    if (out_path.empty()) {
        std::fputs(csv.str().c_str(), stdout);
        return 0;
    }
    std::ofstream of(out_path);
    if (!(of << csv.str())) {
        std::fprintf(stderr, "error: cannot write %s\n", out_path.c_str());
        return 1;
    }
    std::printf("results written to %s\n", out_path.c_str());
    return 0;
}

int run_eb_check(const Args& a) {
    if (a.positional.size() != 2) return usage("eb-check takes a table file and an indices file");
    uint64_t bags = 0, flagged = 0;
    char* text = nullptr;
    const abftlp_status st = abftlp_eb_check_files(a.positional[0].c_str(), a.positional[1].c_str(),
                                                   a.flags.count("skip-validation") ? 1 : 0, &bags, &flagged, &text);
    if (st != ABFTLP_OK) return report_failure(st, "eb-check");
    std::fputs(text, stdout);
    abftlp_string_free(text);
    std::printf("%llu/%llu bags flagged\n", static_cast<unsigned long long>(flagged), static_cast<unsigned long long>(bags));
    return flagged ? 2 : 0;
}

struct Command {
    const char* name;
    std::vector<std::string> valued;
    std::function<int(const Args&)> run;
};

}  // namespace

int main(int argc, char** argv) {
    const std::vector<Command> commands = {
        {"campaign", {"out"}, run_campaign},
        {"analyze", {"m", "n", "k", "d", "pool"}, run_analyze},
        {"bench", {"shapes", "reps", "out", "eb-rows"}, run_bench},
        {"eb-check", {}, run_eb_check},
    };
    if (argc < 2) return usage("a subcommand is required");
    for (const Command& c : commands) {
        if (std::strcmp(argv[1], c.name) != 0) continue;
        Args args;
        std::string err;
        if (!parse_args(argc, argv, 2, c.valued, args, err)) return usage(err.c_str());
        return c.run(args);
    }
    return usage((std::string("unknown subcommand ") + argv[1]).c_str());
}
