// Host side of the fault lab and the reference-compatible tooling: campaign configuration,
// GPU campaign driver, reports, benches, ABEB table files and bag files.
#pragma once
#include <cstdint>
#include <istream>
#include <optional>
#include <string>
#include <vector>

namespace abftk {

// ---- configuration (P:src/fault_lab.hpp:17-50)
enum class FaultTarget { weight_B, intermediate_C, eb_table, none };
enum class FaultModel { single_bit_flip, random_value };
enum class BitRange { all, high4, low4 };

struct FaultSpec {
    FaultTarget target = FaultTarget::none;
    FaultModel model = FaultModel::single_bit_flip;
    BitRange bitRange = BitRange::all;
    uint64_t seed = 0;
};
struct GemmShape {
    uint64_t m = 1, n = 1, k = 1;
};
struct GemmWorkload {
    std::vector<GemmShape> shapes;
    uint64_t trialsPerShape = 100;
};
struct EbWorkload {
    uint64_t tableRows = 100000, tableDim = 64, pooling = 100, batch = 10, trials = 200;
};
struct CampaignConfig {
    std::optional<GemmWorkload> gemm;
    std::optional<EbWorkload> eb;
    FaultSpec fault;
    uint64_t threads = 0;  // accepted for compatibility; trials run as GPU work
};

// ---- report (P:src/fault_lab.hpp:59-85)
struct ShapeStats {
    std::string label;
    uint64_t trials = 0, detected = 0, falsePositives = 0;
};
struct CampaignReport {
    std::string target, model, bitRange;
    uint64_t trials = 0, detected = 0, notDetected = 0, falsePositives = 0;
    std::vector<ShapeStats> perShape;
    std::string notes;
    double detectionRate() const { return trials ? double(detected) / double(trials) : 0.0; }
};
struct WilsonInterval {
    double low = 0.0, high = 0.0;
};

CampaignConfig parse_campaign_config(const std::string& text);  // hostio.cpp
const char* fault_target_name(FaultTarget t);                    // spellings of the config file / report
const char* fault_model_name(FaultModel m);
const char* bit_range_name(BitRange r);
CampaignReport run_campaign(const CampaignConfig& cfg);
CampaignReport run_gemm_campaign(const CampaignConfig& cfg);
CampaignReport run_eb_campaign(const CampaignConfig& cfg);
WilsonInterval wilson_interval(uint64_t successes, uint64_t trials);
std::string report_to_csv(const CampaignReport& r);
std::string report_to_table(const CampaignReport& r);

// ---- benches (P:src/bench.cpp:50-152)
struct BenchTimes {
    double baseline_ns = 0.0, abft_ns = 0.0;
};
BenchTimes bench_gemm(uint64_t m, uint64_t n, uint64_t k, uint64_t reps, uint64_t seed);
BenchTimes bench_eb(uint64_t rows, uint64_t dim, uint64_t pooling, uint64_t batch, uint64_t reps, uint64_t seed);

// ---- ABEB table files and bag files (P:src/embedding_abft.cpp:93-145, P:src/capi.cpp:195-227)
struct HostTable {
    uint64_t rows = 0;
    uint32_t dim = 0;
    std::vector<int8_t> data;
    std::vector<float> scales, biases;
    std::vector<int32_t> rowSums;
};
struct HostBags {
    std::vector<int64_t> offsets{0};
    std::vector<int64_t> indices;
    std::vector<float> weights;
    bool weighted = false;
};
struct EbResultHost {
    double rsum = 0.0, csum = 0.0;
    bool err = false;
};
HostTable load_table_file(const std::string& path);
void save_table_file(const HostTable& t, const std::string& path);
bool parse_bag_lines(std::istream& in, HostBags& bags, std::string& error);
std::vector<EbResultHost> check_bags_on_device(const HostTable& t, const HostBags& bags, bool validate);

}  // namespace abftk
