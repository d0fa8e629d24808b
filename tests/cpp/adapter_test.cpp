// C++ drop-in check: the reference's operator API (through include/abftlp_b200.hpp) on the GPU,
// exercised with the known answers the reference's own suites pin (cited per case). Prints one line per
// case and "ALL OK" at the end; exits non-zero on the first failure. Built by tests/cpp/Makefile and run by
// tests/test_adapter_gpu.py.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "abftlp_b200.hpp"

namespace A = abft_b200;
using A::MatI32;
using A::MatI8;
using A::MatU8;

static int g_fail = 0;
#define EXPECT(cond)                                                                    \
    do {                                                                                \
        if (!(cond)) {                                                                  \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);                 \
            ++g_fail;                                                                   \
        }                                                                               \
    } while (0)
template <typename E, typename F>
static bool throws(F f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

// Small counter-based generator for random inputs (same mixing function as the reference's SplitMix64).
struct Rng {
    uint64_t s;
    explicit Rng(uint64_t seed) : s(seed) {}
    uint64_t next() {
        uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        return z ^ (z >> 31);
    }
    int below(int n) { return static_cast<int>(next() % static_cast<uint64_t>(n)); }
};

static void gemm_cases() {
    using namespace A::gemm;
    using A::quant::IntermediateMatrix;
    using A::quant::QuantI8;
    using A::quant::QuantU8;
    // identity-A hand oracle + forced corruption (P:tests/test_gemm_abft.cpp:107-116)
    {
        QuantU8 a{MatU8(2, 2, {1, 0, 0, 1}), 1.0, 0.0};
        QuantI8 b{MatI8(2, 2, {3, 4, 5, 6}), 1.0, 0.0};
        AbftGemmResult res = abft_gemm(a, PackedEncodedWeight(b, compute_row_checksums(b)));
        EXPECT(res.errCount == 0);
        EXPECT(res.cTemp.data == MatI32(2, 3, {3, 4, 7, 5, 6, 11}));
        res.cTemp.data(0, 1) = 5;
        EXPECT(verify_checksums(res.cTemp) == 1);
        std::printf("gemm identity + forced corruption ok\n");
    }
    // row-level verify incl. aliasing (P:tests/test_gemm_abft.cpp:126-132)
    {
        IntermediateMatrix c{MatI32(3, 3, {3, 4, 7, 3, 4, 6, 200, 181, 0}), true};
        EXPECT(verify_checksums(c) == 1);
        IntermediateMatrix noCol{MatI32(1, 2, {1, 2}), false};
        EXPECT(throws<std::invalid_argument>([&] { verify_checksums(noCol); }));
        std::printf("verify rows ok\n");
    }
    // checksum examples and zero weights (P:tests/test_gemm_abft.cpp:40-51, 98-105)
    {
        QuantI8 b{MatI8(4, 3, {1, 2, 3, -1, -2, -3, 127, 127, 127, -128, -128, -128}), 1.0, 0.0};
        WeightChecksum cs = compute_row_checksums(b);
        for (int i = 0; i < 4; ++i) {
            int64_t s = 0;
            for (int j = 0; j < 3; ++j) s += b.data(i, j);
            EXPECT(cs.values[i] == mod127(s));
        }
        QuantU8 a{MatU8(3, 4, 7), 1.0, 0.0};
        QuantI8 z{MatI8(4, 2, 0), 1.0, 0.0};
        AbftGemmResult r = abft_gemm(a, PackedEncodedWeight(z, compute_row_checksums(z)));
        EXPECT(r.errCount == 0);
        for (int32_t v : r.cTemp.data.data()) EXPECT(v == 0);
        std::printf("checksums + zero weights ok\n");
    }
    // dimension mismatch, empty B, checksum length mismatch (P:tests/test_gemm_abft.cpp:86-96, 118-124)
    {
        QuantU8 a{MatU8(2, 3, 1), 1.0, 0.0};
        QuantI8 b{MatI8(4, 2, 1), 1.0, 0.0};
        EXPECT(throws<std::invalid_argument>([&] { abft_gemm(a, PackedEncodedWeight(b, compute_row_checksums(b))); }));
        QuantI8 e{MatI8(0, 0), 1.0, 0.0};
        EXPECT(throws<std::invalid_argument>([&] { compute_row_checksums(e); }));
        WeightChecksum bad{std::vector<int8_t>(3, 0)};
        EXPECT(throws<std::invalid_argument>([&] { PackedEncodedWeight(b, bad); }));
        std::printf("argument errors ok\n");
    }
    // random soundness + residue congruence + at() round trip + plain == checked columns
    {
        Rng rng(14);
        for (int t = 0; t < 20; ++t) {
            const int m = 1 + rng.below(70), k = 1 + rng.below(300), n = 1 + rng.below(90);
            QuantU8 a{MatU8(m, k), 1.0, 0.0};
            QuantI8 b{MatI8(k, n), 1.0, 0.0};
            for (auto& v : a.data.data()) v = static_cast<uint8_t>(rng.below(256));
            for (auto& v : b.data.data()) v = static_cast<int8_t>(rng.below(256) - 128);
            PackedEncodedWeight pb(b, compute_row_checksums(b));
            AbftGemmResult r = abft_gemm(a, pb);
            EXPECT(r.errCount == 0);
            for (int i = 0; i < m; ++i) {
                int64_t rs = 0;
                for (int j = 0; j < n; ++j) {
                    int64_t ref = 0;
                    for (int p = 0; p < k; ++p) ref += int64_t(a.data(i, p)) * b.data(p, j);
                    if (r.cTemp.data(i, j) != static_cast<int32_t>(ref)) {
                        EXPECT(false);
                        i = m;
                        break;
                    }
                    rs += ref;
                }
                if (i < m) EXPECT(mod127(rs) == mod127(r.cTemp.data(i, n)));
            }
            EXPECT(pb.at(k - 1, n - 1) == b.data(k - 1, n - 1));
            IntermediateMatrix plain = plain_gemm(a, b);
            for (int i = 0; i < m; ++i)
                for (int j = 0; j < n; ++j) EXPECT(plain.data(i, j) == r.cTemp.data(i, j));
            r.cTemp.data(rng.below(m), rng.below(n + 1)) ^= 1 << rng.below(31);
            EXPECT(verify_checksums(r.cTemp) == 1);  // a single flip is never congruent to 0 mod 127
        }
        std::printf("random soundness ok\n");
    }
}

static void eb_cases() {
    using namespace A::eb;
    Rng rng(32);
    auto random_table = [&](int R, int d) {
        QuantEmbeddingTable t;
        t.rows = MatI8(R, d);
        for (auto& v : t.rows.data()) v = static_cast<int8_t>(rng.below(256) - 128);
        for (int r = 0; r < R; ++r) {
            t.scales.push_back(0.001f + 0.009f * static_cast<float>(rng.below(1000)) / 1000.0f);
            t.biases.push_back(-1.0f + 2.0f * static_cast<float>(rng.below(1000)) / 1000.0f);
        }
        t.rowSums = precompute_row_sums(t.rows);
        return t;
    };
    // row sums (P:tests/test_embedding_abft.cpp:44-57)
    EXPECT(precompute_row_sums(MatI8(3, 4, 0)) == std::vector<int32_t>({0, 0, 0}));
    EXPECT(precompute_row_sums(MatI8(1, 3, {1, -1, 5})) == std::vector<int32_t>({5}));
    // empty bag, identity lookup, duplicate index (P:tests/test_embedding_abft.cpp:60-76)
    {
        QuantEmbeddingTable t = random_table(20, 8);
        for (float v : embedding_bag(t, IndexBag{})) EXPECT(v == 0.0f);
        t.scales[3] = 1.0f;
        t.biases[3] = 0.0f;
        auto single = embedding_bag(t, IndexBag{{3}, std::nullopt});
        for (int j = 0; j < 8; ++j) EXPECT(single[j] == static_cast<float>(t.rows(3, j)));
        auto twice = embedding_bag(t, IndexBag{{3, 3}, std::nullopt});
        for (int j = 0; j < 8; ++j) EXPECT(twice[j] == 2.0f * single[j]);
        EXPECT(throws<std::out_of_range>([&] { embedding_bag(t, IndexBag{{20}, std::nullopt}); }));
        EXPECT(throws<std::invalid_argument>([&] { abft_embedding_bag(t, IndexBag{{1, 2}, std::vector<float>{1.0f}}); }));
        std::printf("eb lookups ok\n");
    }
    // integer path exact, error-free under bound, sign flip detected (P:tests/test_embedding_abft.cpp:82-109)
    {
        QuantEmbeddingTable t = random_table(100, 16);
        std::fill(t.scales.begin(), t.scales.end(), 1.0f);
        std::fill(t.biases.begin(), t.biases.end(), 0.0f);
        IndexBag bag;
        for (int i = 0; i < 50; ++i) bag.indices.push_back(rng.below(100));
        EbCheckedResult r = abft_embedding_bag(t, bag);
        EXPECT(r.rSum == r.cSum);
        EXPECT(!r.err);
        QuantEmbeddingTable u = random_table(1000, 64);
        IndexBag b2;
        for (int i = 0; i < 100; ++i) b2.indices.push_back(rng.below(1000));
        EbCheckedResult r2 = abft_embedding_bag(u, b2);
        EXPECT(!r2.err);
        EXPECT(std::abs(r2.rSum - r2.cSum) <= kEbRelativeBound * std::max({std::abs(r2.rSum), std::abs(r2.cSum), 1.0}));
        const std::size_t victim = b2.indices[0];
        u.rows(victim, 5) = static_cast<int8_t>(u.rows(victim, 5) ^ 0x80);  // sign-bit flip after row sums
        EXPECT(abft_embedding_bag(u, b2).err);
        std::printf("eb check ok\n");
    }
    // ABEB round trip + validation (P:src/embedding_abft.cpp:93-145)
    {
        QuantEmbeddingTable t = random_table(50, 12);
        const std::string path = "/tmp/abftlp_adapter_test.abeb";
        save_table(t, path);
        QuantEmbeddingTable l = load_table(path);
        EXPECT(l.rows == t.rows && l.scales == t.scales && l.biases == t.biases && l.rowSums == t.rowSums);
        t.rowSums[7] += 1;
        save_table(t, path);
        EXPECT(throws<std::runtime_error>([&] { load_table(path); }));
        QuantEmbeddingTable stale = load_table(path, false);
        EXPECT(stale.rowSums[7] == t.rowSums[7]);
        std::remove(path.c_str());
        std::printf("eb table file ok\n");
    }
}

int main() {
    try {
        gemm_cases();
        eb_cases();
    } catch (const std::exception& e) {
        std::printf("FAIL exception: %s\n", e.what());
        return 2;
    }
    if (g_fail) {
        std::printf("%d failure(s)\n", g_fail);
        return 1;
    }
    std::printf("ALL OK\n");
    return 0;
}
