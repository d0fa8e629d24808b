// TEST INFRASTRUCTURE ONLY -- never linked into the product library.
//
// extern "C" wrappers around the *reference's own* C++ operators so the
// Python test-suite and bench.py's reference arm can call them through ctypes.
// This file contains no reference code: it includes the reference headers
// straight from /root/reference/proj/src (read-only) and is compiled together
// with the reference's own .cpp files by oracle/Makefile into
// oracle/_ref/libabftlp_ref.so.
//
// Wrapped reference entry points (file:line under /root/reference/proj):
//   compute_row_checksums, PackedEncodedWeight, abft_gemm, plain_gemm,
//   verify_checksums                        src/gemm_abft.hpp:23-74
//   precompute_row_sums, abft_embedding_bag src/embedding_abft.hpp:38-47
//   inject_weight_B / _intermediate_C / _eb_table  src/fault_lab.hpp:101-106
//   SplitMix64                              src/rng.hpp:10-43
//   requantize, row_sums, col_sums          src/quant.hpp:24-71
#include <cstdint>
#include <cstring>
#include <exception>
#include <optional>
#include <stdexcept>
#include <vector>

#include "embedding_abft.hpp"
#include "fault_lab.hpp"
#include "gemm_abft.hpp"
#include "quant.hpp"
#include "rng.hpp"

using namespace abft;

namespace {
template <typename Fn>
int guard(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const std::out_of_range&) {
        return -2;
    } catch (const std::invalid_argument&) {
        return -1;
    } catch (const std::exception&) {
        return -4;
    }
}

quant::QuantU8 make_a(const uint8_t* a, size_t m, size_t k) {
    return {MatU8(m, k, std::vector<uint8_t>(a, a + m * k)), 1.0, 0.0};
}
quant::QuantI8 make_b(const int8_t* b, size_t k, size_t n) {
    return {MatI8(k, n, std::vector<int8_t>(b, b + k * n)), 1.0, 0.0};
}

eb::QuantEmbeddingTable make_table(const int8_t* rows, size_t R, size_t d, const float* scales,
                                   const float* biases, const int32_t* rowSums) {
    eb::QuantEmbeddingTable t;
    t.rows = MatI8(R, d, std::vector<int8_t>(rows, rows + R * d));
    t.scales.assign(scales, scales + R);
    t.biases.assign(biases, biases + R);
    if (rowSums)
        t.rowSums.assign(rowSums, rowSums + R);
    else
        t.rowSums = eb::precompute_row_sums(t.rows);
    return t;
}

std::vector<eb::IndexBag> make_bags(const uint64_t* offsets, const uint64_t* indices,
                                    const float* weights, size_t nbags) {
    std::vector<eb::IndexBag> bags(nbags);
    for (size_t b = 0; b < nbags; ++b) {
        for (uint64_t t = offsets[b]; t < offsets[b + 1]; ++t) bags[b].indices.push_back(indices[t]);
        if (weights)
            bags[b].weights = std::vector<float>(weights + offsets[b], weights + offsets[b + 1]);
    }
    return bags;
}
}  // namespace

extern "C" {

void ref_splitmix64(uint64_t seed, uint64_t stream, uint64_t count, uint64_t* out) {
    lab::SplitMix64 rng(seed, stream);
    for (uint64_t i = 0; i < count; ++i) out[i] = rng.next();
}

int32_t ref_mod127(int64_t v) { return gemm::mod127(v); }

int ref_compute_row_checksums(const int8_t* b, size_t k, size_t n, int8_t* cs_out) {
    return guard([&] {
        auto cs = gemm::compute_row_checksums(make_b(b, k, n));
        std::memcpy(cs_out, cs.values.data(), cs.values.size());
    });
}

// Encoded weight handle: compute_row_checksums + PackedEncodedWeight, built once.
void* ref_gemm_weight_new(const int8_t* b, size_t k, size_t n) {
    try {
        auto qb = make_b(b, k, n);
        return new gemm::PackedEncodedWeight(qb, gemm::compute_row_checksums(qb));
    } catch (...) {
        return nullptr;
    }
}
void ref_gemm_weight_free(void* w) { delete static_cast<gemm::PackedEncodedWeight*>(w); }

// abft_gemm on a pre-encoded weight: cTemp is m x (n+1) row-major.
int ref_abft_gemm_w(const uint8_t* a, size_t m, size_t k, const void* w, int32_t* ctemp,
                    uint64_t* err_count) {
    return guard([&] {
        auto res = gemm::abft_gemm(make_a(a, m, k), *static_cast<const gemm::PackedEncodedWeight*>(w));
        std::memcpy(ctemp, res.cTemp.data.data().data(), res.cTemp.data.data().size() * 4);
        *err_count = res.errCount;
    });
}

int ref_abft_gemm(const uint8_t* a, size_t m, size_t k, const int8_t* b, size_t n, int32_t* ctemp,
                  uint64_t* err_count) {
    return guard([&] {
        auto qb = make_b(b, k, n);
        gemm::PackedEncodedWeight pb(qb, gemm::compute_row_checksums(qb));
        auto res = gemm::abft_gemm(make_a(a, m, k), pb);
        std::memcpy(ctemp, res.cTemp.data.data().data(), res.cTemp.data.data().size() * 4);
        *err_count = res.errCount;
    });
}

int ref_plain_gemm(const uint8_t* a, size_t m, size_t k, const int8_t* b, size_t n, int32_t* c) {
    return guard([&] {
        auto res = gemm::plain_gemm(make_a(a, m, k), make_b(b, k, n));
        std::memcpy(c, res.data.data().data(), res.data.data().size() * 4);
    });
}

// c is rows x cols row-major with the checksum column last (cols = n+1).
int ref_verify_checksums(const int32_t* c, size_t rows, size_t cols, uint64_t* err_count) {
    return guard([&] {
        quant::IntermediateMatrix im{MatI32(rows, cols, std::vector<int32_t>(c, c + rows * cols)), true};
        *err_count = gemm::verify_checksums(im);
    });
}

int ref_precompute_row_sums(const int8_t* rows, size_t R, size_t d, int32_t* out) {
    return guard([&] {
        auto s = eb::precompute_row_sums(MatI8(R, d, std::vector<int8_t>(rows, rows + R * d)));
        std::memcpy(out, s.data(), s.size() * 4);
    });
}

// batch_abft_eb over CSR bags. row_sums may be null (then precomputed).
// r_out: nbags x d floats.
int ref_batch_abft_eb(const int8_t* rows, size_t R, size_t d, const float* scales,
                      const float* biases, const int32_t* row_sums, const uint64_t* offsets,
                      const uint64_t* indices, const float* weights, size_t nbags, float* r_out,
                      double* rsum, double* csum, uint8_t* err) {
    return guard([&] {
        auto t = make_table(rows, R, d, scales, biases, row_sums);
        auto bags = make_bags(offsets, indices, weights, nbags);
        auto res = eb::batch_abft_eb(t, bags);
        for (size_t b = 0; b < nbags; ++b) {
            std::memcpy(r_out + b * d, res[b].r.data(), d * 4);
            rsum[b] = res[b].rSum;
            csum[b] = res[b].cSum;
            err[b] = res[b].err ? 1 : 0;
        }
    });
}

// Unchecked lookups (embedding_bag) for the baseline timing.
int ref_batch_eb(const int8_t* rows, size_t R, size_t d, const float* scales, const float* biases,
                 const uint64_t* offsets, const uint64_t* indices, const float* weights,
                 size_t nbags, float* r_out) {
    return guard([&] {
        auto t = make_table(rows, R, d, scales, biases, nullptr);
        auto bags = make_bags(offsets, indices, weights, nbags);
        for (size_t b = 0; b < nbags; ++b) {
            auto r = eb::embedding_bag(t, bags[b]);
            std::memcpy(r_out + b * d, r.data(), d * 4);
        }
    });
}

// Persistent table handle so timing loops do not re-copy the table.
void* ref_eb_table_new(const int8_t* rows, size_t R, size_t d, const float* scales,
                       const float* biases) {
    try {
        return new eb::QuantEmbeddingTable(make_table(rows, R, d, scales, biases, nullptr));
    } catch (...) {
        return nullptr;
    }
}
void ref_eb_table_free(void* t) { delete static_cast<eb::QuantEmbeddingTable*>(t); }

// Checked lookups for bags [b0, b1) of a CSR batch on a persistent table.
int ref_eb_table_check_range(const void* table, const uint64_t* offsets, const uint64_t* indices,
                             const float* weights, size_t b0, size_t b1, float* r_out,
                             uint8_t* err) {
    return guard([&] {
        const auto& t = *static_cast<const eb::QuantEmbeddingTable*>(table);
        const size_t d = t.dim();
        eb::IndexBag bag;
        for (size_t b = b0; b < b1; ++b) {
            bag.indices.assign(indices + offsets[b], indices + offsets[b + 1]);
            if (weights)
                bag.weights = std::vector<float>(weights + offsets[b], weights + offsets[b + 1]);
            else
                bag.weights.reset();
            auto res = eb::abft_embedding_bag(t, bag);
            std::memcpy(r_out + b * d, res.r.data(), d * 4);
            err[b] = res.err ? 1 : 0;
        }
    });
}

// Fault injectors: target 0 weight_B, 1 intermediate_C, 2 eb_table, 3 none;
// model 0 single_bit_flip, 1 random_value; range 0 all, 1 high4, 2 low4.
// rec = {injected, i, j, before, after}.
static lab::FaultSpec spec_of(int target, int model, int range, uint64_t seed) {
    lab::FaultSpec s;
    s.target = static_cast<lab::FaultTarget>(target);
    s.model = model == 0 ? abft::model::FaultModel::single_bit_flip
                         : abft::model::FaultModel::random_value;
    s.bitRange = static_cast<lab::BitRange>(range);
    s.seed = seed;
    return s;
}

int ref_inject_weight_B(int8_t* b, size_t k, size_t n, int target, int model, int range,
                        uint64_t seed, uint64_t trial, int64_t* rec) {
    return guard([&] {
        MatI8 mb(k, n, std::vector<int8_t>(b, b + k * n));
        auto r = lab::inject_weight_B(mb, spec_of(target, model, range, seed), trial);
        std::memcpy(b, mb.data().data(), k * n);
        rec[0] = r.injected;
        rec[1] = r.before;
        rec[2] = r.after;
    });
}

int ref_inject_intermediate_C(int32_t* c, size_t rows, size_t cols, int target, int model,
                              int range, uint64_t seed, uint64_t trial, int64_t* rec) {
    return guard([&] {
        quant::IntermediateMatrix im{MatI32(rows, cols, std::vector<int32_t>(c, c + rows * cols)), true};
        auto r = lab::inject_intermediate_C(im, spec_of(target, model, range, seed), trial);
        std::memcpy(c, im.data.data().data(), rows * cols * 4);
        rec[0] = r.injected;
        rec[1] = r.before;
        rec[2] = r.after;
    });
}

int ref_inject_eb_table(int8_t* rows, size_t R, size_t d, const uint64_t* offsets,
                        const uint64_t* indices, size_t nbags, int target, int model, int range,
                        uint64_t seed, uint64_t trial, int64_t* rec) {
    return guard([&] {
        std::vector<float> ones(R, 1.0f), zeros(R, 0.0f);
        auto t = make_table(rows, R, d, ones.data(), zeros.data(), nullptr);
        auto bags = make_bags(offsets, indices, nullptr, nbags);
        auto r = lab::inject_eb_table(t, bags, spec_of(target, model, range, seed), trial);
        std::memcpy(rows, t.rows.data().data(), R * d);
        rec[0] = r.injected;
        rec[1] = r.before;
        rec[2] = r.after;
    });
}


int ref_requantize(const int32_t* c, size_t m, size_t n, int with_cs, const int32_t* rs, const int32_t* cs,
                   const double* prm, uint64_t k, uint8_t* out) {
    return guard([&] {
        quant::IntermediateMatrix im;
        const size_t cols = n + (with_cs ? 1 : 0);
        im.data = MatI32(m, cols, std::vector<int32_t>(c, c + m * cols));
        im.hasChecksumColumn = with_cs != 0;
        quant::RequantParams p{prm[0], prm[1], prm[2], prm[3], prm[4], prm[5], static_cast<std::size_t>(k)};
        quant::QuantU8 q = quant::requantize(im, std::vector<int32_t>(rs, rs + m), std::vector<int32_t>(cs, cs + n), p);
        std::memcpy(out, q.data.data().data(), m * n);
    });
}

void ref_row_sums_u8(const uint8_t* a, size_t m, size_t k, int32_t* out) {
    auto v = quant::row_sums(MatU8(m, k, std::vector<uint8_t>(a, a + m * k)));
    std::memcpy(out, v.data(), m * 4);
}

void ref_col_sums_i8(const int8_t* b, size_t k, size_t n, int32_t* out) {
    auto v = quant::col_sums(MatI8(k, n, std::vector<int8_t>(b, b + k * n)));
    std::memcpy(out, v.data(), n * 4);
}
}  // extern "C"
