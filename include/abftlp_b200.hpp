/*
 * abftlp_b200.hpp -- C++ operator adapter over the B200 C ABI (header-only).
 *
 * Mirrors the reference's C++ operator API (P:src/gemm_abft.hpp:10-74, P:src/embedding_abft.hpp:14-52,
 * P:src/quant.hpp:11-44, P:src/matrix.hpp:11-44) name for name, with host matrices in and out, so code
 * written against `namespace abft` switches to the GPU by swapping the namespace (`namespace abft =
 * abft_b200;`). Every operator runs on the GPU through include/abftlp.h + include/abftlp_b200.h; this
 * header only moves host data (H2D/D2H) and maps status codes back to the reference's exception types
 * (invalid_argument / out_of_range / runtime_error, P:src/capi.cpp:28-41 in reverse). Performance work
 * belongs on the device-pointer ABI; this adapter exists for drop-in use and for parity tests.
 *
 * Link: -labftlp_b200 -lcudart (the library itself links the CUDA runtime statically).
 */
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <fstream>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "abftlp_b200.h"

namespace abft_b200 {

// ------------------------------------------------------------------ plumbing
namespace detail {
inline void check(abftlp_status s) {
    if (s == ABFTLP_OK) return;
    const std::string msg = abftlp_last_error() ? abftlp_last_error() : "abftlp error";
    if (s == ABFTLP_ERR_INVALID_ARGUMENT) {
        if (msg.find("out of range") != std::string::npos) throw std::out_of_range(msg);
        throw std::invalid_argument(msg);
    }
    throw std::runtime_error(msg);
}
inline void cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}
// RAII device buffer
struct DBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DBuf() = default;
    explicit DBuf(size_t n) : bytes(n) {
        if (n) cuda(cudaMalloc(&p, n), "cudaMalloc");
    }
    DBuf(const void* host, size_t n) : DBuf(n) {
        if (n) cuda(cudaMemcpy(p, host, n, cudaMemcpyHostToDevice), "cudaMemcpy H2D");
    }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr; o.bytes = 0; }
    DBuf& operator=(DBuf&& o) noexcept {
        if (this != &o) {
            if (p) cudaFree(p);
            p = o.p;
            bytes = o.bytes;
            o.p = nullptr;
            o.bytes = 0;
        }
        return *this;
    }
    ~DBuf() {
        if (p) cudaFree(p);
    }
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
    void to_host(void* dst, size_t n) const {
        if (n) cuda(cudaMemcpy(dst, p, n, cudaMemcpyDeviceToHost), "cudaMemcpy D2H");
    }
};
}  // namespace detail

// ------------------------------------------------------------------ containers (P:src/matrix.hpp, P:src/quant.hpp)
template <typename T>
class Mat {
public:
    Mat() = default;
    Mat(std::size_t rows, std::size_t cols, T fill = T{}) : rows_(rows), cols_(cols), data_(rows * cols, fill) {}
    Mat(std::size_t rows, std::size_t cols, std::vector<T> data) : rows_(rows), cols_(cols), data_(std::move(data)) {
        if (data_.size() != rows_ * cols_) throw std::invalid_argument("matrix data size does not match dimensions");
    }
    std::size_t rows() const { return rows_; }
    std::size_t cols() const { return cols_; }
    bool empty() const { return data_.empty(); }
    T& operator()(std::size_t i, std::size_t j) { return data_[i * cols_ + j]; }
    const T& operator()(std::size_t i, std::size_t j) const { return data_[i * cols_ + j]; }
    std::vector<T>& data() { return data_; }
    const std::vector<T>& data() const { return data_; }
    bool operator==(const Mat& o) const { return rows_ == o.rows_ && cols_ == o.cols_ && data_ == o.data_; }

private:
    std::size_t rows_ = 0, cols_ = 0;
    std::vector<T> data_;
};
using MatI32 = Mat<std::int32_t>;
using MatI8 = Mat<std::int8_t>;
using MatU8 = Mat<std::uint8_t>;

namespace quant {
template <typename T>
struct QuantizedMatrix {
    Mat<T> data;
    double scale = 1.0;
    double bias = 0.0;
    std::size_t rows() const { return data.rows(); }
    std::size_t cols() const { return data.cols(); }
};
using QuantU8 = QuantizedMatrix<std::uint8_t>;
using QuantI8 = QuantizedMatrix<std::int8_t>;
struct IntermediateMatrix {
    MatI32 data;
    bool hasChecksumColumn = false;
    std::size_t rows() const { return data.rows(); }
    std::size_t logicalCols() const { return hasChecksumColumn ? data.cols() - 1 : data.cols(); }
};
}  // namespace quant

// ------------------------------------------------------------------ GEMM (P:src/gemm_abft.hpp:10-74)
namespace gemm {

inline constexpr std::int32_t kChecksumMod = 127;
inline std::int32_t mod127(std::int64_t v) {
    const std::int64_t r = v % kChecksumMod;
    return static_cast<std::int32_t>(r < 0 ? r + kChecksumMod : r);
}

struct WeightChecksum {
    std::vector<std::int8_t> values;
};

// The device layout is fixed by the kernel (K-block-major); the reference's
// BlockLayout is accepted for signature compatibility and validated, not used.
struct BlockLayout {
    std::size_t rowBlock = 64;
    std::size_t colBlock = 16;
};

// B (+ checksums) encoded on the device once; immutable, shareable across threads/streams.
class PackedEncodedWeight {
public:
    PackedEncodedWeight(const quant::QuantI8& b, const WeightChecksum& cs, BlockLayout layout = {})
        : k_(b.rows()), n_(b.cols()), layout_(layout), scale_(b.scale), bias_(b.bias) {
        if (layout.rowBlock == 0 || layout.colBlock == 0)
            throw std::invalid_argument("PackedEncodedWeight: block sizes must be positive");
        if (cs.values.size() != k_) throw std::invalid_argument("PackedEncodedWeight: checksum length mismatch");
        if (b.data.empty()) throw std::invalid_argument("compute_row_checksums: empty matrix");
        detail::DBuf db(b.data.data().data(), k_ * n_);
        detail::check(abftlp_gemm_encode(db.as<int8_t>(), k_, n_, n_, nullptr, &w_));
        detail::DBuf dcs(cs.values.data(), k_);
        detail::check(abftlp_gemm_weight_set_checksums(w_, dcs.as<int8_t>(), nullptr));
        detail::cuda(cudaDeviceSynchronize(), "encode");
    }
    PackedEncodedWeight(const PackedEncodedWeight&) = delete;
    PackedEncodedWeight& operator=(const PackedEncodedWeight&) = delete;
    PackedEncodedWeight(PackedEncodedWeight&& o) noexcept
        : k_(o.k_), n_(o.n_), layout_(o.layout_), scale_(o.scale_), bias_(o.bias_), w_(o.w_),
          logical_(std::move(o.logical_)), blocked_(std::move(o.blocked_)) {
        o.w_ = nullptr;
    }
    ~PackedEncodedWeight() { abftlp_gemm_weight_free(w_); }

    std::size_t k() const { return k_; }
    std::size_t n() const { return n_; }
    const BlockLayout& layout() const { return layout_; }
    double scale() const { return scale_; }
    double bias() const { return bias_; }
    // Element of the logical k x (n+1) encoded matrix (reads the device copy once, then caches).
    std::int8_t at(std::size_t i, std::size_t j) const {
        if (i >= k_ || j > n_) throw std::out_of_range("PackedEncodedWeight::at: index out of range");
        if (logical_.empty()) {
            detail::DBuf d(k_ * (n_ + 1));
            detail::check(abftlp_gemm_weight_read(w_, d.as<int8_t>(), nullptr));
            logical_.resize(k_ * (n_ + 1));
            d.to_host(logical_.data(), logical_.size());
        }
        return logical_[i * (n_ + 1) + j];
    }
    // Host view of [B | cs] in the caller's BlockLayout -- the reference's buffer format (P:src/gemm_abft.hpp:46-48):
    // blocks in row-major order over (row block, column block), rowBlock x colBlock cells each, row-major inside a
    // block, zero padding. Built on first use from the device copy; the device layout itself is fixed.
    std::size_t rowBlocks() const { return (k_ + layout_.rowBlock - 1) / layout_.rowBlock; }
    std::size_t colBlocks() const { return (n_ + 1 + layout_.colBlock - 1) / layout_.colBlock; }
    const std::vector<std::int8_t>& buffer() const {
        if (blocked_.empty()) {
            const std::size_t rb = layout_.rowBlock, cb = layout_.colBlock, cbs = colBlocks();
            blocked_.assign(rowBlocks() * cbs * rb * cb, 0);
            for (std::size_t i = 0; i < k_; ++i)
                for (std::size_t j = 0; j <= n_; ++j)
                    blocked_[((i / rb) * cbs + j / cb) * rb * cb + (i % rb) * cb + j % cb] = at(i, j);
        }
        return blocked_;
    }
    const abftlp_gemm_weight* handle() const { return w_; }
    abftlp_gemm_weight* handle() { return w_; }

private:
    std::size_t k_ = 0, n_ = 0;
    BlockLayout layout_;
    double scale_ = 1.0, bias_ = 0.0;
    abftlp_gemm_weight* w_ = nullptr;
    mutable std::vector<std::int8_t> logical_;
    mutable std::vector<std::int8_t> blocked_;
};

struct AbftGemmResult {
    quant::IntermediateMatrix cTemp;  // m x (n+1), checksum column last
    std::size_t errCount = 0;
};

inline WeightChecksum compute_row_checksums(const quant::QuantI8& b) {
    if (b.data.empty()) throw std::invalid_argument("compute_row_checksums: empty matrix");
    detail::DBuf db(b.data.data().data(), b.rows() * b.cols());
    abftlp_gemm_weight* w = nullptr;
    detail::check(abftlp_gemm_encode(db.as<int8_t>(), b.rows(), b.cols(), b.cols(), nullptr, &w));
    WeightChecksum cs;
    cs.values.resize(b.rows());
    detail::DBuf dcs(b.rows());
    const abftlp_status s = abftlp_gemm_weight_checksums(w, dcs.as<int8_t>(), nullptr);
    abftlp_gemm_weight_free(w);
    detail::check(s);
    dcs.to_host(cs.values.data(), cs.values.size());
    return cs;
}

// Row-checksum verified product: the result is returned even when rows are flagged.
inline AbftGemmResult abft_gemm(const quant::QuantU8& a, const PackedEncodedWeight& pb) {
    if (a.cols() != pb.k()) throw std::invalid_argument("abft_gemm: dimension mismatch");
    const std::size_t m = a.rows(), n = pb.n();
    AbftGemmResult r;
    r.cTemp.hasChecksumColumn = true;
    r.cTemp.data = MatI32(m, n + 1);
    if (m == 0) return r;
    std::vector<int32_t> csum(m);
    uint32_t err = 0;
    detail::check(abftlp_gemm_checked_host(a.data.data().data(), m, a.cols(), pb.handle(), r.cTemp.data.data().data(),
                                           n + 1, csum.data(), nullptr, &err, nullptr));
    for (std::size_t i = 0; i < m; ++i) r.cTemp.data(i, n) = csum[i];
    r.errCount = err;
    return r;
}

// Unchecked baseline over the same kernel (checking compiled out).
inline quant::IntermediateMatrix plain_gemm(const quant::QuantU8& a, const quant::QuantI8& b, BlockLayout layout = {}) {
    if (a.cols() != b.rows()) throw std::invalid_argument("plain_gemm: dimension mismatch");
    if (layout.rowBlock == 0 || layout.colBlock == 0)
        throw std::invalid_argument("PackedEncodedWeight: block sizes must be positive");
    const std::size_t m = a.rows(), k = b.rows(), n = b.cols();
    quant::IntermediateMatrix c;
    c.data = MatI32(m, n);
    if (m == 0 || n == 0) return c;
    detail::DBuf db(b.data.data().data(), k * n);
    abftlp_gemm_weight* w = nullptr;
    detail::check(abftlp_gemm_encode(db.as<int8_t>(), k, n, n, nullptr, &w));
    detail::DBuf da(a.data.data().data(), m * k), dc(m * n * 4);
    const abftlp_status s = abftlp_gemm_unchecked(da.as<uint8_t>(), m, k, w, dc.as<int32_t>(), n, nullptr);
    abftlp_gemm_weight_free(w);
    detail::check(s);
    dc.to_host(c.data.data().data(), m * n * 4);
    return c;
}

inline std::size_t verify_checksums(const quant::IntermediateMatrix& c) {
    if (!c.hasChecksumColumn || c.data.cols() == 0)
        throw std::invalid_argument("verify_checksums: missing checksum column");
    const std::size_t m = c.data.rows(), cols = c.data.cols();
    if (m == 0) return 0;
    detail::DBuf dc(c.data.data().data(), m * cols * 4), cnt(4);
    detail::check(abftlp_gemm_verify(dc.as<int32_t>(), cols, dc.as<int32_t>() + (cols - 1), cols, m, cols - 1, nullptr,
                                     cnt.as<uint32_t>(), nullptr));
    uint32_t h = 0;
    cnt.to_host(&h, 4);
    return h;
}

}  // namespace gemm

// ------------------------------------------------------------------ EmbeddingBag (P:src/embedding_abft.hpp:14-52)
namespace eb {

struct QuantEmbeddingTable {
    MatI8 rows;                         // R x d
    std::vector<float> scales;          // per row
    std::vector<float> biases;          // per row
    std::vector<std::int32_t> rowSums;  // exact integer row sums
    std::size_t numRows() const { return rows.rows(); }
    std::size_t dim() const { return rows.cols(); }
};

struct IndexBag {
    std::vector<std::size_t> indices;
    std::optional<std::vector<float>> weights;
};

struct EbCheckedResult {
    std::vector<float> r;
    double rSum = 0.0;
    double cSum = 0.0;
    bool err = false;
};

inline constexpr double kEbRelativeBound = 1e-5;

// A table resident on the device (rows, scale/bias, the table's stored row sums). Build once and pass
// to the batch overloads to avoid re-uploading per call.
class DeviceTable {
public:
    explicit DeviceTable(const QuantEmbeddingTable& t)
        : rows_(t.rows.data().data(), t.numRows() * t.dim()), sc_(t.scales.data(), 4 * t.numRows()),
          bi_(t.biases.data(), 4 * t.numRows()), R_(t.numRows()), d_(t.dim()) {
        if (t.scales.size() != R_ || t.biases.size() != R_) throw std::invalid_argument("table: per-row vector size");
        const int32_t* sums = nullptr;
        detail::DBuf dsums;
        if (!t.rowSums.empty()) {
            if (t.rowSums.size() != R_) throw std::invalid_argument("table: rowSums size");
            dsums = detail::DBuf(t.rowSums.data(), 4 * R_);
            sums = dsums.as<int32_t>();
        }
        detail::check(abftlp_eb_table_create(ABFTLP_EB_S8, rows_.p, R_, d_, d_, ABFTLP_EB_SCALE_F32, sc_.p, bi_.p, sums,
                                             nullptr, &t_));
        detail::cuda(cudaDeviceSynchronize(), "table");
    }
    DeviceTable(const DeviceTable&) = delete;
    DeviceTable& operator=(const DeviceTable&) = delete;
    ~DeviceTable() { abftlp_eb_table_free(t_); }
    const abftlp_eb_table* handle() const { return t_; }
    std::size_t numRows() const { return R_; }
    std::size_t dim() const { return d_; }

private:
    detail::DBuf rows_, sc_, bi_;
    std::size_t R_, d_;
    abftlp_eb_table* t_ = nullptr;
};

inline std::vector<std::int32_t> precompute_row_sums(const MatI8& rows) {
    std::vector<std::int32_t> sums(rows.rows(), 0);
    if (rows.rows() == 0) return sums;
    if (rows.cols() == 0) return sums;
    detail::DBuf dr(rows.data().data(), rows.rows() * rows.cols()), one(4 * rows.rows()), out(4 * rows.rows());
    std::vector<float> ones(rows.rows(), 1.0f);
    detail::cuda(cudaMemcpy(one.p, ones.data(), 4 * rows.rows(), cudaMemcpyHostToDevice), "cudaMemcpy");
    abftlp_eb_table* t = nullptr;
    detail::check(abftlp_eb_table_create(ABFTLP_EB_S8, dr.p, rows.rows(), rows.cols(), rows.cols(), ABFTLP_EB_SCALE_F32,
                                         one.p, one.p, nullptr, nullptr, &t));
    const abftlp_status s = abftlp_eb_table_row_sums(t, out.as<int32_t>(), nullptr);
    abftlp_eb_table_free(t);
    detail::check(s);
    out.to_host(sums.data(), 4 * sums.size());
    return sums;
}

inline std::vector<EbCheckedResult> batch_abft_eb(const DeviceTable& table, const std::vector<IndexBag>& bags,
                                                  bool checked = true) {
    const std::size_t B = bags.size(), d = table.dim();
    std::vector<int64_t> offsets(B + 1, 0);
    std::vector<int64_t> indices;
    std::vector<float> weights;
    bool any_w = false;
    for (const IndexBag& bag : bags) any_w |= bag.weights.has_value();
    for (std::size_t b = 0; b < B; ++b) {
        const IndexBag& bag = bags[b];
        for (std::size_t idx : bag.indices)  // check_bag order: index range first (P:src/embedding_abft.cpp:16-22)
            if (idx >= table.numRows()) throw std::out_of_range("embedding_bag: index out of range");
        if (bag.weights && bag.weights->size() != bag.indices.size())
            throw std::invalid_argument("embedding_bag: weights length mismatch");
        for (std::size_t t = 0; t < bag.indices.size(); ++t) {
            indices.push_back(static_cast<int64_t>(bag.indices[t]));
            if (any_w) weights.push_back(bag.weights ? (*bag.weights)[t] : 1.0f);  // unweighted: w = 1.0f
        }
        offsets[b + 1] = static_cast<int64_t>(indices.size());
    }
    std::vector<EbCheckedResult> res(B);
    if (B == 0) return res;
    if (indices.empty()) indices.push_back(0);  // a valid (never read) pointer for all-empty batches
    detail::DBuf doff(offsets.data(), 8 * (B + 1)), didx(indices.data(), 8 * indices.size()),
        dw(weights.data(), 4 * weights.size()), dout(4 * B * (d ? d : 1)), dfl(B), drs(8 * B), dcs(8 * B);
    if (checked)
        detail::check(abftlp_eb_checked(table.handle(), doff.as<int64_t>(), didx.as<int64_t>(), B,
                                        any_w ? dw.as<float>() : nullptr, dout.as<float>(), d, dfl.as<uint8_t>(),
                                        drs.as<double>(), dcs.as<double>(), nullptr, nullptr, nullptr));
    else
        detail::check(abftlp_eb_unchecked(table.handle(), doff.as<int64_t>(), didx.as<int64_t>(), B,
                                          any_w ? dw.as<float>() : nullptr, dout.as<float>(), d, nullptr, nullptr));
    std::vector<float> out(B * d);
    dout.to_host(out.data(), 4 * out.size());
    std::vector<uint8_t> fl(B, 0);
    std::vector<double> rs(B, 0.0), cs(B, 0.0);
    if (checked) {
        dfl.to_host(fl.data(), B);
        drs.to_host(rs.data(), 8 * B);
        dcs.to_host(cs.data(), 8 * B);
    }
    for (std::size_t b = 0; b < B; ++b) {
        res[b].r.assign(out.begin() + b * d, out.begin() + (b + 1) * d);
        res[b].rSum = rs[b];
        res[b].cSum = cs[b];
        res[b].err = fl[b] != 0;
    }
    return res;
}

inline std::vector<EbCheckedResult> batch_abft_eb(const QuantEmbeddingTable& table, const std::vector<IndexBag>& bags) {
    DeviceTable dt(table);
    return batch_abft_eb(dt, bags, true);
}
inline EbCheckedResult abft_embedding_bag(const QuantEmbeddingTable& table, const IndexBag& bag) {
    return batch_abft_eb(table, std::vector<IndexBag>{bag}).front();
}
inline std::vector<float> embedding_bag(const QuantEmbeddingTable& table, const IndexBag& bag) {
    DeviceTable dt(table);
    return batch_abft_eb(dt, std::vector<IndexBag>{bag}, false).front().r;
}

// ABEB container: "ABEB", u16 version 1, u64 R, u32 d, R x (d int8, f32 scale, f32 bias), R x i32 row sums;
// little-endian (format of P:src/embedding_abft.hpp:48-50). Row-sum validation runs on the device.
inline void save_table(const QuantEmbeddingTable& t, const std::string& path) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error("cannot open table file for writing: " + path);
    const uint16_t ver = 1;
    const uint64_t R = t.numRows();
    const uint32_t d = static_cast<uint32_t>(t.dim());
    out.write("ABEB", 4);
    out.write(reinterpret_cast<const char*>(&ver), 2);
    out.write(reinterpret_cast<const char*>(&R), 8);
    out.write(reinterpret_cast<const char*>(&d), 4);
    for (uint64_t r = 0; r < R; ++r) {
        out.write(reinterpret_cast<const char*>(&t.rows(r, 0)), d);
        out.write(reinterpret_cast<const char*>(&t.scales[r]), 4);
        out.write(reinterpret_cast<const char*>(&t.biases[r]), 4);
    }
    out.write(reinterpret_cast<const char*>(t.rowSums.data()), 4 * static_cast<std::streamsize>(R));
    if (!out) throw std::runtime_error("failed writing table file: " + path);
}

inline QuantEmbeddingTable load_table(const std::string& path, bool validateRowSums = true) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("cannot open table file: " + path);
    auto rd = [&](void* p, std::size_t n) {
        in.read(static_cast<char*>(p), static_cast<std::streamsize>(n));
        if (!in) throw std::runtime_error("table file truncated");
    };
    char magic[4];
    uint16_t ver = 0;
    uint64_t R = 0;
    uint32_t d = 0;
    in.read(magic, 4);
    if (!in || std::memcmp(magic, "ABEB", 4) != 0) throw std::runtime_error("not an embedding table file: " + path);
    rd(&ver, 2);
    if (ver != 1) throw std::runtime_error("unsupported table file version");
    rd(&R, 8);
    rd(&d, 4);
    if (R == 0 || d == 0) throw std::runtime_error("table file has empty dimensions");
    QuantEmbeddingTable t;
    t.rows = MatI8(R, d);
    t.scales.resize(R);
    t.biases.resize(R);
    t.rowSums.resize(R);
    for (uint64_t r = 0; r < R; ++r) {
        rd(&t.rows(r, 0), d);
        rd(&t.scales[r], 4);
        rd(&t.biases[r], 4);
    }
    rd(t.rowSums.data(), 4 * R);
    if (validateRowSums) {
        DeviceTable dt(QuantEmbeddingTable{t.rows, t.scales, t.biases, {}});
        detail::DBuf ds(t.rowSums.data(), 4 * R);
        uint64_t bad = 0;
        detail::check(abftlp_eb_table_validate(dt.handle(), ds.as<int32_t>(), nullptr, &bad));
        if (bad) throw std::runtime_error("table row-sum checksums do not match contents");
    }
    return t;
}

}  // namespace eb
}  // namespace abft_b200
