// sfd_gpu.hpp -- header-only C++ drop-in over the sfdg C ABI.
//
// Mirrors the reference interface so a caller of sfd::SfdSketcher switches by changing
// the include and the namespace (reference: core/include/sfd/sketch.hpp:9-71,
// shrink.hpp:11-41, sparse.hpp:12-15, dense_matrix.hpp:10-30, common.hpp:14-17):
//
//   sfd_gpu::SketchConfig cfg; cfg.ell = 100; cfg.d = 10000; cfg.seed = 1;
//   sfd_gpu::SfdSketcher s(cfg);          // throws std::invalid_argument like the reference
//   for (auto& row : rows) s.append(row); // SparseRow {indices, values}
//   sfd_gpu::DenseMatrix b = s.finalize();
//
// Exceptions: SFDG_INVALID_ARGUMENT -> std::invalid_argument,
// SFDG_NUMERICAL_ERROR -> sfd_gpu::numerical_error (the reference's sfd::numerical_error),
// SFDG_CUDA_ERROR -> std::runtime_error. Link with paper_1602_00412_b200/libsfdg.so.
#pragma once

#include <cstddef>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "sfdg.h"

namespace sfd_gpu {

class numerical_error : public std::runtime_error {
  public:
    explicit numerical_error(const std::string& what) : std::runtime_error(what) {}
};

inline void check(int code) {
    if (code == SFDG_OK) return;
    const std::string msg = sfdg_last_error();
    if (code == SFDG_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    if (code == SFDG_NUMERICAL_ERROR) throw numerical_error(msg);
    throw std::runtime_error(msg);
}

struct DenseMatrix {  // dense_matrix.hpp:10-30
    std::size_t rows = 0;
    std::size_t cols = 0;
    std::vector<double> data;  // row-major
    DenseMatrix() = default;
    DenseMatrix(std::size_t r, std::size_t c) : rows(r), cols(c), data(r * c, 0.0) {}
    double& operator()(std::size_t i, std::size_t j) { return data[i * cols + j]; }
    double operator()(std::size_t i, std::size_t j) const { return data[i * cols + j]; }
};

struct SparseRow {  // sparse.hpp:12-15
    std::vector<std::uint32_t> indices;
    std::vector<double> values;
};

struct PowerConfig {  // randsvd.hpp:10-14
    double epsilon = 0.25;
    double q_constant = 1.0;
    std::optional<std::size_t> q_override;
    sfdg_power_config c() const {
        return {epsilon, q_constant, q_override ? static_cast<int64_t>(*q_override) : int64_t(-1)};
    }
};

struct SketchConfig {  // sketch.hpp:9-17
    std::size_t ell = 0;
    std::size_t d = 0;
    double delta = 0.1;
    PowerConfig power;
    std::uint64_t seed = 0;
};

struct VerifierState {  // shrink.hpp:11-16
    std::size_t i = 0;
    double delta = 0.1;
    double c_verify = 2.0;
    double delta_spent = 0.0;
};

class SfdSketcher {  // sketch.hpp:22-49
  public:
    explicit SfdSketcher(const SketchConfig& cfg, int device = 0) : cfg_(cfg) {
        sfdg_sketch_config c{cfg.ell, cfg.d, cfg.delta, cfg.power.c(), cfg.seed};
        check(sfdg_sketcher_create(&c, device, &h_));
    }
    ~SfdSketcher() {
        if (h_) sfdg_sketcher_destroy(h_);
    }
    SfdSketcher(const SfdSketcher&) = delete;
    SfdSketcher& operator=(const SfdSketcher&) = delete;
    SfdSketcher(SfdSketcher&& o) noexcept : cfg_(o.cfg_), h_(o.h_) { o.h_ = nullptr; }

    void append(const SparseRow& row) {
        if (row.indices.size() != row.values.size())
            throw std::invalid_argument("append_row: index/value length mismatch");
        const int64_t rp[2] = {0, static_cast<int64_t>(row.indices.size())};
        static const std::uint32_t kNoIdx = 0;
        static const double kNoVal = 0.0;
        check(sfdg_sketcher_append_csr(h_, rp, row.indices.empty() ? &kNoIdx : row.indices.data(),
                                       row.values.empty() ? &kNoVal : row.values.data(), 1, nullptr));
    }
    // Many rows at once (CSR), same per-row trigger semantics as repeated append().
    void append_csr(const int64_t* row_ptr, const std::uint32_t* cols, const double* vals, std::size_t nrows) {
        check(sfdg_sketcher_append_csr(h_, row_ptr, cols, vals, nrows, nullptr));
    }
    DenseMatrix finalize() {
        DenseMatrix b(cfg_.ell, cfg_.d);
        check(sfdg_sketcher_finalize(h_, b.data.data()));
        return b;
    }
    DenseMatrix sketch() const {
        DenseMatrix b(cfg_.ell, cfg_.d);
        check(sfdg_sketcher_get_sketch(h_, b.data.data()));
        return b;
    }
    VerifierState verifier() const {
        const sfdg_stats s = stats();
        return {s.verifier.i, s.verifier.delta, s.verifier.c_verify, s.verifier.delta_spent};
    }
    std::size_t flush_count() const { return stats().flush_count; }
    std::size_t attempt_total() const { return stats().attempt_total; }
    sfdg_stats stats() const {
        sfdg_stats s{};
        check(sfdg_sketcher_stats(h_, &s));
        return s;
    }

  private:
    SketchConfig cfg_;
    sfdg_sketcher* h_ = nullptr;
};

// merge (sketch.hpp:71, sketch.cpp:80-83)
inline DenseMatrix merge(const DenseMatrix& b1, const DenseMatrix& b2, std::size_t ell, int device = 0) {
    if (b1.cols != b2.cols) throw std::invalid_argument("merge: column mismatch");
    DenseMatrix out(ell, b1.cols);
    check(sfdg_merge(b1.data.data(), b1.rows, b2.data.data(), b2.rows, b1.cols, ell, out.data.data(), device));
    return out;
}

// dense_shrink (shrink.hpp:26, shrink.cpp:30-61)
inline DenseMatrix dense_shrink(const DenseMatrix& a, std::size_t ell, int device = 0) {
    DenseMatrix out(ell, a.cols);
    check(sfdg_dense_shrink(a.data.data(), a.rows, a.cols, ell, out.data.data(), device));
    return out;
}

}  // namespace sfd_gpu
