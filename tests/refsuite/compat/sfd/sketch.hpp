// compat/sfd/sketch.hpp -- the sketcher interface (sketch.hpp:9-71) over the sfdg C ABI.
// Accessors that return references (sketch(), buffer(), verifier()) are synchronous views:
// each call refreshes a host copy from the device sketcher.
#pragma once

#include <cstddef>
#include <cstdint>
#include <vector>

#include "sfd/shrink.hpp"
#include "sfdg.h"

namespace sfd {

struct SketchConfig {
    std::size_t ell = 0;
    std::size_t d = 0;
    double delta = 0.1;
    PowerConfig power;
    std::uint64_t seed = 0;

    void validate() const;
};

class SfdSketcher {
  public:
    explicit SfdSketcher(const SketchConfig& cfg);
    ~SfdSketcher();
    SfdSketcher(const SfdSketcher&) = delete;
    SfdSketcher& operator=(const SfdSketcher&) = delete;

    void append(const SparseRow& row);
    DenseMatrix finalize();

    const DenseMatrix& sketch() const;
    const SparseBuffer& buffer() const;
    const VerifierState& verifier() const;
    std::size_t flush_count() const;
    std::size_t attempt_total() const;

  private:
    SketchConfig cfg_;
    sfdg_sketcher* h_ = nullptr;
    mutable DenseMatrix view_b_;
    mutable SparseBuffer view_buf_;
    mutable VerifierState view_ver_;
};

class FdSketcher {
  public:
    FdSketcher(std::size_t ell, std::size_t d);
    ~FdSketcher();
    FdSketcher(const FdSketcher&) = delete;
    FdSketcher& operator=(const FdSketcher&) = delete;

    void append(const std::vector<double>& row);
    DenseMatrix finalize();
    std::size_t shrink_count() const;

  private:
    std::size_t ell_, d_;
    sfdg_fd_sketcher* h_ = nullptr;
};

DenseMatrix merge(const DenseMatrix& b1, const DenseMatrix& b2, std::size_t ell);  // sfdg_merge

}  // namespace sfd
