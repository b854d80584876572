// sfd_compat_io.cpp -- io.hpp over the device build (test infrastructure; see sfd_compat.cpp).
#include <stdexcept>
#include <string>
#include <vector>

#include "../../../tools/sfdg_host_io.hpp"
#include "sfd/io.hpp"
#include "sfdg.h"

namespace sfd {

namespace {

class ParsedStream : public RowStream {
  public:
    ParsedStream(const std::string& path, size_t plain) {
        size_t n = 0, nnz = 0;
        int rc = sfdg_read_row_stream(path.c_str(), plain, &n, &d_, &nnz, nullptr, nullptr, nullptr);
        if (rc != SFDG_OK) {
            // the reference raises header-level errors from open_row_stream (io.cpp:20-40,
            // 170-189) and entry errors from next(); the library reports both at parse time
            const std::string msg = sfdg_last_error();
            if (rc != SFDG_INVALID_ARGUMENT) throw std::runtime_error(msg);
            for (const char* at_open : {"cannot open input", "empty file and no column count",
                                        "unsupported MatrixMarket header", "requires an explicit column count",
                                        "MatrixMarket size line"})
                if (msg.find(at_open) != std::string::npos) throw std::invalid_argument(msg);
            error_ = msg;
            return;
        }
        rp_.assign(n + 1, 0);
        cols_.resize(nnz ? nnz : 1);
        vals_.resize(nnz ? nnz : 1);
        rc = sfdg_read_row_stream(path.c_str(), plain, &n, &d_, &nnz, rp_.data(), cols_.data(), vals_.data());
        if (rc != SFDG_OK) error_ = sfdg_last_error();  // surfaced by next()
    }
    std::size_t cols() const override { return d_; }
    bool next(SparseRow& out) override {
        if (!error_.empty()) throw std::invalid_argument(error_);
        if (pos_ + 1 >= rp_.size()) return false;
        out.indices.assign(cols_.begin() + rp_[pos_], cols_.begin() + rp_[pos_ + 1]);
        out.values.assign(vals_.begin() + rp_[pos_], vals_.begin() + rp_[pos_ + 1]);
        ++pos_;
        return true;
    }

  private:
    size_t d_ = 0, pos_ = 0;
    std::vector<int64_t> rp_;
    std::vector<uint32_t> cols_;
    std::vector<double> vals_;
    std::string error_;
};

sfdg_tools::MetricsLine line_of(const MetricsRow& r) {
    sfdg_tools::MetricsLine l;
    l.algo = r.algo;
    l.n = r.n;
    l.d = r.d;
    l.ell = r.ell;
    l.z = r.z;
    l.k = r.k;
    l.has_proj = r.proj_err.has_value();
    l.proj_err = r.proj_err.value_or(0.0);
    l.cov_err = r.cov_err;
    l.wall_seconds = r.wall_seconds;
    l.seed = r.seed;
    return l;
}

}  // namespace

std::unique_ptr<RowStream> open_row_stream(const std::string& path, std::optional<std::size_t> plain_cols) {
    return std::make_unique<ParsedStream>(path, plain_cols ? *plain_cols : 0);
}

struct MatrixMarketWriter::Impl {
    sfdg_tools::MmWriter w;
    Impl(const std::string& p, size_t r, size_t c, size_t z) : w(p, r, c, z) {}
};

MatrixMarketWriter::MatrixMarketWriter(const std::string& path, std::size_t rows, std::size_t cols, std::size_t nnz)
    : impl_(std::make_unique<Impl>(path, rows, cols, nnz)) {}
MatrixMarketWriter::~MatrixMarketWriter() = default;
void MatrixMarketWriter::append_row(std::size_t row_index, const SparseRow& row) {
    impl_->w.append_row(row_index, row.indices.data(), row.values.data(), row.indices.size());
}
void MatrixMarketWriter::close() { impl_->w.close(); }

void write_sketch_csv(const std::string& path, const DenseMatrix& sketch) {
    sfdg_tools::write_sketch_csv(path, sketch.data.data(), sketch.rows, sketch.cols);
}

DenseMatrix read_sketch_csv(const std::string& path) {
    size_t r = 0, c = 0;
    std::vector<double> v = sfdg_tools::read_sketch_csv(path, r, c);
    DenseMatrix m(r, c);
    m.data = std::move(v);
    return m;
}

void write_metrics_csv(const std::string& path, const std::vector<MetricsRow>& rows) {
    std::vector<sfdg_tools::MetricsLine> lines;
    for (const MetricsRow& r : rows) lines.push_back(line_of(r));
    sfdg_tools::write_metrics_csv(path, lines);
}

std::string metrics_csv_header() { return sfdg_tools::metrics_csv_header(); }
std::string metrics_csv_line(const MetricsRow& row) { return sfdg_tools::metrics_csv_line(line_of(row)); }
void write_manifest(const std::string& output_path, const std::string& json_text) {
    sfdg_tools::write_manifest(output_path, json_text);
}

}  // namespace sfd
