// sfdg_host_io.hpp -- the reference's file writers/readers for CLI outputs (io.cpp:191-301),
// host code shared by the `sfdg` CLI and the reference-suite compat layer (tests/refsuite).
//   MmWriter            MatrixMarketWriter (io.cpp:191-230): header, 1-based "i j %.17g" lines,
//                       rows in order, close() checks the declared entry count
//   write_sketch_csv    io.cpp:232-245, 17 significant digits (round-trips doubles)
//   read_sketch_csv     io.cpp:247-263, blank lines skipped, ragged / empty files rejected
//   metrics_csv_*       io.cpp:265-292, "%.9f" metrics, "nan" for an empty proj_err
//   write_manifest      io.cpp:296-301, <output>.manifest.json
#pragma once

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

namespace sfdg_tools {

class MmWriter {
  public:
    MmWriter(const std::string& path, size_t rows, size_t cols, size_t nnz) : declared_(nnz) {
        f_ = std::fopen(path.c_str(), "w");
        if (!f_) throw std::invalid_argument(path + ": cannot open output");
        buf_ = "%%MatrixMarket matrix coordinate real general\n";
        buf_ += std::to_string(rows) + " " + std::to_string(cols) + " " + std::to_string(nnz) + "\n";
    }
    ~MmWriter() {
        if (f_) {
            flush();
            std::fclose(f_);
        }
    }
    MmWriter(const MmWriter&) = delete;
    MmWriter& operator=(const MmWriter&) = delete;

    // row_index is 0-based; rows must come in nondecreasing order
    void append_row(size_t row_index, const uint32_t* idx, const double* val, size_t n) {
        if (any_ && row_index < last_) throw std::invalid_argument("MatrixMarketWriter: rows must be appended in order");
        any_ = true;
        last_ = row_index;
        char line[96];
        for (size_t k = 0; k < n; ++k) {
            const int len = std::snprintf(line, sizeof line, "%zu %zu %.17g\n", row_index + 1, (size_t)idx[k] + 1, val[k]);
            buf_.append(line, (size_t)len);
            ++written_;
        }
        if (buf_.size() > (1u << 20)) flush();
    }
    void close() {
        if (written_ != declared_)
            throw std::logic_error("MatrixMarketWriter: entry count does not match declared nnz");
        flush();
        std::fclose(f_);
        f_ = nullptr;
    }

  private:
    void flush() {
        if (!buf_.empty()) std::fwrite(buf_.data(), 1, buf_.size(), f_);
        buf_.clear();
    }
    FILE* f_ = nullptr;
    std::string buf_;
    size_t declared_, written_ = 0, last_ = 0;
    bool any_ = false;
};

inline void write_sketch_csv(const std::string& path, const double* b, size_t rows, size_t cols) {
    FILE* f = std::fopen(path.c_str(), "w");
    if (!f) throw std::invalid_argument(path + ": cannot open output");
    char cell[32];
    std::string line;
    for (size_t i = 0; i < rows; ++i) {
        line.clear();
        for (size_t j = 0; j < cols; ++j) {
            std::snprintf(cell, sizeof cell, "%.17g", b[i * cols + j]);
            line += cell;
            if (j + 1 < cols) line += ',';
        }
        line += '\n';
        std::fwrite(line.data(), 1, line.size(), f);
    }
    std::fclose(f);
}

inline std::vector<double> read_sketch_csv(const std::string& path, size_t& rows, size_t& cols) {
    FILE* f = std::fopen(path.c_str(), "r");
    if (!f) throw std::invalid_argument(path + ": cannot open sketch file");
    std::vector<double> m;
    rows = cols = 0;
    std::string line;
    bool eof = false;
    while (!eof) {
        line.clear();
        int ch;
        while ((ch = std::fgetc(f)) != EOF && ch != '\n') line += (char)ch;
        eof = ch == EOF;
        if (line.empty()) continue;
        size_t count = 0, start = 0;
        for (;;) {  // getline(ss, cell, ',') semantics: no cell after a trailing comma
            const size_t comma = line.find(',', start);
            const std::string cell = line.substr(start, comma == std::string::npos ? std::string::npos : comma - start);
            double v;
            try {
                v = std::stod(cell);
            } catch (...) {
                std::fclose(f);
                throw;
            }
            m.push_back(v);
            ++count;
            if (comma == std::string::npos || comma + 1 == line.size()) break;
            start = comma + 1;
        }
        if (rows && count != cols) {
            std::fclose(f);
            throw std::invalid_argument(path + ": ragged sketch file");
        }
        cols = count;
        ++rows;
    }
    std::fclose(f);
    if (!rows) throw std::invalid_argument(path + ": empty sketch file");
    return m;
}

struct MetricsLine {
    std::string algo;
    size_t n = 0, d = 0, ell = 0, z = 0, k = 0;
    bool has_proj = false;
    double proj_err = 0, cov_err = 0, wall_seconds = 0;
    uint64_t seed = 0;
};

inline std::string metrics_csv_header() { return "algo,n,d,ell,z,k,proj_err,cov_err,wall_seconds,seed"; }

inline std::string metrics_csv_line(const MetricsLine& r) {
    char buf[128];
    std::string s = r.algo;
    std::snprintf(buf, sizeof buf, ",%zu,%zu,%zu,%zu,%zu,", r.n, r.d, r.ell, r.z, r.k);
    s += buf;
    if (r.has_proj) {
        std::snprintf(buf, sizeof buf, "%.9f", r.proj_err);
        s += buf;
    } else {
        s += "nan";
    }
    std::snprintf(buf, sizeof buf, ",%.9f,%.6f,%llu", r.cov_err, r.wall_seconds, (unsigned long long)r.seed);
    return s + buf;
}

inline void write_metrics_csv(const std::string& path, const std::vector<MetricsLine>& rows) {
    FILE* f = std::fopen(path.c_str(), "w");
    if (!f) throw std::invalid_argument(path + ": cannot open output");
    std::string text = metrics_csv_header() + "\n";
    for (const MetricsLine& r : rows) text += metrics_csv_line(r) + "\n";
    std::fwrite(text.data(), 1, text.size(), f);
    std::fclose(f);
}

inline void write_manifest(const std::string& output_path, const std::string& json_text) {
    const std::string path = output_path + ".manifest.json";
    FILE* f = std::fopen(path.c_str(), "w");
    if (!f) throw std::invalid_argument(path + ": cannot open manifest output");
    const std::string text = json_text + "\n";
    std::fwrite(text.data(), 1, text.size(), f);
    std::fclose(f);
}

}  // namespace sfdg_tools
