// io.cu -- ingestion of row-stream files into the sketcher.
//
// Reference: open_row_stream (core/src/io.cpp:170-189) over MatrixMarketStream
// (io.cpp:21-104: "matrix coordinate real general", 1-based, entries grouped by
// nondecreasing row, columns sorted per row, duplicates rejected) and PlainStream
// (io.cpp:106-166: one "col:value" row per line, 0-based, '#' comments). The reference
// parses one line at a time through iostreams; at c5 (1e9 nnz, 12.6 GB of text) that is
// the end-to-end bottleneck. Here the file is memory-mapped and cut into windows; each
// window is split at line boundaries and parsed by all host threads in parallel, then
// assembled in file order into CSR batches that go to the device sketcher while the next
// window is parsed. Row contents, order and error classes follow the reference.
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"
#include "io.cuh"

namespace sfdg {

namespace {

struct Mapped {
    const char* p = nullptr;
    size_t n = 0;
    int fd = -1;
    explicit Mapped(const std::string& path) {
        fd = ::open(path.c_str(), O_RDONLY);
        if (fd < 0) throw invalid_argument(path + ": cannot open input");
        struct stat sb;
        if (fstat(fd, &sb) != 0) throw invalid_argument(path + ": cannot open input");
        n = (size_t)sb.st_size;
        if (n > 0) {
            void* m = mmap(nullptr, n, PROT_READ, MAP_PRIVATE, fd, 0);
            if (m == MAP_FAILED) throw invalid_argument(path + ": cannot map input");
            madvise(m, n, MADV_SEQUENTIAL);
            p = static_cast<const char*>(m);
        }
    }
    ~Mapped() {
        if (p) munmap((void*)p, n);
        if (fd >= 0) ::close(fd);
    }
};

inline bool is_space(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f'; }

// istream >> long long: optional sign, digits; the token must end at whitespace/end
bool parse_ll(const char*& s, const char* e, long long& out) {
    while (s < e && is_space(*s)) ++s;
    const char* b = s;
    bool neg = false;
    if (s < e && (*s == '+' || *s == '-')) neg = *s++ == '-';
    const char* d0 = s;
    unsigned long long v = 0;
    while (s < e && *s >= '0' && *s <= '9') {
        v = v * 10 + (unsigned)(*s - '0');
        if (v > (1ull << 62)) return false;
        ++s;
    }
    if (s == d0) {
        s = b;
        return false;
    }
    out = neg ? -(long long)v : (long long)v;
    return true;
}

// istream >> double (strtod on the token, without the inf/nan spellings num_get rejects)
bool parse_double(const char*& s, const char* e, double& out) {
    while (s < e && is_space(*s)) ++s;
    char buf[128];
    size_t k = 0;
    const char* t = s;
    while (t < e && !is_space(*t) && *t != '\n' && k + 1 < sizeof buf) buf[k++] = *t++;
    buf[k] = 0;
    if (k == 0) return false;
    for (size_t i = 0; i < k; ++i)
        if (buf[i] == 'n' || buf[i] == 'N' || buf[i] == 'i' || buf[i] == 'I') return false;
    char* endp = nullptr;
    errno = 0;
    out = std::strtod(buf, &endp);
    if (endp == buf) return false;
    s += (endp - buf);
    return true;
}

struct Entry {
    long long row;  // 0-based
    uint32_t col;
    double val;
};

struct ChunkResult {
    std::vector<Entry> entries;
    std::string error;  // first error in the chunk ("" = none)
};

// MatrixMarket entry lines of [b, e) (whole lines)
void parse_mm_chunk(const char* b, const char* e, long long n, long long d, const std::string& path,
                    ChunkResult& out) {
    const char* s = b;
    while (s < e) {
        const char* le = (const char*)memchr(s, '\n', e - s);
        if (!le) le = e;
        if (le > s && *s != '%') {
            const char* q = s;
            long long r = 0, c = 0;
            double v = 0.0;
            if (!parse_ll(q, le, r) || !parse_ll(q, le, c) || !parse_double(q, le, v)) {
                out.error = path + ": malformed entry line";
                return;
            }
            if (r < 1 || r > n || c < 1 || c > d) {
                out.error = path + ": entry index out of range";
                return;
            }
            out.entries.push_back({r - 1, (uint32_t)(c - 1), v});
        }
        s = le + 1;
    }
}

// plain "col:value" lines of [b, e): one row per non-blank line (io.cpp:113-160)
struct PlainChunk {
    std::vector<int64_t> rp{0};
    std::vector<uint32_t> cols;
    std::vector<double> vals;
    std::string error;
};

void parse_plain_chunk(const char* b, const char* e, size_t d, const std::string& path, PlainChunk& out) {
    const char* s = b;
    while (s < e) {
        const char* le = (const char*)memchr(s, '\n', e - s);
        if (!le) le = e;
        const char* hash = (const char*)memchr(s, '#', le - s);
        const char* ce = hash ? hash : le;
        const char* q = s;
        while (q < ce && (is_space(*q))) ++q;
        if (q < ce) {
            const size_t row_start = out.cols.size();
            while (q < ce) {
                while (q < ce && is_space(*q)) ++q;
                if (q >= ce) break;
                const char* tb = q;
                while (q < ce && !is_space(*q)) ++q;
                const char* colon = (const char*)memchr(tb, ':', q - tb);
                if (!colon) {
                    out.error = path + ": expected col:value token, got '" + std::string(tb, q) + "'";
                    return;
                }
                const char* x = tb;
                long long col = 0;
                if (!parse_ll(x, colon, col)) {
                    out.error = path + ": bad column index in '" + std::string(tb, q) + "'";
                    return;
                }
                const char* y = colon + 1;
                double val = 0.0;
                if (!parse_double(y, q, val)) {
                    out.error = path + ": bad value in '" + std::string(tb, q) + "'";
                    return;
                }
                if (col < 0 || (size_t)col >= d) {
                    out.error = path + ": column index out of range";
                    return;
                }
                if (out.cols.size() > row_start && (uint32_t)col <= out.cols.back()) {
                    out.error = path + ": columns must be strictly increasing";
                    return;
                }
                out.cols.push_back((uint32_t)col);
                out.vals.push_back(val);
            }
            out.rp.push_back((int64_t)out.cols.size());
        }
        s = le + 1;
    }
}

// [b, e) cut into `parts` pieces at line starts
std::vector<const char*> split_lines(const char* b, const char* e, int parts) {
    std::vector<const char*> cut{b};
    for (int i = 1; i < parts; ++i) {
        const char* t = b + (size_t)(e - b) * i / parts;
        if (t <= cut.back()) continue;
        const char* nl = (const char*)memchr(t, '\n', e - t);
        if (!nl) break;
        cut.push_back(nl + 1);
    }
    cut.push_back(e);
    return cut;
}

int host_threads() {
    if (const char* e = std::getenv("SFDG_IO_THREADS")) return std::max(1, std::atoi(e));
    return std::max(1u, std::thread::hardware_concurrency());
}

}  // namespace

void read_row_stream(const std::string& path, size_t plain_cols, size_t window_bytes, size_t* d_out,
                     const std::function<void(const int64_t*, const uint32_t*, const double*, size_t)>& sink) {
    Mapped f(path);
    const char* p = f.p;
    const char* end = p + f.n;
    const int T = host_threads();
    if (window_bytes == 0) window_bytes = (size_t)256 << 20;
    // first line decides the format (io.cpp:174-188)
    const char* nl = f.n ? (const char*)memchr(p, '\n', f.n) : nullptr;
    const char* l1e = nl ? nl : end;
    const std::string first(p ? p : "", p ? (size_t)(l1e - p) : 0);
    if (f.n == 0) {
        if (!plain_cols) throw invalid_argument(path + ": empty file and no column count given");
        *d_out = plain_cols;
        return;
    }
    if (first.rfind("%%MatrixMarket", 0) == 0) {
        if (first.find("matrix coordinate real general") == std::string::npos)
            throw invalid_argument(path +
                                   ": unsupported MatrixMarket header (need 'matrix coordinate real general')");
        // size line (io.cpp:25-37)
        const char* s = nl ? nl + 1 : end;
        long long n = -1, d = -1, nnz = -1;
        bool found = false;
        while (s < end) {
            const char* le = (const char*)memchr(s, '\n', end - s);
            if (!le) le = end;
            if (le > s && *s != '%') {
                const char* q = s;
                if (!parse_ll(q, le, n) || !parse_ll(q, le, d) || !parse_ll(q, le, nnz) || n < 0 || d <= 0 ||
                    nnz < 0)
                    throw invalid_argument(path + ": bad MatrixMarket size line");
                found = true;
                s = le + 1;
                break;
            }
            s = le + 1;
        }
        if (!found) throw invalid_argument(path + ": missing MatrixMarket size line");
        *d_out = (size_t)d;
        // stream the entries window by window; rows are emitted in order, empty rows included
        long long next_row = 0;  // first row not yet emitted
        std::vector<Entry> carry;  // entries of the row still open at a window end
        std::vector<int64_t> rp;
        std::vector<uint32_t> cs;
        std::vector<double> vs;
        std::vector<size_t> order;
        auto emit_rows_until = [&](long long upto, const Entry* eb, const Entry* ee) {
            // entries [eb, ee) all belong to rows < upto (grouped, nondecreasing); emit rows
            // next_row .. upto-1
            rp.assign(1, 0);
            cs.clear();
            vs.clear();
            const Entry* q = eb;
            for (long long r = next_row; r < upto; ++r) {
                const Entry* rb = q;
                while (q < ee && q->row == r) ++q;
                order.resize(q - rb);
                for (size_t i = 0; i < order.size(); ++i) order[i] = i;
                std::sort(order.begin(), order.end(), [&](size_t x, size_t y) { return rb[x].col < rb[y].col; });
                for (size_t i = 0; i < order.size(); ++i) {
                    if (i > 0 && rb[order[i]].col == rb[order[i - 1]].col)
                        throw invalid_argument(path + ": duplicate column within a row");
                    cs.push_back(rb[order[i]].col);
                    vs.push_back(rb[order[i]].val);
                }
                rp.push_back((int64_t)cs.size());
            }
            if (upto > next_row) sink(rp.data(), cs.data(), vs.data(), (size_t)(upto - next_row));
            next_row = upto;
        };
        while (s < end || !carry.empty()) {
            const char* we = s;
            if (s < end) {
                we = s + std::min(window_bytes, (size_t)(end - s));
                if (we < end) {
                    const char* t = (const char*)memchr(we, '\n', end - we);
                    we = t ? t + 1 : end;
                }
            }
            std::vector<const char*> cut = split_lines(s, we, T);
            std::vector<ChunkResult> res(cut.size() - 1);
            std::vector<std::thread> th;
            for (size_t i = 0; i + 1 < cut.size(); ++i)
                th.emplace_back([&, i] { parse_mm_chunk(cut[i], cut[i + 1], n, d, path, res[i]); });
            for (auto& t : th) t.join();
            std::vector<Entry> all;
            all.swap(carry);
            std::string err;
            for (auto& r : res) {
                all.insert(all.end(), r.entries.begin(), r.entries.end());
                if (!r.error.empty()) {
                    err = r.error;
                    break;
                }
            }
            // order check (io.cpp:47-49) over the assembled entries
            long long prev = all.empty() ? next_row : all.front().row;
            size_t good = all.size();
            std::string order_err;
            if (!all.empty() && all.front().row < next_row) good = 0;
            for (size_t i = 0; i < all.size() && good == all.size(); ++i) {
                if (all[i].row < prev) good = i;
                prev = std::max(prev, all[i].row);
            }
            if (good < all.size()) {
                order_err = path + ": entries not grouped by nondecreasing row (streaming input must be row ordered)";
                all.resize(good);
            }
            const bool last = we >= end || !err.empty() || !order_err.empty();
            // rows complete in this window: all rows below the last entry's row (that row may
            // continue in the next window), or everything at the end of the file
            long long upto = last ? (err.empty() && order_err.empty() ? n : (all.empty() ? next_row : all.back().row))
                                  : (all.empty() ? next_row : all.back().row);
            size_t split = all.size();
            while (split > 0 && all[split - 1].row >= upto) --split;
            if (upto > next_row) emit_rows_until(upto, all.data(), all.data() + split);
            carry.assign(all.begin() + split, all.end());
            if (!err.empty()) throw invalid_argument(err);
            if (!order_err.empty()) throw invalid_argument(order_err);
            s = we;
            if (last) break;
        }
        return;
    }
    if (!plain_cols) throw invalid_argument(path + ": plain format input requires an explicit column count");
    *d_out = plain_cols;
    const char* s = p;
    while (s < end) {
        const char* we = s + std::min(window_bytes, (size_t)(end - s));
        if (we < end) {
            const char* t = (const char*)memchr(we, '\n', end - we);
            we = t ? t + 1 : end;
        }
        std::vector<const char*> cut = split_lines(s, we, T);
        std::vector<PlainChunk> res(cut.size() - 1);
        std::vector<std::thread> th;
        for (size_t i = 0; i + 1 < cut.size(); ++i)
            th.emplace_back([&, i] { parse_plain_chunk(cut[i], cut[i + 1], plain_cols, path, res[i]); });
        for (auto& t : th) t.join();
        for (auto& r : res) {
            if (r.rp.size() > 1) sink(r.rp.data(), r.cols.data(), r.vals.data(), r.rp.size() - 1);
            if (!r.error.empty()) throw invalid_argument(r.error);
        }
        s = we;
    }
}

}  // namespace sfdg
