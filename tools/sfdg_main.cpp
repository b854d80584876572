// sfdg_main.cpp -- the reference CLI (tools/sfd_main.cpp) over the device library
// (SURVEY 8(f) rank 4). Four commands, same options, outputs and exit codes:
//
//   sfdg sketch   --input A --output B.csv --ell N [--algo sfd|fd] [--delta X] [--seed N]
//                 [--epsilon X] [--q-const X] [--fast-q] [--q-override N] [--cols D]
//                 (sfd_main.cpp:38-88): SFD or the dense FD baseline over a MatrixMarket or
//                 plain "col:value" file; sketch CSV with 17 significant digits (io.cpp:232-245)
//   sfdg generate --output A.mtx [--n 10000] [--d 1000] [--z 100] [--seed 0]
//                 (sfd_main.cpp:90-111): the synthetic +-1 head/tail row stream
//                 (bench.cpp:13-66), MatrixMarket with %.17g values (io.cpp:191-230)
//   sfdg eval     --matrix A --sketch B.csv --output M.csv [--k 10] [--cols D] [--seed 0]
//                 (sfd_main.cpp:123-155): exact_tail -> proj_err -> cov_err with one Rng,
//                 all three on the device; metrics CSV (io.cpp:265-292)
//   sfdg bench    --sweep n|d|ell|nnz --out-csv M.csv [--scale X] [--seed N] [--fast-q]
//                 (sfd_main.cpp:157-228, timed_run bench.cpp:185-237): fd vs sfd per cell,
//                 wall-clock seconds of the sketch, metrics untimed
//
// Every command also takes --device N. Each writes <output>.manifest.json (io.cpp:296-301)
// with the reference's keys, formatted like nlohmann::json::dump(2) (keys sorted, shortest
// round-trip doubles). Exit codes (sfd_main.cpp:285-298): 0 ok, 1 invalid argument / usage,
// 2 numerical failure, 3 device fault (no reference counterpart).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "../include/sfdg.h"
#include "sfdg_host_io.hpp"
#include "synthetic_rows.hpp"

namespace {

const char* kUsage =
    "usage: sfdg <command> [options]\n"
    "  sketch   --input FILE --output CSV --ell N [--algo sfd|fd] [--delta X] [--seed N]\n"
    "           [--epsilon X] [--q-const X] [--fast-q] [--q-override N] [--cols D]\n"
    "  generate --output MTX [--n N] [--d D] [--z Z] [--seed N]\n"
    "  eval     --matrix FILE --sketch CSV --output CSV [--k K] [--cols D] [--seed N]\n"
    "  bench    --sweep n|d|ell|nnz --out-csv CSV [--scale X] [--seed N] [--fast-q]\n"
    "  (every command: [--device N])\n";

// Failure classes of the reference CLI's catch blocks (sfd_main.cpp:285-298).
struct Usage : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct Invalid : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct Lib {
    int code;
};

void check(int rc) {
    if (rc != SFDG_OK) throw Lib{rc};
}

// ---------------------------------------------------------------- options
struct Opts {
    std::map<std::string, std::string> kv;
    std::map<std::string, bool> flags;

    bool has(const char* k) const { return kv.count(k) != 0; }
    std::string str(const char* k, const std::string& dflt = "") const {
        auto it = kv.find(k);
        return it == kv.end() ? dflt : it->second;
    }
    std::string req(const char* k) const {
        if (!has(k)) throw Usage(std::string(k) + " is required");
        return kv.at(k);
    }
    unsigned long long u64(const char* k, unsigned long long dflt) const {
        if (!has(k)) return dflt;
        const std::string& s = kv.at(k);
        size_t pos = 0;
        unsigned long long v = 0;
        try {
            if (!s.empty() && s[0] == '-') throw 0;
            v = std::stoull(s, &pos);
        } catch (...) {
            pos = 0;
        }
        if (pos == 0 || pos != s.size()) throw Usage(std::string(k) + ": bad value '" + s + "'");
        return v;
    }
    long long i64(const char* k, long long dflt) const {
        if (!has(k)) return dflt;
        const std::string& s = kv.at(k);
        size_t pos = 0;
        long long v = 0;
        try {
            v = std::stoll(s, &pos);
        } catch (...) {
            pos = 0;
        }
        if (pos == 0 || pos != s.size()) throw Usage(std::string(k) + ": bad value '" + s + "'");
        return v;
    }
    double f64(const char* k, double dflt) const {
        if (!has(k)) return dflt;
        const std::string& s = kv.at(k);
        size_t pos = 0;
        double v = 0;
        try {
            v = std::stod(s, &pos);
        } catch (...) {
            pos = 0;
        }
        if (pos == 0 || pos != s.size()) throw Usage(std::string(k) + ": bad value '" + s + "'");
        return v;
    }
};

Opts parse(int argc, char** argv, const std::vector<std::string>& valued, const std::vector<std::string>& flags) {
    Opts o;
    for (int i = 2; i < argc; ++i) {
        const std::string k = argv[i];
        if (std::find(flags.begin(), flags.end(), k) != flags.end()) {
            o.flags[k] = true;
        } else if (std::find(valued.begin(), valued.end(), k) != valued.end()) {
            if (i + 1 >= argc) throw Usage(k + " requires an argument");
            o.kv[k] = argv[++i];
        } else {
            throw Usage("unexpected argument " + k);
        }
    }
    return o;
}

// ---------------------------------------------------------------- manifest (nlohmann dump(2) layout)
// Shortest decimal that round-trips, with ".0" on integral values (how nlohmann prints doubles).
std::string jnum(double v) {
    char buf[64];
    for (int p = 1; p <= 17; ++p) {
        std::snprintf(buf, sizeof buf, "%.*g", p, v);
        if (std::strtod(buf, nullptr) == v) break;
    }
    std::string s = buf;
    if (s.find_first_of(".eE") == std::string::npos && s.find_first_of("0123456789") != std::string::npos)
        s += ".0";
    return s;
}

std::string jstr(const std::string& s) {
    std::string o = "\"";
    for (char c : s) {
        if (c == '"' || c == '\\') o += '\\';
        o += c;
    }
    return o + "\"";
}

// A JSON object of pre-rendered scalars and nested objects; std::map keeps the keys sorted
// like nlohmann::json's default object type.
struct JObj {
    struct Entry {
        std::string scalar;
        std::vector<JObj> nested;  // 0 or 1 element
    };
    std::map<std::string, Entry> v;
    JObj& num(const std::string& k, double x) { return v[k] = {jnum(x), {}}, *this; }
    JObj& uint(const std::string& k, unsigned long long x) { return v[k] = {std::to_string(x), {}}, *this; }
    JObj& str(const std::string& k, const std::string& x) { return v[k] = {jstr(x), {}}, *this; }
    JObj& boolean(const std::string& k, bool x) { return v[k] = {x ? "true" : "false", {}}, *this; }
    JObj& obj(const std::string& k, const JObj& o) { return v[k] = {"", {o}}, *this; }
    std::string dump(int level = 1) const {
        if (v.empty()) return "{}";
        const std::string pad(2 * level, ' ');
        std::string out = "{\n";
        size_t i = 0;
        for (const auto& [k, e] : v) {
            out += pad + jstr(k) + ": " + (e.nested.empty() ? e.scalar : e.nested[0].dump(level + 1));
            out += ++i < v.size() ? ",\n" : "\n";
        }
        return out + std::string(2 * (level - 1), ' ') + "}";
    }
};

void write_manifest(const std::string& output, const JObj& m) { sfdg_tools::write_manifest(output, m.dump()); }

JObj power_json(const sfdg_power_config& p) {
    JObj j;
    j.num("epsilon", p.epsilon).num("q_constant", p.q_constant);
    if (p.q_override >= 0) j.uint("q_override", (unsigned long long)p.q_override);
    return j;
}

// ---------------------------------------------------------------- data
struct Csr {
    size_t n = 0, d = 0;
    std::vector<int64_t> rp{0};
    std::vector<uint32_t> cols;
    std::vector<double> vals;
    size_t nnz() const { return cols.size(); }
};

// open_row_stream(path, plain_cols) read to the end (io.cpp:170-189), parsed by the library.
Csr load_matrix(const std::string& path, long long plain_cols) {
    const size_t pc = plain_cols >= 0 ? (size_t)plain_cols : 0;
    Csr a;
    size_t nnz = 0;
    check(sfdg_read_row_stream(path.c_str(), pc, &a.n, &a.d, &nnz, nullptr, nullptr, nullptr));
    a.rp.assign(a.n + 1, 0);
    a.cols.resize(nnz);
    a.vals.resize(nnz);
    check(sfdg_read_row_stream(path.c_str(), pc, &a.n, &a.d, &nnz, a.rp.data(), a.cols.data(), a.vals.data()));
    return a;
}

Csr synthetic_csr(size_t n, size_t d, size_t z, uint64_t seed) {
    sfdg_tools::SyntheticRows g(n, d, z, 0.9, seed);
    Csr a;
    a.n = n;
    a.d = d;
    a.cols.reserve(n * z);
    a.vals.reserve(n * z);
    std::vector<std::pair<uint32_t, double>> row;
    while (g.more()) {
        g.next(row);
        for (const auto& [c, v] : row) {
            a.cols.push_back(c);
            a.vals.push_back(v);
        }
        a.rp.push_back((int64_t)a.cols.size());
    }
    return a;
}

using sfdg_tools::read_sketch_csv;
using MetricsRow = sfdg_tools::MetricsLine;

void write_sketch_csv(const std::string& path, const std::vector<double>& b, size_t rows, size_t cols) {
    sfdg_tools::write_sketch_csv(path, b.data(), rows, cols);
}

// ---------------------------------------------------------------- sketching and metrics
std::vector<double> sketch_sfd(const Csr& a, const sfdg_sketch_config& cfg, int device) {
    sfdg_sketcher* h = nullptr;
    check(sfdg_sketcher_create(&cfg, device, &h));
    std::vector<double> b(cfg.ell * a.d, 0.0);
    int rc = sfdg_sketcher_append_csr(h, a.rp.data(), a.cols.data(), a.vals.data(), a.n, nullptr);
    if (rc == SFDG_OK) rc = sfdg_sketcher_finalize(h, b.data());
    sfdg_sketcher_destroy(h);
    check(rc);
    return b;
}

std::vector<double> sketch_fd(const Csr& a, size_t ell, int device) {
    sfdg_fd_sketcher* h = nullptr;
    check(sfdg_fd_create(ell, a.d, device, &h));
    std::vector<double> b(ell * a.d, 0.0);
    int rc = sfdg_fd_append_csr(h, a.rp.data(), a.cols.data(), a.vals.data(), a.n);
    if (rc == SFDG_OK) rc = sfdg_fd_finalize(h, b.data());
    sfdg_fd_destroy(h);
    check(rc);
    return b;
}

struct Tail {
    double tail_sq = 0;
    std::vector<double> sigma;
};

Tail exact_tail(const Csr& a, size_t k, sfdg_rng_state& rng, int device) {
    Tail t;
    t.sigma.assign(k ? k : 1, 0.0);
    check(sfdg_exact_tail(a.rp.data(), a.cols.data(), a.vals.data(), a.n, a.d, k, &rng, t.sigma.data(), &t.tail_sq,
                          nullptr, device));
    t.sigma.resize(k);
    return t;
}

void metrics(const Csr& a, const std::vector<double>& b, size_t ell, size_t k, const Tail& tail, sfdg_rng_state& rng,
             int device, MetricsRow& row) {
    if (k >= 1) {
        int has = 0;
        check(sfdg_proj_err(a.rp.data(), a.cols.data(), a.vals.data(), a.n, a.d, b.data(), ell, k, tail.tail_sq,
                            &row.proj_err, &has, device));
        row.has_proj = has != 0;
    }
    check(sfdg_cov_err(a.rp.data(), a.cols.data(), a.vals.data(), a.n, a.d, b.data(), ell, 1000, &rng, &row.cov_err,
                       device));
}

// ---------------------------------------------------------------- commands
int run_sketch(int argc, char** argv) {
    const Opts o = parse(argc, argv,
                         {"--input", "--output", "--algo", "--ell", "--delta", "--seed", "--epsilon", "--q-const",
                          "--q-override", "--cols", "--device"},
                         {"--fast-q"});
    const std::string input = o.req("--input"), output = o.req("--output");
    const std::string algo = o.str("--algo", "sfd");
    if (algo != "sfd" && algo != "fd") throw Usage("--algo: " + algo + " not in {fd,sfd}");
    const size_t ell = (size_t)o.u64("--ell", 0);
    if (!o.has("--ell")) throw Usage("--ell is required");
    const int device = (int)o.i64("--device", 0);

    sfdg_sketch_config cfg{};
    cfg.ell = ell;
    cfg.delta = o.f64("--delta", 0.1);
    cfg.seed = o.u64("--seed", 0);
    cfg.power.epsilon = o.f64("--epsilon", 0.25);
    cfg.power.q_constant = o.f64("--q-const", 1.0);
    cfg.power.q_override = o.flags.count("--fast-q") ? 8 : -1;
    const long long qo = o.i64("--q-override", -1);
    if (qo >= 0) cfg.power.q_override = qo;

    const long long cols = o.i64("--cols", -1);
    std::vector<double> b;
    size_t d = 0;
    if (algo == "fd") {
        // FdSketcher(ell, d) (sketch.cpp:47-52) validates 1 <= ell <= d itself
        const Csr a = load_matrix(input, cols);
        d = a.d;
        b = sketch_fd(a, ell, device);
    } else {
        // streamed: the library parses the file window by window into the sketcher
        size_t n = 0, nnz = 0;
        const size_t pc = cols >= 0 ? (size_t)cols : 0;
        check(sfdg_read_row_stream(input.c_str(), pc, &n, &d, &nnz, nullptr, nullptr, nullptr));
        b.assign(ell * d, 0.0);
        check(sfdg_sketch_file(input.c_str(), pc, &cfg, device, b.data(), nullptr, &d));
    }
    cfg.d = d;  // from the stream (sfd_main.cpp:52)
    write_sketch_csv(output, b, ell, d);

    JObj m;
    m.str("command", "sketch").str("version", sfdg_version()).str("input", input).str("output", output);
    m.str("algo", algo).uint("ell", ell).uint("d", d).num("delta", cfg.delta).uint("seed", cfg.seed);
    m.obj("power", power_json(cfg.power));
    write_manifest(output, m);
    return 0;
}

int run_generate(int argc, char** argv) {
    const Opts o = parse(argc, argv, {"--n", "--d", "--z", "--seed", "--output", "--device"}, {});
    const std::string output = o.req("--output");
    const size_t n = o.u64("--n", 10000), d = o.u64("--d", 1000), z = o.u64("--z", 100);
    const uint64_t seed = o.u64("--seed", 0);
    sfdg_tools::SyntheticRows g(n, d, z, 0.9, seed);

    sfdg_tools::MmWriter writer(output, n, d, n * z);
    std::vector<std::pair<uint32_t, double>> row;
    std::vector<uint32_t> idx;
    std::vector<double> val;
    for (size_t i = 0; g.more(); ++i) {
        g.next(row);
        idx.clear();
        val.clear();
        for (const auto& [c, v] : row) {
            idx.push_back(c);
            val.push_back(v);
        }
        writer.append_row(i, idx.data(), val.data(), idx.size());
    }
    writer.close();

    JObj m;
    m.str("command", "generate").str("version", sfdg_version()).str("output", output);
    m.uint("n", n).uint("d", d).uint("z", z).num("p_head", 0.9).uint("seed", seed);
    write_manifest(output, m);
    return 0;
}

int run_eval(int argc, char** argv) {
    const Opts o = parse(argc, argv, {"--matrix", "--sketch", "--k", "--output", "--cols", "--seed", "--device"}, {});
    const std::string mpath = o.req("--matrix"), spath = o.req("--sketch"), output = o.req("--output");
    const size_t k = o.u64("--k", 10);
    const uint64_t seed = o.u64("--seed", 0);
    const int device = (int)o.i64("--device", 0);

    const Csr a = load_matrix(mpath, o.i64("--cols", -1));
    size_t ell = 0, cols = 0;
    const std::vector<double> b = read_sketch_csv(spath, ell, cols);
    if (cols != a.d) throw Invalid("eval: matrix and sketch dimensions are incompatible");

    sfdg_rng_state rng{seed, 0, 0, 0.0};  // Rng rng(seed), shared by exact_tail and cov_err
    const Tail tail = exact_tail(a, k, rng, device);
    MetricsRow row;
    row.algo = "eval";
    row.n = a.n;
    row.d = a.d;
    row.ell = ell;
    row.z = a.n ? a.nnz() / a.n : 0;
    row.k = k;
    row.seed = seed;
    metrics(a, b, ell, k, tail, rng, device, row);
    sfdg_tools::write_metrics_csv(output, {row});

    JObj m;
    m.str("command", "eval").str("version", sfdg_version()).str("matrix", mpath).str("sketch", spath);
    m.str("output", output).uint("k", k).uint("seed", seed);
    write_manifest(output, m);
    return 0;
}

size_t scaled(size_t v, double scale, size_t lo) {
    return std::max(lo, (size_t)std::llround((double)v * scale));
}

int run_bench(int argc, char** argv) {
    const Opts o = parse(argc, argv, {"--sweep", "--out-csv", "--scale", "--seed", "--device"}, {"--fast-q"});
    const std::string sweep = o.req("--sweep"), out_csv = o.req("--out-csv");
    if (sweep != "n" && sweep != "d" && sweep != "ell" && sweep != "nnz")
        throw Usage("--sweep: " + sweep + " not in {d,ell,n,nnz}");
    const double scale = o.f64("--scale", 1.0);
    const uint64_t seed = o.u64("--seed", 0);
    const bool fast_q = o.flags.count("--fast-q") != 0;
    const int device = (int)o.i64("--device", 0);

    const size_t def_n = scaled(10000, scale, 50), def_d = scaled(1000, scale, 20);
    const size_t def_ell = scaled(50, scale, 4), def_z = scaled(100, scale, 2);
    std::vector<size_t> values;
    if (sweep == "n") {
        for (size_t v : {10000, 20000, 30000, 40000, 50000, 60000}) values.push_back(scaled(v, scale, 50));
    } else if (sweep == "d") {
        for (size_t v : {1000, 2000, 3000, 4000, 5000, 6000}) values.push_back(scaled(v, scale, 20));
    } else if (sweep == "ell") {
        for (size_t v : {5, 10, 25, 50, 75, 100}) values.push_back(scaled(v, scale, 2));
    } else {
        for (size_t v : {5, 25, 50, 100, 250, 500}) values.push_back(scaled(v, scale, 2));
    }

    // bring the device context up before the first timed sketch
    {
        sfdg_fd_sketcher* h = nullptr;
        check(sfdg_fd_create(1, 1, device, &h));
        sfdg_fd_destroy(h);
    }

    std::vector<MetricsRow> rows;
    for (size_t cell = 0; cell < values.size(); ++cell) {
        const size_t v = values[cell];
        size_t n = def_n, d = def_d, ell = def_ell, z = def_z;
        if (sweep == "n") n = v;
        else if (sweep == "d") d = v;
        else if (sweep == "ell") ell = v;
        else z = v;
        z = std::min(z, d);
        ell = std::min(ell, d);
        const size_t k = std::max<size_t>(1, std::min<size_t>(10, ell - 1));
        const uint64_t cseed = seed + 1000 * cell;
        const Csr a = synthetic_csr(n, d, z, cseed);

        sfdg_sketch_config cfg{};
        cfg.ell = ell;
        cfg.d = d;
        cfg.delta = 0.1;
        cfg.seed = cseed;
        cfg.power.epsilon = 0.25;
        cfg.power.q_constant = 1.0;
        cfg.power.q_override = fast_q ? 8 : -1;

        sfdg_rng_state tail_rng{cseed ^ 0x5bf03635ULL, 0, 0, 0.0};
        const Tail tail = exact_tail(a, k, tail_rng, device);
        for (const char* algo : {"fd", "sfd"}) {
            // timed_run (bench.cpp:185-237): the sketch is timed, the metrics are not
            MetricsRow row;
            row.algo = algo;
            row.n = n;
            row.d = d;
            row.ell = ell;
            row.z = z;
            row.k = k;
            row.seed = cseed;
            const auto t0 = std::chrono::steady_clock::now();
            const std::vector<double> b = row.algo == "fd" ? sketch_fd(a, ell, device) : sketch_sfd(a, cfg, device);
            row.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            sfdg_rng_state mrng{cseed ^ 0x9e3779b97f4a7c15ULL, 0, 0, 0.0};
            metrics(a, b, ell, k, tail, mrng, device, row);
            rows.push_back(row);
        }
        std::fprintf(stderr, "bench: %s=%zu done\n", sweep.c_str(), v);
    }
    sfdg_tools::write_metrics_csv(out_csv, rows);

    JObj m;
    m.str("command", "bench").str("version", sfdg_version()).str("sweep", sweep).num("scale", scale);
    m.uint("seed", seed).boolean("fast_q", fast_q).str("out_csv", out_csv);
    write_manifest(out_csv, m);
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    const std::string cmd = argc >= 2 ? argv[1] : "";
    if (cmd == "--help" || cmd == "-h") {
        std::fputs(kUsage, stdout);
        return 0;
    }
    for (int i = 2; i < argc; ++i)
        if (!std::strcmp(argv[i], "--help") || !std::strcmp(argv[i], "-h")) {
            std::fputs(kUsage, stdout);
            return 0;
        }
    try {
        if (cmd == "sketch") return run_sketch(argc, argv);
        if (cmd == "generate") return run_generate(argc, argv);
        if (cmd == "eval") return run_eval(argc, argv);
        if (cmd == "bench") return run_bench(argc, argv);
        throw Usage(cmd.empty() ? "a subcommand is required" : "unknown subcommand " + cmd);
    } catch (const Usage& e) {
        std::fprintf(stderr, "%s\n%s", e.what(), kUsage);
        return 1;
    } catch (const Invalid& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    } catch (const Lib& e) {
        if (e.code == SFDG_NUMERICAL_ERROR) std::fprintf(stderr, "numerical failure: %s\n", sfdg_last_error());
        else std::fprintf(stderr, "error: %s\n", sfdg_last_error());
        return e.code == SFDG_NUMERICAL_ERROR ? 2 : e.code == SFDG_CUDA_ERROR ? 3 : 1;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
}
