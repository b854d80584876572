// sfdg_main.cpp -- `sfdg sketch`: the reference CLI's sketch command (tools/sfd_main.cpp:38-88)
// over the device library. Reads a MatrixMarket or plain "col:value"
// file (--cols for plain), sketches it with SFD (or the dense FD baseline), writes the
// sketch as CSV with 17 significant digits (io.cpp:232-245) and a JSON manifest next to it
// (io.cpp:296-301). Exit codes follow tools/sfd_main.cpp:289-298: 1 = invalid argument,
// 2 = numerical error (3 = device fault).
//
//   sfdg sketch --input A.mtx --output B.csv [--algo sfd|fd] [--ell 50] [--delta 0.1]
//               [--seed 0] [--epsilon 0.25] [--q-const 1] [--fast-q] [--q-override N]
//               [--cols d] [--device 0]
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../include/sfdg.h"

namespace {

struct Args {
    std::string input, output, algo = "sfd";
    size_t ell = 50;
    double delta = 0.1;
    unsigned long long seed = 0;
    double epsilon = 0.25, q_const = 1.0;
    bool fast_q = false;
    long long q_override = -1, cols = -1;
    int device = 0;
};

int usage(const char* msg) {
    std::fprintf(stderr, "sfdg: %s\nusage: sfdg sketch --input FILE --output CSV [--algo sfd|fd] [--ell N] "
                         "[--delta X] [--seed N] [--epsilon X] [--q-const X] [--fast-q] [--q-override N] "
                         "[--cols D] [--device N]\n", msg);
    return 1;
}

int fail(int code) {
    std::fprintf(stderr, "sfdg: %s\n", sfdg_last_error());
    return code;
}

void write_csv(const std::string& path, const std::vector<double>& b, size_t rows, size_t cols) {
    FILE* f = std::fopen(path.c_str(), "w");
    if (!f) throw 1;
    char buf[64];
    for (size_t i = 0; i < rows; ++i) {
        for (size_t j = 0; j < cols; ++j) {
            std::snprintf(buf, sizeof buf, "%.17g", b[i * cols + j]);
            std::fputs(buf, f);
            if (j + 1 < cols) std::fputc(',', f);
        }
        std::fputc('\n', f);
    }
    std::fclose(f);
}

std::string jnum(double v) {
    char buf[64];
    std::snprintf(buf, sizeof buf, "%.17g", v);
    return buf;
}

std::string jstr(const std::string& s) {
    std::string o = "\"";
    for (char c : s) {
        if (c == '"' || c == '\\') o += '\\';
        o += c;
    }
    return o + "\"";
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2 || std::strcmp(argv[1], "sketch") != 0) return usage("expected the 'sketch' command");
    Args a;
    for (int i = 2; i < argc; ++i) {
        const std::string k = argv[i];
        auto val = [&]() -> const char* {
            if (i + 1 >= argc) throw 0;
            return argv[++i];
        };
        try {
            if (k == "--input") a.input = val();
            else if (k == "--output") a.output = val();
            else if (k == "--algo") a.algo = val();
            else if (k == "--ell") a.ell = std::stoull(val());
            else if (k == "--delta") a.delta = std::stod(val());
            else if (k == "--seed") a.seed = std::stoull(val());
            else if (k == "--epsilon") a.epsilon = std::stod(val());
            else if (k == "--q-const") a.q_const = std::stod(val());
            else if (k == "--fast-q") a.fast_q = true;
            else if (k == "--q-override") a.q_override = std::stoll(val());
            else if (k == "--cols") a.cols = std::stoll(val());
            else if (k == "--device") a.device = std::atoi(val());
            else return usage(("unknown option " + k).c_str());
        } catch (...) {
            return usage(("bad value for " + k).c_str());
        }
    }
    if (a.input.empty() || a.output.empty()) return usage("--input and --output are required");
    if (a.algo != "sfd" && a.algo != "fd") return usage("sketch: --algo must be fd or sfd");
    const size_t plain = a.cols >= 0 ? (size_t)a.cols : 0;

    sfdg_sketch_config cfg{};
    cfg.ell = a.ell;
    cfg.d = 0;  // from the file (tools/sfd_main.cpp:52)
    cfg.delta = a.delta;
    cfg.power.epsilon = a.epsilon;
    cfg.power.q_constant = a.q_const;
    cfg.power.q_override = a.fast_q ? 8 : -1;
    if (a.q_override >= 0) cfg.power.q_override = a.q_override;
    cfg.seed = a.seed;

    size_t n = 0, d = 0, nnz = 0;
    std::vector<double> b;
    if (a.algo == "sfd") {
        // the width is needed for the output buffer: parse the header (cheap) first
        int rc = sfdg_read_row_stream(a.input.c_str(), plain, &n, &d, &nnz, nullptr, nullptr, nullptr);
        if (rc != SFDG_OK) return fail(rc);
        b.assign(a.ell * d, 0.0);
        size_t dd = 0;
        rc = sfdg_sketch_file(a.input.c_str(), plain, &cfg, a.device, b.data(), nullptr, &dd);
        if (rc != SFDG_OK) return fail(rc);
    } else {
        int rc = sfdg_read_row_stream(a.input.c_str(), plain, &n, &d, &nnz, nullptr, nullptr, nullptr);
        if (rc != SFDG_OK) return fail(rc);
        std::vector<int64_t> rp(n + 1);
        std::vector<uint32_t> cs(nnz ? nnz : 1);
        std::vector<double> vs(nnz ? nnz : 1);
        rc = sfdg_read_row_stream(a.input.c_str(), plain, &n, &d, &nnz, rp.data(), cs.data(), vs.data());
        if (rc != SFDG_OK) return fail(rc);
        sfdg_fd_sketcher* h = nullptr;
        rc = sfdg_fd_create(a.ell, d, a.device, &h);
        if (rc != SFDG_OK) return fail(rc);
        b.assign(a.ell * d, 0.0);
        if ((rc = sfdg_fd_append_csr(h, rp.data(), cs.data(), vs.data(), n)) != SFDG_OK ||
            (rc = sfdg_fd_finalize(h, b.data())) != SFDG_OK) {
            const int code = fail(rc);
            sfdg_fd_destroy(h);
            return code;
        }
        sfdg_fd_destroy(h);
    }
    try {
        write_csv(a.output, b, a.ell, d);
    } catch (...) {
        std::fprintf(stderr, "sfdg: %s: cannot open output\n", a.output.c_str());
        return 1;
    }
    // manifest (tools/sfd_main.cpp:73-85)
    std::string m = "{\n";
    m += "  \"command\": \"sketch\",\n  \"version\": " + jstr(sfdg_version()) + ",\n";
    m += "  \"input\": " + jstr(a.input) + ",\n  \"output\": " + jstr(a.output) + ",\n";
    m += "  \"algo\": " + jstr(a.algo) + ",\n  \"ell\": " + std::to_string(a.ell) + ",\n";
    m += "  \"d\": " + std::to_string(d) + ",\n  \"delta\": " + jnum(a.delta) + ",\n";
    m += "  \"seed\": " + std::to_string(a.seed) + ",\n";
    m += "  \"power\": {\"epsilon\": " + jnum(a.epsilon) + ", \"q_constant\": " + jnum(a.q_const);
    if (cfg.power.q_override >= 0) m += ", \"q_override\": " + std::to_string(cfg.power.q_override);
    m += "}\n}\n";
    FILE* f = std::fopen((a.output + ".manifest.json").c_str(), "w");
    if (!f) {
        std::fprintf(stderr, "sfdg: %s.manifest.json: cannot open manifest output\n", a.output.c_str());
        return 1;
    }
    std::fputs(m.c_str(), f);
    std::fclose(f);
    return 0;
}
