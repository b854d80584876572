// ref_io_main.cpp -- test helper (oracle side): runs the UNMODIFIED reference reader
// sfd::open_row_stream (core/src/io.cpp:170-189) over a file and writes the rows as binary
// CSR to stdout: int64 n, d, nnz, error flag, message length, message bytes, then
// row_ptr[n+1] (int64), cols[nnz] (uint32), vals[nnz] (double). Rows read before an error
// are included. A separate executable: the reference's iostream code is not dlopen-safe
// inside the Python test process.
//
//   refio PATH [PLAIN_COLS]           read PATH, CSR to stdout
//   refio --gen N D Z SEED OUT        the reference `generate` body (tools/sfd_main.cpp:90-98):
//                                     sfd::SyntheticStream rows through sfd::MatrixMarketWriter
#include <cstdint>
#include <cstdio>
#include <optional>
#include <string>
#include <vector>

#include "sfd/bench.hpp"
#include "sfd/io.hpp"

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    if (std::string(argv[1]) == "--gen") {
        if (argc < 7) return 2;
        try {
            const std::size_t n = std::stoull(argv[2]), d = std::stoull(argv[3]), z = std::stoull(argv[4]);
            sfd::SyntheticSpec spec{n, d, z, 0.9, std::stoull(argv[5])};
            spec.validate();
            sfd::SyntheticStream gen(spec);
            sfd::MatrixMarketWriter writer(argv[6], n, d, n * z);
            std::size_t i = 0;
            while (gen.has_next()) writer.append_row(i++, gen.next());
            writer.close();
        } catch (const std::exception& e) {
            std::fprintf(stderr, "error: %s\n", e.what());
            return 1;
        }
        return 0;
    }
    const std::size_t plain = argc > 2 ? std::stoull(argv[2]) : 0;
    std::vector<int64_t> rp{0};
    std::vector<uint32_t> cs;
    std::vector<double> vs;
    int64_t d = 0, err = 0;
    std::string msg;
    try {
        std::optional<std::size_t> pc;
        if (plain) pc = plain;
        auto st = sfd::open_row_stream(argv[1], pc);
        d = (int64_t)st->cols();
        sfd::SparseRow r;
        while (st->next(r)) {
            cs.insert(cs.end(), r.indices.begin(), r.indices.end());
            vs.insert(vs.end(), r.values.begin(), r.values.end());
            rp.push_back((int64_t)cs.size());
        }
    } catch (const std::exception& e) {
        err = 1;
        msg = e.what();
    }
    const int64_t hdr[5] = {(int64_t)rp.size() - 1, d, (int64_t)cs.size(), err, (int64_t)msg.size()};
    std::fwrite(hdr, sizeof hdr, 1, stdout);
    std::fwrite(msg.data(), 1, msg.size(), stdout);
    std::fwrite(rp.data(), sizeof(int64_t), rp.size(), stdout);
    std::fwrite(cs.data(), sizeof(uint32_t), cs.size(), stdout);
    std::fwrite(vs.data(), sizeof(double), vs.size(), stdout);
    return 0;
}
