// prof.cu -- optional per-kernel-class device timing (CUDA events on the launching stream).
//
// Off by default (zero cost). bench.py turns it on for one extra, untimed-for-throughput
// step to measure each kernel class's average launch duration on the stream it runs
// on, which feeds the roofline numbers (achieved = algorithmic bytes or flops / duration).
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/sfdg.h"
#include "common.cuh"

namespace sfdg {

namespace {
struct Rec {
    const char* cls;
    cudaEvent_t e0, e1;
};
std::mutex g_mu;
std::vector<Rec> g_recs;
}  // namespace

std::atomic<bool> g_prof_on{false};

ProfScope::ProfScope(const char* cls, cudaStream_t st) : st_(st) {
    if (!g_prof_on.load(std::memory_order_relaxed)) return;
    cls_ = cls;
    cudaEventCreate(&e0_);
    cudaEventCreate(&e1_);
    cudaEventRecord(e0_, st_);
}

ProfScope::~ProfScope() {
    if (!cls_) return;
    cudaEventRecord(e1_, st_);
    std::lock_guard<std::mutex> lk(g_mu);
    g_recs.push_back({cls_, e0_, e1_});
}

}  // namespace sfdg

using namespace sfdg;

extern "C" {

int sfdg_profile_begin(void) {
    std::lock_guard<std::mutex> lk(g_mu);
    for (auto& r : g_recs) {
        cudaEventDestroy(r.e0);
        cudaEventDestroy(r.e1);
    }
    g_recs.clear();
    g_prof_on = true;
    return SFDG_OK;
}

// Writes {"class": [total_ms, launches], ...} into buf (NUL-terminated, truncated to n).
int sfdg_profile_end(char* buf, size_t n) {
    g_prof_on = false;
    cudaDeviceSynchronize();
    std::map<std::string, std::pair<double, int>> acc;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        for (auto& r : g_recs) {
            float ms = 0.f;
            if (cudaEventElapsedTime(&ms, r.e0, r.e1) == cudaSuccess) {
                auto& a = acc[r.cls];
                a.first += ms;
                a.second += 1;
            }
            cudaEventDestroy(r.e0);
            cudaEventDestroy(r.e1);
        }
        g_recs.clear();
    }
    cudaGetLastError();
    std::string s = "{";
    bool first = true;
    for (auto& kv : acc) {
        char tmp[160];
        snprintf(tmp, sizeof tmp, "%s\"%s\": [%.6f, %d]", first ? "" : ", ", kv.first.c_str(), kv.second.first,
                 kv.second.second);
        s += tmp;
        first = false;
    }
    s += "}";
    if (buf && n) {
        const size_t k = std::min(n - 1, s.size());
        memcpy(buf, s.data(), k);
        buf[k] = 0;
    }
    return SFDG_OK;
}

}  // extern "C"
