// prof.cu -- optional per-kernel-class device timing (CUDA events on the launching stream).
//
// Off by default (zero cost). bench.py turns it on for one extra, untimed-for-throughput
// step to measure each kernel class's average launch duration on the stream it runs
// on, which feeds the roofline numbers (achieved = algorithmic bytes or flops / duration).
#include <map>
#include <set>
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
    double flops, bytes;
};
std::mutex g_mu;
std::vector<Rec> g_recs;
}  // namespace

std::atomic<bool> g_prof_on{false};

bool first_on_device(const void* key) {
    static std::mutex mu;
    static std::set<std::pair<int, const void*>> seen;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> g(mu);
    return seen.insert({dev, key}).second;
}

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
    g_recs.push_back({cls_, e0_, e1_, flops_, bytes_});
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

// Writes {"class": [total_ms, launches, flops, bytes], ...} into buf (NUL-terminated,
// truncated to n); flops / bytes are the algorithmic work the launchers declared.
int sfdg_profile_end(char* buf, size_t n) {
    g_prof_on = false;
    cudaDeviceSynchronize();
    struct Acc {
        double ms = 0.0;
        int n = 0;
        double flops = 0.0, bytes = 0.0;
    };
    std::map<std::string, Acc> acc;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        for (auto& r : g_recs) {
            float ms = 0.f;
            if (cudaEventElapsedTime(&ms, r.e0, r.e1) == cudaSuccess) {
                auto& a = acc[r.cls];
                a.ms += ms;
                a.n += 1;
                a.flops += r.flops;
                a.bytes += r.bytes;
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
        char tmp[200];
        snprintf(tmp, sizeof tmp, "%s\"%s\": [%.6f, %d, %.6e, %.6e]", first ? "" : ", ", kv.first.c_str(), kv.second.ms,
                 kv.second.n, kv.second.flops, kv.second.bytes);
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
