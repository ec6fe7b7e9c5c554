// C-ABI glue: error reporting, version, launch accounting and kernel timing
// (see include/msfm_b200.h).
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <atomic>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

namespace msfm {
static thread_local char g_err[1024] = "";
static std::atomic<long long> g_launches{0};

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

void count_launches(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// Optional per-kernel CUDA-event timing on the launching stream.
struct ProfRecord {
    std::string name;
    cudaEvent_t start, stop;
};
static std::mutex g_prof_mu;
static bool g_prof_on = false;
static std::vector<ProfRecord> g_prof;

bool profiling() { return g_prof_on; }

void prof_begin(const char* name, cudaStream_t st, void** token) {
    *token = nullptr;
    if (!g_prof_on) return;
    ProfRecord r;
    r.name = name;
    cudaEventCreate(&r.start);
    cudaEventCreate(&r.stop);
    cudaEventRecord(r.start, st);
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof.push_back(r);
    *token = (void*)(g_prof.size());
}

void prof_end(void* token, cudaStream_t st) {
    if (!token) return;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    size_t i = (size_t)token - 1;
    if (i < g_prof.size()) cudaEventRecord(g_prof[i].stop, st);
}
}  // namespace msfm

extern "C" const char* msfm_last_error(void) { return msfm::g_err; }
extern "C" int msfm_version(void) { return 2; }
extern "C" int64_t msfm_launch_count(void) { return msfm::g_launches.load(); }

extern "C" int msfm_profile_enable(int on) {
    std::lock_guard<std::mutex> lk(msfm::g_prof_mu);
    for (auto& r : msfm::g_prof) {
        cudaEventDestroy(r.start);
        cudaEventDestroy(r.stop);
    }
    msfm::g_prof.clear();
    msfm::g_prof_on = on != 0;
    return MSFM_OK;
}

extern "C" int msfm_profile_read(const char* name, double* total_ms, int64_t* launches) {
    if (!name || !total_ms || !launches) {
        msfm::set_error("msfm_profile_read: null argument");
        return MSFM_EINVAL;
    }
    std::lock_guard<std::mutex> lk(msfm::g_prof_mu);
    double tot = 0.0;
    int64_t n = 0;
    for (auto& r : msfm::g_prof) {
        if (r.name != name) continue;
        MSFM_CUDA_TRY(cudaEventSynchronize(r.stop));
        float ms = 0.f;
        MSFM_CUDA_TRY(cudaEventElapsedTime(&ms, r.start, r.stop));
        tot += ms;
        n++;
    }
    *total_ms = tot;
    *launches = n;
    return MSFM_OK;
}
