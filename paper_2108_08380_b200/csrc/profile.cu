// profile.cu — kernel-level tracing for the C ABI (bd_profile_*): a CUDA event pair around
// every kernel launch the library makes while recording is on; totals per kernel name.
#include <nvtx3/nvToolsExt.h>
#include <mutex>
#include <string>
#include <vector>

#include "internal.cuh"

namespace bd {
namespace {

struct Pending {
    int slot;
    cudaEvent_t a, b;
};
struct Slot {
    std::string name;
    int64_t launches = 0;
    double ms = 0.0;
};

std::mutex g_mu;
bool g_on = false;
std::vector<Slot> g_slots;
std::vector<Pending> g_pending;
std::vector<cudaEvent_t> g_free;

cudaEvent_t get_event() {
    if (!g_free.empty()) {
        cudaEvent_t e = g_free.back();
        g_free.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

int slot_of(const char* name) {
    for (size_t i = 0; i < g_slots.size(); ++i)
        if (g_slots[i].name == name) return (int)i;
    g_slots.push_back(Slot{name});
    return (int)g_slots.size() - 1;
}

void drain_locked() {
    for (auto& p : g_pending) {
        float ms = 0.f;
        if (cudaEventSynchronize(p.b) == cudaSuccess && cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) {
            g_slots[p.slot].launches += 1;
            g_slots[p.slot].ms += ms;
        }
        g_free.push_back(p.a);
        g_free.push_back(p.b);
    }
    g_pending.clear();
}

}  // namespace

// Every scope is also an NVTX range (nvtx3, header-only: a no-op unless a tool such as nsys or
// ncu --nvtx injects itself), so external timelines show the library's kernels by C-ABI step.
ProfScope::ProfScope(const char* name, cudaStream_t s) : s_(s), idx_(-1) {
    nvtxRangePushA(name);
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g_on) return;
    Pending p{slot_of(name), get_event(), get_event()};
    cudaEventRecord(p.a, s);
    g_pending.push_back(p);
    idx_ = (int)g_pending.size() - 1;
}

ProfScope::~ProfScope() {
    if (idx_ >= 0) {
        std::lock_guard<std::mutex> lk(g_mu);
        if (idx_ < (int)g_pending.size()) cudaEventRecord(g_pending[idx_].b, s_);
    }
    nvtxRangePop();
}

}  // namespace bd

extern "C" {

int bd_profile_start(void) {
    std::lock_guard<std::mutex> lk(bd::g_mu);
    bd::drain_locked();
    bd::g_slots.clear();
    bd::g_on = true;
    return BD_OK;
}

int bd_profile_stop(void) {
    std::lock_guard<std::mutex> lk(bd::g_mu);
    bd::g_on = false;
    return BD_OK;
}

int bd_profile_query(int i, const char** name, int64_t* launches, double* ms) {
    std::lock_guard<std::mutex> lk(bd::g_mu);
    bd::drain_locked();
    if (i < 0 || i >= (int)bd::g_slots.size()) return BD_EINVAL;
    if (name) *name = bd::g_slots[i].name.c_str();
    if (launches) *launches = bd::g_slots[i].launches;
    if (ms) *ms = bd::g_slots[i].ms;
    return BD_OK;
}

}  // extern "C"
