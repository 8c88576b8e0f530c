// prof.cu -- launch counting and optional per-kernel CUDA-event timing.
//
// Every kernel launch of the library goes through KernelScope, which bumps a
// global launch counter and, when profiling is enabled (tlc_prof_enable),
// brackets the launch with a pair of CUDA events recorded on the launching
// stream.  tlc_prof_collect() synchronizes those events and reports per-kernel
// launch counts and summed device durations -- bench.py uses it for the live
// roofline of the dominant kernel.
#include <atomic>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "tlc_launch.h"

namespace tlc {

static const char *kNames[kNumKernelIds] = {"k1_absmax", "k2_quant_qe", "k3_zre",
                                            "k4_zre_scan", "k5_expand_dequant",
                                            "k5m_aggregate", "k9_flag_barrier",
                                            "k8_scale_mean", "k2s_stoch_qe",
                                            "kq8_int8_quant", "kd8_int8_dequant",
                                            "k6_small_compress", "k7_small_decompress",
                                            "k12_absmax_quant"};

namespace {
struct Rec {
    int id, dev;
    cudaEvent_t a, b;
};
std::atomic<unsigned long long> g_launches{0};
std::atomic<bool> g_on{false};
std::mutex g_mu;
std::vector<Rec> g_recs;
std::vector<cudaEvent_t> g_pool[64];                 // per device: an event records only on its device's streams

cudaEvent_t get_event(int dev) {
    if (!g_pool[dev].empty()) {
        cudaEvent_t e = g_pool[dev].back();
        g_pool[dev].pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}
}  // namespace

KernelScope::KernelScope(int id, cudaStream_t st) : id_(id), st_(st), a_(nullptr) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if (g_on.load(std::memory_order_relaxed)) {
        std::lock_guard<std::mutex> lk(g_mu);
        dev_ = cur_device();
        a_ = get_event(dev_);
        cudaEventRecord((cudaEvent_t)a_, st_);
    }
}

KernelScope::~KernelScope() {
    if (a_) {
        std::lock_guard<std::mutex> lk(g_mu);
        cudaEvent_t b = get_event(dev_);
        cudaEventRecord(b, st_);
        g_recs.push_back(Rec{id_, dev_, (cudaEvent_t)a_, b});
    }
}

// Programmatic dependent launch between the kernels of a call is opt-in
// (TLC_PDL=1): measured on B200 it gained nothing on the 2^28-value step and
// cost ~15 % on the 110-tensor ResNet-110 step (profiles/r01_pdl_ab.txt).
bool pdl_enabled() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("TLC_PDL");
        v = (e && e[0] == '1') ? 1 : 0;
    }
    return v == 1;
}

}  // namespace tlc

using namespace tlc;

extern "C" {

unsigned long long tlc_launch_count(void) { return g_launches.load(); }

void tlc_prof_enable(int on) { g_on.store(on != 0); }

int tlc_prof_collect(tlc_prof_entry *out, int cap) {
    std::lock_guard<std::mutex> lk(g_mu);
    double ms[kNumKernelIds] = {0};
    unsigned long long cnt[kNumKernelIds] = {0};
    for (auto &r : g_recs) {
        float t = 0.f;
        cudaEventSynchronize(r.b);
        cudaEventElapsedTime(&t, r.a, r.b);
        ms[r.id] += t;
        cnt[r.id] += 1;
        g_pool[r.dev].push_back(r.a);
        g_pool[r.dev].push_back(r.b);
    }
    g_recs.clear();
    int k = 0;
    for (int i = 0; i < kNumKernelIds; i++) {
        if (!cnt[i]) continue;
        if (k < cap && out) {
            out[k].name = kNames[i];
            out[k].launches = cnt[i];
            out[k].total_ms = ms[i];
        }
        k++;
    }
    return k;
}

}  // extern "C"
