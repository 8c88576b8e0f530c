// Host-only harness (no GPU): drives the device-side ZRE building blocks of
// paper_1802_07389_b200/csrc/tlc_device.cuh (segment_summary, compose, run_eval,
// segment_emit -- all __host__ __device__) through the same decomposition the
// K3 kernel (compress.cu) uses: `nchunks` contiguous chunks, rows of
// threads x 32-byte segments, in-order tree reductions (phase 1), the carry-in
// composed from per-thread partial compositions of the preceding chunk
// summaries (phase 2), and per-row Hillis-Steele exclusive scans with emission
// at the final offsets (phase 3).  tests/test_zre_scan_host.py compares the
// output with the oracle's zero-run encoding.
#include <algorithm>
#include <array>
#include <cstdint>
#include <cstring>
#include <vector>

#include "../../paper_1802_07389_b200/csrc/tlc_device.cuh"

using namespace tlc;

namespace {
constexpr int NW = 8;
constexpr int SEG = 4 * NW;

RunSum tree_reduce(std::vector<RunSum> v) {   // shfl_down-style in-order tree
    for (size_t d = 1; d < v.size(); d <<= 1)
        for (size_t l = 0; l + d < v.size(); l += 2 * d) v[l] = compose(v[l], v[l + d]);
    return v.empty() ? run_identity() : v[0];
}

int seg_at(const uint8_t *B, uint64_t pos, uint64_t hi, uint32_t (&w)[NW]) {
    const int len = pos < hi ? (int)std::min<uint64_t>(SEG, hi - pos) : 0;
    for (int k = 0; k < NW; k++) {
        uint32_t x = 0;
        for (int c = 0; c < 4; c++) x |= (uint32_t)(4 * k + c < len ? B[pos + 4 * k + c] : 121) << (8 * c);
        w[k] = x;
    }
    return len;
}
}  // namespace

extern "C" uint64_t zre_scan_sim(const uint8_t *B, uint64_t P, int threads, uint64_t nchunks_req, uint8_t *out) {
    const uint64_t row_bytes = (uint64_t)threads * SEG;
    uint64_t chunk = (P + nchunks_req - 1) / nchunks_req;
    chunk = (chunk + SEG - 1) / SEG * SEG;
    const uint64_t nch = (P + chunk - 1) / chunk;
    std::vector<RunSum> agg(nch);
    // phase 1
    for (uint64_t b = 0; b < nch; b++) {
        const uint64_t lo = b * chunk, hi = std::min(P, lo + chunk);
        RunSum a = run_identity();
        for (uint64_t row = lo; row < hi; row += row_bytes) {
            std::vector<RunSum> v(threads);
            for (int t = 0; t < threads; t++) {
                uint32_t s[NW];
                const int len = seg_at(B, row + (uint64_t)SEG * t, hi, s);
                v[t] = segment_summary(s, len);
            }
            a = compose(a, tree_reduce(v));
        }
        agg[b] = a;
    }
    uint64_t total = 0;
    for (uint64_t b = 0; b < nch; b++) {
        const uint64_t lo = b * chunk, hi = std::min(P, lo + chunk);
        // phase 2
        const uint64_t per = (b + threads - 1) / threads;
        std::vector<RunSum> part(threads, run_identity());
        for (int t = 0; t < threads; t++)
            for (uint64_t i = per * t; i < std::min<uint64_t>(b, per * t + per); i++) part[t] = compose(part[t], agg[i]);
        RunSum run = tree_reduce(part);
        if (b == nch - 1) {
            uint64_t cnt;
            uint32_t carry;
            run_eval(compose(run, agg[b]), 0, cnt, carry);
            total = cnt + (carry > 0);
        }
        // phase 3
        for (uint64_t row = lo; row < hi; row += row_bytes) {
            std::vector<RunSum> v(threads), incl(threads);
            std::vector<std::array<uint32_t, NW>> segs(threads);
            std::vector<int> lens(threads);
            for (int t = 0; t < threads; t++) {
                uint32_t s[NW];
                lens[t] = seg_at(B, row + (uint64_t)SEG * t, hi, s);
                std::memcpy(segs[t].data(), s, sizeof(s));
                v[t] = segment_summary(s, lens[t]);
            }
            incl = v;
            for (int d = 1; d < threads; d <<= 1) {
                std::vector<RunSum> nx(incl);
                for (int t = d; t < threads; t++) nx[t] = compose(incl[t - d], incl[t]);
                incl.swap(nx);
            }
            for (int t = 0; t < threads; t++) {
                if (lens[t] <= 0) continue;
                const RunSum ex = t == 0 ? run_identity() : incl[t - 1];
                uint64_t off;
                uint32_t c;
                run_eval(compose(run, ex), 0, off, c);
                uint32_t s[NW];
                std::memcpy(s, segs[t].data(), sizeof(s));
                segment_emit(s, lens[t], c, out, off);
                if (c > 0 && row + (uint64_t)SEG * t + lens[t] == P) out[off++] = run_code(c);
            }
            run = compose(run, incl[threads - 1]);
        }
    }
    return total;
}
