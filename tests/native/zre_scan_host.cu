// Host-only harness (no GPU): drives the device-side ZRE building blocks of
// paper_1802_07389_b200/csrc/tlc_device.cuh (literal_mask, mask_summary,
// mask_emit, compose, run_eval -- all __host__ __device__) through the same
// decomposition as the K3 kernel (compress.cu): `nchunks` contiguous chunks,
// each split into `warps` sub-chunks scanned in rows of 32 lanes x 32 bytes;
// in-order tree reductions (phase 1), the carry-in composed from per-thread
// partial compositions of the preceding chunk summaries (phase 2), per-row
// Hillis-Steele exclusive scans and emission at final offsets (phase 3).
// tests/test_zre_scan_host.py compares the output with the oracle's ZRE.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <vector>

#include "../../paper_1802_07389_b200/csrc/tlc_device.cuh"

using namespace tlc;

namespace {
constexpr int SEG = 32, LANES = 32;

RunSum tree_reduce(std::vector<RunSum> v) {   // shfl_down-style in-order tree
    for (size_t d = 1; d < v.size(); d <<= 1)
        for (size_t l = 0; l + d < v.size(); l += 2 * d) v[l] = compose(v[l], v[l + d]);
    return v.empty() ? run_identity() : v[0];
}

int seg_at(const uint8_t *B, uint64_t pos, uint64_t hi, uint32_t (&w)[8]) {
    const int len = pos < hi ? (int)std::min<uint64_t>(SEG, hi - pos) : 0;
    for (int k = 0; k < 8; k++) {
        uint32_t x = 0;
        for (int c = 0; c < 4; c++) x |= (uint32_t)(4 * k + c < len ? B[pos + 4 * k + c] : 121) << (8 * c);
        w[k] = x;
    }
    return len;
}
}  // namespace

extern "C" uint64_t zre_scan_sim(const uint8_t *B, uint64_t P, int warps, uint64_t nchunks_req, uint8_t *out) {
    uint64_t chunk = (P + nchunks_req - 1) / nchunks_req;
    chunk = (chunk + SEG - 1) / SEG * SEG;
    const uint64_t nch = (P + chunk - 1) / chunk;
    std::vector<RunSum> agg(nch);
    std::vector<std::vector<RunSum>> wagg(nch, std::vector<RunSum>(warps));
    auto bounds = [&](uint64_t b, int w, uint64_t &wlo, uint64_t &whi) {
        const uint64_t lo = b * chunk, hi = std::min(P, lo + chunk);
        const uint64_t sub = ((hi - lo + warps - 1) / warps + SEG - 1) / SEG * SEG;
        wlo = std::min(hi, lo + w * sub);
        whi = std::min(hi, wlo + sub);
    };
    for (uint64_t b = 0; b < nch; b++) {                 // phase 1
        RunSum a = run_identity();
        for (int w = 0; w < warps; w++) {
            uint64_t wlo, whi;
            bounds(b, w, wlo, whi);
            RunSum x = run_identity();
            for (uint64_t row = wlo; row < whi; row += (uint64_t)LANES * SEG) {
                std::vector<RunSum> v(LANES);
                for (int l = 0; l < LANES; l++) {
                    uint32_t s[8];
                    const int len = seg_at(B, row + (uint64_t)SEG * l, whi, s);
                    v[l] = mask_summary(literal_mask(s), len);
                }
                x = compose(x, tree_reduce(v));
            }
            wagg[b][w] = x;
            a = compose(a, x);
        }
        agg[b] = a;
    }
    uint64_t total = 0;
    const int threads = 32 * warps;
    for (uint64_t b = 0; b < nch; b++) {
        const uint64_t per = (b + threads - 1) / threads;   // phase 2
        std::vector<RunSum> part(threads, run_identity());
        for (int t = 0; t < threads; t++)
            for (uint64_t i = per * t; i < std::min<uint64_t>(b, per * t + per); i++) part[t] = compose(part[t], agg[i]);
        const RunSum chunk_in = tree_reduce(part);
        if (b == nch - 1) {
            uint64_t cnt;
            uint32_t carry;
            run_eval(compose(chunk_in, agg[b]), 0, cnt, carry);
            total = cnt + (carry > 0);
        }
        for (int w = 0; w < warps; w++) {                  // phase 3
            RunSum run = chunk_in;
            for (int k = 0; k < w; k++) run = compose(run, wagg[b][k]);
            uint64_t wlo, whi;
            bounds(b, w, wlo, whi);
            for (uint64_t row = wlo; row < whi; row += (uint64_t)LANES * SEG) {
                std::vector<RunSum> v(LANES);
                std::vector<std::vector<uint32_t>> segs(LANES, std::vector<uint32_t>(8));
                std::vector<int> lens(LANES);
                for (int l = 0; l < LANES; l++) {
                    uint32_t s[8];
                    lens[l] = seg_at(B, row + (uint64_t)SEG * l, whi, s);
                    std::memcpy(segs[l].data(), s, sizeof(s));
                    v[l] = mask_summary(literal_mask(s), lens[l]);
                }
                std::vector<RunSum> incl(v);
                for (int d = 1; d < LANES; d <<= 1) {
                    std::vector<RunSum> nx(incl);
                    for (int l = d; l < LANES; l++) nx[l] = compose(incl[l - d], incl[l]);
                    incl.swap(nx);
                }
                for (int l = 0; l < LANES; l++) {
                    if (lens[l] <= 0) continue;
                    const RunSum ex = l == 0 ? run_identity() : incl[l - 1];
                    uint64_t off;
                    uint32_t c;
                    run_eval(compose(run, ex), 0, off, c);
                    uint32_t s[8];
                    std::memcpy(s, segs[l].data(), sizeof(s));
                    mask_emit(s, literal_mask(s), lens[l], c, out, off);
                    if (c > 0 && row + (uint64_t)SEG * l + lens[l] == P) out[off++] = run_code(c);
                }
                run = compose(run, incl[LANES - 1]);
            }
        }
    }
    return total;
}
