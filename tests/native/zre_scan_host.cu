// Host-only harness (no GPU): drives the device-side ZRE scan building blocks of
// paper_1802_07389_b200/csrc/tlc_device.cuh (segment_summary, compose, run_eval,
// segment_emit -- all __host__ __device__) through the same decomposition the
// K2 kernel uses: 8-byte thread segments, Hillis-Steele warp scans, per-tile
// aggregates and a decoupled look-back over windows of 32 predecessors whose
// publication state (aggregate only / inclusive prefix) is drawn at random.
// tests/test_zre_scan_host.py compares its output with the oracle's ZRE.
#include <cstdint>
#include <array>
#include <algorithm>
#include <cstring>
#include <random>
#include <vector>

#include "../../paper_1802_07389_b200/csrc/tlc_device.cuh"

using namespace tlc;

extern "C" uint64_t zre_scan_sim(const uint8_t *B, uint64_t P, int threads, uint64_t seed, uint8_t *out) {
    constexpr int SEG = 8;
    const uint64_t T = (uint64_t)threads * SEG;
    const uint64_t num_tiles = (P + T - 1) / T;
    std::mt19937_64 rng(seed);
    std::vector<RunSum> tile_agg(num_tiles), tile_incl(num_tiles);
    std::vector<int> has_prefix(num_tiles, 0);
    uint64_t total = 0;
    for (uint64_t tile = 0; tile < num_tiles; tile++) {
        const uint64_t j0 = tile * T;
        const int tile_len = (int)std::min<uint64_t>(T, P - j0);
        std::vector<RunSum> mine(threads);
        std::vector<std::array<uint8_t, SEG>> segs(threads);
        std::vector<int> slen(threads);
        for (int th = 0; th < threads; th++) {
            uint8_t b[SEG];
            const int sbeg = th * SEG;
            slen[th] = std::max(0, std::min(SEG, tile_len - sbeg));
            for (int m = 0; m < SEG; m++) b[m] = (m < slen[th]) ? B[j0 + sbeg + m] : 0;
            std::memcpy(segs[th].data(), b, SEG);
            mine[th] = segment_summary(b, slen[th]);
        }
        // warp inclusive scans (Hillis-Steele, as with shfl_up)
        std::vector<RunSum> incl(mine);
        const int nw = (threads + 31) / 32;
        for (int w = 0; w < nw; w++) {
            const int lo = w * 32, hi = std::min(threads, lo + 32);
            for (int d = 1; d < 32; d <<= 1) {
                std::vector<RunSum> nx(incl.begin() + lo, incl.begin() + hi);
                for (int l = lo; l < hi; l++)
                    if (l - lo >= d) nx[l - lo] = compose(incl[l - d], incl[l]);
                std::copy(nx.begin(), nx.end(), incl.begin() + lo);
            }
        }
        std::vector<RunSum> warp_excl(nw);
        RunSum agg = run_identity();
        for (int w = 0; w < nw; w++) {
            warp_excl[w] = agg;
            agg = compose(agg, incl[std::min(threads, w * 32 + 32) - 1]);
        }
        // decoupled look-back over windows of 32 predecessors
        RunSum excl = run_identity();
        if (tile > 0) {
            int64_t pred = (int64_t)tile - 1;
            while (true) {
                RunSum v[32];
                int first = 31;
                bool found = false;
                for (int l = 0; l < 32; l++) {
                    const int64_t idx = pred - l;
                    if (idx < 0) { v[l] = run_identity(); if (!found) { first = l; found = true; } continue; }
                    if (has_prefix[idx]) { v[l] = tile_incl[idx]; if (!found) { first = l; found = true; } }
                    else v[l] = tile_agg[idx];
                }
                for (int l = first + 1; l < 32; l++) v[l] = run_identity();
                for (int d = 1; d < 32; d <<= 1)      // tree reduction as with shfl_down
                    for (int l = 0; l + d < 32; l++) v[l] = compose(v[l + d], v[l]);
                excl = compose(v[0], excl);
                if (found) break;
                pred -= 32;
            }
        }
        tile_agg[tile] = agg;
        tile_incl[tile] = compose(excl, agg);
        has_prefix[tile] = (tile == 0) || (rng() % 3 == 0);   // some tiles publish only aggregates
        // emission
        for (int th = 0; th < threads; th++) {
            if (slen[th] <= 0) continue;
            const int w = th / 32, l = th % 32;
            RunSum texcl = l == 0 ? run_identity() : incl[th - 1];
            RunSum before = compose(excl, compose(warp_excl[w], texcl));
            uint64_t off;
            uint32_t c;
            run_eval(before, 0, off, c);
            uint8_t b[SEG];
            std::memcpy(b, segs[th].data(), SEG);
            segment_emit(b, slen[th], c, out, off);
            if (c > 0 && j0 + th * SEG + slen[th] == P) out[off++] = run_code(c);
            total = std::max(total, off);
        }
        if (tile == num_tiles - 1) {
            uint64_t cnt;
            uint32_t carry;
            run_eval(tile_incl[tile], 0, cnt, carry);
            if (cnt + (carry > 0) != total) return ~0ull;    // header length disagrees
        }
    }
    return total;
}
