// Host-only harness (no GPU): drives the device-side ZRE building blocks of
// paper_1802_07389_b200/csrc/tlc_device.cuh (literal_mask, mask_summary,
// lane_carry_in, row_carry_out, row_summary, compose, run_eval --
// all __host__ __device__) through the same decomposition as the K3 kernel
// (compress.cu): `nchunks` contiguous chunks, each split into `warps`
// sub-chunks scanned in warp rows of 32 lanes x 32 bytes (ballots and shuffles
// emulated serially); phase 1 composes row summaries, phase 2 composes the
// preceding chunk summaries, phase 3 tracks (offset, carry) across rows and
// emits each row from its literal list at the final offsets.
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

struct Row {
    uint32_t w[LANES][8], mask[LANES];
    int len[LANES];
    RunSum ls[LANES];
    uint32_t carry_in[LANES], count[LANES], row_count, carry_out, row_len;
    bool any;
    uint32_t lead;
};

// serial emulation of warp_row (ballot + shuffles)
void warp_row_host(Row &r, uint32_t c_row) {
    uint32_t mixbal = 0, lastpos[LANES];
    for (int l = 0; l < LANES; l++) {
        mixbal |= (uint32_t)(r.mask[l] != 0) << l;
        lastpos[l] = 32u * l + (r.mask[l] ? msb32(r.mask[l]) : 0u);
    }
    r.row_count = 0;
    for (int l = 0; l < LANES; l++) {
        const uint32_t before = mixbal & ((1u << l) - 1u);
        const uint32_t lp = lastpos[before ? msb32(before) : 0];
        r.carry_in[l] = lane_carry_in(l, before != 0, lp, c_row);
        uint64_t cnt;
        uint32_t co;
        run_eval(r.ls[l], r.carry_in[l], cnt, co);
        r.count[l] = r.len[l] > 0 ? (uint32_t)cnt : 0u;
        r.row_count += r.count[l];
    }
    r.any = mixbal != 0;
    r.carry_out = row_carry_out(r.any, lastpos[r.any ? msb32(mixbal) : 0], c_row, r.row_len);
    const uint32_t k0 = r.any ? ctz32(mixbal) : 0u;
    r.lead = (r.mask[k0] ? ctz32(r.mask[k0]) : 0u) + 32u * k0;
}

// K3 phase 3 for one warp row (serial form of the device code): a row without
// literals emits (carry + row_len)/14 full chunks; otherwise the row's literal
// list is walked, literal k preceded by R 121s emitting R/14 codes 255 (the
// prefilled range), a flush code if R%14 > 0 and the literal.
void emit_row_list(const Row &r, uint64_t row, uint64_t P, uint32_t &carry, uint8_t *out, uint64_t &off) {
    std::vector<uint32_t> lit;
    uint8_t bytes[LANES * SEG];
    for (int l = 0; l < LANES; l++)
        for (int m = 0; m < SEG; m++) {
            bytes[SEG * l + m] = (uint8_t)byte_at(r.w[l], m);
            if ((r.mask[l] >> m) & 1u) lit.push_back(SEG * l + m);
        }
    if (lit.empty()) {
        const uint32_t x = carry + r.row_len, cnt = x / kMaxRun;
        for (uint32_t k = 0; k < cnt; k++) out[off + k] = 0xff;
        carry = x - cnt * kMaxRun;
        off += cnt;
        if (carry > 0 && row + r.row_len == P) out[off] = run_code(carry);
        return;
    }
    const uint32_t L = (uint32_t)lit.size(), Rt = r.row_len - 1u - lit[L - 1];
    uint32_t total = 0;
    std::vector<uint32_t> R(L), cost(L);
    for (uint32_t k = 0; k < L; k++) {
        R[k] = lit[k] - (k ? lit[k - 1] + 1u : 0u) + (k ? 0u : carry);
        cost[k] = R[k] / kMaxRun + (R[k] % kMaxRun != 0) + 1u;
        total += cost[k];
    }
    const uint32_t row_count = total + Rt / kMaxRun;
    for (uint32_t k = 0; k < row_count; k++) out[off + k] = 0xff;
    uint64_t ex = 0;
    for (uint32_t k = 0; k < L; k++) {
        uint64_t o = off + ex + R[k] / kMaxRun;
        if (R[k] % kMaxRun) out[o++] = run_code(R[k] % kMaxRun);
        out[o] = bytes[lit[k]];
        ex += cost[k];
    }
    off += row_count;
    carry = Rt % kMaxRun;
    if (carry > 0 && row + r.row_len == P) out[off] = run_code(carry);
}

// K3 phase 3 for a row whose literal list was not kept (dense rows): every lane
// emits its own bytes with lane_emit into a stage prefilled with 255, at its
// exclusive-scanned offset; the row's output is then copied out.
void emit_row_lanes(const Row &r, uint64_t row, uint64_t P, uint32_t &carry, uint8_t *out, uint64_t &off,
                    int lane_mode) {
    uint8_t stage[pad_stage_bytes(LANES * SEG + 16)];
    std::memset(stage, 0xff, sizeof stage);
    const PadStage pst{stage};
    uint32_t o = 0;
    for (int l = 0; l < LANES; l++) {
        const uint32_t end = lane_mode == 5 ? lane_emit<4>(r.w[l], r.mask[l], r.carry_in[l], pst, o)
                             : lane_mode == 4 ? lane_emit<1>(r.w[l], r.mask[l], r.carry_in[l], pst, o)
                             : lane_mode == 3 ? lane_emit<3>(r.w[l], r.mask[l], r.carry_in[l], stage, o)
                             : lane_mode == 2 ? lane_emit<2>(r.w[l], r.mask[l], r.carry_in[l], stage, o)
                                              : lane_emit<1>(r.w[l], r.mask[l], r.carry_in[l], stage, o);
        if (r.len[l] > 0 && end > o + r.count[l]) std::abort();   // lane_emit never writes past its count
        o += r.count[l];
    }
    if (lane_mode >= 4)
        for (uint32_t q = 0; q < r.row_count; q++) out[off + q] = pst[q];   // the padded layout, logical order
    else
        std::memcpy(out + off, stage, r.row_count);
    off += r.row_count;
    carry = r.carry_out;
    if (carry > 0 && row + r.row_len == P) out[off] = run_code(carry);
}

void load_row(const uint8_t *B, uint64_t row, uint64_t whi, Row &r) {
    r.row_len = (uint32_t)std::min<uint64_t>((uint64_t)LANES * SEG, whi - row);
    for (int l = 0; l < LANES; l++) {
        r.len[l] = seg_at(B, row + (uint64_t)SEG * l, whi, r.w[l]);
        r.mask[l] = literal_mask(r.w[l]);
        r.ls[l] = mask_summary(r.mask[l], r.len[l]);
    }
}
}  // namespace

// sub_round: granule of a warp's sub-range (SEG, or a whole row as K3 does since it writes
// seek entries); seek != nullptr: at every row start that is a multiple of 4096 (a K5 tile
// start) record (payload offset << 4) | carry, as K3's phase 3 does
static uint64_t scan_impl(const uint8_t *B, uint64_t P, int warps, uint64_t chunk, uint8_t *out, int lane_mode,
                          uint64_t sub_round, uint64_t *seek) {
    const uint64_t nch = (P + chunk - 1) / chunk;
    std::vector<RunSum> agg(nch);
    std::vector<std::vector<RunSum>> wagg(nch, std::vector<RunSum>(warps));
    auto bounds = [&](uint64_t b, int w, uint64_t &wlo, uint64_t &whi) {
        const uint64_t lo = b * chunk, hi = std::min(P, lo + chunk);
        const uint64_t sub = ((hi - lo + warps - 1) / warps + sub_round - 1) / sub_round * sub_round;
        wlo = std::min(hi, lo + w * sub);
        whi = std::min(hi, wlo + sub);
    };
    static Row r;
    for (uint64_t b = 0; b < nch; b++) {                 // phase 1
        RunSum a = run_identity();
        for (int w = 0; w < warps; w++) {
            uint64_t wlo, whi;
            bounds(b, w, wlo, whi);
            RunSum x = run_identity();
            for (uint64_t row = wlo; row < whi; row += (uint64_t)LANES * SEG) {
                load_row(B, row, whi, r);
                warp_row_host(r, 0);
                x = compose(x, row_summary(r.any, r.lead, r.row_count, r.carry_out, r.row_len));
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
            RunSum before = chunk_in;
            for (int k = 0; k < w; k++) before = compose(before, wagg[b][k]);
            uint64_t off;
            uint32_t carry;
            run_eval(before, 0, off, carry);
            uint64_t wlo, whi;
            bounds(b, w, wlo, whi);
            for (uint64_t row = wlo; row < whi; row += (uint64_t)LANES * SEG) {
                if (seek && row % 4096 == 0) seek[row / 4096] = (off << 4) | carry;
                load_row(B, row, whi, r);
                warp_row_host(r, carry);
                if (lane_mode) emit_row_lanes(r, row, P, carry, out, off, lane_mode);
                else emit_row_list(r, row, P, carry, out, off);
            }
        }
    }
    return total;
}

extern "C" uint64_t zre_scan_sim_mode(const uint8_t *B, uint64_t P, int warps, uint64_t nchunks_req, uint8_t *out,
                                      int lane_mode) {
    uint64_t chunk = (P + nchunks_req - 1) / nchunks_req;
    chunk = (chunk + SEG - 1) / SEG * SEG;
    return scan_impl(B, P, warps, chunk, out, lane_mode, SEG, nullptr);
}

// K3's decomposition as built (chunks of `chunk` bytes, a multiple of 4096; warps take whole
// 1 KiB rows) with the producer seek entries of every K5 tile written to seek[ceil(P/4096)]
extern "C" uint64_t zre_seek_sim(const uint8_t *B, uint64_t P, int warps, uint64_t chunk, uint8_t *out,
                                 uint64_t *seek) {
    return scan_impl(B, P, warps, chunk, out, 0, (uint64_t)LANES * SEG, seek);
}

extern "C" uint64_t zre_scan_sim(const uint8_t *B, uint64_t P, int warps, uint64_t nchunks_req, uint8_t *out) {
    return zre_scan_sim_mode(B, P, warps, nchunks_req, out, 0);
}

// K4's SWAR expansion length of a payload word (tlc_device.cuh word_len), host form
extern "C" uint32_t tlc_word_len(uint32_t w) { return word_len(w); }
