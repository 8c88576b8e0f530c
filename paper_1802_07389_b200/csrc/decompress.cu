// decompress.cu -- the 3LC decompressor on sm_100a (rows a5-a6) over a table of
// tensors (segments, tlc_launch.h).
//
//  K4 tlc_zre_scan_kernel: validates each segment's header (status, n, length,
//     M finite >= +0) and, with ZRE, scans the expansion lengths
//     len(b) = b >= 243 ? b-241 : 1 (inverse of P:545-546) with the chunked
//     single-pass scan of K3 over the sum monoid.  For every output tile start
//     J0 = k*kT5 it writes a seek entry (payload byte covering J0, offset inside
//     it); the chunk holding the last payload byte checks the expansion is
//     exactly P bytes, else FORMAT.
//  K5 tlc_expand_dequant_kernel: output-driven tiles of kT5 quartic bytes =
//     5*kT5 fp32 outputs, so every CTA does the same work whatever the run
//     structure: 121 prefill of shared memory, scatter of the literal bytes of
//     the covering payload window, base-3 decode and Eq. 3
//      through a per-segment table V[i][b] = M*(digit_i(b) - 1),
//     128-bit stores to the five partitions (or, in ACCUMULATE mode, a
//     read-modify-write of the elements whose q != 0, R16).
#include <algorithm>
#include <cstdlib>

#include "tlc_device.cuh"
#include "tlc_launch.h"

namespace tlc {

// ============================================================== K4
constexpr int kK4Threads = kScanThreads;
constexpr int kK4Seg = 16;

// Payload bytes [pos, min(pos+16, hi)) as 4 words and their total expansion
// length; n = the number of bytes present.
__device__ __forceinline__ uint32_t pay16(const uint8_t *__restrict__ p, uint64_t pos, uint64_t hi,
                                          uint32_t (&w)[4], int &n) {
    n = pos < hi ? (int)tmin<uint64_t>(kK4Seg, hi - pos) : 0;
    if (n == kK4Seg && (reinterpret_cast<uintptr_t>(p + pos) & 15u) == 0) {
        const uint4 v = __ldg(reinterpret_cast<const uint4 *>(p + pos));
        w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
        return word_len(w[0]) + word_len(w[1]) + word_len(w[2]) + word_len(w[3]);
    }
    uint32_t sum = 0;
#pragma unroll
    for (int k = 0; k < 4; k++) w[k] = 0;
#pragma unroll
    for (int k = 0; k < kK4Seg; k++)
        if (k < n) {
            const uint32_t b = p[pos + k];
            w[k >> 2] |= b << (8 * (k & 3));
            sum += zre_len(b);
        }
    return sum;
}

// rows of 32 lanes x 16 bytes per warp and chunk (the large item size; small chunks use fewer)
constexpr int kK4Rows = (int)(kLargeItems.c4 / kScanWarps / (32 * kK4Seg));
static_assert(kK4Rows * kScanWarps * 32 * kK4Seg == (int)kLargeItems.c4, "whole rows per warp");
static_assert(kSmallItems.c4 <= kLargeItems.c4, "small chunks need no more rows");

__global__ void __launch_bounds__(kK4Threads)
tlc_zre_scan_kernel(const SegTable T, Ctrl *ctrl, unsigned long long *states, unsigned long long *seek) {
    __shared__ unsigned long long s_warp[kScanWarps];
    __shared__ unsigned long long s_wsum[kScanWarps];
    __shared__ unsigned long long s_id;
    __shared__ uint64_t s_first[kSegCache];
    pdl_trigger();
    seg_index_load<4>(T, s_first);
    while (true) {
        if (threadIdx.x == 0) s_id = atomicAdd(&ctrl->k4_counter, 1ull);
        __syncthreads();
        const uint64_t id = s_id;
        __syncthreads();
        if (id >= T.n4) break;
        const int si = find_seg_c<4>(T, id, s_first);
        const Seg S = get_seg(T, si);
        const uint64_t lc = id - S.k4;
        tlc_header *hdr = S.hdr;
        // Chunks are sized by P (Z is only known on the device); once a chunk of a
        // segment has nothing to scan, neither have the segment's later ones, and
        // no chunk with work waits on them: advance the counter past the segment.
        const uint64_t seg_end = S.k4 + (S.P + T.sz.c4 - 1) / T.sz.c4;
        if (!header_valid(hdr, S.n)) {                    // uniform over the CTA
            if (threadIdx.x == 0) {
                if (lc == 0 && hdr->status == TLC_OK) raise_format(hdr);
                atomicMax(&ctrl->k4_counter, (unsigned long long)seg_end);
            }
            continue;
        }
        const uint64_t P = S.P, Z = hdr->payload_len;
        const uint64_t lo = lc * T.sz.c4, hi = tmin<uint64_t>(Z, lo + T.sz.c4);
        if (!(hdr->flags & TLC_FLAG_ZRE) || lo >= Z) {    // no ZRE (K5 reads the quartic bytes
            if (threadIdx.x == 0)                         // directly) or past the payload
                atomicMax(&ctrl->k4_counter, (unsigned long long)seg_end);
            continue;
        }
        const uint64_t num_out_tiles = (P + kT5 - 1) / kT5;

        // the chunk is split into one sub-range per warp, scanned in warp rows of 32 x 16 bytes
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        constexpr uint64_t kWRow = 32 * kK4Seg;
        const uint64_t sub = ((hi - lo + kScanWarps - 1) / kScanWarps + kK4Seg - 1) / kK4Seg * kK4Seg;
        const uint64_t wlo = tmin<uint64_t>(hi, lo + warp * sub), whi = tmin<uint64_t>(hi, wlo + sub);

        // ---- phase 1: expansion length of each warp's sub-range, then of the chunk.  The
        // rows' loads are all issued before any reduction, and every lane keeps its rows'
        // sums for phase 3 (which then reloads bytes only where an output tile starts).
        uint32_t wv[4];
        int nb;
        uint32_t rsum[kK4Rows];
#pragma unroll
        for (int r = 0; r < kK4Rows; r++)
            rsum[r] = pay16(S.payload, wlo + (uint64_t)r * kWRow + (uint64_t)kK4Seg * lane, whi, wv, nb);
        uint64_t wsum = 0;
#pragma unroll
        for (int r = 0; r < kK4Rows; r++) {
            uint32_t sum = rsum[r];
#pragma unroll
            for (int d = 16; d >= 1; d >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, d);
            wsum += sum;
        }
        if (lane == 0) s_wsum[warp] = wsum;
        __syncthreads();
        uint64_t agg = 0, before = 0;
#pragma unroll
        for (int k = 0; k < kScanWarps; k++) {
            before += k < warp ? s_wsum[k] : 0ull;
            agg += s_wsum[k];
        }
        if (threadIdx.x == 0) st_relaxed_u64(states + id, (lc == 0 ? kPrefix : kReady) | agg);

        // ---- phase 2: quartic position of the chunk's first byte (look-back)
        if (warp == 0) {
            const unsigned long long ex = warp_lookback<SumOp>(states + S.k4, lc);
            if (lane == 0) {
                if (lc > 0) st_relaxed_u64(states + id, kPrefix | (ex + agg));
                s_warp[0] = ex;
            }
        }
        __syncthreads();
        const uint64_t run = s_warp[0];
        if (hi == Z && threadIdx.x == 0 && run + agg != P) raise_format(hdr);

        // ---- phase 3: seek entries (payload byte covering J0 = k*kT5, offset inside it).  A
        // lane's 16 bytes expand to at most 16*14 < kT5 positions: at most one J0 falls in them.
        uint64_t q0 = run + before;                       // position of the warp's first byte
#pragma unroll
        for (int r = 0; r < kK4Rows; r++) {
            const uint64_t row = wlo + (uint64_t)r * kWRow;
            if (row >= whi) break;                        // warp-uniform
            const uint64_t pos0 = row + (uint64_t)kK4Seg * lane;
            const uint32_t sum = rsum[r];
            uint32_t x = sum;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
                if (lane >= d) x += y;
            }
            uint64_t q = q0 + (x - sum);
            const uint64_t kt = (q + kT5 - 1) / kT5, J0 = kt * kT5;
            if (J0 < q + sum && kt < num_out_tiles) {
                pay16(S.payload, pos0, whi, wv, nb);      // this lane's bytes again (L2)
#pragma unroll
                for (int k = 0; k < kK4Seg; k++) {
                    if (k >= nb) break;
                    const uint32_t len = zre_len((wv[k >> 2] >> (8 * (k & 3))) & 0xffu);
                    if (J0 < q + len) {
                        seek[S.k5 + kt] = ((pos0 + k) << 4) | (J0 - q);
                        break;
                    }
                    q += len;
                }
            }
            q0 += __shfl_sync(0xffffffffu, x, 31);
        }
    }
}

// ============================================================== K5
constexpr int kK5Threads = 256;
constexpr int kK5BytesPerThread = kT5 / kK5Threads;   // 16 quartic bytes per thread per tile
constexpr int kK5Words = kK5BytesPerThread / 4;

struct K5Smem {
    alignas(16) uint8_t E[kT5];          // expanded quartic bytes of the tile
    uint32_t V[5][256];                  // Eq. 3 output bits of partition i for byte value b
    uint16_t lut[256];                   // per byte: bit i = (digit_i != 1)
    uint16_t dig[256];                   // per byte: digit_i at bits 2i (no dependence on M)
    unsigned int warp_sum[kK5Threads / 32];
};

// Without ZRE: the quartic bytes as sent, 16 per thread (one 128-bit load when aligned); a
// byte > 242 is not a quartic code -> FORMAT, replaced by 121 meanwhile.  Out of
// line so that the ZRE path's register allocation (and K5's occupancy) is unaffected.
__device__ __noinline__ bool copy_quartic(uint8_t *E, const uint8_t *src, int tl) {
    bool bad = false;
    const int j = kK5BytesPerThread * threadIdx.x;
    if ((reinterpret_cast<uintptr_t>(src) & 15u) == 0 && j + kK5BytesPerThread <= tl) {
        const uint4 v = __ldg(reinterpret_cast<const uint4 *>(src + j));
        uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int c = 0; c < 4; c++) {
            const uint32_t m = __vcmpgtu4(w[c], 0xf2f2f2f2u);   // bytes > 242
            if (m) { bad = true; w[c] = (w[c] & ~m) | (0x79797979u & m); }
        }
        *reinterpret_cast<uint4 *>(E + j) = make_uint4(w[0], w[1], w[2], w[3]);
    } else {
        for (int jl = j; jl < j + kK5BytesPerThread && jl < tl; jl++) {
            uint8_t v = src[jl];
            if (v > 242) { bad = true; v = kZeroGroup; }
            E[jl] = v;
        }
    }
    return bad;
}

// The ZRE expansion of a tile in two halves, so that a caller with several payloads (K5m)
// can have every source's loads in flight before the first scan:
//  expand_load  -- this thread's window words of the payload bytes covering the tile
//                  (seek entries -> payload: two dependent global accesses);
//  expand_scan  -- 121 prefill, expansion-length scan over the block, literal scatter.
constexpr int kK5NW = kK5Words + 1;
struct ExpandWin {
    uint32_t wd[kK5NW];
    int skip, wl, sh;
};

// sk = the tile's seek entry, sk1 = the next tile's (ignored for the last tile, lt + 1 = ntiles)
__device__ __forceinline__ void expand_load_at(ExpandWin &X, const uint8_t *payload, uint64_t Z,
                                               unsigned long long sk, unsigned long long sk1, uint64_t lt,
                                               uint64_t ntiles) {
    const uint64_t bi = sk >> 4;                          // payload byte covering J0
    X.skip = (int)(sk & 15);                              // J0 - (first position of that byte)
    const uint64_t be = lt + 1 < ntiles ? (sk1 >> 4) : Z - 1;   // last byte needed
    X.wl = (int)(be - bi) + 1;                            // <= kT5 + 1
    // thread owns window bytes [16*tid, 16*tid+16) relative to w0 = bi rounded down
    // to 4; the last thread also owns the next 4 bytes, so the <= kT5 bytes from bi
    // on are always covered
    const bool pal = (reinterpret_cast<uintptr_t>(payload) & 3u) == 0;
    const uint64_t w0 = bi & ~3ull;
    X.sh = (int)(bi - w0);
    const int nwords = threadIdx.x == kK5Threads - 1 ? kK5NW : kK5Words;
#pragma unroll
    for (int h = 0; h < kK5NW; h++) {
        X.wd[h] = 0;
        if (h >= nwords) continue;
        const int r = kK5BytesPerThread * threadIdx.x + 4 * h - X.sh;   // window offset of the word
        if (pal && r >= 0 && r + 3 < X.wl) {
            X.wd[h] = __ldg(reinterpret_cast<const uint32_t *>(payload + w0) + kK5Words * threadIdx.x + h);
        } else {
            uint32_t x = 0;
#pragma unroll
            for (int c = 0; c < 4; c++)
                if (r + c >= 0 && r + c < X.wl) x |= (uint32_t)payload[bi + r + c] << (8 * c);
            X.wd[h] = x;
        }
    }
}

__device__ __forceinline__ void expand_load(ExpandWin &X, const uint8_t *payload, uint64_t Z,
                                            const unsigned long long *seek, uint64_t lt, uint64_t ntiles) {
    expand_load_at(X, payload, Z, seek[lt], lt + 1 < ntiles ? seek[lt + 1] : 0ull, lt, ntiles);
}

// true if this thread's window bytes hold a literal other than 121, i.e. a nonzero trit
// in the tile (or in the next tile's first byte: conservative)
__device__ __forceinline__ bool window_nonzero(const ExpandWin &X) {
    const int nwords = threadIdx.x == kK5Threads - 1 ? kK5NW : kK5Words;
    bool nz = false;
#pragma unroll
    for (int m = 0; m < 4 * kK5NW; m++) {
        const int r = kK5BytesPerThread * threadIdx.x + m - X.sh;
        const uint32_t b = (X.wd[m >> 2] >> (8 * (m & 3))) & 0xffu;
        nz |= m < 4 * nwords && r >= 0 && r < X.wl && b < kFirstRunCode && b != kZeroGroup;
    }
    return nz;
}

// kWarpSkip: warps whose bytes all lie past the window only prefill.  Used by the ACCUMULATE
// decoder, which is instruction-bound on sparse tiles (pull apply 0.201 -> 0.185 ms per
// BERT-large W = 1 step); the store-bound OVERWRITE decoder measured 2 % slower with it.
template <bool kWarpSkip = false>
__device__ __forceinline__ void expand_scan(uint8_t *E, unsigned int *warp_sum, const ExpandWin &X, int tl) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    *reinterpret_cast<uint4 *>(E + kK5BytesPerThread * threadIdx.x) =
        make_uint4(0x79797979u, 0x79797979u, 0x79797979u, 0x79797979u);
    const int nwords = threadIdx.x == kK5Threads - 1 ? kK5NW : kK5Words;
    // warp-uniform: does any of the warp's bytes fall in the window?  A sparse tile's window is
    // a few hundred bytes, so most warps only prefill (their bytes would all have length 0)
    const bool wact = !kWarpSkip || kK5BytesPerThread * 32 * warp - X.sh < X.wl;
    // expansion length of window byte m of this thread (0 outside the window); recomputed in
    // the scatter below rather than kept live across the barrier (that spilled)
    auto len = [&](int m) -> uint32_t {
        const int r = kK5BytesPerThread * threadIdx.x + m - X.sh;
        const uint32_t b = (X.wd[m >> 2] >> (8 * (m & 3))) & 0xffu;
        return (m < 4 * nwords && r >= 0 && r < X.wl) ? zre_len(b) : 0u;
    };
    uint32_t sum = 0, x = 0;
    if (wact) {
#pragma unroll
        for (int m = 0; m < 4 * kK5NW; m++) sum += len(m);
        x = sum;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
            if (lane >= d) x += y;
        }
    }
    if (lane == 31) warp_sum[warp] = x;
    __syncthreads();
    if (wact) {
        uint32_t wofs = 0;
#pragma unroll
        for (int w = 0; w < kK5Threads / 32; w++) wofs += (w < warp) ? warp_sum[w] : 0u;
        int p = (int)(wofs + x - sum) - X.skip;   // tile position of this thread's first byte
#pragma unroll
        for (int m = 0; m < 4 * kK5NW; m++) {
            const uint32_t b = (X.wd[m >> 2] >> (8 * (m & 3))) & 0xffu;
            const uint32_t l = len(m);
            if (l == 1 && p >= 0 && p < tl) E[p] = (uint8_t)b;   // literal byte
            p += (int)l;
        }
    }
    __syncthreads();                                      // warp_sum reuse; E complete
}

// Expand the payload bytes covering output tile lt (positions [J0, J0+tl)) into
// E[0, tl): 121 prefill, then only the literal bytes are written at their scanned
// positions (zero-run codes expand to 121s).  seek points at the segment's seek
// entries.  Without ZRE the bytes are copied (a literal > 242 returns true:
// FORMAT).  Ends with E complete and visible to the whole block.
__device__ __forceinline__ bool expand_tile(uint8_t *E, unsigned int *warp_sum, const uint8_t *payload,
                                            bool zre, uint64_t Z, const unsigned long long *seek,
                                            uint64_t lt, uint64_t ntiles, uint64_t J0, int tl) {
    bool bad = false;
    if (zre) {
        ExpandWin X;
        expand_load(X, payload, Z, seek, lt, ntiles);
        expand_scan(E, warp_sum, X, tl);
    } else {
        bad = copy_quartic(E, payload + J0, tl);
    }
    return __syncthreads_or(bad);
}

#ifndef TLC_K5_MINB
#define TLC_K5_MINB 3
#endif
template <int kMode>
__global__ void __launch_bounds__(kK5Threads, TLC_K5_MINB)   // <= 85 registers: 3 CTAs per SM
tlc_expand_dequant_kernel(const SegTable T, const unsigned long long *seek) {
    __shared__ K5Smem sm;
    __shared__ uint64_t s_first[kSegCache];
    // Decoding step 1, "dividing a by a power of 3 and taking the remainder", for
    // the 243 byte values, once per CTA: the digits and the nonzero mask do not depend on M
    for (int v = threadIdx.x; v < 256; v += kK5Threads) {
        uint32_t w = 0, pk = 0, r = v < 243 ? v : 121;
#pragma unroll
        for (int i = 4; i >= 0; i--) {
            const uint32_t d = r % 3u;
            r /= 3u;
            w |= (uint32_t)(d != 1) << i;
            pk |= d << (2 * i);
        }
        sm.lut[v] = (uint16_t)w;
        sm.dig[v] = (uint16_t)pk;
    }
    seg_index_load<5>(T, s_first);                       // (ends with __syncthreads)
    pdl_wait();                                          // K4's seek entries and header checks
    int cur = -1;
    // ACCUMULATE (the exchange's apply over a table of contexts): runs of R consecutive tiles
    // dealt to the CTAs cyclically, so the value tables V are rebuilt at most once per run (with
    // a plain grid stride of ~450 tiles nearly every tile of a 150-context table rebuilt them),
    // while dense and sparse contexts still spread over all CTAs (N = 4 apply 0.207 ms vs 0.224
    // with whole contiguous ranges per CTA and 0.251 with the stride).  OVERWRITE: grid stride.
#ifndef TLC_K5A_RUN
#define TLC_K5A_RUN 8
#endif
    // (a table with fewer than TLC_K5A_RUN tiles per CTA takes shorter runs: every CTA busy)
    const uint64_t R = kMode != TLC_MODE_OVERWRITE
                           ? tmax<uint64_t>(1, tmin<uint64_t>(TLC_K5A_RUN, (T.n5 + gridDim.x - 1) / gridDim.x))
                           : 1u;
    for (uint64_t it = 0;; it++) {
        const uint64_t run = blockIdx.x + (it / R) * gridDim.x;
        if (run * R >= T.n5) break;
        const uint64_t tile = run * R + it % R;
        if (tile >= T.n5) continue;
        const int si = find_seg_c<5>(T, tile, s_first);
        const Seg S = get_seg(T, si);
        const tlc_header *hdr = S.hdr;
        const uint64_t lt = tile - S.k5, ntiles = (S.P + kT5 - 1) / kT5;
        // ACCUMULATE (the exchange's apply): the seek entries are loaded beside the header, not
        // after it -- over peer memory both are the owner's (one remote round trip fewer)
        unsigned long long sk0 = 0, sk1 = 0;
        if (kMode != TLC_MODE_OVERWRITE) {
            const unsigned long long *sp = S.seek ? S.seek : seek + S.k5;
            sk0 = sp[lt];
            if (lt + 1 < ntiles) sk1 = sp[lt + 1];
        }
        if (hdr->status != TLC_OK) continue;             // uniform: FORMAT from K4 or a failed compress
        const float M = hdr->M;
        const bool zre = (hdr->flags & TLC_FLAG_ZRE) != 0;
        const uint64_t Z = hdr->payload_len, P = S.P, n = S.n;
        const uint8_t *__restrict__ payload = S.payload;
        __syncthreads();   // previous tile's readers of sm.E / sm.V are done
        if (si != cur) {
            // Eq. 3 per partition: V[i][b] = M * (digit_i(b) - 1), taken as a selection
            // of {-M, +0, M} -- the bits of the fp32 product (M >= +0, validated by K4)
            const uint32_t mb = __float_as_uint(M), nmb = __float_as_uint(-M);
            for (int v = threadIdx.x; v < 256; v += kK5Threads) {
                const uint32_t pk = sm.dig[v];
#pragma unroll
                for (int i = 0; i < 5; i++) {
                    const uint32_t d = (pk >> (2 * i)) & 3u;
                    sm.V[i][v] = d == 2u ? mb : (d == 0u ? nmb : 0u);
                }
            }
            cur = si;
        }
        const uint64_t J0 = lt * kT5;
        const int tl = (int)tmin<uint64_t>(kT5, P - J0);
        // valid positions of partition i in this tile: e = i*P + J0 + jl < n
        int lim[5];
        float *ob[5];
#pragma unroll
        for (int i = 0; i < 5; i++) {
            const uint64_t e0 = (uint64_t)i * P + J0;
            lim[i] = e0 >= n ? 0 : (int)tmin<uint64_t>(tl, n - e0);
            ob[i] = S.out + e0;
        }
        if (kMode != TLC_MODE_OVERWRITE && zre) {
            // skip-zero (R16): a tile whose payload window holds no literal but 121 leaves
            // out untouched -- the expansion and the decode are skipped
            ExpandWin X;
            expand_load_at(X, payload, Z, sk0, sk1, lt, ntiles);
            if (!__syncthreads_or(window_nonzero(X))) continue;
            expand_scan<true>(sm.E, sm.warp_sum, X, tl);
        }
        const bool bad = (kMode != TLC_MODE_OVERWRITE && zre)
                             ? false : expand_tile(sm.E, sm.warp_sum, payload, zre, Z, S.seek ? S.seek : seek + S.k5, lt, ntiles, J0, tl);
        if (bad) {                                         // literal > 242 without ZRE
            if (threadIdx.x == 0) raise_format(S.hdr);
            continue;
        }
        const bool vec = (S.flags & kSegVec5) != 0;

        if (kMode == TLC_MODE_OVERWRITE && !vec && (reinterpret_cast<uintptr_t>(S.out) & 3u) == 0) {
            // Partitions not 16-byte aligned (P % 4 != 0 or an offset view): shift each
            // partition's groups of four so every float4 store is aligned; the bytes of a
            // group come from shared memory at any offset.
#pragma unroll
            for (int i = 0; i < 5; i++) {
                float *base = ob[i];
                const int sh = (int)((4u - ((reinterpret_cast<uintptr_t>(base) >> 2) & 3u)) & 3u);  // first aligned jl
                if ((int)threadIdx.x < sh && (int)threadIdx.x < lim[i])
                    base[threadIdx.x] = __uint_as_float(sm.V[i][sm.E[threadIdx.x]]);
                for (int jl = sh + 4 * (int)threadIdx.x; jl < lim[i]; jl += 4 * kK5Threads) {
                    if (jl + 3 < lim[i]) {
                        __stcs(reinterpret_cast<uint4 *>(base + jl),
                               make_uint4(sm.V[i][sm.E[jl]], sm.V[i][sm.E[jl + 1]], sm.V[i][sm.E[jl + 2]],
                                          sm.V[i][sm.E[jl + 3]]));
                    } else {
                        for (int c = 0; jl + c < lim[i]; c++) base[jl + c] = __uint_as_float(sm.V[i][sm.E[jl + c]]);
                    }
                }
            }
            continue;
        }

        // ---- base-3 decode + dequantize, 4 consecutive quartic bytes per step
#pragma unroll
        for (int k = 0; k < kK5BytesPerThread / 4; k++) {
            const int jl = 4 * threadIdx.x + 4 * kK5Threads * k;
            if (jl >= tl) break;
            const uint32_t w4 = *reinterpret_cast<const uint32_t *>(sm.E + jl);
            const uint32_t b0 = w4 & 0xffu, b1 = (w4 >> 8) & 0xffu, b2 = (w4 >> 16) & 0xffu, b3 = w4 >> 24;
            if (kMode == TLC_MODE_OVERWRITE) {
                const bool zero4 = w4 == 0x79797979u;   // four all-zero groups: 20 x M*0
#pragma unroll
                for (int i = 0; i < 5; i++) {
                    float *o = ob[i] + jl;
                    uint4 v = zero4 ? make_uint4(sm.V[i][121], sm.V[i][121], sm.V[i][121], sm.V[i][121])
                                    : make_uint4(sm.V[i][b0], sm.V[i][b1], sm.V[i][b2], sm.V[i][b3]);
                    if (vec && jl + 3 < lim[i]) {
                        __stcs(reinterpret_cast<uint4 *>(o), v);
                    } else {
                        const uint32_t vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                        for (int c = 0; c < 4; c++)
                            if (jl + c < lim[i]) o[c] = __uint_as_float(vv[c]);
                    }
                }
            } else {
                if (w4 == 0x79797979u) continue;         // skip-zero: sectors untouched (R16)
                const uint32_t L[4] = {sm.lut[b0], sm.lut[b1], sm.lut[b2], sm.lut[b3]};
                const uint32_t bb[4] = {b0, b1, b2, b3};
#pragma unroll
                for (int i = 0; i < 5; i++) {
                    if ((((L[0] | L[1] | L[2] | L[3]) >> i) & 1u) == 0) continue;
                    float *o = ob[i] + jl;
                    if (vec && jl + 3 < lim[i]) {
                        float4 v = *reinterpret_cast<float4 *>(o);
                        float *vv = reinterpret_cast<float *>(&v);
#pragma unroll
                        for (int c = 0; c < 4; c++)
                            if ((L[c] >> i) & 1u) vv[c] = __fadd_rn(vv[c], __uint_as_float(sm.V[i][bb[c]]));
                        *reinterpret_cast<float4 *>(o) = v;
                    } else {
                        // unaligned partition row: all four loads first, then the adds and stores
                        // (one load-add-store after another was a memory latency per element:
                        // 56 % of the stall samples at s = 1.0, ncu)
                        float v[4];
#pragma unroll
                        for (int c = 0; c < 4; c++)
                            if (jl + c < lim[i] && ((L[c] >> i) & 1u)) v[c] = o[c];
#pragma unroll
                        for (int c = 0; c < 4; c++)
                            if (jl + c < lim[i] && ((L[c] >> i) & 1u))
                                o[c] = __fadd_rn(v[c], __uint_as_float(sm.V[i][bb[c]]));
                    }
                }
            }
        }
    }
}

// ============================================================== K5m (exchange aggregation)
// The owner's fused decompress-aggregate of W pushed payloads per owned
// context (row a6, multi-source variant; reading R15): for each output element
// acc = +0, then for w = 0..W-1 in rank order acc = fl(acc + M_w*q_w) where
// q_w != 0, then mean = fl(acc / W) -- written once.  A = owned contexts (out,
// n); X = the W x |A| received (payload, header) rows, row w*|A| + q, whose
// seek entries K4 wrote.  A source whose header is not OK contributes nothing.
constexpr int kMaxSources = 8;

#ifndef TLC_K5M_G
#define TLC_K5M_G 1
#endif
constexpr int kK5mG = TLC_K5M_G;                    // sources whose loads are in flight together

// Dynamic shared memory, sized for W sources: E[W][kT5] bytes, then
// V[W][5][256] words (V[w][i][b] = M_w * (digit_i(b) - 1): +0 for a zero trit).
struct alignas(16) K5mHead {   // E follows it: 16-byte stores into E need sizeof % 16 == 0
    int ok[kMaxSources];
    unsigned int stat[kMaxSources];   // each source's header status at the tile start
    int poison;                       // the tile's mean is NaN (reading R24)
    unsigned int warp_sum[kK5Threads / 32];
};
constexpr int kK5mSegCache = kSegCache;               // owned contexts (all 150 of BERT-large at W = 1)
static_assert(sizeof(K5mHead) % 16 == 0, "E[] must stay 16-byte aligned");
__host__ __device__ constexpr size_t k5m_smem_bytes(int W) {
    return sizeof(K5mHead) + (size_t)W * kT5 + (size_t)W * 5 * 256 * sizeof(uint32_t);
}

// One source's Eq. 3 table (the same single fp32 multiply as the decoder).
__device__ __forceinline__ void build_values(uint32_t (*V)[256], float M) {
    for (int v = threadIdx.x; v < 256; v += kK5Threads) {
        uint32_t r = v < 243 ? v : 121;
#pragma unroll
        for (int i = 4; i >= 0; i--) {
            V[i][v] = __float_as_uint(__fmul_rn(M, (float)((int)(r % 3u) - 1)));
            r /= 3u;
        }
    }
}

#ifndef TLC_K5M_MINB
#define TLC_K5M_MINB 4                                   // 4 CTAs/SM (64 registers, 28 B spilled): K5m 0.298 -> 0.287 ms at N = 2, 0.370 -> 0.355 at W = 1; 2: 0.43
#endif
__global__ void __launch_bounds__(kK5Threads, TLC_K5M_MINB)
tlc_aggregate_kernel(const SegTable A, const SegTable X, int W, const unsigned long long *seek) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    __shared__ uint64_t s_first[kK5mSegCache];         // owned contexts: few per rank
    seg_index_load<5, kK5mSegCache>(A, s_first);
    pdl_wait();                                          // K4's seek entries
    K5mHead &sm = *reinterpret_cast<K5mHead *>(smem_raw);
    uint8_t(*E)[kT5] = reinterpret_cast<uint8_t(*)[kT5]>(smem_raw + sizeof(K5mHead));
    uint32_t(*V)[5][256] = reinterpret_cast<uint32_t(*)[5][256]>(smem_raw + sizeof(K5mHead) + (size_t)W * kT5);
    // acc / W: for W a power of two the division is the exact scaling acc * (1/W),
    // bitwise equal to the IEEE quotient; otherwise divide
    const bool pow2 = (W & (W - 1)) == 0;
    const float Wf = (float)W, rW = 1.0f / (float)W;
    int cur = -1;
    for (uint64_t tile = blockIdx.x; tile < A.n5; tile += gridDim.x) {
        const int q = find_seg_c<5, kK5mSegCache>(A, tile, s_first);
        const Seg S = get_seg(A, q);
        const uint64_t P = S.P, n = S.n, lt = tile - S.k5, ntiles = (P + kT5 - 1) / kT5;
        const uint64_t J0 = lt * kT5;
        const int tl = (int)tmin<uint64_t>(kT5, P - J0);
        __syncthreads();                                   // previous tile's readers are done
        // R24: a context with a failed push (a source header not OK: NONFINITE/RANGE from its
        // compression, FORMAT from K4) has a NaN mean -- as an fp32 sum would -- so the owner's
        // pull compression raises NONFINITE, which every rank then sees.  One load per
        // source, broadcast through shared memory so the decision is uniform in the CTA.
        if (threadIdx.x < W) sm.stat[threadIdx.x] = get_seg(X, threadIdx.x * A.count + q).hdr->status;
        if (threadIdx.x == 0) sm.poison = 0;
        __syncthreads();
        bool poison = false;
        for (int w = 0; w < W; w++) poison |= sm.stat[w] != TLC_OK;
        // sources in groups of kK5mG: every source's header, seek and payload-window loads of a
        // group are in flight together (in peer-memory mode they cross NVLink), then the scans
        for (int w0 = 0; w0 < W; w0 += kK5mG) {
            ExpandWin Xw[kK5mG];
            bool okw[kK5mG], zw[kK5mG];
            const uint8_t *pw[kK5mG];
            tlc_header *hw[kK5mG];
#pragma unroll
            for (int g = 0; g < kK5mG; g++) {
                const int w = w0 + g;
                okw[g] = false;
                if (w >= W || poison) continue;
                const Seg R = get_seg(X, w * A.count + q);
                hw[g] = R.hdr;
                pw[g] = R.payload;
                okw[g] = true;                              // every source OK (not poisoned)
                zw[g] = (R.hdr->flags & TLC_FLAG_ZRE) != 0;
                if (okw[g] && zw[g]) expand_load(Xw[g], R.payload, R.hdr->payload_len, R.seek ? R.seek : seek + R.k5, lt, ntiles);
            }
#pragma unroll
            for (int g = 0; g < kK5mG; g++) {
                const int w = w0 + g;
                if (w >= W) continue;
                if (threadIdx.x == 0) sm.ok[w] = okw[g];
                if (!okw[g]) continue;
                if (q != cur) build_values(V[w], hw[g]->M);
                bool bad = false;
                if (zw[g]) {
                    // a window without a literal but 121: all trits zero, the source adds +0 only
                    if (__syncthreads_or(window_nonzero(Xw[g]))) expand_scan(E[w], sm.warp_sum, Xw[g], tl);
                    else if (threadIdx.x == 0) sm.ok[w] = 0;
                } else {
                    bad = __syncthreads_or(copy_quartic(E[w], pw[g] + J0, tl));
                }
                if (bad && threadIdx.x == 0) { raise_format(hw[g]); sm.ok[w] = 0; sm.poison = 1; }
            }
        }
        cur = poison ? -1 : q;                                // tables not rebuilt when poisoned
        __syncthreads();
        poison |= sm.poison != 0;                            // a literal > 242 found in this tile
#pragma unroll 1                                         // unrolled: 0.43 vs 0.37 ms (BERT-large W = 1)
        for (int k = 0; k < kK5BytesPerThread / 4; k++) {
            const int jl = 4 * threadIdx.x + 4 * kK5Threads * k;
            if (jl >= tl) break;
            float acc[5][4];
#pragma unroll
            for (int i = 0; i < 5; i++)
#pragma unroll
                for (int c = 0; c < 4; c++) acc[i][c] = 0.0f;     // +0 (R15)
            bool any = false;
            for (int w = 0; w < W; w++) {                          // rank order
                const uint32_t w4 = *reinterpret_cast<const uint32_t *>(E[w] + jl);
                if (!sm.ok[w] || w4 == 0x79797979u) continue;      // all trits zero: adds +0 only
                any = true;
                const uint32_t b[4] = {w4 & 0xffu, (w4 >> 8) & 0xffu, (w4 >> 16) & 0xffu, w4 >> 24};
                // acc is never -0, so adding the +0 of a zero trit leaves it bitwise unchanged:
                // this equals "add M_w*q_w only where q_w != 0"
#pragma unroll
                for (int i = 0; i < 5; i++)
#pragma unroll
                    for (int c = 0; c < 4; c++) acc[i][c] = __fadd_rn(acc[i][c], __uint_as_float(V[w][i][b[c]]));
            }
#pragma unroll
            for (int i = 0; i < 5; i++) {
                float r[4];
#pragma unroll
                for (int c = 0; c < 4; c++)
                    r[c] = poison ? __int_as_float(0x7fc00000)
                                  : !any ? 0.0f : (pow2 ? __fmul_rn(acc[i][c], rW) : __fdiv_rn(acc[i][c], Wf));
                // partition i's positions e = i*P + J0 + jl < n (its row base recomputed here:
                // keeping five row pointers live spilled at 80 registers)
                const uint64_t e0 = (uint64_t)i * P + J0;
                const int lim = e0 >= n ? 0 : (int)tmin<uint64_t>(tl, n - e0);
                float *o = S.out + e0 + jl;
                if (((reinterpret_cast<uintptr_t>(o) & 15u) == 0) && jl + 3 < lim) {
                    __stcs(reinterpret_cast<float4 *>(o), make_float4(r[0], r[1], r[2], r[3]));
                } else {
                    // P % 4 != 0: 32-bit stores (16-byte stores realigned by lane shuffles
                    // measured slower: K5m 0.37 -> 0.44 ms, BERT-large W = 1)
#pragma unroll
                    for (int c = 0; c < 4; c++)
                        if (jl + c < lim) o[c] = r[c];
                }
            }
        }
    }
}

// ---------------------------------------------------------------- K5m, sources in parallel
// The kernel above expands the W sources of a tile one after another with the whole CTA,
// so a tile pays W dependent global round trips (seek entries, then the window; over
// NVLink in peer mode) and 2W block barriers: per owner its time hardly fell as W grew
// (loopback, BERT-large: 0.35 / 0.24 / 0.19 / 0.20 ms per owner at W = 1 / 2 / 4 / 8).
// ncu (W = 8): 85 M warp instructions per owner, mostly every thread walking all its
// byte slots of every source window (window_nonzero, per-byte loads) though a window at
// s = 1.9 holds a few hundred bytes.  Here the CTA splits into WP groups (WP = W rounded
// up to a power of two), group g expands source g -- all groups at once, one round trip
// per tile -- in passes of 16 bytes per thread over only the bytes the window has.
// Loopback, BERT-large, s = 1.9, per owner: 0.195 / 0.108 / 0.080 ms at W = 2 / 4 / 8
// (sequential: 0.242 / 0.192 / 0.202; profiles/r02n_loopback.txt).
// The fold (rank order from +0, skip-zero, IEEE / W, R15; NaN for a failed source, R24)
// is the same as above.
// 4 CTAs/SM where shared memory allows it (W <= 4): per owner 0.180 -> 0.168 ms at W = 2,
// 0.099 -> 0.093 at W = 4 (loopback, profiles/r02y_k5m_minb_ab.txt); W = 8 is held to 3 by its
// shared memory either way
#ifndef TLC_K5P_MINB
#define TLC_K5P_MINB 4
#endif
template <int WP, bool KEYED>
__global__ void __launch_bounds__(kK5Threads, (WP == 8 || KEYED) ? 3 : TLC_K5P_MINB)
tlc_aggregate_par_kernel(const SegTable A, const SegTable X, int W, const unsigned long long *seek,
                         const SegTable K, unsigned int *__restrict__ keys) {
    constexpr int TP = kK5Threads / WP;                  // threads per source
    extern __shared__ __align__(16) uint8_t smem_raw[];
    __shared__ uint64_t s_first[kK5mSegCache];
    __shared__ unsigned int s_stat[kMaxSources];
    __shared__ int s_ok[kMaxSources], s_nz[kMaxSources], s_poison;
    __shared__ unsigned int s_wsum[kK5Threads / 32];
    __shared__ float s_M[kMaxSources];
    seg_index_load<5, kK5mSegCache>(A, s_first);
    pdl_wait();                                          // K4's seek entries
    uint8_t(*E)[kT5] = reinterpret_cast<uint8_t(*)[kT5]>(smem_raw);
    uint32_t(*V)[5][256] = reinterpret_cast<uint32_t(*)[5][256]>(smem_raw + (size_t)WP * kT5);
    const bool pow2 = (W & (W - 1)) == 0;
    const float Wf = (float)W, rW = 1.0f / (float)W;
    const int g = threadIdx.x / TP, tg = threadIdx.x % TP, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int cur = -1;
    // contiguous runs of tiles per CTA: consecutive tiles share a context, so the W value
    // tables are rebuilt only when the context changes (with a grid stride it changed at
    // almost every tile: 5 % of the instructions, ncu W = 4)
    const uint64_t per = (A.n5 + gridDim.x - 1) / gridDim.x;
    const uint64_t t_end = tmin<uint64_t>(A.n5, per * (blockIdx.x + 1));
    for (uint64_t tile = per * blockIdx.x; tile < t_end; tile++) {
        const int q = find_seg_c<5, kK5mSegCache>(A, tile, s_first);
        const Seg S = get_seg(A, q);
        const uint64_t P = S.P, n = S.n, lt = tile - S.k5, ntiles = (P + kT5 - 1) / kT5;
        const uint64_t J0 = lt * kT5;
        const int tl = (int)tmin<uint64_t>(kT5, P - J0);
        // keys: the max key of u = err + mean over this tile (K1 of the owner's pull compress,
        // which then skips K1), err = the pull table's error buffer of the same context
        const float *kerr = KEYED ? get_seg(K, q).err : nullptr;
        unsigned int kmax = 0;
        // every thread of group g reads source g's row (the same addresses: broadcast)
        const bool src = g < W;
        Seg R{};
        unsigned int st = TLC_OK, flags = 0;
        uint64_t Z = 0;
        unsigned long long sk0 = 0, sk1 = 0;
        if (src) {
            R = get_seg(X, g * A.count + q);
            // the seek entries are loaded beside the header, not after it (over peer memory they
            // are the producer's: one remote round trip fewer per tile); used only with ZRE
            const unsigned long long *sp = R.seek ? R.seek : seek + R.k5;   // producer's or K4's
            sk0 = sp[lt];
            if (lt + 1 < ntiles) sk1 = sp[lt + 1];
            st = R.hdr->status;
            flags = R.hdr->flags;
            Z = R.hdr->payload_len;
        }
        __syncthreads();                                   // previous tile's readers of E / V / flags
        if (tg == 0 && src) {
            s_stat[g] = st;
            s_M[g] = R.hdr->M;
            s_nz[g] = 0;
        }
        if (threadIdx.x == 0) s_poison = 0;
        __syncthreads();
        bool poison = false;
        for (int w = 0; w < W; w++) poison |= s_stat[w] != TLC_OK;   // R24
        // ---- expansion of source g's window into E[g] (all groups at once).  A group reads the
        // window in passes of 16 bytes per thread (16*TP bytes), as many as the window needs --
        // one for a sparse window, up to kT5/(16*TP) + 1 for a dense one -- so idle byte slots
        // cost nothing; each pass scans its expansion lengths within the group and scatters the
        // literals.  Groups synchronise on their own named barrier (id 1 + g).
        const bool zre = (flags & TLC_FLAG_ZRE) != 0;
        const bool act0 = src && !poison;
        int wl = 0, sh = 0, skip = 0;
        uint64_t bi = 0;
        if (act0 && zre) {
            bi = sk0 >> 4;
            skip = (int)(sk0 & 15);
            const uint64_t be = lt + 1 < ntiles ? (sk1 >> 4) : Z - 1;
            wl = (int)(be - bi) + 1;                           // <= kT5 + 1
            sh = (int)(bi & 15);                               // passes start at the granule of bi
        }
        auto group_sync = [&]() {
            if (TP == 32) __syncwarp();
            else asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(TP) : "memory");
        };
        // pass 0 doubles as the nonzero test: a window without a literal but 121 adds +0 only
        if (act0) {
            uint8_t *Eg = E[g];
            if (q != cur) {                                    // Eq. 3 values of source g (new context)
                const float M = s_M[g];
                for (int v = tg; v < 256; v += TP) {
                    uint32_t r = v < 243 ? v : 121;
#pragma unroll
                    for (int i = 4; i >= 0; i--) {
                        V[g][i][v] = __float_as_uint(__fmul_rn(M, (float)((int)(r % 3u) - 1)));
                        r /= 3u;
                    }
                }
            }
            for (int k = 16 * tg; k < kT5; k += 16 * TP)      // 121 prefill
                *reinterpret_cast<uint4 *>(Eg + k) = make_uint4(0x79797979u, 0x79797979u, 0x79797979u, 0x79797979u);
            bool nz = false;
            if (zre) {
                const uint8_t *gbase = R.payload + (bi & ~15ull);
                const bool pal = (reinterpret_cast<uintptr_t>(R.payload) & 15u) == 0;
                int pos = -skip;                               // tile position of the pass's first byte
                group_sync();                                  // prefill before any scatter
                for (int base = 0; base < wl + sh; base += 16 * TP) {   // uniform within the group
                    const int r0 = base + 16 * tg - sh;        // window offset of this thread's 16 bytes
                    uint32_t wd[4];
                    if (pal && r0 + 15 >= 0 && r0 < wl) {
                        // the 16-byte granule holding window bytes (bytes outside [0, wl) are
                        // ignored below; a granule with a payload byte lies in mapped memory)
                        const uint4 xv = __ldg(reinterpret_cast<const uint4 *>(gbase + base + 16 * tg));
                        wd[0] = xv.x; wd[1] = xv.y; wd[2] = xv.z; wd[3] = xv.w;
                    } else if (r0 + 15 < 0 || r0 >= wl) {
                        wd[0] = wd[1] = wd[2] = wd[3] = 0;
                    } else {
#pragma unroll
                        for (int h = 0; h < 4; h++) {
                            uint32_t y = 0;
#pragma unroll
                            for (int c = 0; c < 4; c++) {
                                const int rr = r0 + 4 * h + c;
                                if (rr >= 0 && rr < wl) y |= (uint32_t)R.payload[bi + rr] << (8 * c);
                            }
                            wd[h] = y;
                        }
                    }
                    uint32_t lens = 0;
                    if (r0 >= 0 && r0 + 15 < wl) {
                        lens = word_len(wd[0]) + word_len(wd[1]) + word_len(wd[2]) + word_len(wd[3]);
                    } else {
#pragma unroll
                        for (int m = 0; m < 16; m++)
                            if (r0 + m >= 0 && r0 + m < wl) lens += zre_len((wd[m >> 2] >> (8 * (m & 3))) & 0xffu);
                    }
                    // exclusive scan within the group: the warp, then its earlier warps
                    uint32_t x = lens;
#pragma unroll
                    for (int d = 1; d < 32; d <<= 1) {
                        const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
                        if (lane >= d) x += y;
                    }
                    uint32_t wofs = 0, tot = __shfl_sync(0xffffffffu, x, 31);
                    if (TP > 32) {
                        if (lane == 31) s_wsum[warp] = x;
                        group_sync();
                        tot = 0;
                        for (int k = g * (TP / 32); k < (g + 1) * (TP / 32); k++) {
                            const uint32_t v = s_wsum[k];
                            wofs += k < warp ? v : 0u;
                            tot += v;
                        }
                    }
                    int p = pos + (int)(wofs + x - lens);
#pragma unroll
                    for (int m = 0; m < 16; m++) {
                        const int r = r0 + m;
                        if (r < 0 || r >= wl) continue;
                        const uint32_t b = (wd[m >> 2] >> (8 * (m & 3))) & 0xffu;
                        const uint32_t l = zre_len(b);
                        if (l == 1) {
                            nz |= b != kZeroGroup;
                            TLC_CHECK(!(p >= 0 && p < tl) || p < kT5);
                            if (p >= 0 && p < tl) Eg[p] = (uint8_t)b;   // literal byte
                        }
                        p += (int)l;
                    }
                    pos += (int)tot;
                    if (TP > 32) group_sync();                 // s_wsum reuse by the next pass
                }
            } else {
                // quartic bytes as sent (a literal > 242 is FORMAT)
                group_sync();                                  // prefill done (bytes past tl stay 121)
                bool bad = false;
                for (int jl = tg; jl < tl; jl += TP) {
                    uint8_t b = R.payload[J0 + jl];
                    if (b > 242) { bad = true; b = kZeroGroup; }
                    Eg[jl] = b;
                }
                nz = true;
                if (bad) {
                    raise_format(R.hdr);
                    s_poison = 1;
                }
            }
            if (nz) s_nz[g] = 1;
        }
        __syncthreads();                                     // every group's E, V and nonzero flag
        if (threadIdx.x < W) s_ok[threadIdx.x] = !poison && s_nz[threadIdx.x];
        cur = poison ? -1 : q;
        __syncthreads();
        poison |= s_poison != 0;
        uint32_t okmask = 0;                                       // sources with a nonzero trit here
        for (int w = 0; w < W; w++) okmask |= (uint32_t)(s_ok[w] != 0) << w;
#pragma unroll 1
        for (int k = 0; k < kK5BytesPerThread / 4; k++) {
            const int jl = 4 * threadIdx.x + 4 * kK5Threads * k;
            if (jl >= tl) break;
            float acc[5][4];
#pragma unroll
            for (int i = 0; i < 5; i++)
#pragma unroll
                for (int c = 0; c < 4; c++) acc[i][c] = 0.0f;     // +0 (R15)
            // KEYED: the err values of this step's 20 elements, loaded before the fold so their
            // latency hides behind it
            float ev[5][4];
            if (KEYED) {
#pragma unroll
                for (int i = 0; i < 5; i++) {
                    const uint64_t e0 = (uint64_t)i * P + J0;
                    const int lim = e0 >= n ? 0 : (int)tmin<uint64_t>(tl, n - e0);
                    const float *ep = kerr + e0 + jl;
                    if (((reinterpret_cast<uintptr_t>(ep) & 15u) == 0) && jl + 3 < lim) {
                        const float4 v = __ldcg(reinterpret_cast<const float4 *>(ep));
                        ev[i][0] = v.x; ev[i][1] = v.y; ev[i][2] = v.z; ev[i][3] = v.w;
                    } else {
#pragma unroll
                        for (int c = 0; c < 4; c++) ev[i][c] = jl + c < lim ? __ldcg(ep + c) : 0.0f;
                    }
                }
            }
            bool any = false;
            for (uint32_t m = okmask; m; m &= m - 1u) {            // rank order (ascending bits)
                const int w = (int)ctz32(m);
                const uint32_t w4 = *reinterpret_cast<const uint32_t *>(E[w] + jl);
                if (w4 == 0x79797979u) continue;                 // all trits zero: adds +0 only
                any = true;
                const uint32_t b[4] = {w4 & 0xffu, (w4 >> 8) & 0xffu, (w4 >> 16) & 0xffu, w4 >> 24};
#pragma unroll
                for (int i = 0; i < 5; i++)
#pragma unroll
                    for (int c = 0; c < 4; c++) acc[i][c] = __fadd_rn(acc[i][c], __uint_as_float(V[w][i][b[c]]));
            }
            if (poison) {
#pragma unroll
                for (int i = 0; i < 5; i++)
#pragma unroll
                    for (int c = 0; c < 4; c++) acc[i][c] = __int_as_float(0x7fc00000);
            } else if (any) {                                      // +0 / W = +0 otherwise
#pragma unroll
                for (int i = 0; i < 5; i++)
#pragma unroll
                    for (int c = 0; c < 4; c++)
                        acc[i][c] = pow2 ? __fmul_rn(acc[i][c], rW) : __fdiv_rn(acc[i][c], Wf);
            }
#pragma unroll
            for (int i = 0; i < 5; i++) {
                const float *r = acc[i];
                const uint64_t e0 = (uint64_t)i * P + J0;
                const int lim = e0 >= n ? 0 : (int)tmin<uint64_t>(tl, n - e0);
                float *o = S.out + e0 + jl;
                if (((reinterpret_cast<uintptr_t>(o) & 15u) == 0) && jl + 3 < lim) {
                    __stcs(reinterpret_cast<float4 *>(o), make_float4(r[0], r[1], r[2], r[3]));
                } else {
#pragma unroll
                    for (int c = 0; c < 4; c++)
                        if (jl + c < lim) o[c] = r[c];
                }
            }
            if (KEYED) {                                           // step (1) and K1's key, fused
#pragma unroll
                for (int i = 0; i < 5; i++) {
                    const uint64_t e0 = (uint64_t)i * P + J0;
                    const int lim = e0 >= n ? 0 : (int)tmin<uint64_t>(tl, n - e0);
#pragma unroll
                    for (int c = 0; c < 4; c++)
                        if (jl + c < lim)
                            kmax = max(kmax, __float_as_uint(__fadd_rn(ev[i][c], acc[i][c])) & 0x7fffffffu);
                }
            }
        }
        if (KEYED) {
            kmax = __reduce_max_sync(0xffffffffu, kmax);
            if (lane == 0 && kmax) atomicMax(keys + q, kmax);
        }
    }
}

template <int WP>
__host__ __device__ constexpr size_t k5p_smem_bytes() { return (size_t)WP * kT5 + (size_t)WP * 5 * 256 * sizeof(uint32_t); }

template <int WP, bool KEYED>
static void launch_par_k(const SegTable &A, const SegTable &X, int W, const unsigned long long *seek, cudaStream_t st,
                         const SegTable &K, unsigned int *keys) {
    static PerDevice attr;
    static int per_sm = 0;
    if (attr.first()) {
        cudaFuncSetAttribute(tlc_aggregate_par_kernel<WP, KEYED>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)k5p_smem_bytes<WP>());
        if (!per_sm)
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tlc_aggregate_par_kernel<WP, KEYED>, kK5Threads,
                                                          k5p_smem_bytes<WP>());
    }
    const int grid = (int)tmax<uint64_t>(1, tmin<uint64_t>(A.n5, (uint64_t)num_sms() * tmax(1, per_sm)));
    launch_pdl(tlc_aggregate_par_kernel<WP, KEYED>, grid, kK5Threads, k5p_smem_bytes<WP>(), st, A, X, W, seek, K,
               keys);
}
template <int WP>
static void launch_par(const SegTable &A, const SegTable &X, int W, const unsigned long long *seek, cudaStream_t st,
                       const SegTable *K, unsigned int *keys) {
    if (K && keys) launch_par_k<WP, true>(A, X, W, seek, st, *K, keys);
    else launch_par_k<WP, false>(A, X, W, seek, st, A, nullptr);
}

// TLC_K5M_SEQ=1 runs the sources-in-sequence kernel at every W (A/B)
static bool k5m_seq() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("TLC_K5M_SEQ");
        v = (e && e[0] == '1') ? 1 : 0;
    }
    return v == 1;
}

bool aggregate_keyable(int W) { return W > 1 && W <= kMaxSources && !k5m_seq(); }

int launch_aggregate(const SegTable &A, const SegTable &X, int W, void *xws, cudaStream_t st, const SegTable *K,
                     unsigned int *keys) {
    // X: K4 over every received payload (validation + seek entries), then one fused pass
    if (W < 1 || W > kMaxSources) return TLC_ERR_ARG;
    const WsLayout L = ws_layout(X, 0);
    char *base = reinterpret_cast<char *>(xws);
    Ctrl *ctrl = reinterpret_cast<Ctrl *>(base + L.ctrl);
    unsigned long long *states = reinterpret_cast<unsigned long long *>(base + L.k4st);
    unsigned long long *seek = reinterpret_cast<unsigned long long *>(base + L.seek);
    const int sms = num_sms();
    if (!X.all_seek) {                       // producer seek entries: no scan (payloads from K3)
        // K4's counter and chunk states (K5 / K5m use neither: no memsets without K4)
        if (cudaMemsetAsync(base + L.ctrl, 0, sizeof(Ctrl), st) != cudaSuccess) return TLC_ERR_CUDA;
        if (cudaMemsetAsync(states, 0, L.memset_d, st) != cudaSuccess) return TLC_ERR_CUDA;
        KernelScope ks(kK4, st);
        const int grid = (int)tmax<uint64_t>(1, tmin<uint64_t>(X.n4, (uint64_t)sms * 8));
        tlc_zre_scan_kernel<<<grid, kK4Threads, 0, st>>>(X, ctrl, states, seek);
    }
    KernelScope ks(kK6, st);
    // W = 1: the sequential kernel (one source either way; 0.346 vs 0.374 ms, BERT-large)
    if (!k5m_seq() && W > 1) {
        if (W == 2) launch_par<2>(A, X, W, seek, st, K, keys);
        else if (W <= 4) launch_par<4>(A, X, W, seek, st, K, keys);
        else launch_par<8>(A, X, W, seek, st, K, keys);
        return cudaPeekAtLastError() == cudaSuccess ? TLC_OK : TLC_ERR_CUDA;
    }
    if (keys) return TLC_ERR_ARG;                                // keyed only with the parallel kernel
    static PerDevice attr;
    if (attr.first())
        cudaFuncSetAttribute(tlc_aggregate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)k5m_smem_bytes(kMaxSources));
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tlc_aggregate_kernel, kK5Threads, k5m_smem_bytes(W));
    const int grid = (int)tmax<uint64_t>(1, tmin<uint64_t>(A.n5, (uint64_t)sms * tmax(1, per_sm)));
    launch_pdl(tlc_aggregate_kernel, grid, kK5Threads, k5m_smem_bytes(W), st, A, X, W, seek);
    return cudaPeekAtLastError() == cudaSuccess ? TLC_OK : TLC_ERR_CUDA;
}

// ============================================================== host side
static int g_k4_blocks = 0, g_k5_blocks = 0;

int launch_decompress_table(const SegTable &T, int mode, void *ws, cudaStream_t st) {
    if (small_table(T)) return launch_small_decompress(T, mode, st);         // one launch, on chip
    const WsLayout L = ws_layout(T, 0);
    char *base = reinterpret_cast<char *>(ws);
    Ctrl *ctrl = reinterpret_cast<Ctrl *>(base + L.ctrl);
    unsigned long long *states = reinterpret_cast<unsigned long long *>(base + L.k4st);
    unsigned long long *seek = reinterpret_cast<unsigned long long *>(base + L.seek);
    const int sms = num_sms();
    if (!T.all_seek) {                       // producer seek entries: no scan (payloads from K3)
        // K4's counter and chunk states (K5 / K5m use neither: no memsets without K4)
        if (cudaMemsetAsync(base + L.ctrl, 0, sizeof(Ctrl), st) != cudaSuccess) return TLC_ERR_CUDA;
        if (cudaMemsetAsync(states, 0, L.memset_d, st) != cudaSuccess) return TLC_ERR_CUDA;
        KernelScope ks(kK4, st);
        if (!g_k4_blocks)
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_k4_blocks, tlc_zre_scan_kernel, kK4Threads, 0);
        const int grid = (int)tmax<uint64_t>(1, tmin<uint64_t>(T.n4, (uint64_t)sms * tmin(16, tmax(1, g_k4_blocks))));
        tlc_zre_scan_kernel<<<grid, kK4Threads, 0, st>>>(T, ctrl, states, seek);
    }
    KernelScope ks(kK5, st);
    if (!g_k5_blocks)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_k5_blocks, tlc_expand_dequant_kernel<0>, kK5Threads, 0);
    const int grid = (int)tmax<uint64_t>(1, tmin<uint64_t>(T.n5, (uint64_t)sms * tmax(1, g_k5_blocks)));
    if (mode == TLC_MODE_OVERWRITE) launch_pdl(tlc_expand_dequant_kernel<0>, grid, kK5Threads, 0, st, T, seek);
    else launch_pdl(tlc_expand_dequant_kernel<1>, grid, kK5Threads, 0, st, T, seek);
    return cudaPeekAtLastError() == cudaSuccess ? TLC_OK : TLC_ERR_CUDA;
}

int launch_decompress(const uint8_t *payload, tlc_header *hdr, uint64_t n, float *out, int mode, void *ws,
                      cudaStream_t st) {
    uint64_t scratch = 0;
    const SegTable T = single_table(nullptr, nullptr, out, const_cast<uint8_t *>(payload), hdr, n, scratch);
    return launch_decompress_table(T, mode, ws, st);
}

size_t decompress_workspace_bytes(uint64_t n) {
    uint64_t scratch = 0;
    const SegTable T = single_table(nullptr, nullptr, nullptr, nullptr, nullptr, n, scratch);
    return ws_layout(T, 0).total;
}

}  // namespace tlc
