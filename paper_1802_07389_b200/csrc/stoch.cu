// stoch.cu -- "Stoch 3-value + QE", a compared design of the paper (Sec. 5.1,
// P:629-632): TernGrad-like stochastic 3-value quantization ("outputs
// randomized quantization values whose expectation matches their input value")
// without gradient clipping, sparsity multiplier or error buffer, followed by
// the same quartic encoding (and optionally zero-run encoding) as 3LC.
//
// K2s tlc_stoch_qe_kernel: m = max|t| from K1's key; element x of the tensor
// becomes sign(x) with probability |x|/m, drawn from a counter-based generator
// (reading R22): the element's word is word e%4 of Philox4x32-10 at counter
// (e/4, step) under key seed, U = (w >> 8) * 2^-24, p = fl(|x| / m) (IEEE
// division), q = sign(x) iff U < p.  The result depends only on (t, seed,
// step), never on the launch shape.
//
// Layout: a tile of t2 quartic positions [j0, j1) needs the elements
// [i*P + j0, i*P + j1) of each partition i.  Philox blocks are aligned to the
// ELEMENT index (four elements e = 4b..4b+3 per block), so a thread takes
// whole blocks: one 128-bit load of t (16-byte aligned for any P), one Philox
// evaluation, four digits packed in one 32-bit word of a shared-memory digit
// plane (partition i's tile starts at byte lo_i mod 4 of its plane).  After a
// barrier every thread funnel-shifts the five planes' words of four positions
// into place and folds them into four quartic bytes with one SWAR multiply-add
// chain (each byte <= 242, no carries between bytes) and one 32-bit store.
#include "tlc_device.cuh"
#include "tlc_launch.h"

namespace tlc {

constexpr int kK2sThreads = 256;
constexpr int kK2sMaxTile = 4096;            // >= every ItemSizes::t2

struct PhiloxKey {
    uint32_t k0, k1;
};

// Philox4x32-10 (Salmon et al., SC'11): ten rounds of two 32x32->64 multiplies.
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, PhiloxKey k) {
#pragma unroll
    for (int r = 0; r < 10; r++) {
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
        c = make_uint4(hi1 ^ c.y ^ k.k0, lo1, hi0 ^ c.w ^ k.k1, lo0);
        k.k0 += 0x9E3779B9u;
        k.k1 += 0xBB67AE85u;
    }
    return c;
}

// Digit (q + 1) of element x under word w: q = sign(x) iff U = (w >> 8) 2^-24 < fl(|x| / m).
// Fast form (2^-100 <= m <= 2^100): r = fl(|x| * fl(1/m)) lies within 2^-22 of fl(|x|/m)
// (three roundings of a quotient <= 1), so whenever |r - U| > 2^-21 comparing U with r
// decides exactly as the IEEE quotient does.  Both sides are kept scaled by 2^24 (exact:
// inv24 = fl(1/m) 2^24 stays normal): d = fl(|x| inv24) - (w >> 8).  The rare draws with
// |d| <= 8 (probability ~2^-20 each) and every other m take the IEEE division, once per
// block of four elements, out of line.
struct StochQ {
    float m, inv24;
    bool fast;
    __device__ __forceinline__ explicit StochQ(float mm)
        : m(mm), inv24(0.0f), fast(mm >= 0x1p-100f && mm <= 0x1p100f) {
        if (fast) inv24 = __fmul_rn(__frcp_rn(mm), 0x1p24f);
    }
    __device__ __forceinline__ static uint32_t code(bool take, float x) {
        return take ? (signbit(x) ? 0u : 2u) : 1u;            // take implies x != 0
    }
    // fast digit; sets `unsure` when the exact quotient must decide
    __device__ __forceinline__ uint32_t digit_fast(float x, uint32_t w, bool &unsure) const {
        const float d = __fsub_rn(__fmul_rn(fabsf(x), inv24), __uint2float_rn(w >> 8));
        unsure |= !(fabsf(d) > 8.0f);
        return code(d > 0.0f, x);
    }
    __device__ __forceinline__ uint32_t digit_exact(float x, uint32_t w) const {
        const float U = __fmul_rn(__uint2float_rn(w >> 8), 0x1p-24f);
        return code(U < __fdiv_rn(fabsf(x), m), x);
    }
};

__device__ __noinline__ uint32_t stoch_block_exact(const StochQ &Q, float4 v, uint4 w, uint32_t valid) {
    const float x[4] = {v.x, v.y, v.z, v.w};
    const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
    uint32_t d = 0;
#pragma unroll
    for (int c = 0; c < 4; c++)
        d |= (c < (int)valid ? Q.digit_exact(x[c], ww[c]) : 0u) << (8 * c);   // pad: digit 0
    return d;
}

__global__ void __launch_bounds__(kK2sThreads)
tlc_stoch_qe_kernel(const SegTable T, const unsigned int *maxkey, uint32_t seed_lo, uint32_t seed_hi,
                    uint32_t step_lo, uint32_t step_hi, int use_zre, uint8_t *__restrict__ scratch) {
    // digit planes: element e of partition i lands at byte e - 4*floor(lo_i/4), so every
    // Philox block writes one aligned 32-bit word; the tile's first position sits at
    // byte sh_i = lo_i mod 4 of plane i.
    __shared__ __align__(16) uint32_t dig[5][kK2sMaxTile / 4 + 4];
    __shared__ uint64_t s_first[kSegCache];
    pdl_trigger();
    seg_index_load<2>(T, s_first);
    pdl_wait();                                          // K1's max keys
    const PhiloxKey key{seed_lo, seed_hi};
    for (uint64_t tile = blockIdx.x; tile < T.n2; tile += gridDim.x) {
        const int si = find_seg_c<2>(T, tile, s_first);
        const Seg S = get_seg(T, si);
        float m;
        const unsigned int status = scale_from_key(maxkey[si], 1.0f, m);   // m = max|t| (no s)
        const uint64_t lt = tile - S.k2;
        if (lt == 0 && threadIdx.x == 0) {
            tlc_header *h = S.hdr;
            h->M = m;
            h->flags = use_zre ? TLC_FLAG_ZRE : 0u;
            h->n = S.n;
            h->payload_len = (status == TLC_OK && !use_zre) ? S.P : 0;   // ZRE: set by K3
            h->status = status;
            h->reserved = 0;
        }
        if (status != TLC_OK) continue;                  // uniform per tile
        const uint64_t P = S.P, n = S.n;
        const uint64_t j0 = lt * T.sz.t2, j1 = tmin<uint64_t>(P, j0 + T.sz.t2);
        const bool vec = aligned16(S.t);
        const StochQ Q(m);
        // phase A: one Philox block (4 elements, one 128-bit load) per thread and step
#pragma unroll 1
        for (int i = 0; i < 5; i++) {
            const uint64_t lo = (uint64_t)i * P + j0, hi = (uint64_t)i * P + j1;
            const uint64_t b0 = lo / 4;
            const uint32_t nb = (uint32_t)((hi - 1) / 4 - b0 + 1);
            // kU blocks per thread and step: their loads are all in flight before the
            // first Philox round, so each thread keeps 16 kU bytes of t outstanding
            constexpr int kU = 4;
            for (uint32_t lb0 = threadIdx.x; lb0 < nb; lb0 += kU * kK2sThreads) {
                const uint32_t lbl = lb0 + (kU - 1) * kK2sThreads;
                if (vec && Q.fast && lbl < nb && 4 * (b0 + lbl) + 3 < n) {
                    // all kU blocks exist and are aligned: no per-block guards
                    float4 v[kU];
#pragma unroll
                    for (int u = 0; u < kU; u++)
                        v[u] = ld_stream4(reinterpret_cast<const float4 *>(S.t) + (b0 + lb0 + u * kK2sThreads));
                    uint32_t d[kU];
                    uint4 w[kU];
                    bool unsure = false;
#pragma unroll
                    for (int u = 0; u < kU; u++) {
                        const uint64_t b = b0 + lb0 + u * kK2sThreads;
                        w[u] = philox4x32_10(make_uint4((uint32_t)b, (uint32_t)(b >> 32), step_lo, step_hi), key);
                        d[u] = Q.digit_fast(v[u].x, w[u].x, unsure) | (Q.digit_fast(v[u].y, w[u].y, unsure) << 8) |
                               (Q.digit_fast(v[u].z, w[u].z, unsure) << 16) | (Q.digit_fast(v[u].w, w[u].w, unsure) << 24);
                    }
                    if (unsure) {                        // rare: the IEEE quotient decides
#pragma unroll
                        for (int u = 0; u < kU; u++) d[u] = stoch_block_exact(Q, v[u], w[u], 4u);
                    }
#pragma unroll
                    for (int u = 0; u < kU; u++) dig[i][lb0 + u * kK2sThreads] = d[u];
                    continue;
                }
                float4 v[kU];
                uint32_t valid[kU];
#pragma unroll
                for (int u = 0; u < kU; u++) {
                    const uint32_t lb = lb0 + u * kK2sThreads;
                    const uint64_t e0 = 4 * (b0 + lb);
                    valid[u] = lb >= nb ? 0u : e0 + 3 < n ? 4u : (uint32_t)(n - tmin<uint64_t>(n, e0));
                    v[u] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
                    if (vec && valid[u] == 4) {
                        v[u] = ld_stream4(reinterpret_cast<const float4 *>(S.t) + (b0 + lb));
                    } else {                             // tensor end or unaligned t
                        if (valid[u] > 0) v[u].x = ld_stream(S.t + e0);
                        if (valid[u] > 1) v[u].y = ld_stream(S.t + e0 + 1);
                        if (valid[u] > 2) v[u].z = ld_stream(S.t + e0 + 2);
                        if (valid[u] > 3) v[u].w = ld_stream(S.t + e0 + 3);
                    }
                }
#pragma unroll
                for (int u = 0; u < kU; u++) {
                    const uint32_t lb = lb0 + u * kK2sThreads;
                    if (lb >= nb) break;
                    const uint64_t b = b0 + lb;
                    const uint4 w = philox4x32_10(make_uint4((uint32_t)b, (uint32_t)(b >> 32), step_lo, step_hi), key);
                    bool unsure = !Q.fast || valid[u] != 4;
                    uint32_t d = Q.digit_fast(v[u].x, w.x, unsure) | (Q.digit_fast(v[u].y, w.y, unsure) << 8) |
                                 (Q.digit_fast(v[u].z, w.z, unsure) << 16) | (Q.digit_fast(v[u].w, w.w, unsure) << 24);
                    if (unsure) d = stoch_block_exact(Q, v[u], w, valid[u]);
                    dig[i][lb] = d;
                }
            }
        }
        __syncthreads();
        // phase B: B = 81 d0 + 27 d1 + 9 d2 + 3 d3 + d4, four positions per thread
        uint8_t *bytes = (use_zre ? scratch + S.bytes_off : S.payload) + j0;
        const uint32_t len = (uint32_t)(j1 - j0);
        const bool word_ok = use_zre || aligned4(S.payload);
        for (uint32_t g = threadIdx.x; 4 * g < len; g += kK2sThreads) {
            uint32_t v = 0;
#pragma unroll
            for (int i = 0; i < 5; i++) {
                const uint32_t sh = (uint32_t)(((uint64_t)i * P + j0) & 3);     // lo_i mod 4
                v = v * 3u + __funnelshift_r(dig[i][g], dig[i][g + 1], 8 * sh);
            }
            if (word_ok && 4 * g + 4 <= len) {
                reinterpret_cast<uint32_t *>(bytes)[g] = v;
            } else {
                for (uint32_t c = 0; c < 4 && 4 * g + c < len; c++) bytes[4 * g + c] = (uint8_t)(v >> (8 * c));
            }
        }
        __syncthreads();                                 // planes are reused by the next tile
    }
}

void launch_stoch_qe(const SegTable &T, const unsigned int *maxkey, uint64_t seed, uint64_t step, int use_zre,
                     uint8_t *scratch, cudaStream_t st) {
    static int blocks = 0;
    if (!blocks) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, tlc_stoch_qe_kernel, kK2sThreads, 0);
    KernelScope ks(kK2s, st);
    const int grid = (int)tmax<uint64_t>(1, tmin<uint64_t>(T.n2, (uint64_t)num_sms() * tmax(1, blocks)));
    launch_pdl(tlc_stoch_qe_kernel, grid, kK2sThreads, 0, st, T, maxkey, (uint32_t)seed, (uint32_t)(seed >> 32),
               (uint32_t)step, (uint32_t)(step >> 32), use_zre, scratch);
}

}  // namespace tlc
