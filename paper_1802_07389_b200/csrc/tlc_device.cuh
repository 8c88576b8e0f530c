// tlc_device.cuh -- device-side building blocks shared by the sm_100a kernels.
//
// Nothing here is shared with oracle/ (the CPU oracle is an independent
// transcription of the paper); see DESIGN.md section 5 for the kernel designs.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>
#ifdef TLC_DEVICE_CHECKS
#include <cstdio>
#endif

#include "../../include/tlc.h"
#include "tlc_launch.h"

namespace tlc {

// ---------------------------------------------------------------- device checks
// -DTLC_DEVICE_CHECKS (a test build, tests/test_gpu_device_checks.py): bounds of every
// data-dependent store index are asserted on the device; a violation prints its site and
// traps.  compute-sanitizer is not available on the GPU pool this was built on.
#ifdef TLC_DEVICE_CHECKS
#define TLC_CHECK(c)                                                                      \
    do {                                                                                  \
        if (!(c)) {                                                                       \
            printf("TLC_CHECK failed: %s at %s:%d\n", #c, __FILE__, __LINE__);            \
            __trap();                                                                     \
        }                                                                                 \
    } while (0)
#else
#define TLC_CHECK(c) do {} while (0)
#endif

// ---------------------------------------------------------------- constants
constexpr uint8_t kZeroGroup = 121;        // five zero trits
constexpr uint8_t kFirstRunCode = 243;     // 243+(k-2), 2 <= k <= 14
constexpr uint32_t kMaxRun = 14;

// Per-call control block at the start of every workspace (zeroed by a
// cudaMemsetAsync at the start of each call, together with the look-back
// tile states that follow it).
struct Ctrl {
    unsigned long long k3_counter;   // dynamic K3 chunk ids (forward-progress ordering)
    unsigned long long k4_counter;   // dynamic K4 chunk ids
    unsigned long long k12_counter;  // dynamic K12 work items
    unsigned int pad[58];
};
static_assert(sizeof(Ctrl) == 256, "ctrl is one 256-byte block");

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int *p) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned int ld_relaxed_u32(const unsigned int *p) {
    unsigned int v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// PDL: wait for the stream predecessor's results / let the successor be scheduled
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---------------------------------------------------------------- mbarriers and bulk copies
__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long *b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "TLC_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra TLC_WAIT_%=;\n\t}" ::"r"(smem_addr(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes, unsigned long long *b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(b)) : "memory");
}


// Streaming loads of data read exactly once by this kernel.
__device__ __forceinline__ float ld_stream(const float *p) { return __ldcs(p); }
__device__ __forceinline__ float4 ld_stream4(const float4 *p) { return __ldcs(p); }

// ---------------------------------------------------------------- quantizer
// Eq. 2 with round-half-away (R1) and the residual of steps (a),(b), given
// M = fl(max|u| * s).  Three uniform regimes (the branch is the same for the
// whole launch):
//   M == 0           -> q = 0, err = u                                   (R5)
//   M >= 2^-125      -> q = sign(u) * [|u| >= M/2]; M/2 is exact, and
//                       fl(u/M) >= 1/2  <=>  u >= M/2 exactly
//   0 < M < 2^-125   -> q from the IEEE quotient __fdiv_rn(u, M)          (R4)
// IEEE quotient path, out of line: only taken when M < 2^-125 (subnormal M/2),
// which keeps the division's registers out of the streaming loops.
static __device__ __noinline__ int quant_div(float u, float M) {
    const float x = __fdiv_rn(u, M);
    return (x >= 0.5f) - (x <= -0.5f);
}

struct Quant {
    float M, halfM;
    int mode;  // 0: zero, 1: compare, 2: divide
    __device__ __forceinline__ Quant(float m) : M(m), halfM(m * 0.5f) {  // exact when used (M >= 2^-125)
        mode = (m == 0.0f) ? 0 : (m >= 2.350988701644575e-38f /* 2^-125 */ ? 1 : 2);
    }
    __device__ __forceinline__ int q(float u) const {
        if (mode == 1) return fabsf(u) >= halfM ? (u > 0.0f ? 1 : -1) : 0;
        if (mode == 2) return quant_div(u, M);
        return 0;
    }
    // err = u - M*q (exact by Sterbenz when q != 0; u - (+0) == u otherwise)
    __device__ __forceinline__ float residual(float u, int q) const {
        return q == 0 ? u : __fsub_rn(u, q > 0 ? M : -M);
    }
};

// The common regime (M >= 2^-125) only: the compare form of Eq. 2.
struct QuantCmp {
    float M, halfM;
    __device__ __forceinline__ explicit QuantCmp(const Quant &Q) : M(Q.M), halfM(Q.halfM) {}
    __device__ __forceinline__ int q(float u) const { return fabsf(u) >= halfM ? (u > 0.0f ? 1 : -1) : 0; }
    __device__ __forceinline__ float residual(float u, int q) const {
        return q == 0 ? u : __fsub_rn(u, q > 0 ? M : -M);
    }
};

// ---------------------------------------------------------------- ZRE run summary monoid
// Zero-run encoding (greedy chunks of <= 14 from the run start, R11)
// is produced left to right with one carry: c = number of 121 bytes seen but
// not yet emitted (0..13).  A 121 byte increments c and emits 255 when c hits
// 14; any other byte first flushes a pending chunk (121 if c == 1, else
// 243+(c-2)) and then emits itself; the end of the stream flushes too.  A
// stretch of quartic bytes therefore acts on the incoming carry as
//     ALL (every byte is 121, length L = 14*div + mod):
//         count(c) = div + [c+mod >= 14],               carry' = (c+mod) mod 14
//     MIX (contains a non-121 byte; leading 121-run of length 14a + r0):
//         count(c) = cnt + ceil((c+r0)/14),             carry' = tr
// with cnt = a + emissions from the first non-121 byte on, tr = trailing run
// length mod 14.  Composition of these transfer functions is associative and
// needs only adds and compares (every sum of residues is < 28), so the encoder
// is a scan over this monoid.
//
// Packing (64 bit): bits 0..43 div|cnt, 45..48 mod|r0, 49..52 tr, bit 53 kind
// (1 = MIX), bit 62 "published" flag of the chunk scans.
struct RunSum {
    uint64_t v;   // ALL: L div 14; MIX: cnt
    uint32_t r0;  // ALL: L mod 14; MIX: leading run mod 14
    uint32_t tr;  // MIX: trailing run mod 14
    bool mix;
};

__host__ __device__ __forceinline__ unsigned long long pack(const RunSum &s) {
    return (s.v & ((1ull << 44) - 1)) | ((unsigned long long)s.r0 << 45) |
           ((unsigned long long)s.tr << 49) | ((unsigned long long)s.mix << 53);
}
__host__ __device__ __forceinline__ RunSum unpack(unsigned long long w) {
    RunSum s;
    s.v = w & ((1ull << 44) - 1);
    s.r0 = (uint32_t)(w >> 45) & 15u;
    s.tr = (uint32_t)(w >> 49) & 15u;
    s.mix = (w >> 53) & 1;
    return s;
}
__host__ __device__ __forceinline__ RunSum run_identity() { return RunSum{0, 0, 0, false}; }

__host__ __device__ __forceinline__ uint32_t mod14(uint32_t x) { return x >= kMaxRun ? x - kMaxRun : x; }  // x < 28

// a then b
__host__ __device__ __forceinline__ RunSum compose(const RunSum &a, const RunSum &b) {
    RunSum r;
    if (!a.mix) {
        const uint32_t x = a.r0 + b.r0;          // ALL . ALL, or a's 121s extend b's leading run
        r.v = a.v + b.v + (x >= kMaxRun);
        r.r0 = mod14(x);
        r.tr = b.tr;
        r.mix = b.mix;
        return r;
    }
    r = a;
    const uint32_t x = a.tr + b.r0;
    if (!b.mix) {                                // MIX . ALL
        r.v = a.v + b.v + (x >= kMaxRun);
        r.tr = mod14(x);
    } else {                                     // MIX . MIX: b's first literal flushes a's tail
        r.v = a.v + b.v + (x > 0) + (x > kMaxRun);
        r.tr = b.tr;
    }
    return r;
}

// (emitted count, carry) of a stretch entered with carry c
__host__ __device__ __forceinline__ void run_eval(const RunSum &s, uint32_t c, uint64_t &count,
                                                  uint32_t &carry) {
    const uint32_t x = c + s.r0;
    if (!s.mix) {
        count = s.v + (x >= kMaxRun);
        carry = mod14(x);
    } else {
        count = s.v + (x > 0) + (x > kMaxRun);
        carry = s.tr;
    }
}

// ZRE byte for a pending chunk of c (1..14) zero groups (R12)
__host__ __device__ __forceinline__ uint8_t run_code(uint32_t c) {
    return c == 1 ? kZeroGroup : (uint8_t)(kFirstRunCode + (c - 2));
}

__host__ __device__ __forceinline__ uint32_t byte_at(const uint32_t *w, int m) {
    return (w[m >> 2] >> (8 * (m & 3))) & 0xffu;
}

// ---------------------------------------------------------------- 32-byte segments as bit masks
// The zero-run encoder only needs to know which quartic bytes are literals
// (!= 121): a 32-byte segment becomes a 32-bit mask and its run summary and
// emission follow from ctz/clz/popc over that mask.
__host__ __device__ __forceinline__ uint32_t ctz32(uint32_t x) {
#ifdef __CUDA_ARCH__
    return (uint32_t)(__ffs(x) - 1);
#else
    return (uint32_t)__builtin_ctz(x);
#endif
}
__host__ __device__ __forceinline__ uint32_t msb32(uint32_t x) {
#ifdef __CUDA_ARCH__
    return 31u - (uint32_t)__clz(x);
#else
    return 31u - (uint32_t)__builtin_clz(x);
#endif
}
__host__ __device__ __forceinline__ uint32_t popc32(uint32_t x) {
#ifdef __CUDA_ARCH__
    return (uint32_t)__popc(x);
#else
    return (uint32_t)__builtin_popcount(x);
#endif
}
// bit c of the result = (byte c of w != 121)
__host__ __device__ __forceinline__ uint32_t literal_nibble(uint32_t w) {
#ifdef __CUDA_ARCH__
    const uint32_t t = __vcmpne4(w, 0x79797979u) & 0x01010101u;
#else
    uint32_t t = 0;
    for (int c = 0; c < 4; c++) t |= (uint32_t)(((w >> (8 * c)) & 0xffu) != kZeroGroup) << (8 * c);
#endif
    return (t * 0x01020408u) >> 24;   // gathers bits 0, 8, 16, 24 into bits 0..3
}
__host__ __device__ __forceinline__ uint32_t literal_mask(const uint32_t (&w)[8]) {
    uint32_t m = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) m |= literal_nibble(w[k]) << (4 * k);
    return m;
}

// Run summary of the first len (1..32) bytes of a segment with literal mask `mask`.
__host__ __device__ __forceinline__ RunSum mask_summary(uint32_t mask, int len) {
    RunSum s = run_identity();
    if (len <= 0) return s;
    if (len < 32) mask &= (1u << len) - 1u;
    if (mask == 0) {
        s.v = (uint64_t)(len / (int)kMaxRun);
        s.r0 = (uint32_t)(len % (int)kMaxRun);
        return s;
    }
    const uint32_t lead = ctz32(mask), hi = msb32(mask);
    const uint32_t T = (uint32_t)len - 1u - hi;                       // trailing run
    uint32_t cnt = popc32(mask);                                       // literals
    // inner runs between literals: a run of L (1..13) 121s costs one flush byte;
    // runs of 14 or more (rare) are counted exactly below.
    const uint32_t inner = hi > lead ? ((~mask) & (((2u << hi) - 1u) ^ ((2u << lead) - 1u))) : 0u;
    uint32_t y = inner;
    y &= y >> 1; y &= y >> 2; y &= y >> 4; y &= y >> 6;               // bit set at runs >= 14
    if (y == 0) {
        cnt += popc32(mask & ~(mask << 1) & (mask - 1u));
    } else {
        uint32_t m = mask & (mask - 1u);
        uint32_t prev = lead;
        while (m) {
            const uint32_t p = ctz32(m);
            m &= m - 1u;
            const uint32_t L = p - prev - 1u;
            cnt += L / kMaxRun + (L % kMaxRun != 0);
            prev = p;
        }
    }
    cnt += T / kMaxRun + lead / kMaxRun;
    s.mix = true;
    s.v = cnt;
    s.r0 = lead % kMaxRun;
    s.tr = T % kMaxRun;
    return s;
}


// ---------------------------------------------------------------- warp rows of 32 x 32 bytes
// A warp row: lane l holds the bytes [32 l, 32 l + len_l) of a row (len_l = 32
// except at the end of a stream), reduced to its literal mask.  The carry a
// lane enters with is fixed by where the last literal before it sits (or by the
// row's incoming carry c_row if there is none), so per-lane carries need one
// ballot and one shuffle instead of a scan over the run monoid.  The three
// formulas below are __host__ __device__ so tests/native can drive them.

// carry entering lane `lane`; lp = row position of the last literal before it
__host__ __device__ __forceinline__ uint32_t lane_carry_in(uint32_t lane, bool has_before, uint32_t lp,
                                                           uint32_t c_row) {
    return (has_before ? (32u * lane - lp - 1u) : (c_row + 32u * lane)) % kMaxRun;
}
// carry leaving a row of row_len bytes; lp_all = position of its last literal
__host__ __device__ __forceinline__ uint32_t row_carry_out(bool any, uint32_t lp_all, uint32_t c_row,
                                                           uint32_t row_len) {
    return (any ? (row_len - lp_all - 1u) : (c_row + row_len)) % kMaxRun;
}
// run summary of a row from its count and carry-out at c_row = 0 and its leading run
__host__ __device__ __forceinline__ RunSum row_summary(bool any, uint32_t lead, uint32_t count0,
                                                       uint32_t carry_out0, uint32_t row_len) {
    RunSum s = run_identity();
    if (!any) {
        s.v = row_len / kMaxRun;
        s.r0 = row_len % kMaxRun;
        return s;
    }
    s.mix = true;
    s.r0 = lead % kMaxRun;
    s.v = count0 - (s.r0 > 0);             // count(c) = v + ceil((c + r0)/14)
    s.tr = carry_out0;
    return s;
}

struct WarpRow {
    uint32_t carry_in;    // this lane's incoming carry
    uint32_t count;       // ZRE bytes this lane emits (given carry_in)
    uint32_t row_count;   // all lanes: ZRE bytes the whole row emits
    uint32_t carry_out;   // all lanes: carry leaving the row
    uint32_t mixbal;      // lanes holding a literal
};

__device__ __forceinline__ WarpRow warp_row(uint32_t mask, int len, const RunSum &lane_sum, uint32_t c_row,
                                            uint32_t row_len) {
    const uint32_t lane = threadIdx.x & 31;
    WarpRow r;
    r.mixbal = __ballot_sync(0xffffffffu, mask != 0);
    const uint32_t lastpos = 32u * lane + (mask ? msb32(mask) : 0u);
    const uint32_t before = r.mixbal & ((1u << lane) - 1u);
    const uint32_t lp = __shfl_sync(0xffffffffu, lastpos, before ? (int)msb32(before) : 0);
    r.carry_in = lane_carry_in(lane, before != 0, lp, c_row);
    uint64_t cnt;
    uint32_t co;
    run_eval(lane_sum, r.carry_in, cnt, co);
    r.count = len > 0 ? (uint32_t)cnt : 0u;
    uint32_t tot = r.count;
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, d);
    r.row_count = tot;
    const uint32_t lp_all = __shfl_sync(0xffffffffu, lastpos, r.mixbal ? (int)msb32(r.mixbal) : 0);
    r.carry_out = row_carry_out(r.mixbal != 0, lp_all, c_row, row_len);
    return r;
}

// Run summary of a whole warp row (as a function of its incoming carry).
__device__ __forceinline__ RunSum warp_row_summary(uint32_t mask, int len, const RunSum &lane_sum,
                                                   uint32_t row_len) {
    const WarpRow r = warp_row(mask, len, lane_sum, 0u, row_len);
    const uint32_t k0 = r.mixbal ? ctz32(r.mixbal) : 0u;
    const uint32_t lead = __shfl_sync(0xffffffffu, mask ? ctz32(mask) : 0u, (int)k0) + 32u * k0;
    return row_summary(r.mixbal != 0, lead, r.row_count, r.carry_out, row_len);
}

// ZRE bytes of one lane's 32 quartic bytes of a warp row, given the zero groups
// pending before them (carry_in < 14, from warp_row): per literal (bit of `mask`), the
// code of the pending zero groups that do not fill a chunk of 14 (full chunks are
// skipped -- their 255 bytes are the caller's prefill), then the literal itself
// (P:545-546).  Writes dst[o, ...) and returns the end offset.
//
// Common case ("simple": no run of 14 or more zero groups before a literal of the lane):
// every literal m lands at o + (literals before m) + (codes up to m), a code right
// before literal m whose preceding run is non-empty -- one running offset, no division,
// the same instructions in every lane (SIMT: a per-byte branchy loop made the warp run
// both paths).  A word of four literals without codes is stored as a unit when the
// whole warp has one there.  The codes' values (run lengths) follow in a short loop
// over the code bits.  Other lanes take the general byte loop.
__host__ __device__ __forceinline__ bool lane_simple(uint32_t mask, uint32_t carry_in) {
    if (!mask) return true;
    const uint32_t lead = ctz32(mask), hi = msb32(mask);
    if (lead + carry_in >= kMaxRun) return false;
    uint32_t y = hi > lead ? ((~mask) & (((2u << hi) - 1u) ^ ((2u << lead) - 1u))) : 0u;
    y &= y >> 1; y &= y >> 2; y &= y >> 4; y &= y >> 6;             // a run of >= 14 zero groups
    return y == 0;
}

// vote among the lanes currently executing together (lane_emit's lanes may have split on
// lane_simple); only ever used where p itself makes the voted path correct for the lane
__host__ __device__ __forceinline__ bool warp_all(bool p) {
#ifdef __CUDA_ARCH__
    return __all_sync(__activemask(), p);
#else
    return p;                                // host emulation: lanes run one at a time
#endif
}

// The general form: one byte at a time, zero groups pending in c.
template <class Dst>
__host__ __device__ __forceinline__ uint32_t lane_emit_bytes(const uint32_t (&w)[8], uint32_t mask, uint32_t c,
                                                             Dst dst, uint32_t o) {
#pragma unroll
    for (int k = 0; k < 8; k++) {
        const uint32_t mk = (mask >> (4 * k)) & 0xfu;
#pragma unroll
        for (int q = 0; q < 4; q++) {
            if ((mk >> q) & 1u) {
                o += c / kMaxRun;
                const uint32_t rem = c % kMaxRun;
                if (rem) dst[o++] = run_code(rem);
                c = 0;
                dst[o++] = (uint8_t)(w[k] >> (8 * q));
            } else {
                c++;
            }
        }
    }
    return o;
}

// Variants (A/B by -DTLC_EMIT_V; the host harness checks all three against the oracle):
//  1  a word of four literals with nothing pending is stored as a unit, other words go
//     byte by byte (divergent: a warp runs both paths when its lanes differ);
//  2  simple lanes: one running offset, predicated byte stores (a serial add chain);
//  3  simple lanes: every byte's offset from popcounts of the masks below it (no chain);
//  4  variant 1 for simple lanes without the division (pending zero groups < 14).
#ifndef TLC_EMIT_V
#define TLC_EMIT_V 1
#endif
template <int V = TLC_EMIT_V, class Dst>
__host__ __device__ __forceinline__ uint32_t lane_emit(const uint32_t (&w)[8], uint32_t mask, uint32_t carry_in,
                                                       Dst dst, uint32_t o) {
    if (V == 1) {
        uint32_t c = carry_in;
#pragma unroll
        for (int k = 0; k < 8; k++) {
            const uint32_t mk = (mask >> (4 * k)) & 0xfu;
            if (mk == 0xfu && c == 0) {
                dst[o] = (uint8_t)w[k];
                dst[o + 1] = (uint8_t)(w[k] >> 8);
                dst[o + 2] = (uint8_t)(w[k] >> 16);
                dst[o + 3] = (uint8_t)(w[k] >> 24);
                o += 4;
                continue;
            }
#pragma unroll
            for (int q = 0; q < 4; q++) {
                if ((mk >> q) & 1u) {
                    o += c / kMaxRun;
                    const uint32_t rem = c % kMaxRun;
                    if (rem) dst[o++] = run_code(rem);
                    c = 0;
                    dst[o++] = (uint8_t)(w[k] >> (8 * q));
                } else {
                    c++;
                }
            }
        }
        return o;
    }
    if (!lane_simple(mask, carry_in)) return lane_emit_bytes(w, mask, carry_in, dst, o);
    if (V == 4) {
        // variant 1's word fast path; simple lanes never hold 14 pending zero groups, so a
        // flush is one code of the pending count c (< 14), no division
        uint32_t c = carry_in;
#pragma unroll
        for (int k = 0; k < 8; k++) {
            const uint32_t mk = (mask >> (4 * k)) & 0xfu;
            if (mk == 0xfu && c == 0) {
                dst[o] = (uint8_t)w[k];
                dst[o + 1] = (uint8_t)(w[k] >> 8);
                dst[o + 2] = (uint8_t)(w[k] >> 16);
                dst[o + 3] = (uint8_t)(w[k] >> 24);
                o += 4;
                continue;
            }
#pragma unroll
            for (int q = 0; q < 4; q++) {
                if ((mk >> q) & 1u) {
                    if (c) dst[o++] = run_code(c);
                    c = 0;
                    dst[o++] = (uint8_t)(w[k] >> (8 * q));
                } else {
                    c++;
                }
            }
        }
        return o;
    }
    // code flags: a literal whose previous byte is a zero group, or the lane's first
    // byte when zero groups are pending from before the lane
    const uint32_t cf = mask & ((~mask << 1) | (carry_in ? 1u : 0u));
    if (V == 2) {
        uint32_t off = o;
#pragma unroll
        for (int k = 0; k < 8; k++) {
            const uint32_t nib = (mask >> (4 * k)) & 0xfu, cnib = (cf >> (4 * k)) & 0xfu;
            if (warp_all(nib == 0xfu && cnib == 0u)) {
                dst[off] = (uint8_t)w[k];
                dst[off + 1] = (uint8_t)(w[k] >> 8);
                dst[off + 2] = (uint8_t)(w[k] >> 16);
                dst[off + 3] = (uint8_t)(w[k] >> 24);
                off += 4;
                continue;
            }
#pragma unroll
            for (int q = 0; q < 4; q++) {
                off += (cnib >> q) & 1u;
                if ((nib >> q) & 1u) dst[off] = (uint8_t)(w[k] >> (8 * q));
                off += (nib >> q) & 1u;
            }
        }
    } else {
#pragma unroll
        for (int k = 0; k < 8; k++) {
            const uint32_t lt = (1u << (4 * k)) - 1u;
            const uint32_t base = o + popc32(mask & lt) + popc32(cf & lt);
            const uint32_t nib = (mask >> (4 * k)) & 0xfu, cnib = (cf >> (4 * k)) & 0xfu;
#pragma unroll
            for (int q = 0; q < 4; q++)
                if ((nib >> q) & 1u)
                    dst[base + popc32(nib & ((1u << q) - 1u)) + popc32(cnib & ((2u << q) - 1u))] =
                        (uint8_t)(w[k] >> (8 * q));
        }
    }
    for (uint32_t cm = cf; cm; cm &= cm - 1u) {
        const uint32_t m = ctz32(cm), lt = (1u << m) - 1u, below = mask & lt;
        const uint32_t R = below ? m - msb32(below) - 1u : m + carry_in;   // 1..13
        dst[o + popc32(below) + popc32(cf & lt)] = run_code(R);
    }
    return o + popc32(mask) + popc32(cf);
}

// The warp's emission stage in shared memory with 4 bytes of padding after every 128:
// a lane of a dense row writes near byte 32*lane, i.e. word 8*lane, and 32 lanes hit
// only 4 banks (8-way conflicts on every byte store); with the padding lane l's word is
// 8*l + l/4, 32 distinct banks.  Logical byte q lives at q + 4*(q/128).
struct PadStage {
    uint8_t *p;
    uint32_t cap;                    // physical bytes (checked in TLC_DEVICE_CHECKS builds)
    __host__ __device__ __forceinline__ uint8_t &operator[](uint32_t q) const {
#if defined(TLC_DEVICE_CHECKS) && defined(__CUDA_ARCH__)
        TLC_CHECK(q + ((q >> 7) << 2) < cap);
#endif
#ifdef TLC_NO_PAD
        return p[q];                                   // A/B: unpadded stage
#else
        return p[q + ((q >> 7) << 2)];
#endif
    }
};
#ifdef TLC_NO_PAD
__host__ __device__ constexpr uint32_t pad_stage_bytes(uint32_t n) { return n; }
#else
__host__ __device__ constexpr uint32_t pad_stage_bytes(uint32_t n) { return n + ((n + 127) >> 7) * 4; }
#endif

// Prefill logical bytes [0, n) of a padded stage with 255 (32-bit stores).
__device__ __forceinline__ void pad_stage_fill(const PadStage &st, uint32_t n) {
    for (uint32_t q = 4 * (threadIdx.x & 31); q < n; q += 128)
        *reinterpret_cast<uint32_t *>(&st[q]) = ~0u;
}

// A warp copies logical bytes [a, a+n) of a padded stage to dst, where dst is congruent
// to stage byte a modulo 4: head and tail bytes singly, the middle with 32-bit stores
// (a 4-byte-aligned logical word never straddles a padding gap).
__device__ __forceinline__ void warp_copy_padded(uint8_t *dst, const PadStage &st, uint32_t a, uint32_t n) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t head = tmin<uint32_t>(n, (4u - (uint32_t)(reinterpret_cast<uintptr_t>(dst) & 3u)) & 3u);
    if (lane < head) dst[lane] = st[a + lane];
    const uint32_t nw = (n - head) / 4u;
    for (uint32_t q = lane; q < nw; q += 32)
        reinterpret_cast<uint32_t *>(dst + head)[q] = *reinterpret_cast<const uint32_t *>(&st[a + head + 4 * q]);
    const uint32_t t0 = head + 4u * nw;
    if (t0 + lane < n) dst[t0 + lane] = st[a + t0 + lane];
}

// A warp copies n bytes from shared memory to global memory where src and dst are
// congruent modulo 16: head and tail bytes singly, the middle with 16-byte stores.
__device__ __forceinline__ void warp_copy_congruent(uint8_t *dst, const uint8_t *src, uint32_t n) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t head = tmin<uint32_t>(n, (16u - (uint32_t)(reinterpret_cast<uintptr_t>(dst) & 15u)) & 15u);
    if (lane < head) dst[lane] = src[lane];
    const uint32_t nv = (n - head) / 16u;
    for (uint32_t q = lane; q < nv; q += 32)
        reinterpret_cast<uint4 *>(dst + head)[q] = reinterpret_cast<const uint4 *>(src + head)[q];
    const uint32_t t0 = head + 16u * nv;
    if (t0 + lane < n) dst[t0 + lane] = src[t0 + lane];
}

// A warp stores code 255 to payload[a, b): head and tail bytes singly, the
// 16-byte-aligned middle with vector stores.  Callers __syncwarp() before
// overwriting any of these bytes.
__device__ __forceinline__ void warp_fill_full_chunks(uint8_t *payload, uint64_t a, uint64_t b) {
    const uint32_t lane = threadIdx.x & 31;
    const uintptr_t lo = reinterpret_cast<uintptr_t>(payload + a), hi = reinterpret_cast<uintptr_t>(payload + b);
    const uintptr_t lo16 = tmin<uintptr_t>(hi, (lo + 15) & ~uintptr_t(15));
    const uintptr_t hi16 = tmax<uintptr_t>(lo16, hi & ~uintptr_t(15));
    if (lo + lane < lo16) *reinterpret_cast<uint8_t *>(lo + lane) = 0xff;
    if (hi16 + lane < hi) *reinterpret_cast<uint8_t *>(hi16 + lane) = 0xff;
    for (uintptr_t q = lo16 + 16 * lane; q < hi16; q += 16 * 32)
        *reinterpret_cast<uint4 *>(q) = make_uint4(~0u, ~0u, ~0u, ~0u);
}

// ---------------------------------------------------------------- segment lookup
template <int F>
__device__ __forceinline__ uint64_t seg_first(const Seg &s) {
    return F == 1 ? s.k1 : F == 2 ? s.k2 : F == 3 ? s.k3 : F == 4 ? s.k4 : s.k5;
}
// segment holding global item `item` of kernel F
template <int F>
__device__ __forceinline__ int find_seg(const SegTable &T, uint64_t item) {
    if (T.count == 1) return 0;
    int lo = 0, hi = T.count - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (seg_first<F>(T.d[mid]) <= item) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}
__device__ __forceinline__ Seg get_seg(const SegTable &T, int i) { return T.count == 1 ? T.one : T.d[i]; }

// Per-CTA shared-memory copy of a kernel's first-item array (tables of up to
// kSegCache segments): the per-item segment search then costs shared loads, not
// a chain of dependent global loads.
constexpr int kSegCache = 512;
template <int F, int C = kSegCache>
__device__ __forceinline__ void seg_index_load(const SegTable &T, uint64_t *sf) {
    if (T.count > 1 && T.count <= C) {
        for (int i = threadIdx.x; i < T.count; i += blockDim.x) sf[i] = T.first[F - 1][i];
    }
    __syncthreads();
}
template <int F, int C = kSegCache>
__device__ __forceinline__ int find_seg_c(const SegTable &T, uint64_t item, const uint64_t *sf) {
    if (T.count == 1) return 0;
    if (T.count > C) return find_seg<F>(T, item);
    int lo = 0, hi = T.count - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (sf[mid] <= item) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// M and the compressor status of a segment from its max key (Eq. 1, R6)
__device__ __forceinline__ unsigned int scale_from_key(unsigned int key, float s, float &M) {
    M = 0.0f;
    if (key >= 0x7f800000u) return TLC_ERR_NONFINITE;      // NaN or Inf in u
    M = __fmul_rn(__uint_as_float(key), s);
    if (isinf(M)) { M = 0.0f; return TLC_ERR_RANGE; }
    return TLC_OK;
}

// ---------------------------------------------------------------- decoder helpers
__device__ __forceinline__ void raise_format(tlc_header *hdr) {
    atomicCAS(&hdr->status, (unsigned int)TLC_OK, (unsigned int)TLC_ERR_FORMAT);
}

// expansion length of a payload byte (inverse of P:545-546)
__host__ __device__ __forceinline__ uint32_t zre_len(uint32_t b) { return b >= kFirstRunCode ? b - 241u : 1u; }

// Expansion length of the 4 payload bytes of a word, SWAR: bytes >= 243 are the
// ones whose low seven bits plus 13 carry into bit 7 while bit 7 is set (no carry
// crosses a byte: 127 + 13 < 256); their excess b - 242 is summed with one dp4a.
__host__ __device__ __forceinline__ uint32_t word_len(uint32_t w) {
    const uint32_t hi = w & ((w & 0x7f7f7f7fu) + 0x0d0d0d0du) & 0x80808080u;   // bit 7 of codes >= 243
    const uint32_t x = w & ((hi >> 7) * 0xffu);                                   // their bytes
#ifdef __CUDA_ARCH__
    return 4u + __dp4a(x, 0x01010101u, 0u) - 242u * (uint32_t)__popc(hi);
#else
    const uint32_t sum = (x & 0xffu) + ((x >> 8) & 0xffu) + ((x >> 16) & 0xffu) + (x >> 24);
    return 4u + sum - 242u * (uint32_t)__builtin_popcount(hi);
#endif
}

// Header checks of the decoder: compressor status OK, n matches, 1 <= Z <= P,
// Z == P without ZRE, and M finite and >= +0 (Eq. 1, R6; anything else R21).
__device__ __forceinline__ bool header_valid(const tlc_header *hdr, uint64_t n) {
    const uint64_t P = (n + 4) / 5;
    const uint64_t Z = hdr->payload_len;
    const bool zre = (hdr->flags & TLC_FLAG_ZRE) != 0;
    const uint32_t Mb = __float_as_uint(hdr->M);
    return hdr->status == TLC_OK && hdr->n == n && Z <= P && Z >= 1 && (zre || Z == P) &&
           (Mb >> 31) == 0 && Mb < 0x7f800000u;
}

// ---------------------------------------------------------------- chunked scans
constexpr int kScanThreads = 256;                   // K4's block; K3 has 8 scanning warps + 1
constexpr int kScanWarps = kScanThreads / 32;

constexpr unsigned long long kReady = 1ull << 62;

constexpr unsigned long long kPrefix = 1ull << 63;   // the state holds the inclusive prefix
constexpr unsigned long long kStateFlags = kReady | kPrefix;

// Monoids of the chunked scans, on packed 62-bit values (identity packs to 0).
struct SumOp {
    __device__ __forceinline__ static unsigned long long combine(unsigned long long a, unsigned long long b) {
        return a + b;
    }
};
struct RunOp {   // a then b
    __device__ __forceinline__ static unsigned long long combine(unsigned long long a, unsigned long long b) {
        return pack(compose(unpack(a), unpack(b)));
    }
};

// Decoupled look-back by one full warp: the composition of chunk states
// st[0..lc), each published as kReady|aggregate or kPrefix|inclusive prefix.
// Each round reads the 4*32 newest unread predecessors (lane l holds four
// consecutive ones, lane 0 the newest), stops at the newest inclusive prefix
// and reduces the window in order.
template <class Op>
__device__ __forceinline__ unsigned long long warp_lookback(const unsigned long long *st, uint64_t lc) {
    constexpr int V = 4;
    const int lane = threadIdx.x & 31;
    unsigned long long excl = 0;
    int64_t j = (int64_t)lc - 1;
    while (j >= 0) {
        unsigned long long w[V];                            // w[0] newest
#pragma unroll
        for (int k = 0; k < V; k++) {
            const int64_t idx = j - (int64_t)(V * lane + k);
            w[k] = idx >= 0 ? ld_relaxed_u64(st + idx) : kPrefix;
        }
#pragma unroll
        for (int k = 0; k < V; k++)
            while (!(w[k] & kStateFlags)) {
                __nanosleep(64);
                w[k] = ld_relaxed_u64(st + (j - (int64_t)(V * lane + k)));
            }
        int kp = V;                                         // newest prefix in this lane
#pragma unroll
        for (int k = V - 1; k >= 0; k--)
            if (w[k] & kPrefix) kp = k;
        const uint32_t pre = __ballot_sync(0xffffffffu, kp < V);
        const int first = pre ? __ffs(pre) - 1 : 31;       // lane of the newest prefix
        unsigned long long v = 0;                            // this lane's part, oldest first
        if (lane <= first) {
            const int kmax = lane == first && pre ? kp : V - 1;
#pragma unroll
            for (int k = V - 1; k >= 0; k--)
                if (k <= kmax) v = Op::combine(v, w[k] & ~kStateFlags);
        }
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {                 // lane L + d is older than lane L
            const unsigned long long o = __shfl_down_sync(0xffffffffu, v, d);
            if (lane + d < 32) v = Op::combine(o, v);
        }
        excl = Op::combine(__shfl_sync(0xffffffffu, v, 0), excl);
        if (pre) break;
        j -= 32 * V;
    }
    return excl;
}

}  // namespace tlc
