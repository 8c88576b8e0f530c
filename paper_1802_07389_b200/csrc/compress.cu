// compress.cu -- the 3LC compressor on sm_100a over a table of tensors
// ("segments", tlc_launch.h): a single tlc_compress call is a one-segment table,
// a batch of per-layer tensors is a device table, and every kernel covers all
// segments in one launch.
//
//  K1 tlc_absmax_kernel  (row a1): u = err + t (not stored); max of
//     bits(u) & 0x7fffffff as uint32 per segment, which orders |u| and flags
//     NaN/Inf in one integer max (atomicMax per CTA and segment).
//  K2 tlc_quant_qe_kernel (rows a2-a3): a streaming pass -- recompute u,
//     M = fl(max|u| * s) (Eq. 1) from the segment's key, quantize (Eq. 2),
//     write err = u - M*q (steps a,b) and fold the five strided trits of each
//     quartic position into its byte (step 3), written to the payload (no ZRE)
//     or to the quartic scratch.  The CTA owning a segment's first tile writes
//     its header.
//  K3 tlc_zre_kernel (row a4): zero-run encoding (step 4) of the quartic bytes
//     as a chunked single-pass scan over the run-carry monoid of
//     tlc_device.cuh (section 5.3 of DESIGN.md).
//
// Paper: P:372-410 (Sec. 3.1), P:495-510 (Sec. 3.2), P:538-548 (Sec. 3.3).
#include <algorithm>
#include <cstdlib>

#include <vector>

#include "tlc_device.cuh"
#include "tlc_launch.h"

namespace tlc {

// ============================================================== K1
constexpr int kK1Threads = 512;

#ifdef TLC_K1_L2HINT
__device__ __forceinline__ float4 ld_l2hint4(const float4 *p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}
#endif
#ifndef TLC_K1_U
#define TLC_K1_U 4
#endif

__device__ __forceinline__ unsigned int absmax_key(float t, float e) {
    float u = __fadd_rn(e, t);                       // step (1): u = buffer + T_in
    return __float_as_uint(u) & 0x7fffffffu;         // |u| as ordered uint; NaN > Inf
}

__device__ __forceinline__ void k1_flush(unsigned int m, unsigned int *maxkey, int si, unsigned int *s_warp) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    m = __reduce_max_sync(0xffffffffu, m);
    if (lane == 0) s_warp[warp] = m;
    __syncthreads();
    if (warp == 0) {
        m = lane < kK1Threads / 32 ? s_warp[lane] : 0u;
        m = __reduce_max_sync(0xffffffffu, m);
        if (lane == 0) atomicMax(maxkey + si, m);
    }
    __syncthreads();
}

// kErr = false: the codecs without an error buffer (stochastic 3-value, 8-bit
// int) take max|t| -- the same key without the add.
template <bool kErr>
__device__ __forceinline__ unsigned int k1_key(float t, float e) {
    if constexpr (kErr) return absmax_key(t, e);
    else return __float_as_uint(t) & 0x7fffffffu;
}

template <bool kErr>
__global__ void __launch_bounds__(kK1Threads, 1)
tlc_absmax_kernel(const SegTable T, unsigned int *__restrict__ maxkey) {
    __shared__ unsigned int s_warp[kK1Threads / 32];
    __shared__ uint64_t s_first[kSegCache];
    pdl_trigger();
    seg_index_load<1>(T, s_first);
    unsigned int m = 0;
    int cur = -1;
    for (uint64_t tile = blockIdx.x; tile < T.n1; tile += gridDim.x) {
        const int si = find_seg_c<1>(T, tile, s_first);
        if (si != cur) {                                  // uniform: flush the previous segment
            if (cur >= 0) k1_flush(m, maxkey, cur, s_warp);
            m = 0;
            cur = si;
        }
        const Seg S = get_seg(T, si);
        const uint64_t lo = (tile - S.k1) * T.sz.t1, hi = tmin<uint64_t>(S.n, lo + T.sz.t1);
        uint64_t tail = lo;
        if (S.flags & kSegVec1) {
            const float4 *t4 = reinterpret_cast<const float4 *>(S.t);
            const float4 *e4 = reinterpret_cast<const float4 *>(S.err);
            const uint64_t a = lo / 4, b = hi / 4;             // lo is a multiple of 4
            constexpr int U = TLC_K1_U;
            uint64_t i = a + threadIdx.x;
            for (; i + (U - 1) * kK1Threads < b; i += U * kK1Threads) {
                float4 x[U], y[U];
#pragma unroll
                for (int k = 0; k < U; k++) {
#ifdef TLC_K1_L2HINT
                    x[k] = ld_l2hint4(t4 + i + k * kK1Threads);
                    y[k] = ld_l2hint4(e4 + i + k * kK1Threads);
#else
                    x[k] = ld_stream4(t4 + i + k * kK1Threads);
                    if constexpr (kErr) y[k] = __ldcg(e4 + i + k * kK1Threads);
                    else y[k] = x[k];
#endif
                }
#pragma unroll
                for (int k = 0; k < U; k++) {
                    m = max(m, k1_key<kErr>(x[k].x, y[k].x));
                    m = max(m, k1_key<kErr>(x[k].y, y[k].y));
                    m = max(m, k1_key<kErr>(x[k].z, y[k].z));
                    m = max(m, k1_key<kErr>(x[k].w, y[k].w));
                }
            }
            for (; i < b; i += kK1Threads) {
                const float4 x = ld_stream4(t4 + i);
                float4 y = x;
                if constexpr (kErr) y = __ldcg(e4 + i);
                m = max(m, k1_key<kErr>(x.x, y.x));
                m = max(m, k1_key<kErr>(x.y, y.y));
                m = max(m, k1_key<kErr>(x.z, y.z));
                m = max(m, k1_key<kErr>(x.w, y.w));
            }
            tail = 4 * b;
        }
        for (uint64_t i = tail + threadIdx.x; i < hi; i += kK1Threads)
            m = max(m, k1_key<kErr>(ld_stream(S.t + i), kErr ? __ldcg(S.err + i) : 0.0f));
    }
    if (cur >= 0) k1_flush(m, maxkey, cur, s_warp);
}

// ============================================================== K2
constexpr int kK2Threads = 256;

// K2's loads of t and err (read once): streaming (.cs, LP = 0), or through an L2 cache-policy
// operand (LP = 1: K12's quantize items demote the lines its max items kept, TLC_K12_HINT=2)
template <int LP>
__device__ __forceinline__ float4 ldq4(const float4 *p, uint64_t pol) {
    if (LP == 0) return __ldcs(p);
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "l"(pol));
    return v;
}
template <int LP>
__device__ __forceinline__ float ldq(const float *p, uint64_t pol) {
    if (LP == 0) return __ldcs(p);
    float v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
    return v;
}

// One quartic position j, any alignment: the five strided elements e = i*P + j
// (partition i), residuals stored, byte returned (pad positions -> digit 0).
template <class QT, int LP = 0>
__device__ __forceinline__ uint32_t quant_qe_one(const float *__restrict__ t, float *__restrict__ err,
                                                 uint64_t n, uint64_t P, uint64_t j, const QT &Q, uint64_t pol = 0) {
    float tv[5], ev[5];
#pragma unroll
    for (int i = 0; i < 5; i++) {
        const uint64_t e = (uint64_t)i * P + j;
        tv[i] = e < n ? ldq<LP>(t + e, pol) : 0.0f;
        ev[i] = e < n ? ldq<LP>(err + e, pol) : 0.0f;
    }
    uint32_t b = 0;
#pragma unroll
    for (int i = 0; i < 5; i++) {
        const uint64_t e = (uint64_t)i * P + j;
        const float u = __fadd_rn(ev[i], tv[i]);            // step (1)
        const int q = Q.q(u);                                // Eq. 2
        if (e < n) __stcs(err + e, Q.residual(u, q));       // steps (a),(b)
        b = b * 3u + (e < n ? (uint32_t)(q + 1) : 0u);       // steps 1,4,6 (pad digit 0)
    }
    return b;
}

// One group of 4 consecutive quartic positions 4g..4g+3 whose 20 elements all
// exist: one float4 of t and of err per partition.
template <class QT, int LP = 0>
__device__ __forceinline__ void quant_qe_group(const float4 *__restrict__ t4, float4 *__restrict__ e4,
                                               uint32_t *__restrict__ b4, uint64_t P4, uint64_t g,
                                               const QT &Q, uint64_t pol = 0) {
    float4 tv[5], ev[5];
#pragma unroll
    for (int i = 0; i < 5; i++) {
        tv[i] = ldq4<LP>(t4 + g + i * P4, pol);
        ev[i] = ldq4<LP>(e4 + g + i * P4, pol);
    }
    uint32_t by[4] = {0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < 5; i++) {
        float r[4];
        const float tt[4] = {tv[i].x, tv[i].y, tv[i].z, tv[i].w};
        const float ee[4] = {ev[i].x, ev[i].y, ev[i].z, ev[i].w};
#pragma unroll
        for (int c = 0; c < 4; c++) {
            const float u = __fadd_rn(ee[c], tt[c]);        // step (1)
            const int q = Q.q(u);                            // Eq. 2
            r[c] = Q.residual(u, q);                         // steps (a),(b)
            by[c] = by[c] * 3u + (uint32_t)(q + 1);          // steps 1, 6
        }
        __stcs(e4 + g + i * P4, make_float4(r[0], r[1], r[2], r[3]));
    }
    b4[g] = by[0] | (by[1] << 8) | (by[2] << 16) | (by[3] << 24);
}

// Four quartic positions j + 256k (k = 0..3), any alignment: all 40 loads are
// issued before any arithmetic so that 160 bytes per thread are in flight.
template <class QT, int LP = 0>
__device__ __forceinline__ void quant_qe_four(const float *__restrict__ t, float *__restrict__ err, uint64_t n,
                                              uint64_t P, uint64_t j, uint64_t jend, uint8_t *__restrict__ bytes,
                                              const QT &Q, uint64_t pol = 0) {
    float tv[4][5], ev[4][5];
#pragma unroll
    for (int k = 0; k < 4; k++) {
        const uint64_t jj = j + (uint64_t)k * kK2Threads;
#pragma unroll
        for (int i = 0; i < 5; i++) {
            const uint64_t e = (uint64_t)i * P + jj;
            const bool ok = jj < jend && e < n;
            tv[k][i] = ok ? ldq<LP>(t + e, pol) : 0.0f;
            ev[k][i] = ok ? ldq<LP>(err + e, pol) : 0.0f;
        }
    }
#pragma unroll
    for (int k = 0; k < 4; k++) {
        const uint64_t jj = j + (uint64_t)k * kK2Threads;
        if (jj >= jend) break;
        uint32_t b = 0;
#pragma unroll
        for (int i = 0; i < 5; i++) {
            const uint64_t e = (uint64_t)i * P + jj;
            const float u = __fadd_rn(ev[k][i], tv[k][i]);      // step (1)
            const int q = Q.q(u);                                // Eq. 2
            if (e < n) __stcs(err + e, Q.residual(u, q));       // steps (a),(b)
            b = b * 3u + (e < n ? (uint32_t)(q + 1) : 0u);       // steps 1,4,6 (pad digit 0)
        }
        bytes[jj] = (uint8_t)b;
    }
}

template <class QT, int LP = 0>
__device__ __forceinline__ void quant_qe_tile(const Seg &S, uint8_t *bytes, uint64_t j0, uint64_t t2, const QT &Q,
                                              uint64_t pol = 0) {
    const uint64_t P = S.P, n = S.n;
    const uint64_t jend = tmin<uint64_t>(P, j0 + t2);
    if (S.flags & kSegVec2) {
        // groups g with 4P + 4g + 3 < n are complete in all five partitions
        const uint64_t full = n >= 4 * P + 3 ? tmin<uint64_t>(P / 4, (n - 4 * P) / 4) : 0;
        const uint64_t g0 = j0 / 4, g1 = tmax<uint64_t>(g0, tmin<uint64_t>(jend / 4, full));
        const float4 *t4 = reinterpret_cast<const float4 *>(S.t);
        float4 *e4 = reinterpret_cast<float4 *>(S.err);
        uint32_t *b4 = reinterpret_cast<uint32_t *>(bytes);
        for (uint64_t g = g0 + threadIdx.x; g < g1; g += kK2Threads)
            quant_qe_group<QT, LP>(t4, e4, b4, P / 4, g, Q, pol);
        for (uint64_t j = 4 * g1 + threadIdx.x; j < jend; j += kK2Threads)
            bytes[j] = (uint8_t)quant_qe_one<QT, LP>(S.t, S.err, n, P, j, Q, pol);
    } else {
        for (uint64_t j = j0 + threadIdx.x; j < jend; j += 4 * kK2Threads)
            quant_qe_four<QT, LP>(S.t, S.err, n, P, j, jend, bytes, Q, pol);
    }
}

#ifndef TLC_K2_MINB
#define TLC_K2_MINB 2
#endif
__global__ void __launch_bounds__(kK2Threads, TLC_K2_MINB)
tlc_quant_qe_kernel(const SegTable T, const unsigned int *maxkey, float s, int use_zre,
                    uint8_t *__restrict__ scratch, uint64_t tile_begin, int skip_bulk) {
    __shared__ uint64_t s_first[kSegCache];
    pdl_trigger();
    seg_index_load<2>(T, s_first);
    pdl_wait();                                          // K1's max keys (or the bulk kernel's tiles)
    // skip_bulk: the bulk kernel took the tiles of T.bulk_list; this kernel takes T.rest_list
    const uint64_t nwork = skip_bulk ? T.n_rest : T.n2 - tile_begin;
    for (uint64_t w = blockIdx.x; w < nwork; w += gridDim.x) {
        const uint64_t tile = skip_bulk ? T.rest_list[w] : tile_begin + w;
        const int si = find_seg_c<2>(T, tile, s_first);
        const Seg S = get_seg(T, si);
        float M;
        const unsigned int status = scale_from_key(maxkey[si], s, M);   // Eq. 1, R6
        const uint64_t lt = tile - S.k2;
        if (lt == 0 && threadIdx.x == 0) {
            tlc_header *h = S.hdr;
            h->M = M;
            h->flags = use_zre ? TLC_FLAG_ZRE : 0u;
            h->n = S.n;
            h->payload_len = (status == TLC_OK && !use_zre) ? S.P : 0;   // ZRE: set by K3
            h->status = status;
            h->reserved = 0;
        }
        if (status != TLC_OK) continue;                  // err untouched (R6)
        uint8_t *bytes = use_zre ? scratch + S.bytes_off : S.payload;
        const Quant Q(M);
        if (Q.mode == 1) quant_qe_tile(S, bytes, lt * T.sz.t2, T.sz.t2, QuantCmp(Q));   // uniform branch
        else quant_qe_tile(S, bytes, lt * T.sz.t2, T.sz.t2, Q);
    }
}

// ---- K2 bulk path: the same computation on tiles staged in shared memory by the
// Blackwell bulk-copy (TMA) engine.  One CTA per SM keeps kBulkStages tiles of
// t and err (10 contiguous 4 KiB partition segments each) in flight behind
// mbarrier transaction counts, so the memory system never waits for a thread;
// threads read their four positions per partition with 128-bit shared loads
// and store err and the quartic bytes straight to global memory.  Used for the
// complete tiles of a single aligned tensor (P % 4 == 0); the ragged tail and
// tensor batches go through tlc_quant_qe_kernel.
constexpr int kBulkPos = 1024;                                   // quartic positions per tile
#ifndef TLC_K2_STAGES
#define TLC_K2_STAGES 4                                  // 5 measured slower (C3 K2 0.518 -> 0.523 ms)
#endif
constexpr int kBulkStages = TLC_K2_STAGES;
constexpr int kBulkRow = kBulkPos + 4;                          // + up to 3 leading elements (alignment)
constexpr uint32_t kBulkPart = kBulkPos * 4;                     // bytes per partition segment
constexpr uint32_t kBulkPartU = kBulkRow * 4;                    // ... of an unaligned partition (superset)

// A stage holds the ten partition segments (t, err) back to back, kBulkPos floats apart for
// aligned partitions and kBulkRow apart for supersets (row(i) below).
struct BulkSmem {
    float buf[kBulkStages][10 * kBulkRow];
    unsigned long long bar[kBulkStages];
};

// kAligned: P % 4 == 0, every partition segment starts 16-byte aligned.  Otherwise the
// copy engine fetched the aligned superset starting sh_i = (i P) mod 4 elements early:
// shared reads are scalar at offset sh_i and err goes back with 32-bit stores.
template <bool kAligned, class QT>
__device__ __forceinline__ void bulk_compute(const float *buf, float *err, uint64_t P, uint64_t j0,
                                             uint8_t *bytes, const QT &Q) {
    const int g = threadIdx.x;                       // group: positions j0 + 4g .. j0 + 4g + 3
    uint32_t by[4] = {0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < 5; i++) {
        const int sh = kAligned ? 0 : (int)(((uint64_t)i * P) & 3);
        float tt[4], ee[4];
        if (kAligned) {
            const float4 tv = *reinterpret_cast<const float4 *>(&buf[i * kBulkPos + 4 * g]);
            const float4 ev = *reinterpret_cast<const float4 *>(&buf[(5 + i) * kBulkPos + 4 * g]);
            tt[0] = tv.x; tt[1] = tv.y; tt[2] = tv.z; tt[3] = tv.w;
            ee[0] = ev.x; ee[1] = ev.y; ee[2] = ev.z; ee[3] = ev.w;
        } else {
#pragma unroll
            for (int c = 0; c < 4; c++) {
                tt[c] = buf[i * kBulkRow + sh + 4 * g + c];
                ee[c] = buf[(5 + i) * kBulkRow + sh + 4 * g + c];
            }
        }
        float r[4];
#pragma unroll
        for (int c = 0; c < 4; c++) {
            const float u = __fadd_rn(ee[c], tt[c]);        // step (1)
            const int q = Q.q(u);                            // Eq. 2
            r[c] = Q.residual(u, q);                         // steps (a),(b)
            by[c] = by[c] * 3u + (uint32_t)(q + 1);          // steps 1, 6
        }
        if (kAligned) {
            __stcs(reinterpret_cast<float4 *>(err + (uint64_t)i * P + j0 + 4 * g), make_float4(r[0], r[1], r[2], r[3]));
        } else {                                     // 32-bit stores (a lane-shuffled realignment
            float *eo = err + (uint64_t)i * P + j0 + 4 * g;   // to 16-byte stores measured slower)
#pragma unroll
            for (int c = 0; c < 4; c++) __stcs(eo + c, r[c]);
        }
    }
    reinterpret_cast<uint32_t *>(bytes + j0)[g] = by[0] | (by[1] << 8) | (by[2] << 16) | (by[3] << 24);
}

template <bool kAligned>                                // P % 4 == 0: no superset, no shifts
__global__ void __launch_bounds__(kK2Threads, 1)
tlc_quant_qe_bulk_kernel(const SegTable T, const unsigned int *maxkey, float s, int use_zre,
                         uint8_t *__restrict__ scratch, uint64_t nbulk) {
    static_assert(kBulkPos == 4 * kK2Threads, "one group of four positions per thread");
    extern __shared__ __align__(128) uint8_t smem_raw[];
    BulkSmem &sm = *reinterpret_cast<BulkSmem *>(smem_raw);
    pdl_trigger();
    if (threadIdx.x == 0) {                              // barrier setup overlaps K1's tail
        for (int st = 0; st < kBulkStages; st++) mbar_init(&sm.bar[st], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    pdl_wait();                                          // K1's max keys
    const Seg S = T.one;
    float M;
    const unsigned int status = scale_from_key(maxkey[0], s, M);   // Eq. 1, R6
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        tlc_header *h = S.hdr;
        h->M = M;
        h->flags = use_zre ? TLC_FLAG_ZRE : 0u;
        h->n = S.n;
        h->payload_len = (status == TLC_OK && !use_zre) ? S.P : 0;
        h->status = status;
        h->reserved = 0;
    }
    if (status != TLC_OK) return;
    uint8_t *bytes = use_zre ? scratch + S.bytes_off : S.payload;
    const uint64_t P = S.P;
    const uint64_t mine = nbulk > blockIdx.x ? (nbulk - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    __syncthreads();
    constexpr uint32_t part = kAligned ? kBulkPart : kBulkPartU;
    constexpr int row = kAligned ? kBulkPos : kBulkRow;
    auto issue = [&](uint64_t k) {
        const int st = (int)(k % kBulkStages);
        const uint64_t j0 = (blockIdx.x + k * gridDim.x) * (uint64_t)kBulkPos;
        mbar_expect_tx(&sm.bar[st], 10 * part);
#pragma unroll
        for (int i = 0; i < 5; i++) {
            const uint64_t a = kAligned ? (uint64_t)i * P + j0 : ((uint64_t)i * P + j0) & ~uint64_t(3);
            bulk_load(&sm.buf[st][i * row], S.t + a, part, &sm.bar[st]);
            bulk_load(&sm.buf[st][(5 + i) * row], S.err + a, part, &sm.bar[st]);
        }
    };
    if (threadIdx.x == 0)
        for (uint64_t k = 0; k < mine && k < kBulkStages; k++) issue(k);
    const Quant Q(M);
    for (uint64_t k = 0; k < mine; k++) {
        const int st = (int)(k % kBulkStages);
        mbar_wait(&sm.bar[st], (uint32_t)((k / kBulkStages) & 1));
        const uint64_t j0 = (blockIdx.x + k * gridDim.x) * (uint64_t)kBulkPos;
        if (Q.mode == 1) bulk_compute<kAligned>(sm.buf[st], S.err, P, j0, bytes, QuantCmp(Q));
        else bulk_compute<kAligned>(sm.buf[st], S.err, P, j0, bytes, Q);
        __syncthreads();                                 // every thread is done with this stage
        if (threadIdx.x == 0 && k + kBulkStages < mine) issue(k + kBulkStages);
    }
}

// The bulk kernel over a segment table: work item q is bulk tile q % kBulkPer of K2 tile
// list[q / kBulkPer] (tiles of kLargeItems.t2 positions, chosen on the host by
// bulk_tile_ok; tlc_quant_qe_kernel skips them).
// Thread 0 resolves each item's segment when it issues the copies and leaves what the
// compute needs in shared memory for that stage.  Everything on that thread's per-item path
// is shared-memory reads and shifts: the other warps wait for it at the stage barrier.
struct BulkItem {
    float *err;
    uint8_t *bytes;                                      // quartic bytes: payload or ZRE scratch
    tlc_header *hdr;
    uint64_t n, P, j0;
    float M;
    unsigned int status;
    int first;
};
constexpr uint64_t kBulkT2 = kLargeItems.t2;             // the launch requires T.sz.t2 == kBulkT2
constexpr uint32_t kBulkPer = (uint32_t)(kBulkT2 / kBulkPos);   // bulk tiles per K2 tile
static_assert(kBulkT2 % kBulkPos == 0, "K2 tile of whole bulk tiles");
// K2 tiles of a CTA's contiguous run of items held in shared memory (BERT-large: ~111 per
// CTA), loaded before K1 finishes: the per-item list read from global memory was a dependent
// load on every item's critical path (0.78 -> 0.73 ms per BERT-large K2)
constexpr int kBulkTileCache = 1024;

// TLC_K2T_WS (default; -DTLC_K2T_NO_WS for the single-role kernel): a ninth (producer) warp
// issues the copies; consumers release a stage by arriving on its `empty` mbarrier instead of
// a block barrier, so they never wait for the issuing thread (40 % of the stall samples were
// at that barrier: BERT-large W = 1 K2 1.415 -> 1.368 ms per step, tools/k2t_ws_check.sh).
#if !defined(TLC_K2T_WS) && !defined(TLC_K2T_NO_WS)
#define TLC_K2T_WS 1
#endif
#ifdef TLC_K2T_WS
constexpr int kK2TThreads = kK2Threads + 32;
#else
constexpr int kK2TThreads = kK2Threads;
#endif
__global__ void __launch_bounds__(kK2TThreads, 1)
tlc_quant_qe_bulk_table_kernel(const SegTable T, const unsigned int *maxkey, float s, int use_zre,
                               uint8_t *__restrict__ scratch) {
    extern __shared__ __align__(128) uint8_t smem_raw[];
    BulkSmem &sm = *reinterpret_cast<BulkSmem *>(smem_raw);
    __shared__ BulkItem s_item[kBulkStages];
    __shared__ uint64_t s_first[kSegCache];
    __shared__ uint64_t s_tiles[kBulkTileCache];
#ifdef TLC_K2T_WS
    __shared__ unsigned long long s_empty[kBulkStages];
#endif
    pdl_trigger();
    if (threadIdx.x == 0) {
        for (int st = 0; st < kBulkStages; st++) mbar_init(&sm.bar[st], 1);
#ifdef TLC_K2T_WS
        for (int st = 0; st < kBulkStages; st++) mbar_init(&s_empty[st], kK2Threads / 32);
#endif
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // a CTA takes a contiguous run of items, so consecutive items mostly share a segment and
    // thread 0 re-reads the segment's descriptor and max key only when it changes
    const uint64_t nitems = kBulkPer * T.n_bulk;
    const uint64_t chunk = (nitems + gridDim.x - 1) / gridDim.x;
    const uint64_t q0 = blockIdx.x * chunk;
    const uint64_t mine = q0 < nitems ? tmin<uint64_t>(chunk, nitems - q0) : 0;
    const uint64_t tl0 = q0 / kBulkPer;                  // first list entry of the run
    const uint64_t ntl = mine ? (q0 + mine - 1) / kBulkPer - tl0 + 1 : 0;
    for (uint64_t i = threadIdx.x; i < ntl && i < kBulkTileCache; i += blockDim.x) s_tiles[i] = T.bulk_list[tl0 + i];
    seg_index_load<2>(T, s_first);                       // (ends with __syncthreads)
    pdl_wait();                                          // K1's max keys
    uint64_t cur_k2 = 1, cur_end = 0;                    // K2 tiles [cur_k2, cur_end) of the current segment
    BulkItem cur{};
    const float *cur_t = nullptr;
    auto issue = [&](uint64_t k) {                       // thread 0
        const int st = (int)(k % kBulkStages);
        const uint64_t q = q0 + k;
        const uint64_t e = q / kBulkPer - tl0;
        const uint64_t tile = e < kBulkTileCache ? s_tiles[e] : T.bulk_list[q / kBulkPer];
        if (tile < cur_k2 || tile >= cur_end) {          // segment change: global reads
            const int si = find_seg_c<2>(T, tile, s_first);
            const Seg S = get_seg(T, si);
            cur_t = S.t;
            cur.err = S.err;
            cur.bytes = use_zre ? scratch + S.bytes_off : S.payload;
            cur.hdr = S.hdr;
            cur.n = S.n;
            cur.P = S.P;
            cur.status = scale_from_key(maxkey[si], s, cur.M);   // Eq. 1, R6
            cur_k2 = S.k2;
            cur_end = S.k2 + (S.P + kBulkT2 - 1) / kBulkT2;
        }
        const uint64_t lt = tile - cur_k2;
        cur.j0 = lt * kBulkT2 + (q % kBulkPer) * (uint64_t)kBulkPos;
        cur.first = lt == 0 && (q % kBulkPer) == 0;
        s_item[st] = cur;
        const uint64_t P = cur.P;
        const uint32_t part = (P & 3) == 0 ? kBulkPart : kBulkPartU;
        const int row = (P & 3) == 0 ? kBulkPos : kBulkRow;
        mbar_expect_tx(&sm.bar[st], 10 * part);
#pragma unroll
        for (int i = 0; i < 5; i++) {
            const uint64_t a = ((uint64_t)i * P + cur.j0) & ~uint64_t(3);   // 16-byte aligned start
            bulk_load(&sm.buf[st][i * row], cur_t + a, part, &sm.bar[st]);
            bulk_load(&sm.buf[st][(5 + i) * row], cur.err + a, part, &sm.bar[st]);
        }
    };
#ifdef TLC_K2T_WS
    if (threadIdx.x >= kK2Threads) {                     // producer warp
        if (threadIdx.x == kK2Threads)
            for (uint64_t k = 0; k < mine; k++) {
                if (k >= kBulkStages)                    // consumers released the stage's last use
                    mbar_wait(&s_empty[k % kBulkStages], (uint32_t)(((k / kBulkStages) - 1) & 1));
                issue(k);
            }
        return;
    }
#else
    if (threadIdx.x == 0)
        for (uint64_t k = 0; k < mine && k < kBulkStages; k++) issue(k);
#endif
    for (uint64_t k = 0; k < mine; k++) {
        const int st = (int)(k % kBulkStages);
        mbar_wait(&sm.bar[st], (uint32_t)((k / kBulkStages) & 1));
        const BulkItem &it = s_item[st];
        const float M = it.M;
        const unsigned int status = it.status;
        if (it.first && threadIdx.x == 0) {
            tlc_header *h = it.hdr;
            h->M = M;
            h->flags = use_zre ? TLC_FLAG_ZRE : 0u;
            h->n = it.n;
            h->payload_len = (status == TLC_OK && !use_zre) ? it.P : 0;
            h->status = status;
            h->reserved = 0;
        }
        if (status == TLC_OK) {                          // else err untouched (R6)
            const Quant Q(M);
            if ((it.P & 3) == 0) {
                if (Q.mode == 1) bulk_compute<true>(sm.buf[st], it.err, it.P, it.j0, it.bytes, QuantCmp(Q));
                else bulk_compute<true>(sm.buf[st], it.err, it.P, it.j0, it.bytes, Q);
            } else {
                if (Q.mode == 1) bulk_compute<false>(sm.buf[st], it.err, it.P, it.j0, it.bytes, QuantCmp(Q));
                else bulk_compute<false>(sm.buf[st], it.err, it.P, it.j0, it.bytes, Q);
            }
        }
#ifdef TLC_K2T_WS
        __syncwarp();                                    // the warp is done with this stage
        if ((threadIdx.x & 31) == 0)
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(&s_empty[st])) : "memory");
#else
        __syncthreads();                                 // every thread is done with this stage
        if (threadIdx.x == 0 && k + kBulkStages < mine) issue(k + kBulkStages);
#endif
    }
}

// ============================================================== K12
// K1 and K2 fused for tables of several tensors (the exchange's push and pull tables, BERT-
// large's 150 tensors): one persistent launch takes work items in order from a counter; the
// host list (k12_plan_build) interleaves the max tiles (K1) and the quantize tiles (K2) of
// consecutive windows of tensors of <= ~32 MB of t + err: K1(w0) K1(w1) K2(w0) K1(w2) K2(w1)
// ...  A window's K2 tiles then re-read t and err while they are still in the 126 MB L2
// (K1 of the next window is the only traffic in between), so HBM sees 12n + P/5 per
// compress instead of K1's 8n plus K2's 12n + P/5.  A quantize item waits (one thread,
// acquire load) until every max item of its tensor has folded its key; max items never
// wait, and every item waits only on items dispensed before it, so the smallest unfinished
// item can always run: no deadlock.  Same tiles, keys and arithmetic as K1 + K2: the same
// bits.
constexpr int kK12Threads = 256;
static_assert(kK12Threads == kK2Threads, "the quantize items run K2's tile code");

// L2 policy of the max items' loads: 0 normal (default), 1 evict_last through a cache-policy
// operand (A/B, TLC_K12_HINT=1)
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
template <int HINT>
__device__ __forceinline__ float4 ld_keep4(const float4 *p, uint64_t pol) {
    float4 v;
    if (HINT >= 1)
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                     : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "l"(pol));
    else
        asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}
template <int HINT>
__device__ __forceinline__ float ld_keep(const float *p, uint64_t pol) {
    float v;
    if (HINT >= 1)
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
    else asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}

// max key of the elements of K2 tile [j0, j0 + t2) (all five partitions).  The tile's part of
// partition i is the run [i P + j0, i P + jend) of the flat arrays: aligned float4 groups
// covering it (elements outside the run masked out: the key is a max, so any cover works),
// all five runs' loads in flight together.
template <int HINT>
__device__ __forceinline__ unsigned int absmax_tile(const Seg &S, uint64_t j0, uint64_t t2) {
    const uint64_t P = S.P, n = S.n;
    const uint64_t jend = tmin<uint64_t>(P, j0 + t2);
    unsigned int m = 0;
    const uint64_t pol = HINT >= 1 ? policy_evict_last() : 0;
    if (S.flags & kSegVec1) {
        const float4 *t4 = reinterpret_cast<const float4 *>(S.t);
        const float4 *e4 = reinterpret_cast<const float4 *>(S.err);
        uint64_t lo[5], hi[5], g0[5];
        uint32_t ng = 0;
#pragma unroll
        for (int i = 0; i < 5; i++) {
            lo[i] = tmin<uint64_t>(n, (uint64_t)i * P + j0);
            hi[i] = tmin<uint64_t>(n, (uint64_t)i * P + jend);
            g0[i] = lo[i] / 4;
            ng = max(ng, (uint32_t)(hi[i] / 4 > g0[i] ? hi[i] / 4 - g0[i] : 0));
        }
        // whole float4 inside [4 g0, hi) (the head's extra elements masked), then the tail
        // elements past the last whole float4 (< 4 per partition) one by one
        if (threadIdx.x < 20) {
            const int i = threadIdx.x >> 2;
            const uint64_t l = i == 0 ? lo[0] : i == 1 ? lo[1] : i == 2 ? lo[2] : i == 3 ? lo[3] : lo[4];
            const uint64_t h = i == 0 ? hi[0] : i == 1 ? hi[1] : i == 2 ? hi[2] : i == 3 ? hi[3] : hi[4];
            const uint64_t e = h / 4 * 4 + (threadIdx.x & 3);
            if (e >= l && e < h) m = max(m, absmax_key(ld_keep<HINT>(S.t + e, pol), ld_keep<HINT>(S.err + e, pol)));
        }
        for (uint32_t k = threadIdx.x; k < ng; k += kK12Threads) {
            float4 tv[5], ev[5];
#pragma unroll
            for (int i = 0; i < 5; i++) {
                const uint64_t g = g0[i] + k;
                const bool ok = g < hi[i] / 4;
                tv[i] = ok ? ld_keep4<HINT>(t4 + g, pol) : make_float4(0.f, 0.f, 0.f, 0.f);
                ev[i] = ok ? ld_keep4<HINT>(e4 + g, pol) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int i = 0; i < 5; i++) {
                const uint64_t e = 4 * (g0[i] + k);
                const float tt[4] = {tv[i].x, tv[i].y, tv[i].z, tv[i].w};
                const float ee[4] = {ev[i].x, ev[i].y, ev[i].z, ev[i].w};
#pragma unroll
                for (int c = 0; c < 4; c++)
                    if (e + c >= lo[i] && e + c < hi[i]) m = max(m, absmax_key(tt[c], ee[c]));
            }
        }
        return m;
    }
    for (uint64_t j = j0 + threadIdx.x; j < jend; j += kK12Threads) {
        float tv[5], ev[5];
#pragma unroll
        for (int i = 0; i < 5; i++) {
            const uint64_t e = (uint64_t)i * P + j;
            tv[i] = e < n ? ld_keep<HINT>(S.t + e, pol) : 0.0f;
            ev[i] = e < n ? ld_keep<HINT>(S.err + e, pol) : 0.0f;
        }
#pragma unroll
        for (int i = 0; i < 5; i++) m = max(m, absmax_key(tv[i], ev[i]));   // pads: key 0
    }
    return m;
}

template <int HINT>
__global__ void __launch_bounds__(kK12Threads, 2)
tlc_absmax_quant_kernel(const SegTable T, unsigned int *__restrict__ maxkey, unsigned int *__restrict__ done,
                        Ctrl *ctrl, float s, int use_zre, uint8_t *__restrict__ scratch) {
    __shared__ uint64_t s_first[kSegCache];
    __shared__ unsigned int s_red[kK12Threads / 32];
    __shared__ uint32_t s_it[2];
    __shared__ unsigned int s_key;
    extern __shared__ __align__(128) float s_buf[];             // 2 stages of 10 superset rows (bulk copies)
    __shared__ __align__(8) unsigned long long s_bar[2];
    uint32_t bphase = 0;                                          // the stages' mbarrier phases (CTA-uniform)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        s_it[0] = (uint32_t)atomicAdd(&ctrl->k12_counter, 1ull);
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    seg_index_load<2>(T, s_first);                          // (ends with a block barrier)
    for (int b = 0;; b ^= 1) {
        const uint32_t it = s_it[b];
        if (it >= T.k12_n) break;
        if (threadIdx.x == 0) s_it[b ^ 1] = (uint32_t)atomicAdd(&ctrl->k12_counter, 1ull);   // the next, early
        const uint32_t item = T.k12[it];
        const uint64_t tile = item >> 1;
        const int si = find_seg_c<2>(T, tile, s_first);
        const Seg S = get_seg(T, si);
        const uint64_t lt = tile - S.k2;
        if ((item & 1u) == 0) {
            // ---- K1 on this tile: max of bits(u) & 0x7fffffff, folded into the tensor's key
            unsigned int m = absmax_tile<HINT>(S, lt * T.sz.t2, T.sz.t2);
            m = __reduce_max_sync(0xffffffffu, m);
            if (lane == 0) s_red[warp] = m;
            __syncthreads();
            if (warp == 0) {
                m = __reduce_max_sync(0xffffffffu, lane < kK12Threads / 32 ? s_red[lane] : 0u);
                if (lane == 0) {
                    atomicMax(maxkey + si, m);
                    __threadfence();                        // the key before the count (release)
                    atomicAdd(done + si, 1u);
                }
            }
        } else {
            // ---- K2 on this tile once every max tile of the tensor is in
            if (threadIdx.x == 0) {
                const unsigned int need = (unsigned int)((S.P + T.sz.t2 - 1) / T.sz.t2);
                while (ld_acquire_u32(done + si) < need) __nanosleep(64);
                s_key = ld_relaxed_u32(maxkey + si);
            }
            __syncthreads();
            float M;
            const unsigned int status = scale_from_key(s_key, s, M);   // Eq. 1, R6
            if (lt == 0 && threadIdx.x == 0) {
                tlc_header *h = S.hdr;
                h->M = M;
                h->flags = use_zre ? TLC_FLAG_ZRE : 0u;
                h->n = S.n;
                h->payload_len = (status == TLC_OK && !use_zre) ? S.P : 0;   // ZRE: set by K3
                h->status = status;
                h->reserved = 0;
            }
            if (status == TLC_OK) {                          // else err untouched (R6)
                uint8_t *bytes = use_zre ? scratch + S.bytes_off : S.payload;
                const Quant Q(M);
                constexpr int LP = HINT == 2 ? 1 : 0;
                const uint64_t pol = LP ? policy_evict_first() : 0;
                const uint64_t j0 = lt * T.sz.t2, jend = tmin<uint64_t>(S.P, j0 + T.sz.t2);
                if (!(S.flags & kSegVec2) && (S.flags & kSegVec1) && (use_zre || aligned4(S.payload))) {
                    // partitions not aligned to each other: the bulk-copy engine stages each
                    // 1024-position sub-tile's ten rows as 16-byte aligned supersets (two stages,
                    // the next sub-tile in flight while this one is quantized), then K2's bulk
                    // compute; a sub-tile whose superset would cross the tensor's end goes
                    // through the register path
                    const uint64_t P = S.P, n = S.n;
                    const int nsub = (int)((jend - j0 + kBulkPos - 1) / kBulkPos);
                    auto whole = [&](int k) {
                        const uint64_t js = j0 + (uint64_t)k * kBulkPos;
                        return js + kBulkPos <= P && ((4 * P + js) & ~uint64_t(3)) + kBulkRow <= n;
                    };
                    auto issue = [&](int k) {                    // thread 0
                        const int st = k & 1;
                        const uint64_t js = j0 + (uint64_t)k * kBulkPos;
                        mbar_expect_tx(&s_bar[st], 10 * kBulkPartU);
#pragma unroll
                        for (int i = 0; i < 5; i++) {
                            const uint64_t a = ((uint64_t)i * P + js) & ~uint64_t(3);
                            bulk_load(s_buf + (size_t)st * 10 * kBulkRow + i * kBulkRow, S.t + a, kBulkPartU, &s_bar[st]);
                            bulk_load(s_buf + (size_t)st * 10 * kBulkRow + (5 + i) * kBulkRow, S.err + a, kBulkPartU,
                                      &s_bar[st]);
                        }
                    };
                    if (threadIdx.x == 0)
                        for (int k = 0; k < 2 && k < nsub; k++)
                            if (whole(k)) issue(k);
                    for (int k = 0; k < nsub; k++) {
                        const int st = k & 1;
                        const uint64_t js = j0 + (uint64_t)k * kBulkPos;
                        if (whole(k)) {
                            mbar_wait(&s_bar[st], (bphase >> st) & 1u);
                            bphase ^= 1u << st;
                            const float *buf = s_buf + (size_t)st * 10 * kBulkRow;
                            if (Q.mode == 1) bulk_compute<false>(buf, S.err, P, js, bytes, QuantCmp(Q));
                            else bulk_compute<false>(buf, S.err, P, js, bytes, Q);
                        } else {
                            if (Q.mode == 1) quant_qe_tile<QuantCmp, LP>(S, bytes, js, kBulkPos, QuantCmp(Q), pol);
                            else quant_qe_tile<Quant, LP>(S, bytes, js, kBulkPos, Q, pol);
                        }
                        __syncthreads();                         // the stage is free again
                        if (threadIdx.x == 0 && k + 2 < nsub && whole(k + 2)) issue(k + 2);
                    }
                } else {
                    if (Q.mode == 1) quant_qe_tile<QuantCmp, LP>(S, bytes, j0, T.sz.t2, QuantCmp(Q), pol);
                    else quant_qe_tile<Quant, LP>(S, bytes, j0, T.sz.t2, Q, pol);
                }
            }
        }
        __syncthreads();                                     // s_it[b ^ 1], s_red, s_key
    }
}

// ============================================================== K3
// Chunked single-pass scan over chunks of kCH3 quartic bytes, numbered globally
// segment after segment and taken in order from an atomic counter.  Each chunk
// is split into one sub-range per warp.
//   phase 1  each warp folds its sub-range (rows of 32 lanes x 32 bytes, each
//            lane's bytes reduced to a literal bit mask) into a run summary; the
//            CTA publishes the composition of its 8 warps;
//   phase 2  it composes the summaries of the segment's preceding chunks (taken
//            earlier, never waiting on a later one: no deadlock) -> carry-in;
//   phase 3  each warp re-reads its sub-range (L2-resident) and writes every ZRE
//            byte at its final offset; the segment's last chunk writes the length.
#ifdef TLC_K3_TRACE
// development instrumentation: %globaltimer at phase boundaries of every K3 chunk
__device__ unsigned long long g_k3_trace[1 << 14][8];
__device__ unsigned long long g_k3_cta[4096][2];           // per CTA: entry, exit
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define K3_TRACE(id, slot) \
    do { if ((threadIdx.x & 31) == 0 && (id) < (1u << 14)) g_k3_trace[(id)][slot] = gtimer(); } while (0)
#else
#define K3_TRACE(id, slot) do {} while (0)
#endif

constexpr int kK3Workers = kScanWarps;                       // warps scanning the chunk
constexpr int kK3LookWarp = kK3Workers;                      // + one warp for the look-back
constexpr int kK3Threads = 32 * (kK3Workers + 1);
constexpr int kK3Seg = 32;                                   // bytes per lane per row
constexpr int kK3WarpRow = 32 * kK3Seg;                      // 1 KiB per warp row

// true if the lane's 32 bytes are all 121 (padding included)
__device__ __forceinline__ bool plain_lane(const uint32_t (&w)[8]) {
    uint32_t x = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) x |= w[k] ^ 0x79797979u;
    return x == 0;
}

constexpr int kK3RowsPerWarp = (int)(kLargeItems.c3 / kScanWarps / kK3WarpRow);   // rows of a sub-range
static_assert(kT5 % kK3WarpRow == 0 && kLargeItems.c3 % kT5 == 0 && kSmallItems.c3 % kT5 == 0,
              "K5 tile starts are warp-row starts (K3 writes the producer seek entries there)");
#ifndef TLC_K3_LITCAP
#define TLC_K3_LITCAP 512
#endif
constexpr int kK3LitCap = TLC_K3_LITCAP;   // list entries a warp keeps per chunk between phases 1 and 3
constexpr uint32_t kRowNotKept = 1u << 31;

// K3 is software-pipelined over the chunks a CTA takes: phase 1 of chunk j runs
// while the look-back warp resolves the carry-in of the previous chunk i, whose
// phase 3 then works from its kept literal lists alone (the chunk buffer already
// holds j).  A kept entry of literal k of a row: the literal byte (bits 8-15)
// and, for k > 0, the flush code remainder R_k % 14 (bits 0-3) and the output
// offset relative to the end of literal 0's bytes (bits 16-31); literal 0's
// position is in the row's metadata, its bytes depend on the row's carry.
constexpr uint32_t kK3Stage = (uint32_t)(kLargeItems.c3 / kK3Workers);   // phase-3 stage per warp
static_assert(kK3Stage >= pad_stage_bytes(kK3WarpRow + 1 + 3), "a row's output (<= row + 1 bytes) fits the stage");
struct K3Smem {
    uint8_t chunk[kLargeItems.c3];                       // the chunk's quartic bytes; phase-3 stages
    uint32_t lit[2][kScanWarps][kK3LitCap];               // literal lists, row after row
    uint4 rowmeta[2][kScanWarps][kK3RowsPerWarp];         // (L | base << 16, rest | cout << 16, p0, -)
    unsigned long long bar;
};

// Literal list of a warp row held as 32 bytes per lane: the row positions of
// its bytes != 121 in ascending order, written to lit[0..L) if L <= cap
// (load_seg_s pads with 121, so positions past the end of the data are clear).
// Returns L in all lanes.
__device__ __forceinline__ uint32_t row_literals(const uint32_t (&w)[8], uint32_t *lit, uint32_t cap,
                                                 bool &stored) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t mask = literal_mask(w);
    const uint32_t nl = popc32(mask);
    uint32_t b = nl;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, b, d);
        if (lane >= d) b += y;
    }
    const uint32_t L = __shfl_sync(0xffffffffu, b, 31);
    stored = L <= cap;
    if (stored) {
        b -= nl;
        for (uint32_t m = mask; m; m &= m - 1u) lit[b++] = kK3Seg * lane + ctz32(m);
    }
    __syncwarp();
    return L;
}

// ZRE bytes of a literal preceded by R zero groups: R/14 full
// chunks, one flush code if R % 14 > 0, the literal itself.
__device__ __forceinline__ uint32_t lit_cost(uint32_t R) { return R / kMaxRun + (R % kMaxRun != 0) + 1u; }

// Load [pos, min(pos+32, hi)) from global memory as 8 words, padding with 121.  A full
// 16-byte-aligned segment takes two 16-byte loads (byte loads from lanes 32 bytes apart
// touched 32 sectors per instruction).
__device__ __forceinline__ int load_seg_g(const uint8_t *bytes, uint64_t pos, uint64_t hi, uint32_t (&w)[8]) {
    const int len = pos < hi ? (int)tmin<uint64_t>(kK3Seg, hi - pos) : 0;
    if (len == kK3Seg && aligned16(bytes + pos)) {
        const uint4 a = __ldg(reinterpret_cast<const uint4 *>(bytes + pos));
        const uint4 b = __ldg(reinterpret_cast<const uint4 *>(bytes + pos) + 1);
        w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w;
        w[4] = b.x; w[5] = b.y; w[6] = b.z; w[7] = b.w;
        return len;
    }
#pragma unroll
    for (int k = 0; k < 8; k++) {
        uint32_t x = 0;
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const int m = 4 * k + q;
            x |= (uint32_t)(m < len ? bytes[pos + m] : kZeroGroup) << (8 * q);
        }
        w[k] = x;
    }
    return len;
}

// Load chunk bytes [rel, min(rel+32, rhi)) from shared memory as 8 words,
// padding with 121 (0x79); rel is a multiple of 32.
__device__ __forceinline__ int load_seg_s(const uint8_t *c, uint32_t rel, uint32_t rhi, uint32_t (&w)[8]) {
    const int len = rel < rhi ? (int)tmin<uint32_t>(kK3Seg, rhi - rel) : 0;
    if (len == kK3Seg) {
        const uint4 a = *reinterpret_cast<const uint4 *>(c + rel);
        const uint4 b = *reinterpret_cast<const uint4 *>(c + rel + 16);
        w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w;
        w[4] = b.x; w[5] = b.y; w[6] = b.z; w[7] = b.w;
    } else {
#pragma unroll
        for (int k = 0; k < 8; k++) {
            uint32_t x = 0;
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const int m = 4 * k + q;
                x |= (uint32_t)(m < len ? c[rel + m] : kZeroGroup) << (8 * q);
            }
            w[k] = x;
        }
    }
    return len;
}

// Geometry of chunk `id` of a K3 launch as seen by warp `warp`.
struct K3Chunk {
    uint64_t id, lc, nch, lo, hi, wlo, whi, P;
    int si;
    bool ok;
};
__device__ __forceinline__ K3Chunk k3_chunk(const SegTable &T, uint64_t id, const uint64_t *s_first,
                                            const unsigned int *maxkey, float s, int warp) {
    K3Chunk c{};
    c.id = id;
    c.ok = id < T.n3;
    if (!c.ok) return c;
    c.si = find_seg_c<3>(T, id, s_first);
    const Seg S = get_seg(T, c.si);
    float M;
    c.ok = scale_from_key(maxkey[c.si], s, M) == TLC_OK;     // else the segment failed in K1
    c.P = S.P;
    c.lc = id - S.k3;
    c.nch = (S.P + T.sz.c3 - 1) / T.sz.c3;
    c.lo = c.lc * T.sz.c3;
    c.hi = tmin<uint64_t>(S.P, c.lo + T.sz.c3);
    // whole 1 KiB rows per warp: every quartic position that is a multiple of kT5 (a K5 tile
    // start) is then the start of some warp's row, where phase 3 knows (offset, carry)
    const uint64_t sub = ((c.hi - c.lo + kK3Workers - 1) / kK3Workers + kK3WarpRow - 1) / kK3WarpRow * kK3WarpRow;
    c.wlo = warp < kK3Workers ? tmin<uint64_t>(c.hi, c.lo + warp * sub) : c.hi;
    c.whi = tmin<uint64_t>(c.hi, c.wlo + sub);
    return c;
}

#ifndef TLC_K3_MINB
#define TLC_K3_MINB 4
#endif
__global__ void __launch_bounds__(kK3Threads, TLC_K3_MINB)
tlc_zre_kernel(const SegTable T, const unsigned int *maxkey, float s,
               const uint8_t *scratch, Ctrl *ctrl, unsigned long long *states) {
    __shared__ unsigned long long s_wagg[kK3Workers];
    __shared__ unsigned long long s_incl[2][kK3Workers];  // warps 0..w of a chunk composed
    __shared__ unsigned long long s_off[kK3Workers + 1];  // offset entering each warp's sub-range, end
    __shared__ uint32_t s_carry[kK3Workers + 1];
    __shared__ unsigned long long s_id;
    extern __shared__ __align__(128) uint8_t k3_smem_raw[];
    K3Smem &sm = *reinterpret_cast<K3Smem *>(k3_smem_raw);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wk = tmin(warp, kK3Workers - 1);
    uint32_t w[8];
    __shared__ uint64_t s_first[kSegCache];
#ifdef TLC_K3_TRACE
    if (threadIdx.x == 0 && blockIdx.x < 4096) g_k3_cta[blockIdx.x][0] = gtimer();
#endif
    if (threadIdx.x == 0) {
        mbar_init(&sm.bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    seg_index_load<3>(T, s_first);                       // (ends with __syncthreads)
    uint32_t parity = 0;
    pdl_wait();                                          // K2's quartic bytes and headers
    uint64_t pend_id = ~0ull;                            // chunk awaiting phase 3 (~0: none)
    int jb = 0;                                          // buffer of the new chunk
    bool more = true;
    while (more || pend_id != ~0ull) {
        if (threadIdx.x == 0) s_id = more ? atomicAdd(&ctrl->k3_counter, 1ull) : ~0ull;
        __syncthreads();
        const uint64_t jid = s_id;
        __syncthreads();
        more = jid < T.n3;
        const int ib = jb ^ 1;
        if (threadIdx.x == 0) {
            K3_TRACE(jid, 0);
#ifdef TLC_K3_TRACE
            unsigned int smid;
            asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
            if (jid < (1u << 14)) { g_k3_trace[jid][6] = smid; g_k3_trace[jid][7] = blockIdx.x; }
#endif
        }

        if (warp == kK3LookWarp) {
            // ---- phase 2 of the pending chunk, concurrent with phase 1 of the new one
            const K3Chunk pend = k3_chunk(T, pend_id, s_first, maxkey, s, warp);
            unsigned long long ex = 0;
            if (pend.ok) ex = warp_lookback<RunOp>(states + get_seg(T, pend.si).k3, pend.lc);
            if (pend.ok) K3_TRACE(pend.id, 1);
            __syncthreads();                                         // B1: phase 1 of cj done
            if (pend.ok) {
                const Seg S = get_seg(T, pend.si);
                RunSum bw = unpack(ex);
                if (lane > 0 && lane <= kK3Workers) bw = compose(bw, unpack(s_incl[ib][lane - 1]));
                const unsigned long long agg = s_incl[ib][kK3Workers - 1];
                if (lane == 0 && pend.lc > 0) st_relaxed_u64(states + pend.id, kPrefix | RunOp::combine(ex, agg));
                uint64_t o;
                uint32_t c;
                run_eval(bw, 0, o, c);
                if (lane <= kK3Workers) {
                    s_off[lane] = o;
                    s_carry[lane] = c;
                }
                const uint64_t o_begin = __shfl_sync(0xffffffffu, o, 0);
                const uint64_t o_end = __shfl_sync(0xffffffffu, o, kK3Workers);
                const uint32_t c_end = __shfl_sync(0xffffffffu, c, kK3Workers);
                if (pend.lc == pend.nch - 1 && lane == 0) S.hdr->payload_len = o_end + (c_end > 0);
                // every byte of the chunk's output that is not a flush code or a literal
                // is a full chunk (255): fill the range before phase 3 stores the rest
                warp_fill_full_chunks(S.payload, o_begin, o_end);
                K3_TRACE(pend.id, 4);
            }
            __syncthreads();                                         // B2
            pend_id = jid;
            jb ^= 1;
            continue;
        }

        {
            const K3Chunk cj = k3_chunk(T, jid, s_first, maxkey, s, warp);
            if (cj.ok) {
            // the chunk's bytes to shared memory with one bulk copy (16-byte multiple:
            // a segment's scratch is padded to 16 bytes; the loaders pad past whi)
            const Seg S = get_seg(T, cj.si);
            const uint32_t rwhi = (uint32_t)(cj.whi - cj.lo);
            if (threadIdx.x == 0) {
                const uint32_t nb = (uint32_t)((cj.hi - cj.lo + 15) & ~uint64_t(15));
                // the previous phase 3 wrote its stages here with generic stores
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_expect_tx(&sm.bar, nb);
                bulk_load(sm.chunk, scratch + S.bytes_off + cj.lo, nb, &sm.bar);
            }
            mbar_wait(&sm.bar, parity);
            parity ^= 1u;
            if (threadIdx.x == 0) K3_TRACE(cj.id, 2);

            // ---- phase 1: run summary of the warp's sub-range (one per 1 KiB row); rows'
            // literal lists with their output offsets are kept while the list space lasts
            RunSum wagg = run_identity();
            uint32_t *lit = sm.lit[jb][wk];
            uint32_t used = 0;
            bool keep = true;
            int r = 0;
            for (uint64_t row = cj.wlo; row < cj.whi; row += kK3WarpRow, r++) {
                const uint32_t rel = (uint32_t)(row - cj.lo);
                const int len = load_seg_s(sm.chunk, rel + kK3Seg * lane, rwhi, w);
                const uint32_t row_len = (uint32_t)tmin<uint64_t>(kK3WarpRow, cj.whi - row);
                if (__all_sync(0xffffffffu, plain_lane(w))) {        // no literal: one ALL run
                    wagg = compose(wagg, RunSum{row_len / kMaxRun, row_len % kMaxRun, 0u, false});
                    if (lane == 0) sm.rowmeta[jb][wk][r] = make_uint4(0u, 0u, 0u, 0u);
                    continue;
                }
                bool stored = false;
                // once a list has not fit, the warp's later rows of the chunk take the mask
                // form directly (they could not be kept in order anyway)
                const uint32_t L = keep ? row_literals(w, lit + used, kK3LitCap - used, stored) : 0u;
                if (!stored) {                                        // list space exhausted: mask form
                    keep = false;
                    const uint32_t mask = literal_mask(w);
                    wagg = compose(wagg, warp_row_summary(mask, len, mask_summary(mask, len), row_len));
                    if (lane == 0) sm.rowmeta[jb][wk][r] = make_uint4(kRowNotKept | 1u, 0u, 0u, 0u);   // L != 0
                    continue;
                }
                // literal k > 0 is preceded by R_k = p_k - p_{k-1} - 1 zero groups and costs
                // lit_cost(R_k) bytes; literal 0's cost depends on the row's carry
                const uint8_t *rowb = sm.chunk + rel;
                uint32_t *e = lit + used;
                uint32_t run = 0, plast = 0, p0 = 0;
                for (uint32_t k0 = 0; k0 < L; k0 += 32) {
                    const uint32_t k = k0 + lane;
                    const uint32_t p = k < L ? e[k] : 0u;
                    uint32_t pp = __shfl_up_sync(0xffffffffu, p, 1);
                    if (lane == 0) pp = plast;
                    plast = __shfl_sync(0xffffffffu, p, (int)tmin<uint32_t>(31u, L - 1u - k0));
                    if (k0 == 0) p0 = __shfl_sync(0xffffffffu, p, 0);
                    const bool inner = k > 0 && k < L;
                    const uint32_t R = inner ? p - pp - 1u : 0u;
                    const uint32_t q = R / kMaxRun, rem = R - q * kMaxRun;
                    const uint32_t cost = inner ? q + (rem != 0) + 1u : 0u;
                    uint32_t x = cost;
#pragma unroll
                    for (int d = 1; d < 32; d <<= 1) {
                        const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
                        if (lane >= d) x += y;
                    }
                    if (k < L) e[k] = ((uint32_t)rowb[p] << 8) | (inner ? rem | ((run + x - cost + q) << 16) : 0u);
                    run += __shfl_sync(0xffffffffu, x, 31);
                }
                const uint32_t Rt = row_len - 1u - plast;                 // trailing zero groups
                const uint32_t rest = run + Rt / kMaxRun;                 // bytes after literal 0's
                wagg = compose(wagg, RunSum{1u + p0 / kMaxRun + rest, p0 % kMaxRun, Rt % kMaxRun, true});
                if (lane == 0)
                    sm.rowmeta[jb][wk][r] = make_uint4(L | (used << 16), rest | ((Rt % kMaxRun) << 16), p0, 0u);
                used += L;
            }
            if (lane == 0) s_wagg[warp] = pack(wagg);
            asm volatile("bar.sync 1, %0;" ::"r"(32 * kK3Workers) : "memory");   // the scanning warps
            if (warp == 0) {                                 // publish the chunk aggregate at once
                RunSum incl = run_identity();
#pragma unroll
                for (int k = 0; k < kK3Workers; k++)
                    if (k <= lane) incl = compose(incl, unpack(s_wagg[k]));
                if (lane < kK3Workers) s_incl[jb][lane] = pack(incl);
                if (lane == 31) st_relaxed_u64(states + cj.id, (cj.lc == 0 ? kPrefix : kReady) | pack(incl));
                K3_TRACE(cj.id, 3);
            }
            }
        }
        __syncthreads();                                     // B1
        __syncthreads();                                     // B2: pending chunk's offsets known, 255s filled

        const K3Chunk pend = k3_chunk(T, pend_id, s_first, maxkey, s, warp);
        if (pend.ok) {
            // ---- phase 3 of the pending chunk: the sparse stores (flush codes and literals)
            const Seg S = get_seg(T, pend.si);
            const uint8_t *bytes = scratch + S.bytes_off;
            const uint32_t *lit = sm.lit[ib][wk];
            uint64_t off = s_off[warp];
            uint32_t carry = s_carry[warp];
            int r = 0;
            for (uint64_t row = pend.wlo; row < pend.whi; row += kK3WarpRow, r++) {
                const uint32_t row_len = (uint32_t)tmin<uint64_t>(kK3WarpRow, pend.whi - row);
                const uint4 meta = sm.rowmeta[ib][wk][r];
                const uint32_t L = meta.x & 0xffffu;
                uint8_t *out = S.payload + off;
                // K5 tile start: the next byte emitted starts `carry` positions before `row`
                // (the pending run's 255 or flush code, or the literal when carry = 0) -- K4's
                // entry, except that a literal at `row` after pending zero groups is reached
                // through their flush code, fully skipped (reading R25)
                if (S.seek && lane == 0 && row % kT5 == 0) S.seek[row / kT5] = (off << 4) | carry;
                if (L == 0) {                             // no literal: the run grows by row_len
                    const uint32_t x = carry + row_len;
                    off += x / kMaxRun;
                    carry = x % kMaxRun;
                } else if (!(meta.x & kRowNotKept)) {     // kept list: offsets known up to literal 0's cost
                    const uint32_t *e = lit + (meta.x >> 16);
                    const uint32_t R0 = meta.z + carry;
                    const uint32_t cost0 = lit_cost(R0);
                    for (uint32_t k = lane; k < L; k += 32) {
                        const uint32_t u = e[k];
                        uint32_t o, rem;
                        if (k == 0) {
                            o = R0 / kMaxRun;
                            rem = R0 % kMaxRun;
                        } else {
                            o = cost0 + (u >> 16);
                            rem = u & 0xfu;
                        }
                        TLC_CHECK(off + o + (rem ? 1 : 0) < pend.P);
                        if (rem) out[o++] = run_code(rem);
                        out[o] = (uint8_t)(u >> 8);
                    }
                    off += cost0 + (meta.y & 0xffffu);
                    carry = meta.y >> 16;
                } else {
                    // not kept (a dense row: its list did not fit): every lane emits its
                    // bytes into the warp's stage in shared memory (the chunk buffer is free
                    // in phase 3), prefilled with 255 for the full chunks, placed congruent
                    // to the output modulo 16; the warp then copies the row's output out with
                    // 16-byte stores (byte stores from lanes 32 bytes apart wrote 32 sectors
                    // per instruction: 0.31 ms on dense stochastic trits)
                    const int len = load_seg_g(bytes, row + kK3Seg * lane, pend.whi, w);
                    const uint32_t mask = literal_mask(w);
                    const WarpRow wr = warp_row(mask, len, mask_summary(mask, len), carry, row_len);
                    uint32_t x = wr.count;
#pragma unroll
                    for (int d = 1; d < 32; d <<= 1) {
                        const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
                        if (lane >= d) x += y;
                    }
                    const PadStage stage{sm.chunk + (size_t)wk * kK3Stage, kK3Stage};
                    const uint32_t sh = (uint32_t)(reinterpret_cast<uintptr_t>(out) & 3u);
                    pad_stage_fill(stage, sh + wr.row_count);
                    __syncwarp();
                    lane_emit(w, mask, wr.carry_in, stage, sh + x - wr.count);
                    __syncwarp();
                    TLC_CHECK(off + wr.row_count <= pend.P);
                    warp_copy_padded(out, stage, sh, wr.row_count);
                    __syncwarp();                         // the stage is reused by the next row
                    off += wr.row_count;
                    carry = wr.carry_out;
                }
                if (lane == 0 && carry > 0 && row + row_len == pend.P) {
                    TLC_CHECK(off < pend.P);
                    S.payload[off] = run_code(carry);
                }
            }
            if (warp == 0) K3_TRACE(pend.id, 5);
        }
        pend_id = jid;
        jb ^= 1;
    }
#ifdef TLC_K3_TRACE
    if (threadIdx.x == 0 && blockIdx.x < 4096) g_k3_cta[blockIdx.x][1] = gtimer();
#endif
}

// ============================================================== host side
static int g_k2_blocks = 0, g_k3_blocks = 0;

// Complete bulk tiles of a one-segment table: positions j < min(P, n - 4P) have all five
// elements; the bulk kernel takes whole K2 tiles of them (kT2 = 4 bulk tiles).
// Complete bulk tiles of a one-segment table (aligned t and err): tiles of positions whose
// five elements exist, with 4 elements of slack at the end of the last partition (an
// unaligned partition is fetched as an aligned superset of up to 3 more elements); the
// bulk kernel takes whole K2 tiles of them (kT2 = 4 bulk tiles).
static uint64_t bulk_tiles(const SegTable &T, int use_zre) {
    if (T.count != 1) return 0;
    const Seg &S = T.one;
    if (!aligned16(S.t) || !aligned16(S.err)) return 0;
    if (!use_zre && !aligned4(S.payload)) return 0;
    const uint64_t complete = S.n >= 4 * S.P + 4 ? tmin<uint64_t>(S.P, S.n - 4 * S.P - 4) : 0;
    return (complete / T.sz.t2) * (T.sz.t2 / kBulkPos);
}

// TLC_NO_BULK=1 disables the bulk-copy K2 path (A/B measurements)
static bool use_bulk() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("TLC_NO_BULK");
        v = (e && e[0] == '1') ? 0 : 1;
    }
    return v == 1;
}

void launch_absmax(const SegTable &T, unsigned int *maxkey, bool has_err, cudaStream_t st) {
    KernelScope ks(kK1, st);
    const int grid = (int)tmax<uint64_t>(1, tmin<uint64_t>(T.n1, (uint64_t)num_sms() * kK1BlocksPerSm));
    if (has_err) tlc_absmax_kernel<true><<<grid, kK1Threads, 0, st>>>(T, maxkey);
    else tlc_absmax_kernel<false><<<grid, kK1Threads, 0, st>>>(T, maxkey);
}

// K1 (max key), then `k2` (the quantizer + quartic pass of the codec), then K3 (ZRE).
template <class K2Launch>
static int compress_pipeline(const SegTable &T, float s, int use_zre, bool has_err, void *ws, cudaStream_t st,
                             const K2Launch &k2, bool fused_k1 = false, bool zeroed = false) {
    const WsLayout L = ws_layout(T, 0);
    char *base = reinterpret_cast<char *>(ws);
    Ctrl *ctrl = reinterpret_cast<Ctrl *>(base + L.ctrl);
    unsigned int *maxkey = reinterpret_cast<unsigned int *>(base + L.maxkey);
    unsigned long long *states = reinterpret_cast<unsigned long long *>(base + L.k3st);
    uint8_t *scratch = reinterpret_cast<uint8_t *>(base + L.bytes);
    const int sms = num_sms();
    if (!zeroed && cudaMemsetAsync(ws, 0, L.memset_c, st) != cudaSuccess) return TLC_ERR_CUDA;
    if (!fused_k1) launch_absmax(T, maxkey, has_err, st);   // K12 / the keyed aggregate fold K1 in
    k2(maxkey, scratch);
    if (use_zre) {
        KernelScope ks(kK3, st);
        static PerDevice k3attr;
        if (k3attr.first())
            cudaFuncSetAttribute(tlc_zre_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(K3Smem));
        if (!g_k3_blocks)
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_k3_blocks, tlc_zre_kernel, kK3Threads, sizeof(K3Smem));
        const int grid = (int)tmax<uint64_t>(1, tmin<uint64_t>(T.n3, (uint64_t)sms * tmin(16, tmax(1, g_k3_blocks))));
        launch_pdl(tlc_zre_kernel, grid, kK3Threads, sizeof(K3Smem), st, T, maxkey, s, scratch, ctrl, states);
    }
    return cudaPeekAtLastError() == cudaSuccess ? TLC_OK : TLC_ERR_CUDA;
}

// A second stream per device (and two events) for the table path's K2 register-tail kernel:
// it needs only K1's keys, so it runs beside the bulk table kernel instead of after it.
// Stream capture records the fork and the join as graph edges.
struct SideStream {
    cudaStream_t s = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
};
static SideStream *side_stream() {
    static SideStream ss[64];
    int dev = 0;
    cudaGetDevice(&dev);
    SideStream &x = ss[dev & 63];
    if (!x.s) {
        cudaStreamCreateWithFlags(&x.s, cudaStreamNonBlocking);
        cudaEventCreateWithFlags(&x.fork, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&x.join, cudaEventDisableTiming);
    }
    return &x;
}

// TLC_NO_FORK=1 keeps the K2 tail on the caller's stream (A/B)
static bool fork_enabled() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("TLC_NO_FORK");
        v = (e && e[0] == '1') ? 0 : 1;
    }
    return v == 1;
}

// K12 is opt-in (TLC_K12=1; measured in round 2): it cuts K2's HBM reads
// (profiles/r04a: 2.66 instead of 4.3 GB per compress of 64 x 4M values) and is 14 % faster
// than K1 + K2 on tables of 16-byte aligned partitions (P % 4 == 0), but its register-staged
// quantize loses to the bulk-copy K2 on unaligned partitions (+20 %), and BERT-large's
// exchange (mostly P % 4 != 0) is 10 % slower with it (profiles/r04f, r04g).
// TLC_K12_WIN=<M values> sets the window (default 4: 32 MB of t + err); TLC_K12_HINT: L2
// policy of the max items' loads (1 default: evict_last; 0 none; 2 also evict_first on the
// quantize items' loads).
static int env_int(const char *name, int dflt) {
    const char *e = getenv(name);
    return e && e[0] ? atoi(e) : dflt;
}
static int k12_mode() {
    static int v = -1;
    if (v < 0) v = env_int("TLC_K12", 0) != 0 ? 1 : 0;
    return v;
}
static bool k12_enabled() { return k12_mode() != 0; }

int k12_plan_build(SegTable &T, const std::vector<Seg> &host, uint32_t **d_k12) {
    T.k12 = nullptr;
    T.k12_n = 0;
    if (!k12_enabled() || host.size() < 2) return TLC_OK;
    const uint64_t win = (uint64_t)tmax(1, env_int("TLC_K12_WIN", 4)) << 20;   // values per window
    std::vector<std::pair<size_t, size_t>> wins;            // [first, last) tensors
    for (size_t i = 0; i < host.size();) {
        size_t j = i;
        uint64_t sum = 0;
        while (j < host.size() && (j == i || sum + host[j].n <= win)) sum += host[j++].n;
        wins.push_back({i, j});
        i = j;
    }
    const uint64_t upos = T.sz.t2, R = 1;                    // items are K2 tiles
    std::vector<uint32_t> items;
    auto emit = [&](size_t w, uint32_t kind) {
        for (size_t i = wins[w].first; i < wins[w].second; i++) {
            const uint64_t nt = (host[i].P + upos - 1) / upos;
            for (uint64_t lt = 0; lt < nt; lt++) items.push_back((uint32_t)((host[i].k2 * R + lt) << 1) | kind);
        }
    };
    emit(0, 0u);
    for (size_t w = 0; w < wins.size(); w++) {              // K1(w+1) then K2(w)
        if (w + 1 < wins.size()) emit(w + 1, 0u);
        emit(w, 1u);
    }
    if (T.n2 * R >= (1ull << 31)) return TLC_OK;            // item ids are 31-bit units: keep K1 + K2
    const size_t nitems = items.size();
    if (cudaMalloc((void **)d_k12, items.size() * sizeof(uint32_t)) != cudaSuccess) return TLC_ERR_CUDA;
    if (cudaMemcpy(*d_k12, items.data(), items.size() * sizeof(uint32_t), cudaMemcpyHostToDevice) != cudaSuccess)
        return TLC_ERR_CUDA;
    T.k12 = *d_k12;
    T.k12_n = (uint32_t)nitems;
    return TLC_OK;
}

static int g_k12_blocks = 0;

static int launch_compress_table_impl(const SegTable &T, float s, int use_zre, void *ws, cudaStream_t st, bool keyed);

int launch_compress_table(const SegTable &T, float s, int use_zre, void *ws, cudaStream_t st) {
    return launch_compress_table_impl(T, s, use_zre, ws, st, false);
}

// the keyed pull compress (keys folded by K5m) runs K2 after them: any table off the small path
bool compress_runs_k1(const SegTable &T) { return !small_table(T); }

int prepare_keyed_compress(const SegTable &T, void *ws, cudaStream_t st, unsigned int **keys) {
    const WsLayout L = ws_layout(T, 0);
    if (cudaMemsetAsync(ws, 0, L.memset_c, st) != cudaSuccess) return TLC_ERR_CUDA;
    *keys = reinterpret_cast<unsigned int *>(reinterpret_cast<char *>(ws) + L.maxkey);
    return TLC_OK;
}

int launch_compress_table_keyed(const SegTable &T, float s, int use_zre, void *ws, cudaStream_t st) {
    if (!compress_runs_k1(T)) return TLC_ERR_ARG;
    return launch_compress_table_impl(T, s, use_zre, ws, st, true);
}

static int launch_compress_table_impl(const SegTable &T, float s, int use_zre, void *ws, cudaStream_t st, bool keyed) {
    if (small_table(T)) return launch_small_compress(T, s, use_zre, st);    // one launch, on chip
    const int sms = num_sms();
    if (T.k12 && k12_enabled() && !keyed) {
        static const int hint = env_int("TLC_K12_HINT", 1);
        const WsLayout L = ws_layout(T, 0);
        char *base = reinterpret_cast<char *>(ws);
        unsigned int *done = reinterpret_cast<unsigned int *>(base + L.k12done);
        Ctrl *ctrl = reinterpret_cast<Ctrl *>(base + L.ctrl);
        return compress_pipeline(T, s, use_zre, true, ws, st, [&](unsigned int *maxkey, uint8_t *scratch) {
            KernelScope ks(kK12, st);
            constexpr size_t smem = 2 * 10 * kBulkRow * sizeof(float);   // two bulk stages
            static PerDevice k12attr;
            if (k12attr.first()) {
                cudaFuncSetAttribute(tlc_absmax_quant_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                cudaFuncSetAttribute(tlc_absmax_quant_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                cudaFuncSetAttribute(tlc_absmax_quant_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            }
            if (!g_k12_blocks)
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_k12_blocks, tlc_absmax_quant_kernel<0>, kK12Threads, smem);
            const int grid = (int)tmin<uint64_t>(T.k12_n, (uint64_t)sms * tmax(1, g_k12_blocks));
            if (hint == 2)
                tlc_absmax_quant_kernel<2><<<grid, kK12Threads, smem, st>>>(T, maxkey, done, ctrl, s, use_zre, scratch);
            else if (hint == 1)
                tlc_absmax_quant_kernel<1><<<grid, kK12Threads, smem, st>>>(T, maxkey, done, ctrl, s, use_zre, scratch);
            else
                tlc_absmax_quant_kernel<0><<<grid, kK12Threads, smem, st>>>(T, maxkey, done, ctrl, s, use_zre, scratch);
        }, true);
    }
    return compress_pipeline(T, s, use_zre, true, ws, st, [&](unsigned int *maxkey, uint8_t *scratch) {
        KernelScope ks(kK2, st);
        const uint64_t nbulk = use_bulk() ? bulk_tiles(T, use_zre) : 0;
        uint64_t tile_begin = 0;
        int skip_bulk = 0;
        static PerDevice attr;
        if (attr.first()) {
            cudaFuncSetAttribute(tlc_quant_qe_bulk_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sizeof(BulkSmem));
            cudaFuncSetAttribute(tlc_quant_qe_bulk_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sizeof(BulkSmem));
            cudaFuncSetAttribute(tlc_quant_qe_bulk_table_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sizeof(BulkSmem));
        }
        if (nbulk) {
            const int grid = (int)tmin<uint64_t>(nbulk, (uint64_t)sms);
            if ((T.one.P & 3) == 0)
                launch_pdl(tlc_quant_qe_bulk_kernel<true>, grid, kK2Threads, sizeof(BulkSmem), st, T, maxkey, s,
                           use_zre, scratch, nbulk);
            else
                launch_pdl(tlc_quant_qe_bulk_kernel<false>, grid, kK2Threads, sizeof(BulkSmem), st, T, maxkey, s,
                           use_zre, scratch, nbulk);
            tile_begin = nbulk * kBulkPos / T.sz.t2;
        } else if (use_bulk() && T.count > 1 && T.n_bulk && (use_zre || T.bulk_nozre_ok) &&
                   T.sz.t2 == kLargeItems.t2) {
            skip_bulk = 1;
        }
        const uint64_t nreg = skip_bulk ? T.n_rest : T.n2 - tile_begin;
        if (!g_k2_blocks) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_k2_blocks, tlc_quant_qe_kernel, kK2Threads, 0);
        const int rgrid = (int)tmax<uint64_t>(1, tmin<uint64_t>(nreg, (uint64_t)sms * tmax(1, g_k2_blocks)));
        const bool fork = skip_bulk && nreg > 0 && fork_enabled();
        SideStream *ss = fork ? side_stream() : nullptr;
        if (fork) {
            // the ragged tail tiles of the table (register kernel) beside the bulk kernel
            cudaEventRecord(ss->fork, st);
            cudaStreamWaitEvent(ss->s, ss->fork, 0);
            tlc_quant_qe_kernel<<<rgrid, kK2Threads, 0, ss->s>>>(T, maxkey, s, use_zre, scratch, tile_begin, skip_bulk);
            cudaEventRecord(ss->join, ss->s);
        }
        if (skip_bulk) {
            // large tables only: below 32M values (ResNet-50) the register kernel at 2 CTAs/SM
            // measured faster (0.44 vs 0.49 ms per W=1 exchange step) than the 1-CTA/SM bulk one
            const int grid = (int)tmin<uint64_t>(T.n_bulk * (T.sz.t2 / kBulkPos), (uint64_t)sms);
            launch_pdl(tlc_quant_qe_bulk_table_kernel, grid, kK2TThreads, sizeof(BulkSmem), st, T, maxkey, s, use_zre,
                       scratch);
        }
        if (fork) {
            cudaStreamWaitEvent(st, ss->join, 0);
        } else if (nreg > 0) {
            launch_pdl(tlc_quant_qe_kernel, rgrid, kK2Threads, 0, st, T, maxkey, s, use_zre, scratch, tile_begin,
                       skip_bulk);
        }
    }, keyed, keyed);
}

// "Stoch 3-value + QE": K1 over t alone (m = max|t|, s = 1), the
// stochastic quantizer + quartic pass of stoch.cu, K3 when ZRE is asked for.
int launch_stoch_compress_table(const SegTable &T, uint64_t seed, uint64_t step, int use_zre, void *ws,
                                cudaStream_t st) {
    return compress_pipeline(T, 1.0f, use_zre, false, ws, st, [&](unsigned int *maxkey, uint8_t *scratch) {
        launch_stoch_qe(T, maxkey, seed, step, use_zre, scratch, st);
    });
}

int launch_compress(const float *t, float *err, uint64_t n, float s, int use_zre, uint8_t *payload,
                    tlc_header *hdr, void *ws, cudaStream_t st) {
    uint64_t scratch = 0;
    const SegTable T = single_table(t, err, nullptr, payload, hdr, n, scratch);
    return launch_compress_table(T, s, use_zre, ws, st);
}

size_t compress_workspace_bytes(uint64_t n) {
    uint64_t scratch = 0;
    const SegTable T = single_table(nullptr, nullptr, nullptr, nullptr, nullptr, n, scratch);
    return ws_layout(T, scratch).total;
}

}  // namespace tlc

#ifdef TLC_K3_TRACE
extern "C" int tlc_debug_k3_trace(void *host, size_t bytes) {
    return cudaMemcpyFromSymbol(host, tlc::g_k3_trace, bytes) == cudaSuccess ? 0 : 1;
}
extern "C" int tlc_debug_k3_cta(void *host, size_t bytes) {
    return cudaMemcpyFromSymbol(host, tlc::g_k3_cta, bytes) == cudaSuccess ? 0 : 1;
}
#endif
