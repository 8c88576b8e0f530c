// small.cu -- the small-tensor regime (SURVEY 8(a) "K6/K7"; BASELINE configs[1] and
// [3]: the 110 per-layer ResNet-110 tensors, <= 36,864 values each).  At these sizes the
// streaming kernels K1-K5 are bound by launch gaps and chains of dependent global
// accesses (ncu on the C2 table: 8-12 us per kernel for 14 MB), not by bandwidth.  Here
// one CTA owns one tensor and runs the whole method on chip, one launch per direction:
//
//  K6 tlc_small_compress_kernel (rows a1-a4): t and err are read ONCE into
//     u = err + t in shared memory (step 1), the CTA reduces max|u| (Eq. 1),
//     quantizes from shared memory writing err (Eq. 2, steps a, b), folds the quartic
//     bytes (step 3) into shared memory and zero-run encodes them (step 4) with the
//     warp-row machinery of K3: one warp per 1 KiB row, the row summaries composed
//     in order by one thread, then every lane emits its flush codes and literals at
//     their offsets over a 255 prefill.  HBM traffic 12n + Z: the two-pass bound of
//     the large path (20n) disappears because the tensor fits on chip.
//  K7 tlc_small_decompress_kernel (rows a5-a6): header checks, the payload to shared
//     memory, a block scan of the expansion lengths (FORMAT unless they sum to P),
//     expansion into the quartic bytes, base-3 decode and Eq. 3 through a per-partition
//     value table, overwrite or skip-zero accumulate (R16).  Nothing is written on
//     FORMAT.
//
// Same results, byte for byte, as the large path (the payload, err, header and output
// are defined by the method, not by the kernels).
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "tlc_device.cuh"
#include "tlc_launch.h"

namespace tlc {

constexpr int kSmThreads = 512;
constexpr uint32_t kK3WarpRowS = 1024;                  // K3's warp row: 32 lanes x 32 bytes
constexpr int kSmWarps = kSmThreads / 32;
static_assert(kSmallMaxN <= 5 * 1024 * kSmWarps, "one warp row per 1 KiB of quartic bytes");

__device__ __forceinline__ unsigned int block_max(unsigned int m, unsigned int *s_red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    m = __reduce_max_sync(0xffffffffu, m);
    if (lane == 0) s_red[warp] = m;
    __syncthreads();
    if (warp == 0) {
        m = __reduce_max_sync(0xffffffffu, lane < kSmWarps ? s_red[lane] : 0u);
        if (lane == 0) s_red[kSmWarps] = m;
    }
    __syncthreads();
    return s_red[kSmWarps];
}

#ifdef TLC_K6C_TRACE
// development instrumentation: %globaltimer at the phase boundaries of every CTA (K6, K6x, K6c)
__device__ unsigned long long g_k6c_trace[1024][8];
#define K6C_TRACE(slot)                                                                     \
    do {                                                                                    \
        if (threadIdx.x == 0 && blockIdx.x < 1024) {                                        \
            unsigned long long t_;                                                          \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                         \
            g_k6c_trace[blockIdx.x][slot] = t_;                                             \
            if (slot == 0) {                                                                \
                unsigned int sm_;                                                           \
                asm volatile("mov.u32 %0, %%smid;" : "=r"(sm_));                           \
                g_k6c_trace[blockIdx.x][7] = sm_;                                           \
            }                                                                               \
        }                                                                                   \
    } while (0)
#else
#define K6C_TRACE(slot) do {} while (0)
#endif

template <class QT>
__device__ __forceinline__ void small_quantize(const Seg &S, const float *u, uint8_t *dst, const QT &Q) {
    const uint64_t P = S.P, n = S.n;
    for (uint32_t j = threadIdx.x; j < P; j += kSmThreads) {
        uint32_t b = 0;
#pragma unroll
        for (int i = 0; i < 5; i++) {
            const uint32_t e = (uint32_t)(i * P) + j;
            uint32_t d = 0;                                      // pad digit (R10)
            if (e < n) {
                const float x = u[e];
                const int q = Q.q(x);                            // Eq. 2
                __stcs(S.err + e, Q.residual(x, q));             // steps (a),(b)
                d = (uint32_t)(q + 1);
            }
            b = b * 3u + d;                                      // steps 1, 4, 6
        }
        dst[j] = (uint8_t)b;
    }
}

__global__ void __launch_bounds__(kSmThreads, 1)
tlc_small_compress_kernel(const SegTable T, float s, int use_zre) {
    extern __shared__ __align__(16) uint8_t sm_raw[];
    __shared__ unsigned int s_red[kSmWarps + 1];
    __shared__ unsigned long long s_row[kSmWarps];
    __shared__ uint32_t s_off[kSmWarps + 1], s_carry[kSmWarps + 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int si = blockIdx.x; si < T.count; si += gridDim.x) {
        K6C_TRACE(0);
        const Seg S = get_seg(T, si);
        const uint32_t n = (uint32_t)S.n, P = (uint32_t)S.P;
        float *u = reinterpret_cast<float *>(sm_raw);
        uint8_t *B = sm_raw + 4 * ((n + 3) & ~3u);
        // ---- step (1): u = buffer + T_in into shared memory, and the max key of |u|
        unsigned int m = 0;
        const bool vec = aligned16(S.t) && aligned16(S.err);
        uint32_t head = 0;
        if (vec) {
            const uint32_t n4 = n / 4;
            const float4 *t4 = reinterpret_cast<const float4 *>(S.t);
            const float4 *e4 = reinterpret_cast<const float4 *>(S.err);
            constexpr int kU = 8;                            // 256 bytes of t and err in flight per thread
            for (uint32_t g0 = threadIdx.x; g0 < n4; g0 += kU * kSmThreads) {
                float4 tv[kU], ev[kU];
#pragma unroll
                for (int k = 0; k < kU; k++) {
                    const uint32_t g = g0 + k * kSmThreads;
                    if (g < n4) { tv[k] = ld_stream4(t4 + g); ev[k] = __ldcs(e4 + g); }
                }
#pragma unroll
                for (int k = 0; k < kU; k++) {
                    const uint32_t g = g0 + k * kSmThreads;
                    if (g >= n4) break;
                    const float4 x = make_float4(__fadd_rn(ev[k].x, tv[k].x), __fadd_rn(ev[k].y, tv[k].y),
                                                 __fadd_rn(ev[k].z, tv[k].z), __fadd_rn(ev[k].w, tv[k].w));
                    reinterpret_cast<float4 *>(u)[g] = x;
                    m = max(m, max(max(__float_as_uint(x.x) & 0x7fffffffu, __float_as_uint(x.y) & 0x7fffffffu),
                                   max(__float_as_uint(x.z) & 0x7fffffffu, __float_as_uint(x.w) & 0x7fffffffu)));
                }
            }
            head = 4 * n4;
        }
        for (uint32_t e = head + threadIdx.x; e < n; e += kSmThreads) {
            const float x = __fadd_rn(__ldcs(S.err + e), ld_stream(S.t + e));
            u[e] = x;
            m = max(m, __float_as_uint(x) & 0x7fffffffu);
        }
        m = block_max(m, s_red);                                 // also orders the u stores
        K6C_TRACE(1);
        float M;
        const unsigned int status = scale_from_key(m, s, M);     // Eq. 1, R6
        if (threadIdx.x == 0) {
            tlc_header *h = S.hdr;
            h->M = M;
            h->flags = use_zre ? TLC_FLAG_ZRE : 0u;
            h->n = S.n;
            h->payload_len = (status == TLC_OK && !use_zre) ? S.P : 0;
            h->status = status;
            h->reserved = 0;
        }
        if (status != TLC_OK) continue;                          // err untouched (R6)
        // ---- Eq. 2, steps (a),(b), quartic steps 1-6
        uint8_t *dst = use_zre ? B : S.payload;
        const Quant Q(M);
        if (Q.mode == 1) small_quantize(S, u, dst, QuantCmp(Q));
        else small_quantize(S, u, dst, Q);
        if (!use_zre) { __syncthreads(); continue; }
        __syncthreads();
        K6C_TRACE(2);
        // ---- step (4): zero-run encoding, one warp per 1 KiB row
        const uint32_t nrows = (P + kK3WarpRowS - 1) / kK3WarpRowS;
        uint32_t w[8], mask = 0;
        int len = 0;
        RunSum lane_sum = run_identity();
        uint32_t row_len = 0;
        if ((uint32_t)warp < nrows) {
            const uint32_t base = (uint32_t)warp * kK3WarpRowS;
            row_len = min(kK3WarpRowS, P - base);
            const uint32_t rel = base + 32u * lane;
            len = rel < P ? (int)min(32u, P - rel) : 0;
#pragma unroll
            for (int k = 0; k < 8; k++) {
                uint32_t x = 0;
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    const int mm = 4 * k + q;
                    x |= (uint32_t)(mm < len ? B[rel + mm] : kZeroGroup) << (8 * q);
                }
                w[k] = x;
            }
            mask = literal_mask(w);
            lane_sum = mask_summary(mask, len);
            const RunSum rs = warp_row_summary(mask, len, lane_sum, row_len);
            if (lane == 0) s_row[warp] = pack(rs);
        }
        __syncthreads();
        if (threadIdx.x == 0) {                                  // rows in order: offset, carry
            RunSum acc = run_identity();
            for (uint32_t r = 0; r <= nrows; r++) {
                uint64_t o;
                uint32_t c;
                run_eval(acc, 0, o, c);
                s_off[r] = (uint32_t)o;
                s_carry[r] = c;
                if (r < nrows) acc = compose(acc, unpack(s_row[r]));
            }
            S.hdr->payload_len = s_off[nrows] + (s_carry[nrows] > 0);
        }
        __syncthreads();
        K6C_TRACE(3);
        // full chunks (255) everywhere first; flush codes and literals overwrite
        const uint32_t total = s_off[nrows];
        for (uint32_t q = threadIdx.x; q < total; q += kSmThreads) S.payload[q] = 0xff;
        __syncthreads();
        K6C_TRACE(4);
        if ((uint32_t)warp < nrows) {
            const WarpRow wr = warp_row(mask, len, lane_sum, s_carry[warp], row_len);
            uint32_t x = wr.count;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
                if (lane >= d) x += y;
            }
            uint8_t *out = S.payload + s_off[warp];
            uint32_t o = x - wr.count, c = wr.carry_in;
            int prev = -1;
            for (uint32_t mk = mask; mk; mk &= mk - 1u) {
                const int q = (int)ctz32(mk);
                const uint32_t R = (uint32_t)(q - prev - 1) + c;
                c = 0;
                o += R / kMaxRun;
                TLC_CHECK(s_off[warp] + o + (R % kMaxRun ? 1 : 0) < P);
                if (R % kMaxRun) out[o++] = run_code(R % kMaxRun);
                uint32_t word = w[0];
#pragma unroll
                for (int k = 1; k < 8; k++) word = (k == (q >> 2)) ? w[k] : word;
                out[o++] = (uint8_t)(word >> (8 * (q & 3)));
                prev = q;
            }
        }
        TLC_CHECK(!(threadIdx.x == 0 && s_carry[nrows] > 0) || total < P);
        if (threadIdx.x == 0 && s_carry[nrows] > 0) S.payload[total] = run_code(s_carry[nrows]);
        __syncthreads();                                         // shared memory reuse
        K6C_TRACE(5);
    }
}

// ============================================================== K6g (clusters)
// K6 with each tensor cut into slices of whole 1 KiB ZRE rows (at most kGRows rows, at most
// CL slices), the slices of one tensor in one thread-block cluster of CL CTAs, several small
// tensors sharing a cluster (host plan, small_group_plan_build).  One SM stores at most
// ~61 GB/s and loads ~130-200 GB/s (profiles/r03l_sm_bw.txt), so the 36,864-value layers of
// ResNet-110 (442 KB each) are too much for one CTA: K6's CTA spends 12 us on one of them
// (profiles/r03k_trace.txt).  The group's CTAs exchange their max keys (cluster barrier 1)
// and their ZRE run summaries (cluster barrier 2) by stores into each other's shared memory
// (DSMEM) before the barriers, so nothing remote is touched after the second barrier and
// every global store -- err, payload, header -- comes after it (a release barrier waits for
// outstanding stores).  Same results bit for bit as K6.
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// store v into the same shared variable of CTA `rank` of this cluster
__device__ __forceinline__ void dsmem_store_u64(unsigned long long *local, uint32_t rank, unsigned long long v) {
    uint32_t a = (uint32_t)__cvta_generic_to_shared(local), ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
    asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(ra), "l"(v) : "memory");
}
__device__ __forceinline__ void dsmem_store_u32(unsigned int *local, uint32_t rank, unsigned int v) {
    uint32_t a = (uint32_t)__cvta_generic_to_shared(local), ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(ra), "r"(v) : "memory");
}

// DSMEM store that completes `bytes` of the receiving CTA's mbarrier transaction count
__device__ __forceinline__ void st_async_u32(unsigned int *local_dst, uint32_t rank, unsigned int v,
                                             unsigned long long *local_mbar) {
    uint32_t ra, rm;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_addr(local_dst)), "r"(rank));
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rm) : "r"(smem_addr(local_mbar)), "r"(rank));
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];"
                 ::"r"(ra), "r"(v), "r"(rm) : "memory");
}
__device__ __forceinline__ void st_async_u64(unsigned long long *local_dst, uint32_t rank, unsigned long long v,
                                             unsigned long long *local_mbar) {
    uint32_t ra, rm;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_addr(local_dst)), "r"(rank));
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rm) : "r"(smem_addr(local_mbar)), "r"(rank));
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];"
                 ::"r"(ra), "l"(v), "r"(rm) : "memory");
}

constexpr int kGThreads = 256;
constexpr int kGWarps = kGThreads / 32;

template <int NW>
__device__ __forceinline__ unsigned int block_max_n(unsigned int m, unsigned int *s_red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    m = __reduce_max_sync(0xffffffffu, m);
    if (lane == 0) s_red[warp] = m;
    __syncthreads();
    if (warp == 0) {
        m = __reduce_max_sync(0xffffffffu, lane < NW ? s_red[lane] : 0u);
        if (lane == 0) s_red[NW] = m;
    }
    __syncthreads();
    return s_red[NW];
}

// thread x < 40 of the 16-byte-aligned case: element (i, jj) of partition i's scalar head
// (slots 0-3, up to the first 16-byte boundary) or tail (slots 4-7, after the float4 groups)
__device__ __forceinline__ bool slice_edge(uint32_t x, uint32_t P, uint32_t j0, uint32_t len, uint32_t n,
                                           uint32_t &i, uint32_t &jj) {
    if (x >= 40) return false;
    i = x >> 3;
    const uint32_t r = x & 7, e0 = i * P + j0;
    const uint32_t lim = e0 >= n ? 0u : min(len, n - e0);
    const uint32_t hd = min((4u - (e0 & 3u)) & 3u, lim), body = hd + (lim - hd) / 4 * 4;
    jj = r < 4 ? r : body + (r - 4);
    return r < 4 ? r < hd : jj < lim;
}

template <class QT>
__device__ __forceinline__ void slice_quantize(float *u, uint8_t *B, uint32_t j0, uint32_t len, uint32_t Ls,
                                               const uint32_t (&sh)[5], uint32_t P, uint32_t n, const QT &Q) {
    for (uint32_t jj = threadIdx.x; jj < len; jj += kGThreads) {
        float x[5];
#pragma unroll
        for (int i = 0; i < 5; i++) x[i] = u[(uint32_t)i * Ls + sh[i] + jj];   // all five loads first
        uint32_t b = 0;
#pragma unroll
        for (int i = 0; i < 5; i++) {
            const bool in = (uint32_t)i * P + j0 + jj < n;
            const int q = in ? Q.q(x[i]) : 0;                      // Eq. 2
            x[i] = Q.residual(x[i], q);                            // steps (a), (b): u becomes err
            b = b * 3u + (in ? (uint32_t)(q + 1) : 0u);            // steps 1, 4, 6; pad digit (R10)
        }
#pragma unroll
        for (int i = 0; i < 5; i++) u[(uint32_t)i * Ls + sh[i] + jj] = x[i];
        B[jj] = (uint8_t)b;
    }
}

__device__ __forceinline__ void bulk_store(void *gdst, const void *ssrc, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_addr(ssrc)),
                 "r"(bytes) : "memory");
}

// plan record: GrpRec (tlc_launch.h).  BULK: t and err rows arrive by bulk copies (every
// partition row of the slice in flight at once; one SM keeps ~40 KB in flight with
// registers, profiles/r03o_trace.txt) into rows of Ls floats placed so that the 16-byte
// aligned interiors land 16-byte aligned (row i starts at i*Ls + (e0_i & 3)), and err leaves
// by bulk stores from the same rows.
// AS (default): the keys and the run summaries travel by st.async into the receivers' shared
// memory, each receiver waiting on its own mbarrier for exactly the bytes it is owed; the only
// cluster barrier is the one that publishes the mbarriers' initialisation (arrived at the
// start, waited on before the first remote store), so err is stored right after the
// quantization and nobody waits for the slowest member of the cluster.  !AS: two cluster
// barriers, every global store after the second (TLC_K6G_SYNC=1, A/B).
template <int CL, bool BULK, bool AS>
__global__ void __launch_bounds__(kGThreads, 2)
tlc_small_group_compress_kernel(const SegTable T, float s, int use_zre) {
    extern __shared__ __align__(16) uint8_t sm_raw[];
    __shared__ unsigned int s_red[kGWarps + 1];
    __shared__ unsigned long long s_row[kGWarps];
    __shared__ uint32_t s_off[kGWarps + 1], s_carry[kGWarps + 1];
    __shared__ unsigned int s_keys[CL];
    __shared__ unsigned long long s_aggs[CL];
    __shared__ __align__(8) unsigned long long s_mbar;
    __shared__ __align__(8) unsigned long long s_mb_keys, s_mb_aggs;   // AS: incoming keys / summaries
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    K6C_TRACE(0);
    const GrpRec S = T.grp[blockIdx.x];                        // one 64-byte record: no table walk
    const bool idle = S.seg == ~0u;
    const uint32_t g0 = S.g0, gcnt = S.gcnt, grank = S.grank;
    if (AS) {
        if (threadIdx.x == 0) {
            mbar_init(&s_mb_keys, 1);
            mbar_init(&s_mb_aggs, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            // the bytes this CTA is owed: every other member's key, every earlier slice's summary
            mbar_expect_tx(&s_mb_keys, idle ? 0u : 4u * (gcnt - 1));
            mbar_expect_tx(&s_mb_aggs, idle || !use_zre ? 0u : 8u * grank);
        }
        __syncthreads();
        asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");   // waited on below
    }
    const uint32_t n = S.n, P = S.P, j0 = S.j0, len = idle ? 0u : S.len;
    const bool vec = aligned16(S.t) && aligned16(S.err);
    const bool bulk = BULK && vec;
    const uint32_t Ls = bulk ? ((len + 3) & ~3u) + 4 : len;   // floats per partition row
    float *u = reinterpret_cast<float *>(sm_raw);             // u[i * Ls + sh_i + j - j0]
    float *tt = u + 5 * Ls;                                    // BULK: T_in rows
    uint8_t *B = reinterpret_cast<uint8_t *>(u + (bulk ? 10 : 5) * Ls);
    B = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(B) + 15) & ~uintptr_t(15));
    // ---- step (1): u = buffer + T_in of the slice into shared memory; its max key.
    // Partition i of the slice is the global run [e0_i = i*P + j0, +lim_i): a scalar head up
    // to a 16-byte boundary, float4 groups, a scalar tail.
    unsigned int m = 0;
    uint32_t hd[5], gc[5], sh[5], lim[5], gmax = 0;
#pragma unroll
    for (int i = 0; i < 5; i++) {
        const uint32_t e0 = (uint32_t)i * P + j0;
        lim[i] = e0 >= n ? 0u : min(len, n - e0);
        sh[i] = bulk ? (e0 & 3u) : 0u;
        hd[i] = vec ? min((4u - (e0 & 3u)) & 3u, lim[i]) : lim[i];
        gc[i] = (lim[i] - hd[i]) / 4;
        gmax = max(gmax, gc[i]);
    }
    if (bulk) {
        if (threadIdx.x == 0) {
            mbar_init(&s_mbar, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t bytes = 0;
#pragma unroll
            for (int i = 0; i < 5; i++) bytes += 32u * gc[i];
            mbar_expect_tx(&s_mbar, bytes);
#pragma unroll
            for (int i = 0; i < 5; i++)
                if (gc[i]) {
                    const uint32_t o = (uint32_t)i * Ls + sh[i] + hd[i], e = (uint32_t)i * P + j0 + hd[i];
                    bulk_load(u + o, S.err + e, 16u * gc[i], &s_mbar);
                    bulk_load(tt + o, S.t + e, 16u * gc[i], &s_mbar);
                }
        }
        uint32_t jj, i;                                        // heads and tails (< 8 per row)
        if (slice_edge(threadIdx.x - 32u, P, j0, len, n, i, jj)) {
            const uint32_t e = i * P + j0 + jj, o = i * Ls + (((i * P + j0) & 3u)) + jj;
            u[o] = __ldcs(S.err + e);
            tt[o] = ld_stream(S.t + e);
        }
        mbar_wait(&s_mbar, 0);
        __syncthreads();
#pragma unroll
        for (int i = 0; i < 5; i++)
            for (uint32_t jj = threadIdx.x; jj < lim[i]; jj += kGThreads) {
                const uint32_t o = (uint32_t)i * Ls + sh[i] + jj;
                const float x = __fadd_rn(u[o], tt[o]);
                u[o] = x;
                m = max(m, __float_as_uint(x) & 0x7fffffffu);
            }
    } else {
        for (uint32_t k = threadIdx.x; k < gmax; k += kGThreads) {
            float4 tv[5], ev[5];
#pragma unroll
            for (int i = 0; i < 5; i++)
                if (k < gc[i]) {
                    const uint32_t g = ((uint32_t)i * P + j0 + hd[i]) / 4 + k;
                    tv[i] = ld_stream4(reinterpret_cast<const float4 *>(S.t) + g);
                    ev[i] = __ldcs(reinterpret_cast<const float4 *>(S.err) + g);
                }
#pragma unroll
            for (int i = 0; i < 5; i++)
                if (k < gc[i]) {
                    float *d = u + (uint32_t)i * Ls + hd[i] + 4 * k;
                    d[0] = __fadd_rn(ev[i].x, tv[i].x); d[1] = __fadd_rn(ev[i].y, tv[i].y);
                    d[2] = __fadd_rn(ev[i].z, tv[i].z); d[3] = __fadd_rn(ev[i].w, tv[i].w);
                    m = max(m, max(max(__float_as_uint(d[0]) & 0x7fffffffu, __float_as_uint(d[1]) & 0x7fffffffu),
                                   max(__float_as_uint(d[2]) & 0x7fffffffu, __float_as_uint(d[3]) & 0x7fffffffu)));
                }
        }
        if (vec) {                                             // heads and tails: < 4 + 4 per partition
            uint32_t jj, i;
            if (slice_edge(threadIdx.x, P, j0, len, n, i, jj)) {
                const uint32_t e = i * P + j0 + jj;
                const float x = __fadd_rn(__ldcs(S.err + e), ld_stream(S.t + e));
                u[i * Ls + jj] = x;
                m = max(m, __float_as_uint(x) & 0x7fffffffu);
            }
        } else {
            for (uint32_t i = 0; i < 5; i++) {
                const uint32_t e0 = i * P + j0;
                for (uint32_t jj = threadIdx.x; jj < lim[i]; jj += kGThreads) {
                    const float x = __fadd_rn(__ldcs(S.err + e0 + jj), ld_stream(S.t + e0 + jj));
                    u[i * Ls + jj] = x;
                    m = max(m, __float_as_uint(x) & 0x7fffffffu);
                }
            }
        }
    }
    m = block_max_n<kGWarps>(m, s_red);
    K6C_TRACE(1);
    if (AS) {
        asm volatile("barrier.cluster.wait.aligned;" ::: "memory");   // every member's mbarriers are live
        if (idle) return;
        if (threadIdx.x < gcnt) {
            if (threadIdx.x == grank) s_keys[grank] = m;
            else st_async_u32(&s_keys[grank], g0 + threadIdx.x, m, &s_mb_keys);
        }
        mbar_wait(&s_mb_keys, 0);
        __syncthreads();                                       // the local key
    } else {
        // the key to every CTA of the group (its own copy included)
        if (!idle && threadIdx.x < gcnt) dsmem_store_u32(&s_keys[grank], g0 + threadIdx.x, m);
        cluster_sync_all();                                    // 1: the group's keys
        if (idle) {
            cluster_sync_all();
            return;
        }
    }
    K6C_TRACE(2);
    for (uint32_t q = 0; q < gcnt; q++) m = max(m, s_keys[q]);
    float M;
    const unsigned int status = scale_from_key(m, s, M);      // Eq. 1, R6
    const Quant Q(M);
    // ---- Eq. 2, steps (a),(b) in shared memory (u becomes err), quartic steps 1-6
    if (status == TLC_OK) {
        if (Q.mode == 1) slice_quantize(u, B, j0, len, Ls, sh, P, n, QuantCmp(Q));
        else slice_quantize(u, B, j0, len, Ls, sh, P, n, Q);
        if (bulk) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // u rows -> bulk stores
    }
    __syncthreads();
    K6C_TRACE(3);
    // the residuals (steps a, b) from shared memory to err: now (AS) or after the last barrier
    auto store_err = [&]() {
        if (bulk) {
            if (threadIdx.x == 0) {
#pragma unroll
                for (int i = 0; i < 5; i++)
                    if (gc[i]) {
                        const uint32_t o = (uint32_t)i * Ls + sh[i] + hd[i];
                        bulk_store(S.err + (uint32_t)i * P + j0 + hd[i], u + o, 16u * gc[i]);
                    }
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            uint32_t jj, i;
            if (slice_edge(threadIdx.x - 32u, P, j0, len, n, i, jj))
                __stcs(S.err + i * P + j0 + jj, u[i * Ls + ((i * P + j0) & 3u) + jj]);
        } else {
            for (uint32_t k = threadIdx.x; k < gmax; k += kGThreads) {
#pragma unroll
                for (int i = 0; i < 5; i++)
                    if (k < gc[i]) {
                        const float *d = u + (uint32_t)i * Ls + hd[i] + 4 * k;
                        __stcs(reinterpret_cast<float4 *>(S.err) + ((uint32_t)i * P + j0 + hd[i]) / 4 + k,
                               make_float4(d[0], d[1], d[2], d[3]));
                    }
            }
            if (vec) {
                uint32_t jj, i;
                if (slice_edge(threadIdx.x, P, j0, len, n, i, jj)) __stcs(S.err + i * P + j0 + jj, u[i * Ls + jj]);
            } else {
                for (uint32_t i = 0; i < 5; i++)
                    for (uint32_t jj = threadIdx.x; jj < lim[i]; jj += kGThreads)
                        __stcs(S.err + i * P + j0 + jj, u[i * Ls + jj]);
            }
        }
    };
    if (AS && status == TLC_OK) store_err();
    // ---- step (4): run summaries of the slice's rows (one warp per 1 KiB row)
    const uint32_t nrows = (len + kK3WarpRowS - 1) / kK3WarpRowS;
    uint32_t w[8] = {0, 0, 0, 0, 0, 0, 0, 0}, mask = 0;
    int lenl = 0;
    RunSum lane_sum = run_identity();
    uint32_t row_len = 0;
    if (status == TLC_OK && use_zre && (uint32_t)warp < nrows) {
        const uint32_t base = (uint32_t)warp * kK3WarpRowS;
        row_len = min(kK3WarpRowS, len - base);
        const uint32_t rel = base + 32u * lane;
        lenl = rel < len ? (int)min(32u, len - rel) : 0;
        // 32 bytes per lane as two 16-byte loads (B is 16-byte aligned, padded by 32 bytes)
        if (lenl > 0) {
            const uint4 a = *reinterpret_cast<const uint4 *>(B + rel), b = *reinterpret_cast<const uint4 *>(B + rel + 16);
            w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w; w[4] = b.x; w[5] = b.y; w[6] = b.z; w[7] = b.w;
        }
        if (lenl < 32) {
#pragma unroll
            for (int k = 0; k < 8; k++) {
#pragma unroll
                for (int q = 0; q < 4; q++)
                    if (4 * k + q >= lenl) w[k] = (w[k] & ~(0xffu << (8 * q))) | ((uint32_t)kZeroGroup << (8 * q));
            }
        }
        mask = literal_mask(w);
        lane_sum = mask_summary(mask, lenl);
        const RunSum rs = warp_row_summary(mask, lenl, lane_sum, row_len);
        if (lane == 0) s_row[warp] = pack(rs);
    }
    __syncthreads();
    if (threadIdx.x == 0 && use_zre && status == TLC_OK) {    // the slice's summary to the later slices
        RunSum acc = run_identity();
        for (uint32_t r = 0; r < nrows; r++) acc = compose(acc, unpack(s_row[r]));
        const unsigned long long v = pack(acc);
        for (uint32_t q = grank + 1; q < gcnt; q++) {
            if (AS) st_async_u64(&s_aggs[grank], g0 + q, v, &s_mb_aggs);
            else dsmem_store_u64(&s_aggs[grank], g0 + q, v);
        }
    }
    K6C_TRACE(4);
    // the earlier slices' summaries (a failed compress sends none: the whole group has the
    // same key, hence the same status, and nothing is owed to it)
    if (AS) { if (status == TLC_OK) mbar_wait(&s_mb_aggs, 0); }
    else cluster_sync_all();                                   // 2: the earlier slices' summaries
    K6C_TRACE(5);
    const bool last = grank + 1 == gcnt;                       // holds the tensor's last row
    if (status != TLC_OK) {                                    // err untouched (R6)
        if (grank == 0 && threadIdx.x == 0) {
            S.hdr->M = M; S.hdr->flags = use_zre ? TLC_FLAG_ZRE : 0u; S.hdr->n = n;
            S.hdr->payload_len = 0; S.hdr->status = status; S.hdr->reserved = 0;
        }
        return;
    }
    if (!AS) store_err();                                      // err first (bulk: in flight meanwhile)
    if (!use_zre) {
        for (uint32_t jj = threadIdx.x; jj < len; jj += kGThreads) S.payload[j0 + jj] = B[jj];
    } else {
        if (threadIdx.x == 0) {                                // rows in order: offset, carry
            RunSum acc = run_identity();
            for (uint32_t q = 0; q < grank; q++) acc = compose(acc, unpack(s_aggs[q]));
            for (uint32_t r = 0; r <= nrows; r++) {
                uint64_t o;
                uint32_t c;
                run_eval(acc, 0, o, c);
                s_off[r] = (uint32_t)o;
                s_carry[r] = c;
                if (r < nrows) acc = compose(acc, unpack(s_row[r]));
            }
            if (last) S.hdr->payload_len = s_off[nrows] + (s_carry[nrows] > 0);
        }
        __syncthreads();
        if ((uint32_t)warp < nrows) {
            // every lane writes its whole output range [x - count, x): full chunks (255), flush
            // codes and literals in order (no prefill pass, no block barrier)
            const WarpRow wr = warp_row(mask, lenl, lane_sum, s_carry[warp], row_len);
            uint32_t x = wr.count;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
                if (lane >= d) x += y;
            }
            uint8_t *out = S.payload + s_off[warp];
            uint32_t o = x - wr.count, c = wr.carry_in;
            int prev = -1;
            for (uint32_t mk = mask; mk; mk &= mk - 1u) {
                const int q = (int)ctz32(mk);
                const uint32_t R = (uint32_t)(q - prev - 1) + c;
                c = 0;
                for (uint32_t f = R / kMaxRun; f; f--) out[o++] = 0xff;
                TLC_CHECK(s_off[warp] + o + (R % kMaxRun ? 1 : 0) < P);
                if (R % kMaxRun) out[o++] = run_code(R % kMaxRun);
                uint32_t word = w[0];
#pragma unroll
                for (int k = 1; k < 8; k++) word = (k == (q >> 2)) ? w[k] : word;
                out[o++] = (uint8_t)(word >> (8 * (q & 3)));
                prev = q;
            }
            while (o < x) out[o++] = 0xff;                     // chunks completed in the trailing run
        }
        if (last && threadIdx.x == 0 && s_carry[nrows] > 0) {
            TLC_CHECK(s_off[nrows] < P);
            S.payload[s_off[nrows]] = run_code(s_carry[nrows]);
        }
    }
    if (grank == 0 && threadIdx.x == 0) {
        tlc_header *h = S.hdr;
        h->M = M;
        h->flags = use_zre ? TLC_FLAG_ZRE : 0u;
        h->n = n;
        if (!use_zre) h->payload_len = P;
        h->status = status;
        h->reserved = 0;
    }
    if (bulk && threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");   // smem in use
    K6C_TRACE(6);
}

// TLC_K6G=0 keeps one CTA per tensor (K6); 4 (default): clusters of 4, slices of <= 2 rows;
// 8: clusters of 8, slices of 1 row (A/B)
static int group_mode() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("TLC_K6G");
        v = e ? atoi(e) : 4;
        if (v != 0 && v != 4 && v != 8 && v != 2) v = 4;
    }
    return v;
}

int small_group_plan_build(SegTable &T, const std::vector<Seg> &host, GrpRec **d_grp, std::vector<uint4> &layout) {
    T.grp = nullptr;
    const int CL = group_mode();
    if (CL == 0) return TLC_OK;
    const uint32_t max_rows = CL == 8 ? 1u : 2u;               // rows per slice
    struct Group { int seg; uint32_t k; };
    std::vector<Group> groups;
    for (int i = 0; i < (int)host.size(); i++) {
        const uint32_t rows = (uint32_t)((host[i].P + kK3WarpRowS - 1) / kK3WarpRowS);
        const uint32_t k = std::min<uint32_t>((uint32_t)CL, (rows + max_rows - 1) / max_rows);
        groups.push_back({i, std::max<uint32_t>(k, 1u)});
    }
    std::stable_sort(groups.begin(), groups.end(), [](const Group &a, const Group &b) { return a.k > b.k; });
    // best fit: open clusters by free slots
    std::vector<std::vector<uint4>> clusters;
    std::vector<std::vector<int>> open(CL + 1);              // open[f]: clusters with f free slots
    uint32_t max_len = 0;
    for (const Group &g : groups) {
        int c = -1;
        for (int f = (int)g.k; f < CL && c < 0; f++)
            if (!open[f].empty()) { c = open[f].back(); open[f].pop_back(); }
        if (c < 0) { c = (int)clusters.size(); clusters.emplace_back(); }
        std::vector<uint4> &cl = clusters[c];
        const Seg &S = host[g.seg];
        const uint32_t P = (uint32_t)S.P, rows = (P + kK3WarpRowS - 1) / kK3WarpRowS;
        const uint32_t base = rows / g.k, extra = rows % g.k, first = (uint32_t)cl.size();
        uint32_t r0 = 0;
        for (uint32_t q = 0; q < g.k; q++) {
            const uint32_t nr = base + (q < extra ? 1u : 0u);
            const uint32_t j0 = r0 * kK3WarpRowS, j1 = std::min(P, (r0 + nr) * kK3WarpRowS);
            cl.push_back(make_uint4((uint32_t)g.seg, j0, j1 - j0, first | (g.k << 8) | (q << 16)));
            max_len = std::max(max_len, j1 - j0);
            r0 += nr;
        }
        const int f = CL - (int)cl.size();
        if (f > 0) open[f].push_back(c);
    }
    layout.clear();
    for (auto &cl : clusters) {
        for (const uint4 &r : cl) layout.push_back(r);
        for (size_t q = cl.size(); q < (size_t)CL; q++) layout.push_back(make_uint4(~0u, 0, 0, 0));
    }
    if (cudaMalloc((void **)d_grp, layout.size() * sizeof(GrpRec)) != cudaSuccess) return TLC_ERR_CUDA;
    T.grp = *d_grp;
    T.grp_grid = (int)layout.size();
    T.grp_cl = CL;
    T.grp_maxlen = max_len;
    return TLC_OK;
}

int small_group_plan_refresh(const SegTable &T, const std::vector<Seg> &host, const std::vector<uint4> &layout) {
    std::vector<GrpRec> recs(layout.size());
    for (size_t c = 0; c < layout.size(); c++) {
        const uint4 &l = layout[c];
        GrpRec &r = recs[c];
        r = GrpRec{};
        r.seg = l.x;
        if (l.x == ~0u) continue;
        const Seg &S = host[l.x];
        r.t = S.t; r.err = S.err; r.payload = S.payload; r.hdr = S.hdr;
        r.n = (uint32_t)S.n; r.P = (uint32_t)S.P; r.j0 = l.y; r.len = l.z;
        r.g0 = l.w & 0xffu; r.gcnt = (l.w >> 8) & 0xffu; r.grank = (l.w >> 16) & 0xffu;
    }
    return cudaMemcpy(const_cast<GrpRec *>(T.grp), recs.data(), recs.size() * sizeof(GrpRec),
                      cudaMemcpyHostToDevice) == cudaSuccess ? TLC_OK : TLC_ERR_CUDA;
}

// TLC_K6G_BULK=1: K6g moves t and err in by bulk copies and err out by bulk stores instead
// of through registers (A/B: 19.3 vs 20.1 us cold at s = 1.75 in favour of registers,
// profiles/r03t_c2.txt; cp.async 16-byte copies were slower than both, r03r)
static bool group_bulk() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("TLC_K6G_BULK");
        v = (e && e[0] == '1') ? 1 : 0;
    }
    return v == 1;
}

// TLC_K6G_SYNC=1: K6g's two cluster barriers instead of st.async + mbarriers (A/B)
static bool group_async() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("TLC_K6G_SYNC");
        v = (e && e[0] == '1') ? 0 : 1;
    }
    return v == 1;
}

template <int CL, bool BULK, bool AS>
static int launch_group(const SegTable &T, float s, int use_zre, cudaStream_t st) {
    // u (and the T_in rows when copied in bulk), then B
    const uint32_t smem = (BULK ? 2u : 1u) * 4u * 5u * (((T.grp_maxlen + 3) & ~3u) + 4u) + T.grp_maxlen + 64u;
    static uint32_t attr[64] = {};                             // per device (tlc_launch.h PerDevice)
    const int dv = cur_device();
    if (smem > attr[dv]) {
        cudaFuncSetAttribute(tlc_small_group_compress_kernel<CL, BULK, AS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        attr[dv] = smem;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(T.grp_grid);
    cfg.blockDim = dim3(kGThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = CL;
    a[0].val.clusterDim.y = 1;
    a[0].val.clusterDim.z = 1;
    cfg.attrs = a;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, tlc_small_group_compress_kernel<CL, BULK, AS>, T, s, use_zre) == cudaSuccess
               ? TLC_OK : TLC_ERR_CUDA;
}

// ============================================================== K6c
// The small-table compressor as ONE cooperative launch over all SMs (tables of many
// small tensors: the 110 ResNet-110 layers).  K6 gave each tensor one CTA, so the 35
// tensors of 36,864 values each streamed ~440 KB through a single SM (22 us, DRAM 9 %).
// Here every tensor is cut into slices of kSlice quartic positions (5 * kSlice values),
// the slices are dealt to the CTAs in contiguous runs of about equal size, and the method
// runs in three phases separated by two grid barriers:
//   A  t and err of the CTA's slices -> shared memory with cp.async (every load in
//      flight at once), u = err + t (step 1), the max key of each slice, atomicMax into
//      its tensor's key (Eq. 1 needs the whole tensor's max);
//   B  M per tensor (Eq. 1, R6), quantize from shared memory writing err (Eq. 2, steps
//      a, b), quartic bytes into shared memory (step 3), the run summary of every slice
//      (one warp per slice) published for its tensor's later slices;
//   C  each slice composes the summaries of its tensor's earlier slices (<= 15) into
//      its output offset and carry and emits its zero-run bytes (step 4) through a
//      255-prefilled stage; the tensor's last slice writes the length.
// Results are identical to K6 / K1-K5 (the payload, err and header are defined by the
// method).  A tensor's key is reset to 0 after barrier 2 for the next launch.
constexpr uint32_t kSlice = 512;                        // quartic positions per slice
constexpr int kSlots = kSmWarps;                        // <= 16 slices per CTA (one warp each)
constexpr uint32_t kStage = 544;                        // per-warp padded stage: <= kSlice + 1 bytes + 3
static_assert(kStage >= pad_stage_bytes(kSlice + 1 + 3), "a slice's output fits the stage");

// All CTAs of the (cooperative) launch: arrive, then wait until every CTA has arrived.
// The counter only grows; each barrier waits for the next multiple of the grid size.
__device__ __forceinline__ void grid_barrier(unsigned long long *ctr) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned long long G = gridDim.x;
        const unsigned long long old = atomicAdd(ctr, 1ull);
        const unsigned long long target = (old / G + 1) * G;
        unsigned long long v;
        do {
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
        } while (v < target);
    }
    __syncthreads();
}

// Phase A's copy of one partition row of a slice: elements [i*P + j0, +m) of t (or err),
// fetched as the 16-byte-aligned superset of its bytes (a bulk copy needs 16-byte
// addresses and sizes; the granules around a valid byte lie in the same mapped page).
struct RowCopy {
    uint32_t dst, bytes, shift;      // smem byte offset, superset bytes, elements before the row
};
__device__ __forceinline__ RowCopy row_copy(const float *base, uint32_t e0, uint32_t m, uint32_t dst) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(base + e0), a0 = a & ~uintptr_t(15);
    const uintptr_t a1 = (a + 4ull * m + 15) & ~uintptr_t(15);
    return RowCopy{dst, (uint32_t)(a1 - a0), (uint32_t)((a - a0) >> 2)};
}
// bytes one slice row can take in the stage: 4 * kSlice + two partial granules
constexpr uint32_t kRowBytes = 4 * kSlice + 32;


__global__ void __launch_bounds__(kSmThreads, 1)
tlc_small_coop_compress_kernel(const SegTable T, float s, int use_zre) {
    extern __shared__ __align__(16) uint8_t sm_raw[];        // bulk-copy destinations: 16-byte aligned
    __shared__ SliceRec s_sl[kSlots];
    __shared__ uint32_t s_row[kSlots][5][2];               // t / err row: smem offset (bytes) | shift << 24
    __shared__ unsigned int s_key[kSlots];
    __shared__ float s_M[kSlots];
    __shared__ unsigned int s_st[kSlots];
    __shared__ __align__(8) unsigned long long s_bar;
    K6C_TRACE(0);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t c0 = T.sl_cta[blockIdx.x], ns = T.sl_cta[blockIdx.x + 1] - c0;
    // the CTA's slice records (pointers included) in one round trip
    if (threadIdx.x < ns * (sizeof(SliceRec) / 16))
        reinterpret_cast<uint4 *>(s_sl)[threadIdx.x] = reinterpret_cast<const uint4 *>(T.sl + c0)[threadIdx.x];
    if (threadIdx.x < kSlots) s_key[threadIdx.x] = 0;
    if (threadIdx.x == 0) {
        mbar_init(&s_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint8_t *stage = sm_raw + (size_t)ns * 10 * kRowBytes + (size_t)warp * kStage;
    uint8_t *Bs = sm_raw + (size_t)ns * 10 * kRowBytes + kSmWarps * kStage;   // kSlots x kSlice quartic bytes

    // ---- A: every row of t and err of every slice with one bulk copy each (the copy
    // engine keeps them all in flight); u = err + t; per-slice max keys
    if (threadIdx.x == 0) {
        uint32_t total = 0;
        for (uint32_t r = 0; r < ns * 10; r++) {
            const SliceRec &sl = s_sl[r / 10];
            const uint32_t i = (r % 10) >> 1, e0 = i * sl.P + sl.j0;
            const uint32_t m = e0 < sl.n ? min(sl.len, sl.n - e0) : 0u;
            const RowCopy rc = m ? row_copy((r & 1) ? sl.err : sl.t, e0, m, r * kRowBytes) : RowCopy{r * kRowBytes, 0u, 0u};
            s_row[r / 10][i][r & 1] = rc.dst | (rc.shift << 24);
            total += rc.bytes;
        }
        mbar_expect_tx(&s_bar, total);
    }
    __syncthreads();
    if (threadIdx.x < ns * 10) {
        const uint32_t r = threadIdx.x;
        const SliceRec &sl = s_sl[r / 10];
        const uint32_t i = (r % 10) >> 1, e0 = i * sl.P + sl.j0;
        const uint32_t m = e0 < sl.n ? min(sl.len, sl.n - e0) : 0u;
        if (m) {
            const float *src = (r & 1) ? sl.err : sl.t;
            const RowCopy rc = row_copy(src, e0, m, r * kRowBytes);
            bulk_load(sm_raw + rc.dst, reinterpret_cast<const void *>(reinterpret_cast<uintptr_t>(src + e0) & ~uintptr_t(15)),
                      rc.bytes, &s_bar);
        }
    }
    mbar_wait(&s_bar, 0);
    K6C_TRACE(1);
    const uint32_t jj = threadIdx.x;                        // thread j: quartic position j0 + j of each slice
    static_assert(kSlice == kSmThreads, "one quartic position per thread and slice");
    for (uint32_t k = 0; k < ns; k++) {
        const SliceRec &sl = s_sl[k];
        unsigned int m = 0;
        if (jj < sl.len) {
#pragma unroll
            for (uint32_t i = 0; i < 5; i++) {
                const uint32_t e = i * sl.P + sl.j0 + jj;
                float *tu = reinterpret_cast<float *>(sm_raw + (s_row[k][i][0] & 0xffffffu)) + (s_row[k][i][0] >> 24) + jj;
                float x = 0.0f;                                   // pad positions: digit 0 below
                if (e < sl.n) {
                    const float ev = reinterpret_cast<const float *>(sm_raw + (s_row[k][i][1] & 0xffffffu))[(s_row[k][i][1] >> 24) + jj];
                    x = __fadd_rn(ev, *tu);                       // step (1)
                    m = max(m, __float_as_uint(x) & 0x7fffffffu);
                }
                *tu = x;                                          // u replaces t in place
            }
        }
        m = __reduce_max_sync(0xffffffffu, m);
        if (lane == 0 && m) atomicMax(&s_key[k], m);
    }
    __syncthreads();
    if (threadIdx.x < ns && s_key[threadIdx.x]) atomicMax(T.sl_key + s_sl[threadIdx.x].seg, s_key[threadIdx.x]);
    K6C_TRACE(2);
    grid_barrier(T.sl_bar);
    K6C_TRACE(3);

    // ---- B: M (Eq. 1), quantization + residual (Eq. 2, steps a, b), quartic bytes (step 3)
    if (threadIdx.x < ns) {
        float M;
        s_st[threadIdx.x] = scale_from_key(__ldcg(T.sl_key + s_sl[threadIdx.x].seg), s, M);
        s_M[threadIdx.x] = M;
    }
    __syncthreads();
    for (uint32_t k = 0; k < ns; k++) {
        const SliceRec &sl = s_sl[k];
        const unsigned int st = s_st[k];
        if (sl.k == 0 && threadIdx.x == 0) {                      // the tensor's first slice: header
            tlc_header *h = sl.hdr;
            h->M = s_M[k];
            h->flags = use_zre ? TLC_FLAG_ZRE : 0u;
            h->n = sl.n;
            h->status = st;
            h->reserved = 0;
            if (!use_zre || st != TLC_OK) h->payload_len = (st == TLC_OK) ? sl.P : 0;
        }
        if (st != TLC_OK) continue;                               // err untouched (R6)
        const Quant Q(s_M[k]);
        if (jj < sl.len) {
            uint32_t b = 0;
#pragma unroll
            for (int i = 0; i < 5; i++) {
                const uint32_t e = (uint32_t)i * sl.P + sl.j0 + jj;
                uint32_t d = 0;                                   // pad digit (R10)
                if (e < sl.n) {
                    const float x = reinterpret_cast<const float *>(sm_raw + (s_row[k][i][0] & 0xffffffu))[(s_row[k][i][0] >> 24) + jj];
                    const int q = Q.q(x);                         // Eq. 2
                    __stcs(sl.err + e, Q.residual(x, q));         // steps (a), (b)
                    d = (uint32_t)(q + 1);
                }
                b = b * 3u + d;                                   // steps 1, 4, 6
            }
            Bs[k * kSlice + jj] = (uint8_t)b;
            if (!use_zre) sl.payload[sl.j0 + jj] = (uint8_t)b;
        }
    }
    __syncthreads();
    // run summary of slice `warp` (one warp row of <= kSlice bytes), kept in registers for C
    uint32_t w[8] = {0, 0, 0, 0, 0, 0, 0, 0}, mask = 0;
    int len_l = 0;
    RunSum lane_sum = run_identity();
    const bool mine = use_zre && (uint32_t)warp < ns && s_st[warp] == TLC_OK;
    uint32_t row_len = 0;
    if (mine) {
        row_len = s_sl[warp].len;
        const uint32_t rel = 32u * lane;
        len_l = rel < row_len ? (int)min(32u, row_len - rel) : 0;
#pragma unroll
        for (int k = 0; k < 8; k++) {
            uint32_t x = 0;
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const int mm = 4 * k + q;
                x |= (uint32_t)(mm < len_l ? Bs[warp * kSlice + rel + mm] : kZeroGroup) << (8 * q);
            }
            w[k] = x;
        }
        mask = literal_mask(w);
        lane_sum = mask_summary(mask, len_l);
        const RunSum rs = warp_row_summary(mask, len_l, lane_sum, row_len);
        if (lane == 0) st_relaxed_u64(T.sl_sum + c0 + warp, pack(rs));
    }
    K6C_TRACE(4);
    grid_barrier(T.sl_bar);
    K6C_TRACE(5);

    // ---- C: offsets from the tensor's earlier slices, zero-run emission (step 4)
    if (mine) {
        const SliceRec &sl = s_sl[warp];
        const uint32_t kk = sl.k;
        const unsigned long long pv = lane < (int)kk ? ld_relaxed_u64(T.sl_sum + sl.first + lane) : 0ull;
        RunSum acc = lane < (int)kk ? unpack(pv) : run_identity();
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {                      // in-order tree: lane 0 = slices 0..kk-1
            const RunSum o = unpack(__shfl_down_sync(0xffffffffu, pack(acc), d));
            if (lane + d < 32) acc = compose(acc, o);
        }
        acc = unpack(__shfl_sync(0xffffffffu, pack(acc), 0));
        uint64_t o0;
        uint32_t c_in;
        run_eval(acc, 0, o0, c_in);
        const WarpRow wr = warp_row(mask, len_l, lane_sum, c_in, row_len);
        uint32_t x = wr.count;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
            if (lane >= d) x += y;
        }
        uint8_t *out = sl.payload + o0;
        const uint32_t sh = (uint32_t)(reinterpret_cast<uintptr_t>(out) & 3u);
        const PadStage pst{stage, kStage};
        TLC_CHECK(o0 + wr.row_count + (sl.last && wr.carry_out > 0) <= sl.P);
        pad_stage_fill(pst, sh + wr.row_count);
        __syncwarp();
        lane_emit(w, mask, wr.carry_in, pst, sh + x - wr.count);
        __syncwarp();
        warp_copy_padded(out, pst, sh, wr.row_count);
        if (sl.last && lane == 0) {                              // the tensor's last slice
            if (wr.carry_out > 0) out[wr.row_count] = run_code(wr.carry_out);
            sl.hdr->payload_len = o0 + wr.row_count + (wr.carry_out > 0);
        }
    }
    // every read of the keys happened before barrier 2: reset them for the next launch
    if (threadIdx.x < ns && s_sl[threadIdx.x].k == 0) T.sl_key[s_sl[threadIdx.x].seg] = 0;
    __syncthreads();
    K6C_TRACE(6);
}

int small_plan_build(SegTable &T, const std::vector<Seg> &host, void **d_small, std::vector<uint4> &layout) {
    // slices in segment order, then contiguous runs of about total/G values per CTA
    layout.clear();
    std::vector<uint32_t> w;                                      // values per slice
    std::vector<uint32_t> first;
    for (int si = 0; si < (int)host.size(); si++) {
        const Seg &S = host[si];
        const uint32_t P = (uint32_t)S.P, nsl = (P + kSlice - 1) / kSlice;
        for (uint32_t k = 0; k < nsl; k++) {
            const uint32_t j0 = k * kSlice, len = min(kSlice, P - j0);
            layout.push_back(make_uint4((uint32_t)si, j0, len, k | ((k + 1 == nsl ? 1u : 0u) << 16)));
            w.push_back(5 * len);
        }
    }
    const int G = (int)tmin<uint64_t>((uint64_t)num_sms(), layout.size());
    uint64_t total = 0;
    for (uint32_t x : w) total += x;
    std::vector<uint32_t> cta(G + 1, 0);
    uint64_t acc = 0;
    int g = 0;
    for (size_t k = 0; k < layout.size(); k++) {
        // open the next CTA's run once this one has reached its share (and slices remain)
        while (g + 1 < G && acc >= (total * (uint64_t)(g + 1)) / G && cta[g + 1] == 0 && k > cta[g]) cta[++g] = (uint32_t)k;
        acc += w[k];
    }
    for (int q = g + 1; q <= G; q++) cta[q] = (uint32_t)layout.size();
    uint32_t max_ns = 0;
    for (int q = 0; q < G; q++) max_ns = max(max_ns, cta[q + 1] - cta[q]);
    if (max_ns > (uint32_t)kSlots) { layout.clear(); return TLC_OK; }   // too many slices per CTA: K6
    const size_t smem = (size_t)max_ns * 10 * kRowBytes + kSmWarps * kStage + kSlots * kSlice;
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (smem + 4096 > (size_t)optin) { layout.clear(); return TLC_OK; }   // does not fit: K6
    const size_t b_sl = align256(layout.size() * sizeof(SliceRec)), b_cta = align256((G + 1) * sizeof(uint32_t));
    const size_t b_key = align256(host.size() * sizeof(unsigned int));
    const size_t b_sum = align256(layout.size() * sizeof(unsigned long long)), b_bar = 256;
    char *d = nullptr;
    if (cudaMalloc((void **)&d, b_sl + b_cta + b_key + b_sum + b_bar) != cudaSuccess) return TLC_ERR_CUDA;
    *d_small = d;
    if (cudaMemcpy(d + b_sl, cta.data(), cta.size() * sizeof(uint32_t), cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemset(d + b_sl + b_cta, 0, b_key + b_sum + b_bar) != cudaSuccess)
        return TLC_ERR_CUDA;
    T.sl = reinterpret_cast<const SliceRec *>(d);
    T.sl_cta = reinterpret_cast<const uint32_t *>(d + b_sl);
    T.sl_key = reinterpret_cast<unsigned int *>(d + b_sl + b_cta);
    T.sl_sum = reinterpret_cast<unsigned long long *>(d + b_sl + b_cta + b_key);
    T.sl_bar = reinterpret_cast<unsigned long long *>(d + b_sl + b_cta + b_key + b_sum);
    T.sl_grid = G;
    T.sl_smem = (uint32_t)smem;
    return TLC_OK;
}

int small_plan_refresh(const SegTable &T, const std::vector<Seg> &host, const std::vector<uint4> &layout) {
    std::vector<SliceRec> rec(layout.size());
    uint32_t first = 0;
    for (size_t q = 0; q < layout.size(); q++) {
        const uint4 &L = layout[q];
        const Seg &S = host[L.x];
        if ((L.w & 0xffffu) == 0) first = (uint32_t)q;
        rec[q] = SliceRec{S.t, S.err, S.payload, S.hdr, (uint32_t)S.n, (uint32_t)S.P, L.y, L.z,
                          first, L.w & 0xffffu, L.w >> 16, L.x};
    }
    return cudaMemcpy(const_cast<SliceRec *>(T.sl), rec.data(), rec.size() * sizeof(SliceRec),
                      cudaMemcpyHostToDevice) == cudaSuccess ? TLC_OK : TLC_ERR_CUDA;
}

// K6c is opt-in (TLC_COOP=1): on the ResNet-110 table it measured 31 us against K6's 22 us
// (tools/k6c_trace.py: every phase takes 3-5 us)
bool small_coop_enabled() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("TLC_COOP");
        v = (e && e[0] == '1') ? 1 : 0;
    }
    return v == 1;
}

// A tensor's decode is split into parts of kSmPart >> sub_log2 quartic positions, one CTA
// each (the 36,864-value ResNet-110 tensors would otherwise keep one SM busy while most
// idle; one SM stores at most ~61 GB/s, profiles/r03l_sm_bw.txt): every part scans the
// whole payload (<= P bytes, on chip) and expands / decodes only its range.
constexpr uint32_t kSmPart = (uint32_t)kT5;   // the K5 tile: parts are numbered like K5's tiles (Seg::k5)

template <int kMode>
__global__ void __launch_bounds__(kSmThreads)
tlc_small_decompress_kernel(const SegTable T, int sub_log2) {
    extern __shared__ __align__(16) uint8_t sm_raw[];
    __shared__ uint16_t dig[256];                                // digit_i(b) at bits 2i
    __shared__ uint32_t s_wsum[kSmWarps + 1];
    __shared__ int s_bad;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // exactly the parts that exist (K5's tile numbering): no CTA for the empty parts of the
    // smaller tensors (round 1 launched count x max-parts CTAs, most of them idle)
    __shared__ uint64_t s_first[kSegCache];
    seg_index_load<5>(T, s_first);
    bool table = false;
    const uint32_t sub_len = kSmPart >> sub_log2;
    for (uint64_t it = blockIdx.x; it < (T.n5 << sub_log2); it += gridDim.x) {
        const uint64_t item = it >> sub_log2;                    // K5 tile, and the sub-part of it
        const uint32_t sub = (uint32_t)(it & ((1u << sub_log2) - 1u));
        const int si = find_seg_c<5>(T, item, s_first);
        const Seg S = get_seg(T, si);
        const uint32_t part = (uint32_t)(item - S.k5) * (1u << sub_log2) + sub;
        tlc_header *hdr = S.hdr;
        const uint32_t jr0 = part * sub_len;
        if (jr0 >= S.P) continue;                                // no positions in this part
        const bool hv = header_valid(hdr, S.n);
        if (!table) {
            // Decoding step 1 for the 243 byte values, once per CTA (no dependence on M), built
            // while the segment and header loads above are in flight: Eq. 3 is then
            // M * (d - 1) in {-M, +0, M}, taken by selection (the same bits as the product)
            for (int v = threadIdx.x; v < 256; v += kSmThreads) {
                uint32_t r = v < 243 ? v : 121, pk = 0;
#pragma unroll
                for (int i = 4; i >= 0; i--) {
                    pk |= (r % 3u) << (2 * i);
                    r /= 3u;
                }
                dig[v] = (uint16_t)pk;
            }
            __syncthreads();
            table = true;
        }
        if (!hv) {                                               // uniform over the CTA
            if (threadIdx.x == 0 && part == 0 && hdr->status == TLC_OK) raise_format(hdr);
            continue;
        }
        const uint32_t n = (uint32_t)S.n, P = (uint32_t)S.P, Z = (uint32_t)hdr->payload_len;
        const uint32_t jr1 = min(P, jr0 + sub_len), pl = jr1 - jr0;
        const bool zre = (hdr->flags & TLC_FLAG_ZRE) != 0;
        const float M = hdr->M, negM = -M;
        uint8_t *E = sm_raw;                                     // quartic bytes [jr0, jr1)
        if (threadIdx.x == 0) s_bad = 0;
        if (zre) {
            // this thread's 16 payload bytes straight to registers (one 16-byte load when
            // aligned), expansion lengths by SWAR, block exclusive scan
            constexpr int kPer = 16;
            static_assert((kSmallMaxN + 4) / 5 <= kPer * kSmThreads, "every payload byte has a thread");
            const uint32_t b0 = kPer * threadIdx.x;
            uint32_t wv[4] = {0, 0, 0, 0}, lens = 0;
            if (b0 + kPer <= Z && aligned16(S.payload)) {
                const uint4 v = __ldg(reinterpret_cast<const uint4 *>(S.payload + b0));
                wv[0] = v.x; wv[1] = v.y; wv[2] = v.z; wv[3] = v.w;
                lens = word_len(wv[0]) + word_len(wv[1]) + word_len(wv[2]) + word_len(wv[3]);
            } else {
#pragma unroll
                for (int k = 0; k < kPer; k++)
                    if (b0 + k < Z) {
                        const uint32_t b = S.payload[b0 + k];
                        wv[k >> 2] |= b << (8 * (k & 3));
                        lens += zre_len(b);
                    }
            }
            uint32_t x = lens;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
                if (lane >= d) x += y;
            }
            if (lane == 31) s_wsum[warp] = x;
            for (uint32_t q = 16 * threadIdx.x; q < pl; q += 16 * kSmThreads) {   // 121 prefill
                if (q + 16 <= pl) *reinterpret_cast<uint4 *>(E + q) = make_uint4(0x79797979u, 0x79797979u,
                                                                                 0x79797979u, 0x79797979u);
                else for (uint32_t r = q; r < pl; r++) E[r] = kZeroGroup;
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                uint32_t acc = 0;
                for (int k = 0; k < kSmWarps; k++) { const uint32_t v = s_wsum[k]; s_wsum[k] = acc; acc += v; }
                s_wsum[kSmWarps] = acc;
                if (acc != P) s_bad = 1;
            }
            __syncthreads();
            if (s_bad) {
                if (threadIdx.x == 0 && part == 0) raise_format(hdr);
                __syncthreads();
                continue;
            }
            uint32_t p = s_wsum[warp] + x - lens;
            if (p < jr1 && p + lens > jr0) {
#pragma unroll
                for (int k = 0; k < kPer; k++) {
                    const uint32_t b = (wv[k >> 2] >> (8 * (k & 3))) & 0xffu;
                    if (b0 + k < Z && b < kFirstRunCode && p >= jr0 && p < jr1) E[p - jr0] = (uint8_t)b;   // literal
                    p += b0 + k < Z ? zre_len(b) : 0u;
                }
            }
        } else {
            for (uint32_t q = threadIdx.x; q < pl; q += kSmThreads) {
                const uint8_t b = S.payload[jr0 + q];
                if (b > 242) s_bad = 1;
                E[q] = b;
            }
            __syncthreads();
            if (s_bad) {
                if (threadIdx.x == 0) raise_format(hdr);
                __syncthreads();
                continue;
            }
        }
        __syncthreads();
        // ---- decoding steps 1-4 and Eq. 3: out = M * (d - 1) (bits of the fp32 product)
        for (uint32_t jl = threadIdx.x; jl < pl; jl += kSmThreads) {
            const uint32_t pk = dig[E[jl]];
#pragma unroll
            for (int i = 0; i < 5; i++) {
                const uint32_t e = (uint32_t)(i * P) + jr0 + jl;
                if (e >= n) break;
                const uint32_t d = (pk >> (2 * i)) & 3u;
                const float v = d == 2u ? M : (d == 0u ? negM : 0.0f);
                if (kMode == TLC_MODE_OVERWRITE) __stcs(S.out + e, v);
                else if (d != 1u) S.out[e] = __fadd_rn(S.out[e], v);   // q != 0 (R16)
            }
        }
        __syncthreads();                                         // E reuse
    }
}

// K7 over per-CTA records (default for small tables): the CTA's part, pointers and sizes
// in one 48-byte record, so the header load is the first global access instead of the third
// (no first-item table, no segment descriptor); otherwise the same steps as above.
template <int kMode>
__global__ void __launch_bounds__(kSmThreads)
tlc_small_decompress_rec_kernel(const SegTable T) {
    extern __shared__ __align__(16) uint8_t sm_raw[];
    __shared__ uint16_t dig[256];                                // digit_i(b) at bits 2i
    __shared__ uint32_t s_wsum[kSmWarps + 1];
    __shared__ int s_bad;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const DecRec R = T.dec[blockIdx.x];
    tlc_header *hdr = R.hdr;
    const uint32_t n = R.n, P = R.P, jr0 = R.jr0, pl = R.pl;
    const bool hv = header_valid(hdr, n);
    // decoding step 1 for the 243 byte values while the header is in flight (as above)
    for (int v = threadIdx.x; v < 256; v += kSmThreads) {
        uint32_t r = v < 243 ? v : 121, pk = 0;
#pragma unroll
        for (int i = 4; i >= 0; i--) {
            pk |= (r % 3u) << (2 * i);
            r /= 3u;
        }
        dig[v] = (uint16_t)pk;
    }
    if (threadIdx.x == 0) s_bad = 0;
    __syncthreads();
    if (!hv) {                                                   // uniform over the CTA
        if (threadIdx.x == 0 && R.first && hdr->status == TLC_OK) raise_format(hdr);
        return;
    }
    const uint32_t Z = (uint32_t)hdr->payload_len, jr1 = jr0 + pl;
    const bool zre = (hdr->flags & TLC_FLAG_ZRE) != 0;
    const float M = hdr->M, negM = -M;
    uint8_t *E = sm_raw;                                         // quartic bytes [jr0, jr1)
    if (zre) {
        constexpr int kPer = 16;
        const uint32_t b0 = kPer * threadIdx.x;
        uint32_t wv[4] = {0, 0, 0, 0}, lens = 0;
        if (b0 + kPer <= Z && aligned16(R.payload)) {
            const uint4 v = __ldg(reinterpret_cast<const uint4 *>(R.payload + b0));
            wv[0] = v.x; wv[1] = v.y; wv[2] = v.z; wv[3] = v.w;
            lens = word_len(wv[0]) + word_len(wv[1]) + word_len(wv[2]) + word_len(wv[3]);
        } else {
#pragma unroll
            for (int k = 0; k < kPer; k++)
                if (b0 + k < Z) {
                    const uint32_t b = R.payload[b0 + k];
                    wv[k >> 2] |= b << (8 * (k & 3));
                    lens += zre_len(b);
                }
        }
        uint32_t x = lens;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
            if (lane >= d) x += y;
        }
        if (lane == 31) s_wsum[warp] = x;
        for (uint32_t q = 16 * threadIdx.x; q < pl; q += 16 * kSmThreads) {   // 121 prefill
            if (q + 16 <= pl) *reinterpret_cast<uint4 *>(E + q) = make_uint4(0x79797979u, 0x79797979u,
                                                                             0x79797979u, 0x79797979u);
            else for (uint32_t r = q; r < pl; r++) E[r] = kZeroGroup;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t acc = 0;
            for (int k = 0; k < kSmWarps; k++) { const uint32_t v = s_wsum[k]; s_wsum[k] = acc; acc += v; }
            s_wsum[kSmWarps] = acc;
            if (acc != P) s_bad = 1;
        }
        __syncthreads();
        if (s_bad) {
            if (threadIdx.x == 0 && R.first) raise_format(hdr);
            return;
        }
        uint32_t p = s_wsum[warp] + x - lens;
        if (p < jr1 && p + lens > jr0) {
#pragma unroll
            for (int k = 0; k < kPer; k++) {
                const uint32_t b = (wv[k >> 2] >> (8 * (k & 3))) & 0xffu;
                if (b0 + k < Z && b < kFirstRunCode && p >= jr0 && p < jr1) E[p - jr0] = (uint8_t)b;   // literal
                p += b0 + k < Z ? zre_len(b) : 0u;
            }
        }
    } else {
        for (uint32_t q = threadIdx.x; q < pl; q += kSmThreads) {
            const uint8_t b = R.payload[jr0 + q];
            if (b > 242) s_bad = 1;
            E[q] = b;
        }
        __syncthreads();
        if (s_bad) {
            if (threadIdx.x == 0) raise_format(hdr);
            return;
        }
    }
    __syncthreads();
    // ---- decoding steps 1-4 and Eq. 3: out = M * (d - 1) (bits of the fp32 product)
    for (uint32_t jl = threadIdx.x; jl < pl; jl += kSmThreads) {
        const uint32_t pk = dig[E[jl]];
#pragma unroll
        for (int i = 0; i < 5; i++) {
            const uint32_t e = (uint32_t)(i * P) + jr0 + jl;
            if (e >= n) break;
            const uint32_t d = (pk >> (2 * i)) & 3u;
            const float v = d == 2u ? M : (d == 0u ? negM : 0.0f);
            if (kMode == TLC_MODE_OVERWRITE) __stcs(R.out + e, v);
            else if (d != 1u) R.out[e] = __fadd_rn(R.out[e], v);   // q != 0 (R16)
        }
    }
}

// TLC_K7_REC=0: K7 walks the segment table instead of taking per-CTA records (A/B)
static bool dec_rec_enabled() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("TLC_K7_REC");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1;
}

int small_dec_plan_build(SegTable &T, const std::vector<Seg> &host, DecRec **d_dec, std::vector<uint4> &layout) {
    T.dec = nullptr;
    if (!dec_rec_enabled()) return TLC_OK;
    // 2048 positions per CTA (as sub_log2 = 1); TLC_K7_PART=1024 / 4096 for A/B
    const char *pe = getenv("TLC_K7_PART");
    const uint32_t part = pe && (atoi(pe) == 1024 || atoi(pe) == 4096) ? (uint32_t)atoi(pe) : kSmPart >> 1;
    layout.clear();
    for (size_t i = 0; i < host.size(); i++) {
        const uint32_t P = (uint32_t)host[i].P;
        for (uint32_t j = 0; j < P; j += part) layout.push_back(make_uint4((uint32_t)i, j, std::min(part, P - j), j == 0));
    }
    if (layout.empty() || layout.size() > 65535) return TLC_OK;
    if (cudaMalloc((void **)d_dec, layout.size() * sizeof(DecRec)) != cudaSuccess) return TLC_ERR_CUDA;
    T.dec = *d_dec;
    T.dec_grid = (int)layout.size();
    return TLC_OK;
}

int small_dec_plan_refresh(const SegTable &T, const std::vector<Seg> &host, const std::vector<uint4> &layout) {
    std::vector<DecRec> recs(layout.size());
    for (size_t c = 0; c < layout.size(); c++) {
        const uint4 &l = layout[c];
        const Seg &S = host[l.x];
        DecRec &r = recs[c];
        r = DecRec{};
        r.payload = S.payload; r.hdr = S.hdr; r.out = S.out;
        r.n = (uint32_t)S.n; r.P = (uint32_t)S.P; r.jr0 = l.y; r.pl = l.z; r.first = l.w; r.seg = l.x;
    }
    return cudaMemcpy(const_cast<DecRec *>(T.dec), recs.data(), recs.size() * sizeof(DecRec),
                      cudaMemcpyHostToDevice) == cudaSuccess ? TLC_OK : TLC_ERR_CUDA;
}

static size_t small_smem_compress(uint64_t max_n) {
    return 4 * ((max_n + 3) & ~3ull) + ((max_n + 4) / 5 + 16);
}
static size_t small_smem_decompress(uint64_t) { return kSmPart; }

// TLC_NO_SMALL=1 routes small tables through K1-K5 (A/B measurements)
bool small_enabled() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("TLC_NO_SMALL");
        v = (e && e[0] == '1') ? 0 : 1;
    }
    return v == 1;
}

bool small_table(const SegTable &T) { return T.max_n <= kSmallMaxN && small_enabled(); }

int launch_small_compress(const SegTable &T, float s, int use_zre, cudaStream_t st) {
    if (T.sl && small_coop_enabled()) {
        static PerDevice cattr;
        if (cattr.first()) {
            int dev = 0, optin = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
            cudaFuncSetAttribute(tlc_small_coop_compress_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 optin - 4096);
        }
        KernelScope ks(kK6s, st);
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(T.sl_grid);
        cfg.blockDim = dim3(kSmThreads);
        cfg.dynamicSmemBytes = T.sl_smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeCooperative;   // every CTA co-resident: the grid barriers
        attr[0].val.cooperative = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        const cudaError_t e = cudaLaunchKernelEx(&cfg, tlc_small_coop_compress_kernel, T, s, use_zre);
        return e == cudaSuccess ? TLC_OK : TLC_ERR_CUDA;
    }
    if (T.grp) {
        KernelScope ks(kK6s, st);
        const bool b = group_bulk(), a = group_async();
        if (T.grp_cl == 8)
            return b ? (a ? launch_group<8, true, true>(T, s, use_zre, st) : launch_group<8, true, false>(T, s, use_zre, st))
                     : (a ? launch_group<8, false, true>(T, s, use_zre, st) : launch_group<8, false, false>(T, s, use_zre, st));
        if (T.grp_cl == 2)
            return b ? (a ? launch_group<2, true, true>(T, s, use_zre, st) : launch_group<2, true, false>(T, s, use_zre, st))
                     : (a ? launch_group<2, false, true>(T, s, use_zre, st) : launch_group<2, false, false>(T, s, use_zre, st));
        return b ? (a ? launch_group<4, true, true>(T, s, use_zre, st) : launch_group<4, true, false>(T, s, use_zre, st))
                 : (a ? launch_group<4, false, true>(T, s, use_zre, st) : launch_group<4, false, false>(T, s, use_zre, st));
    }
    static PerDevice attr;
    if (attr.first())
        cudaFuncSetAttribute(tlc_small_compress_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)small_smem_compress(kSmallMaxN));
    KernelScope ks(kK6s, st);
    const int grid = (int)tmin<uint64_t>((uint64_t)T.count, 65535);
    tlc_small_compress_kernel<<<grid, kSmThreads, small_smem_compress(T.max_n), st>>>(T, s, use_zre);
    return cudaPeekAtLastError() == cudaSuccess ? TLC_OK : TLC_ERR_CUDA;
}

// K7 parts per K5 tile, log2 (TLC_K7_SUB=0..3 for A/B; default 1: 2048 positions per CTA)
static int k7_sub_log2() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("TLC_K7_SUB");
        v = (e && e[0] >= '0' && e[0] <= '3') ? e[0] - '0' : 1;
    }
    return v;
}

int launch_small_decompress(const SegTable &T, int mode, cudaStream_t st) {
    static PerDevice attr;
    if (attr.first()) {
        cudaFuncSetAttribute(tlc_small_decompress_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)small_smem_decompress(kSmallMaxN));
        cudaFuncSetAttribute(tlc_small_decompress_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)small_smem_decompress(kSmallMaxN));
    }
    KernelScope ks(kK7s, st);
    if (T.dec) {
        if (mode == TLC_MODE_OVERWRITE) tlc_small_decompress_rec_kernel<0><<<T.dec_grid, kSmThreads, kSmPart, st>>>(T);
        else tlc_small_decompress_rec_kernel<1><<<T.dec_grid, kSmThreads, kSmPart, st>>>(T);
        return cudaPeekAtLastError() == cudaSuccess ? TLC_OK : TLC_ERR_CUDA;
    }
    const int sl = k7_sub_log2();
    const int grid = (int)tmin<uint64_t>(T.n5 << sl, 65535);
    const size_t smem = small_smem_decompress(T.max_n);
    if (mode == TLC_MODE_OVERWRITE) tlc_small_decompress_kernel<0><<<grid, kSmThreads, smem, st>>>(T, sl);
    else tlc_small_decompress_kernel<1><<<grid, kSmThreads, smem, st>>>(T, sl);
    return cudaPeekAtLastError() == cudaSuccess ? TLC_OK : TLC_ERR_CUDA;
}

}  // namespace tlc

#ifdef TLC_K6C_TRACE
extern "C" int tlc_debug_k6c_trace(void *host, size_t bytes) {
    return cudaMemcpyFromSymbol(host, tlc::g_k6c_trace, bytes < sizeof(tlc::g_k6c_trace) ? bytes : sizeof(tlc::g_k6c_trace)) ==
                   cudaSuccess ? 0 : 1;
}
#endif
