// compress.cu -- the 3LC compressor on sm_100a: two HBM passes.
//
//  K1 tlc_absmax_kernel  (row a1): u = err + t (not stored); grid max of
//     bits(u) & 0x7fffffff as uint32, which orders |u| and flags NaN/Inf in one
//     integer max; last CTA turns it into M = fl(a*s) and the header.
//  K2 tlc_quant_qe_kernel (rows a2-a3): a pure streaming pass -- recompute u,
//     quantize (Eq. 2), write err = u - M*q (steps a,b) and fold the five
//     strided trits of each quartic position into its byte (step 3), written
//     to the payload (no ZRE) or to a P-byte scratch in the workspace.
//  K3 tlc_zre_kernel (row a4): zero-run encoding (step 4) of the quartic bytes
//     as one scan over the run-carry monoid of tlc_device.cuh with decoupled
//     look-back across tiles (dynamic tile ids keep it deadlock-free); each
//     thread emits its payload bytes at their final offsets and the last tile
//     writes hdr->payload_len.
//
// Paper: P:372-410 (Sec. 3.1), P:495-510 (Sec. 3.2), P:538-548 (Sec. 3.3).
#include "tlc_device.cuh"
#include "tlc_launch.h"

namespace tlc {

// ============================================================== K1
constexpr int kK1Threads = 512;

__device__ __forceinline__ unsigned int absmax_key(float t, float e) {
    float u = __fadd_rn(e, t);                       // step (1): u = buffer + T_in
    return __float_as_uint(u) & 0x7fffffffu;         // |u| as ordered uint; NaN > Inf
}

template <bool kVec>
__global__ void __launch_bounds__(kK1Threads, 1)
tlc_absmax_kernel(const float *__restrict__ t, const float *__restrict__ err, uint64_t n,
                  float s, int use_zre, unsigned int *__restrict__ partial, Ctrl *ctrl,
                  tlc_header *hdr) {
    unsigned int m = 0;
    const uint64_t gtid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t tail_start = 0;
    if (kVec) {
        const uint64_t n4 = n / 4;
        const float4 *t4 = reinterpret_cast<const float4 *>(t);
        const float4 *e4 = reinterpret_cast<const float4 *>(err);
        constexpr int U = 4;
        uint64_t i = gtid;
        for (; i + (U - 1) * stride < n4; i += U * stride) {
            float4 a[U], b[U];
#pragma unroll
            for (int k = 0; k < U; k++) {
                a[k] = ld_stream4(t4 + i + k * stride);
                b[k] = __ldcg(e4 + i + k * stride);
            }
#pragma unroll
            for (int k = 0; k < U; k++) {
                m = max(m, absmax_key(a[k].x, b[k].x));
                m = max(m, absmax_key(a[k].y, b[k].y));
                m = max(m, absmax_key(a[k].z, b[k].z));
                m = max(m, absmax_key(a[k].w, b[k].w));
            }
        }
        for (; i < n4; i += stride) {
            float4 a = ld_stream4(t4 + i), b = __ldcg(e4 + i);
            m = max(m, absmax_key(a.x, b.x));
            m = max(m, absmax_key(a.y, b.y));
            m = max(m, absmax_key(a.z, b.z));
            m = max(m, absmax_key(a.w, b.w));
        }
        tail_start = n4 * 4;
    }
    for (uint64_t i = tail_start + gtid; i < n; i += stride)
        m = max(m, absmax_key(ld_stream(t + i), __ldcg(err + i)));

    // block reduction: warp redux, then one warp over the warp maxima
    __shared__ unsigned int s_warp[kK1Threads / 32];
    __shared__ bool s_last;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    m = __reduce_max_sync(0xffffffffu, m);
    if (lane == 0) s_warp[warp] = m;
    __syncthreads();
    if (warp == 0) {
        m = lane < (kK1Threads / 32) ? s_warp[lane] : 0u;
        m = __reduce_max_sync(0xffffffffu, m);
        if (lane == 0) {
            partial[blockIdx.x] = m;
            __threadfence();
            unsigned int ticket = atomicAdd(&ctrl->done_counter, 1u);
            s_last = (ticket == gridDim.x - 1);
        }
    }
    __syncthreads();
    if (!s_last) return;

    // last CTA: reduce the per-CTA maxima, derive M (Eq. 1) and the status
    __threadfence();
    m = 0;
    for (unsigned int i = threadIdx.x; i < gridDim.x; i += blockDim.x)
        m = max(m, __ldcg(partial + i));
    m = __reduce_max_sync(0xffffffffu, m);
    if (lane == 0) s_warp[warp] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned int key = 0;
        for (int w = 0; w < kK1Threads / 32; w++) key = max(key, s_warp[w]);
        unsigned int status = TLC_OK;
        float M = 0.0f;
        if (key >= 0x7f800000u) {
            status = TLC_ERR_NONFINITE;                       // NaN or Inf in u (R6)
        } else {
            M = __fmul_rn(__uint_as_float(key), s);           // Eq. 1
            if (isinf(M)) { status = TLC_ERR_RANGE; M = 0.0f; }
        }
        ctrl->maxkey = key;
        ctrl->M = M;
        ctrl->status = status;
        const uint64_t P = (n + 4) / 5;
        hdr->M = M;
        hdr->flags = use_zre ? TLC_FLAG_ZRE : 0u;
        hdr->n = n;
        hdr->payload_len = (status == TLC_OK && !use_zre) ? P : 0;
        hdr->status = status;
        hdr->reserved = 0;
    }
}

// ============================================================== K2
constexpr int kK2Threads = 256;

// One quartic position j, any alignment: the five strided elements e = i*P + j
// (partition i), residuals stored, byte returned (pad positions -> digit 0).
__device__ __forceinline__ uint32_t quant_qe_one(const float *__restrict__ t, float *__restrict__ err,
                                                 uint64_t n, uint64_t P, uint64_t j, const Quant &Q) {
    float tv[5], ev[5];
#pragma unroll
    for (int i = 0; i < 5; i++) {
        const uint64_t e = (uint64_t)i * P + j;
        tv[i] = e < n ? ld_stream(t + e) : 0.0f;
        ev[i] = e < n ? __ldcs(err + e) : 0.0f;
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

// ---- vector path (P % 4 == 0, 16-byte aligned t/err/bytes): one thread per
// group of 4 consecutive quartic positions j..j+3, one float4 per partition.
// Groups whose 20 elements all exist run without bounds checks; the few
// positions of the last group(s) of partition 4 go through quant_qe_one.
template <class QT>
__device__ __forceinline__ void quant_qe_groups(const float4 *__restrict__ t4, float4 *__restrict__ e4,
                                                uint32_t *__restrict__ b4, uint64_t P4,
                                                uint64_t full_groups, const QT &Q) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < full_groups; g += stride) {
        float4 tv[5], ev[5];
#pragma unroll
        for (int i = 0; i < 5; i++) {
            tv[i] = ld_stream4(t4 + g + i * P4);
            ev[i] = __ldcs(e4 + g + i * P4);
        }
        uint32_t by[4] = {0, 0, 0, 0};
#pragma unroll
        for (int i = 0; i < 5; i++) {
            float r[4];
            const float tt[4] = {tv[i].x, tv[i].y, tv[i].z, tv[i].w};
            const float ee[4] = {ev[i].x, ev[i].y, ev[i].z, ev[i].w};
#pragma unroll
            for (int c = 0; c < 4; c++) {
                const float u = __fadd_rn(ee[c], tt[c]);    // step (1)
                const int q = Q.q(u);                        // Eq. 2
                r[c] = Q.residual(u, q);                     // steps (a),(b)
                by[c] = by[c] * 3u + (uint32_t)(q + 1);      // steps 1, 6
            }
            __stcs(e4 + g + i * P4, make_float4(r[0], r[1], r[2], r[3]));
        }
        b4[g] = by[0] | (by[1] << 8) | (by[2] << 16) | (by[3] << 24);
    }
}

#ifndef TLC_K2_MINB
#define TLC_K2_MINB 2
#endif
__global__ void __launch_bounds__(kK2Threads, TLC_K2_MINB)
tlc_quant_qe_vec_kernel(const float *__restrict__ t, float *__restrict__ err, uint64_t n,
                        uint8_t *__restrict__ bytes, const Ctrl *__restrict__ ctrl) {
    if (ctrl->status != TLC_OK) return;           // K1 raised NONFINITE / RANGE: err untouched
    const Quant Q(ctrl->M);
    const uint64_t P = (n + 4) / 5;
    const uint64_t P4 = P / 4;                     // partition stride in float4
    // group g is complete iff 4P + 4g + 3 < n
    const uint64_t full_groups = n >= 4 * P + 3 ? tmin<uint64_t>(P4, (n - 4 * P) / 4) : 0;
    const float4 *t4 = reinterpret_cast<const float4 *>(t);
    float4 *e4 = reinterpret_cast<float4 *>(err);
    uint32_t *b4 = reinterpret_cast<uint32_t *>(bytes);
    if (Q.mode == 1) quant_qe_groups(t4, e4, b4, P4, full_groups, QuantCmp(Q));   // uniform branch
    else quant_qe_groups(t4, e4, b4, P4, full_groups, Q);
    // tail: quartic positions of the incomplete groups
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t j = 4 * full_groups + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < P; j += stride)
        bytes[j] = (uint8_t)quant_qe_one(t, err, n, P, j, Q);
}

// ---- scalar path (any alignment, any P): one thread per quartic position j.
__global__ void __launch_bounds__(kK2Threads)
tlc_quant_qe_scalar_kernel(const float *__restrict__ t, float *__restrict__ err, uint64_t n,
                           uint8_t *__restrict__ bytes, const Ctrl *__restrict__ ctrl) {
    if (ctrl->status != TLC_OK) return;
    const Quant Q(ctrl->M);
    const uint64_t P = (n + 4) / 5;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < P;
         j += (uint64_t)gridDim.x * blockDim.x)
        bytes[j] = (uint8_t)quant_qe_one(t, err, n, P, j, Q);
}

// ============================================================== K3
// Chunked single-pass scan: the grid splits the P quartic bytes into one
// contiguous chunk per CTA (chunk ids taken in order from an atomic counter),
// and each CTA splits its chunk into one sub-chunk per warp.
//   phase 1  each warp folds its sub-chunk (rows of 32 lanes x 32 bytes, each
//            lane's 32 bytes reduced to a literal bit mask) into a run
//            summary; the CTA publishes the composition of its 8 warps;
//   phase 2  the CTA composes the summaries of all preceding chunks (they
//            never wait on later chunks, so this cannot deadlock) -> carry-in;
//   phase 3  each warp re-reads its sub-chunk (L2-resident: P <= 0.2 n bytes),
//            scans it and emits every ZRE byte at its final offset.
// The dependency depth between chunks is one publication, not a chain.
constexpr int kK3Threads = kScanThreads;
constexpr int kK3Seg = 32;                                   // bytes per lane per row
constexpr int kK3WarpRow = 32 * kK3Seg;                      // 1 KiB per warp row

// Load [pos, min(pos+32, hi)) as 8 words, padding with 121 (0x79).
__device__ __forceinline__ int load_seg(const uint8_t *__restrict__ bytes, uint64_t pos, uint64_t hi,
                                        uint32_t (&w)[8]) {
    const int len = pos < hi ? (int)tmin<uint64_t>(kK3Seg, hi - pos) : 0;
    if (len == kK3Seg && (reinterpret_cast<uintptr_t>(bytes + pos) & 15u) == 0) {
        const uint4 a = *reinterpret_cast<const uint4 *>(bytes + pos);
        const uint4 b = *reinterpret_cast<const uint4 *>(bytes + pos + 16);
        w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w;
        w[4] = b.x; w[5] = b.y; w[6] = b.z; w[7] = b.w;
    } else {
#pragma unroll
        for (int k = 0; k < 8; k++) {
            uint32_t x = 0;
#pragma unroll
            for (int c = 0; c < 4; c++) {
                const int m = 4 * k + c;
                x |= (uint32_t)(m < len ? bytes[pos + m] : kZeroGroup) << (8 * c);
            }
            w[k] = x;
        }
    }
    return len;
}

__global__ void __launch_bounds__(kK3Threads)
tlc_zre_kernel(const uint8_t *__restrict__ bytes, uint64_t P, uint64_t chunk,
               uint8_t *__restrict__ payload, Ctrl *ctrl, unsigned long long *states, tlc_header *hdr) {
    __shared__ unsigned long long s_warp[kScanWarps];
    __shared__ unsigned long long s_wagg[kScanWarps];
    __shared__ unsigned int s_id;
    if (ctrl->status != TLC_OK) return;
    const uint64_t nchunks = (P + chunk - 1) / chunk;
    if (threadIdx.x == 0) s_id = atomicAdd(&ctrl->tile_counter, 1u);
    __syncthreads();
    const uint64_t b = s_id;
    if (b >= nchunks) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t lo = b * chunk, hi = tmin<uint64_t>(P, lo + chunk);
    const uint64_t sub = ((hi - lo + kScanWarps - 1) / kScanWarps + kK3Seg - 1) / kK3Seg * kK3Seg;
    const uint64_t wlo = tmin<uint64_t>(hi, lo + warp * sub), whi = tmin<uint64_t>(hi, wlo + sub);
    uint32_t w[8];

    // ---- phase 1: run summary of the warp's sub-chunk (one per 1 KiB row), then of the chunk
    RunSum wagg = run_identity();
    for (uint64_t row = wlo; row < whi; row += kK3WarpRow) {
        const int len = load_seg(bytes, row + (uint64_t)kK3Seg * lane, whi, w);
        const uint32_t mask = literal_mask(w);
        const uint32_t row_len = (uint32_t)tmin<uint64_t>(kK3WarpRow, whi - row);
        wagg = compose(wagg, warp_row_summary(mask, len, mask_summary(mask, len), row_len));
    }
    if (lane == 0) s_wagg[warp] = pack(wagg);
    __syncthreads();
    RunSum agg = run_identity();
#pragma unroll
    for (int k = 0; k < kScanWarps; k++) agg = compose(agg, unpack(s_wagg[k]));
    if (threadIdx.x == 0) st_relaxed_u64(states + b, kReady | pack(agg));

    // ---- phase 2: carry-in = composition of all preceding chunk summaries
    RunSum part = run_identity();
    const uint64_t per = (b + kK3Threads - 1) / kK3Threads;
    const uint64_t i0 = per * threadIdx.x, i1 = tmin<uint64_t>(b, i0 + per);
    for (uint64_t i = i0; i < i1; i++) part = compose(part, unpack(wait_ready(states + i) & ~kReady));
    const RunSum chunk_in = block_reduce_runs(part, s_warp);
    if (b == nchunks - 1 && threadIdx.x == 0) {
        uint64_t total;
        uint32_t carry;
        run_eval(compose(chunk_in, agg), 0, total, carry);
        hdr->payload_len = total + (carry > 0);   // the end of the stream flushes
    }

    // ---- phase 3: emission at the final payload offsets
    RunSum before = chunk_in;
    for (int k = 0; k < warp; k++) before = compose(before, unpack(s_wagg[k]));
    uint64_t off;
    uint32_t carry;
    run_eval(before, 0, off, carry);              // payload offset and carry at the sub-chunk start
    for (uint64_t row = wlo; row < whi; row += kK3WarpRow) {
        const uint64_t pos = row + (uint64_t)kK3Seg * lane;
        const int len = load_seg(bytes, pos, whi, w);
        const uint32_t mask = literal_mask(w);
        const uint32_t row_len = (uint32_t)tmin<uint64_t>(kK3WarpRow, whi - row);
        const WarpRow r = warp_row(mask, len, mask_summary(mask, len), carry, row_len);
        uint32_t ex = r.count;                    // exclusive prefix of the lane counts
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, ex, d);
            if (lane >= d) ex += y;
        }
        ex -= r.count;
        if (len > 0) {
            uint64_t o = off + ex;
            uint32_t c = r.carry_in;
            mask_emit(w, mask, len, c, payload, o);
            if (c > 0 && pos + len == P) payload[o] = run_code(c);
        }
        off += r.row_count;
        carry = r.carry_out;
    }
}

// ============================================================== host launchers
struct CompressWs {
    Ctrl *ctrl;
    unsigned long long *states;
    unsigned int *partial;
    uint8_t *bytes;
    size_t memset_bytes;
};

static CompressWs carve_compress_ws(void *ws) {
    const uint64_t tiles = (uint64_t)kMaxSms * 16;       // K3 chunk summaries
    CompressWs w;
    char *p = reinterpret_cast<char *>(ws);
    w.ctrl = reinterpret_cast<Ctrl *>(p);
    w.states = reinterpret_cast<unsigned long long *>(p + sizeof(Ctrl));
    const size_t o1 = sizeof(Ctrl) + align256(tiles * sizeof(unsigned long long));
    w.partial = reinterpret_cast<unsigned int *>(p + o1);
    const size_t o2 = o1 + align256((size_t)kMaxSms * kK1BlocksPerSm * sizeof(unsigned int));
    w.bytes = reinterpret_cast<uint8_t *>(p + o2);
    w.memset_bytes = sizeof(Ctrl) + tiles * sizeof(unsigned long long);
    return w;
}

size_t compress_workspace_bytes(uint64_t n) {
    const uint64_t P = (n + 4) / 5;
    const uint64_t tiles = (uint64_t)kMaxSms * 16;
    return sizeof(Ctrl) + align256(tiles * sizeof(unsigned long long)) +
           align256((size_t)kMaxSms * kK1BlocksPerSm * sizeof(unsigned int)) + align256(P);
}

static int g_k2_vec_blocks = 0, g_k2_sc_blocks = 0, g_k3_blocks = 0;

int launch_compress(const float *t, float *err, uint64_t n, float s, int use_zre, uint8_t *payload,
                    tlc_header *hdr, void *ws, cudaStream_t st) {
    const uint64_t P = (n + 4) / 5;
    const CompressWs w = carve_compress_ws(ws);
    const int sms = num_sms();
    if (cudaMemsetAsync(ws, 0, w.memset_bytes, st) != cudaSuccess) return TLC_ERR_CUDA;

    const bool vec1 = aligned16(t) && aligned16(err);
    const uint64_t work1 = vec1 ? (n + 3) / 4 : n;
    const int grid1 = (int)tmin<uint64_t>((uint64_t)sms * kK1BlocksPerSm,
                                          tmax<uint64_t>(1, (work1 + kK1Threads * 4 - 1) / (kK1Threads * 4)));
    {
        KernelScope ks(kK1, st);
        if (vec1) tlc_absmax_kernel<true><<<grid1, kK1Threads, 0, st>>>(t, err, n, s, use_zre, w.partial, w.ctrl, hdr);
        else tlc_absmax_kernel<false><<<grid1, kK1Threads, 0, st>>>(t, err, n, s, use_zre, w.partial, w.ctrl, hdr);
    }

    uint8_t *bytes = use_zre ? w.bytes : payload;
    const bool vec2 = (P % 4 == 0) && aligned16(t) && aligned16(err) && aligned4(bytes);
    {
        KernelScope ks(kK2, st);
        if (vec2) {
            if (!g_k2_vec_blocks)
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_k2_vec_blocks, tlc_quant_qe_vec_kernel, kK2Threads, 0);
            const uint64_t groups = P / 4;
            const int grid = (int)tmin<uint64_t>((groups + kK2Threads - 1) / kK2Threads,
                                                 (uint64_t)sms * tmax(1, g_k2_vec_blocks));
            tlc_quant_qe_vec_kernel<<<tmax(grid, 1), kK2Threads, 0, st>>>(t, err, n, bytes, w.ctrl);
        } else {
            if (!g_k2_sc_blocks)
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_k2_sc_blocks, tlc_quant_qe_scalar_kernel, kK2Threads, 0);
            const int grid = (int)tmin<uint64_t>((P + kK2Threads - 1) / kK2Threads,
                                                 (uint64_t)sms * tmax(1, g_k2_sc_blocks));
            tlc_quant_qe_scalar_kernel<<<tmax(grid, 1), kK2Threads, 0, st>>>(t, err, n, bytes, w.ctrl);
        }
    }
    if (use_zre) {
        KernelScope ks(kK3, st);
        if (!g_k3_blocks)
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_k3_blocks, tlc_zre_kernel, kK3Threads, 0);
        const uint64_t rows = (P + kScanWarps * kK3WarpRow - 1) / (kScanWarps * kK3WarpRow);
        const uint64_t grid = tmax<uint64_t>(1, tmin<uint64_t>(rows, (uint64_t)sms * tmin(16, tmax(1, g_k3_blocks))));
        const uint64_t chunk = ((P + grid - 1) / grid + kK3Seg - 1) / kK3Seg * kK3Seg;
        const uint64_t nch = (P + chunk - 1) / chunk;
        tlc_zre_kernel<<<(unsigned)nch, kK3Threads, 0, st>>>(w.bytes, P, chunk, payload, w.ctrl, w.states, hdr);
    }
    return cudaPeekAtLastError() == cudaSuccess ? TLC_OK : TLC_ERR_CUDA;
}

}  // namespace tlc
