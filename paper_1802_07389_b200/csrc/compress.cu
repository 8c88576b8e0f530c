// compress.cu -- the 3LC compressor on sm_100a: two HBM passes.
//
//  K1 tlc_absmax_kernel  (row a1): u = err + t (not stored); grid max of
//     bits(u) & 0x7fffffff as uint32, which orders |u| and flags NaN/Inf in one
//     integer max; last CTA turns it into M = fl(a*s) and the header.
//  K2 tlc_quant_qe_zre_kernel (rows a2-a4): per tile of kTile quartic bytes,
//     recompute u, quantize (Eq. 2), write err = u - M*q (steps a,b), fold the
//     five strided trits into quartic bytes (step 3) in shared memory, then
//     zero-run encode the tile (step 4) as a scan with decoupled look-back over
//     the run-carry monoid of tlc_device.cuh and write the payload bytes at
//     their final offsets.  Dynamic tile ids keep the look-back deadlock-free.
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
__global__ void __launch_bounds__(kK1Threads)
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
constexpr int kK2BytesPerThread = 8;
constexpr int kTile = kK2Threads * kK2BytesPerThread;    // 2048 quartic bytes per tile
constexpr int kK2Warps = kK2Threads / 32;

struct K2Smem {
    alignas(16) uint8_t B[kTile];        // quartic bytes of the tile
    unsigned long long warp_incl[kK2Warps];
    unsigned long long tile_excl;
    unsigned int tile;
};

// One quartic byte from the five strided elements e_i = i*P + j.
// Loads are issued by the caller; this folds digits d_i = q_i + 1 (pad -> 0).
__device__ __forceinline__ uint32_t fold_byte(const float (&tv)[5], const float (&ev)[5],
                                              const bool (&ok)[5], const Quant &Q,
                                              float (&rv)[5]) {
    uint32_t b = 0;
#pragma unroll
    for (int i = 0; i < 5; i++) {
        float u = __fadd_rn(ev[i], tv[i]);
        int q = Q.q(u);
        rv[i] = Q.residual(u, q);
        uint32_t d = ok[i] ? (uint32_t)(q + 1) : 0u;   // step 4: pad digit 0 (R10)
        b = b * 3u + d;                                 // step 6: p0*81+...+p4
    }
    return b;
}

// ---- phase A, scalar path: thread handles j = j0 + k*256 + tid, k = 0..7
template <bool kWritePayload>
__device__ __forceinline__ void k2_phase_a_scalar(const float *__restrict__ t, float *__restrict__ err,
                                                  uint64_t n, uint64_t P, uint64_t j0, int tile_len,
                                                  const Quant &Q, uint8_t *sB,
                                                  uint8_t *__restrict__ payload) {
    constexpr int KU = 4;
#pragma unroll
    for (int kb = 0; kb < kK2BytesPerThread; kb += KU) {
        float tv[KU][5], ev[KU][5];
        bool ok[KU][5];
#pragma unroll
        for (int kk = 0; kk < KU; kk++) {
            const int jl = (kb + kk) * kK2Threads + threadIdx.x;
            const uint64_t j = j0 + jl;
#pragma unroll
            for (int i = 0; i < 5; i++) {
                const uint64_t e = (uint64_t)i * P + j;
                ok[kk][i] = (jl < tile_len) && (e < n);
                tv[kk][i] = ok[kk][i] ? ld_stream(t + e) : 0.0f;
                ev[kk][i] = ok[kk][i] ? __ldcs(err + e) : 0.0f;
            }
        }
#pragma unroll
        for (int kk = 0; kk < KU; kk++) {
            const int jl = (kb + kk) * kK2Threads + threadIdx.x;
            const uint64_t j = j0 + jl;
            float rv[5];
            uint32_t b = fold_byte(tv[kk], ev[kk], ok[kk], Q, rv);
#pragma unroll
            for (int i = 0; i < 5; i++)
                if (ok[kk][i]) __stcs(err + (uint64_t)i * P + j, rv[i]);
            if (jl < tile_len) {
                if (kWritePayload) payload[j] = (uint8_t)b;
                else sB[jl] = (uint8_t)b;
            }
        }
    }
}

// ---- phase A, vector path (P % 4 == 0, 16-byte aligned t/err): thread handles
// 4 consecutive j at j0 + 4*tid + 1024*g, g = 0..1, one float4 per partition.
template <bool kWritePayload>
__device__ __forceinline__ void k2_phase_a_vec(const float *__restrict__ t, float *__restrict__ err,
                                               uint64_t n, uint64_t P, uint64_t j0, int tile_len,
                                               const Quant &Q, uint8_t *sB,
                                               uint8_t *__restrict__ payload) {
    constexpr int G = kK2BytesPerThread / 4;   // 2 groups of 4 bytes
    float4 tv[G][5], ev[G][5];
    bool full[G][5];
#pragma unroll
    for (int g = 0; g < G; g++) {
        const int jl = 4 * threadIdx.x + g * 4 * kK2Threads;
        const uint64_t j = j0 + jl;
#pragma unroll
        for (int i = 0; i < 5; i++) {
            const uint64_t e = (uint64_t)i * P + j;
            full[g][i] = (jl + 3 < tile_len) && (e + 3 < n);
            if (full[g][i]) {
                tv[g][i] = ld_stream4(reinterpret_cast<const float4 *>(t + e));
                ev[g][i] = __ldcs(reinterpret_cast<const float4 *>(err + e));
            } else {
                float a[4], b[4];
#pragma unroll
                for (int c = 0; c < 4; c++) {
                    bool ok = (jl + c < tile_len) && (e + c < n);
                    a[c] = ok ? ld_stream(t + e + c) : 0.0f;
                    b[c] = ok ? __ldcs(err + e + c) : 0.0f;
                }
                tv[g][i] = make_float4(a[0], a[1], a[2], a[3]);
                ev[g][i] = make_float4(b[0], b[1], b[2], b[3]);
            }
        }
    }
#pragma unroll
    for (int g = 0; g < G; g++) {
        const int jl = 4 * threadIdx.x + g * 4 * kK2Threads;
        const uint64_t j = j0 + jl;
        uint32_t bytes[4] = {0, 0, 0, 0};
#pragma unroll
        for (int i = 0; i < 5; i++) {
            const uint64_t e = (uint64_t)i * P + j;
            const float tt[4] = {tv[g][i].x, tv[g][i].y, tv[g][i].z, tv[g][i].w};
            const float ee[4] = {ev[g][i].x, ev[g][i].y, ev[g][i].z, ev[g][i].w};
            float r[4];
#pragma unroll
            for (int c = 0; c < 4; c++) {
                const bool ok = full[g][i] || ((jl + c < tile_len) && (e + c < n));
                float u = __fadd_rn(ee[c], tt[c]);
                int q = Q.q(u);
                r[c] = Q.residual(u, q);
                bytes[c] = bytes[c] * 3u + (ok ? (uint32_t)(q + 1) : 0u);
            }
            if (full[g][i]) {
                __stcs(reinterpret_cast<float4 *>(err + e), make_float4(r[0], r[1], r[2], r[3]));
            } else {
#pragma unroll
                for (int c = 0; c < 4; c++)
                    if ((jl + c < tile_len) && (e + c < n)) __stcs(err + e + c, r[c]);
            }
        }
        if (jl + 3 < tile_len) {
            uint32_t w = bytes[0] | (bytes[1] << 8) | (bytes[2] << 16) | (bytes[3] << 24);
            if (kWritePayload) {
                // payload + j is 4-aligned when the payload base is (checked on host)
                *reinterpret_cast<uint32_t *>(payload + j) = w;
            } else {
                *reinterpret_cast<uint32_t *>(sB + jl) = w;
            }
        } else {
#pragma unroll
            for (int c = 0; c < 4; c++)
                if (jl + c < tile_len) {
                    if (kWritePayload) payload[j + c] = (uint8_t)bytes[c];
                    else sB[jl + c] = (uint8_t)bytes[c];
                }
        }
    }
}

template <bool kVec, bool kZre>
__global__ void __launch_bounds__(kK2Threads)
tlc_quant_qe_zre_kernel(const float *__restrict__ t, float *__restrict__ err, uint64_t n,
                        uint8_t *__restrict__ payload, Ctrl *ctrl, unsigned long long *states,
                        tlc_header *hdr) {
    __shared__ K2Smem sm;
    if (ctrl->status != TLC_OK) return;           // K1 raised NONFINITE / RANGE: err untouched
    const Quant Q(ctrl->M);
    const uint64_t P = (n + 4) / 5;
    const uint64_t num_tiles = (P + kTile - 1) / kTile;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

    while (true) {
        if (threadIdx.x == 0) sm.tile = atomicAdd(&ctrl->tile_counter, 1u);
        __syncthreads();
        const uint64_t tile = sm.tile;
        if (tile >= num_tiles) break;
        const uint64_t j0 = tile * kTile;
        const int tile_len = (int)tmin<uint64_t>(kTile, P - j0);

        // ---------------- phase A: quantize, residual, quartic bytes
        if (kVec) k2_phase_a_vec<!kZre>(t, err, n, P, j0, tile_len, Q, sm.B, payload);
        else k2_phase_a_scalar<!kZre>(t, err, n, P, j0, tile_len, Q, sm.B, payload);

        if (kZre) {
            __syncthreads();

            // ---------------- phase B: per-thread run summaries, block scan
            const int sbeg = threadIdx.x * kK2BytesPerThread;
            const int slen = max(0, min(kK2BytesPerThread, tile_len - sbeg));
            uint8_t b[kK2BytesPerThread];
            {
                uint2 w = *reinterpret_cast<const uint2 *>(sm.B + sbeg);
#pragma unroll
                for (int m = 0; m < 4; m++) b[m] = (w.x >> (8 * m)) & 0xff;
#pragma unroll
                for (int m = 0; m < 4; m++) b[4 + m] = (w.y >> (8 * m)) & 0xff;
            }
            const RunSum mine = segment_summary(b, slen);

            // warp inclusive scan
            unsigned long long x = pack(mine);
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                unsigned long long y = shfl_up64(x, d);
                if (lane >= d) x = pack(compose(unpack(y), unpack(x)));
            }
            unsigned long long thread_excl = shfl_up64(x, 1);
            if (lane == 0) thread_excl = pack(run_identity());
            if (lane == 31) sm.warp_incl[warp] = x;
            __syncthreads();

            // ---------------- tile aggregate + decoupled look-back (warp 0)
            if (warp == 0) {
                RunSum agg = run_identity();
#pragma unroll
                for (int w = 0; w < kK2Warps; w++) agg = compose(agg, unpack(sm.warp_incl[w]));
                RunSum excl = run_identity();
                if (tile == 0) {
                    if (lane == 0) st_relaxed_u64(states + tile, kStatusPrefix | pack(agg));
                } else {
                    if (lane == 0) st_relaxed_u64(states + tile, kStatusAgg | pack(agg));
                    int64_t pred = (int64_t)tile - 1;
                    while (true) {
                        const int64_t idx = pred - lane;
                        unsigned long long w =
                            idx >= 0 ? ld_relaxed_u64(states + idx) : (kStatusPrefix | pack(run_identity()));
                        const unsigned int st = (unsigned int)(w >> 62);
                        const unsigned int pref = __ballot_sync(0xffffffffu, st == 2u);
                        const unsigned int inval = __ballot_sync(0xffffffffu, st == 0u);
                        const int first = pref ? (__ffs(pref) - 1) : 31;
                        const unsigned int window = (first == 31) ? 0xffffffffu : ((2u << first) - 1u);
                        if (inval & window) { __nanosleep(32); continue; }
                        unsigned long long v = (lane <= first) ? (w & ~kStatusMask) : pack(run_identity());
#pragma unroll
                        for (int d = 1; d < 32; d <<= 1) {
                            unsigned long long o = shfl_down64(v, d);
                            if (lane + d < 32) v = pack(compose(unpack(o), unpack(v)));
                        }
                        v = __shfl_sync(0xffffffffu, v, 0);
                        excl = compose(unpack(v), excl);
                        if (pref) break;
                        pred -= 32;
                    }
                    if (lane == 0) st_relaxed_u64(states + tile, kStatusPrefix | pack(compose(excl, agg)));
                }
                if (lane == 0) {
                    sm.tile_excl = pack(excl);
                    if (tile == num_tiles - 1) {
                        uint64_t total;
                        uint32_t carry;
                        run_eval(compose(excl, agg), 0, total, carry);
                        hdr->payload_len = total + (carry > 0);   // end of stream flushes
                    }
                }
                // warp exclusive prefixes for the block: reuse warp_incl as exclusive
                __syncwarp();
                if (lane == 0) {
                    RunSum acc = run_identity();
                    for (int w = 0; w < kK2Warps; w++) {
                        RunSum nx = compose(acc, unpack(sm.warp_incl[w]));
                        sm.warp_incl[w] = pack(acc);
                        acc = nx;
                    }
                }
            }
            __syncthreads();

            // ---------------- emission at final payload offsets
            if (slen > 0) {
                RunSum before = compose(unpack(sm.tile_excl),
                                        compose(unpack(sm.warp_incl[warp]), unpack(thread_excl)));
                uint64_t off;
                uint32_t c;
                run_eval(before, 0, off, c);
                segment_emit(b, slen, c, payload, off);
                // the thread holding the last byte of the stream flushes the pending run
                if (c > 0 && j0 + sbeg + slen == P) payload[off] = run_code(c);
            }
        }
        __syncthreads();   // sm.B / sm.tile reuse
    }
}

// ============================================================== host launchers
static int g_k2_blocks_vec = 0, g_k2_blocks_sc = 0;

int launch_compress(const float *t, float *err, uint64_t n, float s, int use_zre, uint8_t *payload,
                    tlc_header *hdr, void *ws, cudaStream_t st) {
    const uint64_t P = (n + 4) / 5;
    const uint64_t num_tiles = (P + kTile - 1) / kTile;
    Ctrl *ctrl = reinterpret_cast<Ctrl *>(ws);
    unsigned long long *states = reinterpret_cast<unsigned long long *>((char *)ws + sizeof(Ctrl));
    unsigned int *partial = reinterpret_cast<unsigned int *>(
        (char *)ws + sizeof(Ctrl) + align256(num_tiles * sizeof(unsigned long long)));

    const int sms = num_sms();
    if (cudaMemsetAsync(ws, 0, sizeof(Ctrl) + num_tiles * sizeof(unsigned long long), st) != cudaSuccess)
        return TLC_ERR_CUDA;

    const bool vec1 = aligned16(t) && aligned16(err);
    const uint64_t work1 = vec1 ? (n + 3) / 4 : n;
    int grid1 = (int)tmin<uint64_t>((uint64_t)sms * kK1BlocksPerSm, tmax<uint64_t>(1, (work1 + kK1Threads * 4 - 1) / (kK1Threads * 4)));
    {
        KernelScope ks(kK1, st);
        if (vec1) tlc_absmax_kernel<true><<<grid1, kK1Threads, 0, st>>>(t, err, n, s, use_zre, partial, ctrl, hdr);
        else tlc_absmax_kernel<false><<<grid1, kK1Threads, 0, st>>>(t, err, n, s, use_zre, partial, ctrl, hdr);
    }

    const bool vec2 = (P % 4 == 0) && aligned16(t) && aligned16(err) && (use_zre || aligned4(payload));
    int per_sm = 0;
    if (vec2) {
        if (!g_k2_blocks_vec)
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_k2_blocks_vec, tlc_quant_qe_zre_kernel<true, true>, kK2Threads, 0);
        per_sm = g_k2_blocks_vec;
    } else {
        if (!g_k2_blocks_sc)
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_k2_blocks_sc, tlc_quant_qe_zre_kernel<false, true>, kK2Threads, 0);
        per_sm = g_k2_blocks_sc;
    }
    int grid2 = (int)tmin<uint64_t>(num_tiles, (uint64_t)sms * max(1, per_sm));
    KernelScope ks(kK2, st);
    if (vec2) {
        if (use_zre) tlc_quant_qe_zre_kernel<true, true><<<grid2, kK2Threads, 0, st>>>(t, err, n, payload, ctrl, states, hdr);
        else tlc_quant_qe_zre_kernel<true, false><<<grid2, kK2Threads, 0, st>>>(t, err, n, payload, ctrl, states, hdr);
    } else {
        if (use_zre) tlc_quant_qe_zre_kernel<false, true><<<grid2, kK2Threads, 0, st>>>(t, err, n, payload, ctrl, states, hdr);
        else tlc_quant_qe_zre_kernel<false, false><<<grid2, kK2Threads, 0, st>>>(t, err, n, payload, ctrl, states, hdr);
    }
    return cudaPeekAtLastError() == cudaSuccess ? TLC_OK : TLC_ERR_CUDA;
}

size_t compress_workspace_bytes(uint64_t n) {
    const uint64_t P = (n + 4) / 5;
    const uint64_t num_tiles = (P + kTile - 1) / kTile;
    return sizeof(Ctrl) + align256(num_tiles * sizeof(unsigned long long)) +
           align256((size_t)kMaxSms * kK1BlocksPerSm * sizeof(unsigned int));
}

}  // namespace tlc
