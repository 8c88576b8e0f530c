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
#include <cstdlib>

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
        // full chunks (255) everywhere first; flush codes and literals overwrite
        const uint32_t total = s_off[nrows];
        for (uint32_t q = threadIdx.x; q < total; q += kSmThreads) S.payload[q] = 0xff;
        __syncthreads();
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
                if (R % kMaxRun) out[o++] = run_code(R % kMaxRun);
                uint32_t word = w[0];
#pragma unroll
                for (int k = 1; k < 8; k++) word = (k == (q >> 2)) ? w[k] : word;
                out[o++] = (uint8_t)(word >> (8 * (q & 3)));
                prev = q;
            }
        }
        if (threadIdx.x == 0 && s_carry[nrows] > 0) S.payload[total] = run_code(s_carry[nrows]);
        __syncthreads();                                         // shared memory reuse
    }
}

// A tensor's decode is split into parts of kSmPart quartic positions, one CTA each (the
// 36,864-value ResNet-110 tensors would otherwise keep one SM busy while most idle): every
// part scans the whole payload (<= P bytes, on chip) and expands / decodes only its range.
constexpr uint32_t kSmPart = 2048;

template <int kMode>
__global__ void __launch_bounds__(kSmThreads)
tlc_small_decompress_kernel(const SegTable T, uint32_t parts) {
    extern __shared__ __align__(16) uint8_t sm_raw[];
    __shared__ uint32_t V[5][256];
    __shared__ uint16_t lut[256];
    __shared__ uint32_t s_wsum[kSmWarps + 1];
    __shared__ int s_bad;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t items = (uint64_t)T.count * parts;
    for (uint64_t item = blockIdx.x; item < items; item += gridDim.x) {
        const int si = (int)(item / parts);
        const uint32_t part = (uint32_t)(item % parts);
        const Seg S = get_seg(T, si);
        tlc_header *hdr = S.hdr;
        const uint32_t jr0 = part * kSmPart;
        if (jr0 >= S.P) continue;                                // no positions in this part
        if (!header_valid(hdr, S.n)) {                           // uniform over the CTA
            if (threadIdx.x == 0 && part == 0 && hdr->status == TLC_OK) raise_format(hdr);
            continue;
        }
        const uint32_t n = (uint32_t)S.n, P = (uint32_t)S.P, Z = (uint32_t)hdr->payload_len;
        const uint32_t jr1 = min(P, jr0 + kSmPart), pl = jr1 - jr0;
        const bool zre = (hdr->flags & TLC_FLAG_ZRE) != 0;
        const float M = hdr->M;
        uint8_t *E = sm_raw;                                     // quartic bytes [jr0, jr1)
        uint8_t *Y = sm_raw + kSmPart;                           // the payload (ZRE)
        if (threadIdx.x == 0) s_bad = 0;
        // value table: Eq. 3 per partition, V[i][b] = M * (digit_i(b) - 1)
        for (int v = threadIdx.x; v < 256; v += kSmThreads) {
            uint32_t wd = 0, r = v < 243 ? v : 121;
#pragma unroll
            for (int i = 4; i >= 0; i--) {
                const uint32_t d = r % 3u;
                r /= 3u;
                wd |= (uint32_t)(d != 1) << i;
                V[i][v] = __float_as_uint(__fmul_rn(M, (float)((int)d - 1)));
            }
            lut[v] = (uint16_t)wd;
        }
        __syncthreads();
        if (zre) {
            for (uint32_t q = threadIdx.x; q < Z; q += kSmThreads) Y[q] = S.payload[q];
            __syncthreads();
            // expansion lengths of bytes [16t, 16t+16), block exclusive scan
            constexpr int kPer = 16;
            static_assert((kSmallMaxN + 4) / 5 <= kPer * kSmThreads, "every payload byte has a thread");
            uint32_t lens = 0;
            const uint32_t b0 = kPer * threadIdx.x;
#pragma unroll
            for (int k = 0; k < kPer; k++) lens += b0 + k < Z ? zre_len(Y[b0 + k]) : 0u;
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
#pragma unroll
            for (int k = 0; k < kPer; k++) {
                if (b0 + k >= Z || p >= jr1) break;
                const uint32_t b = Y[b0 + k];
                if (b < kFirstRunCode && p >= jr0) E[p - jr0] = (uint8_t)b;   // literal
                p += zre_len(b);
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
        // ---- decoding steps 1-4 and Eq. 3
        for (uint32_t jl = threadIdx.x; jl < pl; jl += kSmThreads) {
            const uint32_t b = E[jl];
            const uint32_t nz = lut[b];
#pragma unroll
            for (int i = 0; i < 5; i++) {
                const uint32_t e = (uint32_t)(i * P) + jr0 + jl;
                if (e >= n) break;
                const float v = __uint_as_float(V[i][b]);
                if (kMode == TLC_MODE_OVERWRITE) __stcs(S.out + e, v);
                else if ((nz >> i) & 1u) S.out[e] = __fadd_rn(S.out[e], v);   // q != 0 (R16)
            }
        }
        __syncthreads();                                         // tables / buffers reuse
    }
}

static size_t small_smem_compress(uint64_t max_n) {
    return 4 * ((max_n + 3) & ~3ull) + ((max_n + 4) / 5 + 16);
}
static size_t small_smem_decompress(uint64_t max_n) {
    const uint64_t P = (max_n + 4) / 5;
    return kSmPart + ((P + 15) & ~15ull);
}

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
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(tlc_small_compress_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)small_smem_compress(kSmallMaxN));
        attr = true;
    }
    KernelScope ks(kK6s, st);
    const int grid = (int)tmin<uint64_t>((uint64_t)T.count, 65535);
    tlc_small_compress_kernel<<<grid, kSmThreads, small_smem_compress(T.max_n), st>>>(T, s, use_zre);
    return cudaPeekAtLastError() == cudaSuccess ? TLC_OK : TLC_ERR_CUDA;
}

int launch_small_decompress(const SegTable &T, int mode, cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(tlc_small_decompress_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)small_smem_decompress(kSmallMaxN));
        cudaFuncSetAttribute(tlc_small_decompress_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)small_smem_decompress(kSmallMaxN));
        attr = true;
    }
    KernelScope ks(kK7s, st);
    const uint32_t parts = (uint32_t)(((T.max_n + 4) / 5 + kSmPart - 1) / kSmPart);
    const int grid = (int)tmin<uint64_t>((uint64_t)T.count * parts, 65535);
    const size_t smem = small_smem_decompress(T.max_n);
    if (mode == TLC_MODE_OVERWRITE) tlc_small_decompress_kernel<0><<<grid, kSmThreads, smem, st>>>(T, parts);
    else tlc_small_decompress_kernel<1><<<grid, kSmThreads, smem, st>>>(T, parts);
    return cudaPeekAtLastError() == cudaSuccess ? TLC_OK : TLC_ERR_CUDA;
}

}  // namespace tlc
