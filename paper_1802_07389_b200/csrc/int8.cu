// int8.cu -- "8-bit int", a compared design of the paper (Sec. 5.1):
// "255 distinct values ([-127,127], leaving -128 unused)".  Reading R23:
// scale = fl(max|t| / 127); code = clamp(round_half_away(fl(t / scale)), -127, 127);
// dequant = fl(scale * code).  No error buffer.
//
// Kq8 tlc_int8_quant_kernel: after K1<no err> (max|t|), one streaming pass:
//     per warp step 512 elements, lane l taking float4 number base + l + 32k
//     (k = 0..3, four coalesced 512-byte loads in flight) and storing its 4 codes
//     as one 32-bit word (coalesced 128-byte stores).  4n read + n written.
// Kd8 tlc_int8_dequant_kernel: the mirror image, 32-bit code loads and float4
//     stores with the same lane mapping: n read + 4n written (accumulate: + 4n).
// Both are plain HBM streams; grid = SMs x resident CTAs, grid-stride.
#include "tlc_device.cuh"
#include "tlc_launch.h"

namespace tlc {

constexpr int kI8Threads = 256;

__device__ __forceinline__ int8_t int8_code(float x, float scale) {
    if (scale == 0.0f) return 0;                          // max = 0 or an underflowed scale (R23)
    float c = roundf(__fdiv_rn(x, scale));                // half away from zero (R1)
    c = fminf(fmaxf(c, -127.0f), 127.0f);                 // -128 unused
    return (int8_t)(int)c;
}

// The same codes without the XU pipe (the IEEE quotient costs MUFU.RCP, roundf FRND, the
// cast F2I: three quarter-rate XU ops per element): for 2^-100 <= scale <= 2^100,
// r = fl(x * fl(1/scale)) lies within 3 * 2^-24 |x/scale| <= 2^-15 of fl(x/scale)
// (|x/scale| <= 127 (1 + 2^-23)), so unless r is within 2^-14 of a half-integer both
// round to the same integer -- computed by adding 1.5 * 2^23 (the sum's last mantissa bit
// is the units place, any rounding of a non-tie lands on the nearest integer).  Near a
// half-integer the IEEE form decides (probability ~2^-13 per element).
struct Int8Q {
    float scale, inv;
    bool fast;
    __device__ __forceinline__ explicit Int8Q(float sc)
        : scale(sc), inv(0.0f), fast(sc >= 0x1p-100f && sc <= 0x1p100f) {
        if (fast) inv = __frcp_rn(sc);
    }
    // code of x as a byte; `unsure` set when the IEEE form must decide
    __device__ __forceinline__ uint32_t code_fast(float x, bool &unsure) const {
        const float r = __fmul_rn(x, inv);
        const float y = __fadd_rn(r, 12582912.0f);                     // 1.5 * 2^23
        const float k = __fsub_rn(y, 12582912.0f);                     // nearest integer (exact)
        unsure |= !(fabsf(__fsub_rn(r, k)) < 0.5f - 0x1p-14f);
        const int c = max(-127, min(127, (int)(__float_as_uint(y) - 0x4b400000u)));
        return (uint32_t)c & 0xffu;
    }
    __device__ __forceinline__ uint32_t pack4(float4 v) const {
        bool unsure = !fast;
        const uint32_t w = code_fast(v.x, unsure) | (code_fast(v.y, unsure) << 8) | (code_fast(v.z, unsure) << 16) |
                           (code_fast(v.w, unsure) << 24);
        if (!unsure) return w;
        return (uint32_t)(uint8_t)int8_code(v.x, scale) | ((uint32_t)(uint8_t)int8_code(v.y, scale) << 8) |
               ((uint32_t)(uint8_t)int8_code(v.z, scale) << 16) | ((uint32_t)(uint8_t)int8_code(v.w, scale) << 24);
    }
};

__global__ void __launch_bounds__(kI8Threads)
tlc_int8_quant_kernel(const float *__restrict__ t, uint64_t n, int8_t *__restrict__ codes, tlc_header *hdr,
                      const unsigned int *maxkey, int vec) {
    const unsigned int key = maxkey[0];
    const unsigned int status = key >= 0x7f800000u ? (unsigned int)TLC_ERR_NONFINITE : (unsigned int)TLC_OK;
    const float scale = status == TLC_OK ? __fdiv_rn(__uint_as_float(key), 127.0f) : 0.0f;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        hdr->M = scale;
        hdr->flags = TLC_FLAG_INT8;
        hdr->n = n;
        hdr->payload_len = status == TLC_OK ? n : 0;
        hdr->status = status;
        hdr->reserved = 0;
    }
    if (status != TLC_OK) return;
    const Int8Q Q(scale);
    const uint64_t stride = (uint64_t)gridDim.x * kI8Threads;
    uint64_t head = 0;
    if (vec) {
        // warp step ws covers float4 numbers 128 ws + 32 k + lane, k = 0..3
        const uint64_t n4 = n / 4;
        const float4 *t4 = reinterpret_cast<const float4 *>(t);
        uint32_t *c32 = reinterpret_cast<uint32_t *>(codes);
        const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        const uint64_t nw = n4 / 128;                                         // 128 float4 per warp step
        const uint64_t wstride = (uint64_t)gridDim.x * (kI8Threads / 32);
        for (uint64_t ws = (uint64_t)blockIdx.x * (kI8Threads / 32) + warp; ws < nw; ws += wstride) {
            float4 v[4];
#pragma unroll
            for (int k = 0; k < 4; k++) v[k] = ld_stream4(t4 + 128 * ws + 32 * k + lane);
#pragma unroll
            for (int k = 0; k < 4; k++) __stcs(c32 + 128 * ws + 32 * k + lane, Q.pack4(v[k]));
        }
        head = 4 * 128 * nw;
    }
    for (uint64_t i = head + (uint64_t)blockIdx.x * kI8Threads + threadIdx.x; i < n; i += stride)
        codes[i] = int8_code(ld_stream(t + i), scale);
}

__device__ __forceinline__ float dq(int8_t c, float scale) { return __fmul_rn(scale, (float)c); }

__device__ __forceinline__ float4 dq4(uint32_t w, float scale, float4 o, int mode) {
    const int8_t c0 = (int8_t)(w & 0xff), c1 = (int8_t)((w >> 8) & 0xff), c2 = (int8_t)((w >> 16) & 0xff),
                 c3 = (int8_t)(w >> 24);
    if (mode == TLC_MODE_OVERWRITE) return make_float4(dq(c0, scale), dq(c1, scale), dq(c2, scale), dq(c3, scale));
    // accumulate: add only where code != 0 (R16); other elements keep their bits
    return make_float4(c0 ? __fadd_rn(o.x, dq(c0, scale)) : o.x, c1 ? __fadd_rn(o.y, dq(c1, scale)) : o.y,
                       c2 ? __fadd_rn(o.z, dq(c2, scale)) : o.z, c3 ? __fadd_rn(o.w, dq(c3, scale)) : o.w);
}

__global__ void __launch_bounds__(kI8Threads)
tlc_int8_dequant_kernel(const int8_t *__restrict__ codes, tlc_header *hdr, uint64_t n, float *__restrict__ out,
                        int mode, int vec) {
    // header checks: the producer's n, the int8 flag, a finite scale >= +0 (R21, R23)
    const float scale = hdr->M;
    const bool ok = hdr->status == TLC_OK && hdr->n == n && (hdr->flags & TLC_FLAG_INT8) &&
                    hdr->payload_len == n && !signbit(scale) && isfinite(scale);
    if (!ok) {
        if (blockIdx.x == 0 && threadIdx.x == 0 && hdr->status == TLC_OK) raise_format(hdr);
        return;
    }
    const uint64_t stride = (uint64_t)gridDim.x * kI8Threads;
    uint64_t head = 0;
    if (vec) {
        const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        const uint64_t nw = n / 512;                                          // 128 code words per warp step
        const uint64_t wstride = (uint64_t)gridDim.x * (kI8Threads / 32);
        const uint32_t *c32 = reinterpret_cast<const uint32_t *>(codes);
        float4 *o4 = reinterpret_cast<float4 *>(out);
        for (uint64_t ws = (uint64_t)blockIdx.x * (kI8Threads / 32) + warp; ws < nw; ws += wstride) {
            uint32_t w[4];
#pragma unroll
            for (int k = 0; k < 4; k++) w[k] = __ldcs(c32 + 128 * ws + 32 * k + lane);
#pragma unroll
            for (int k = 0; k < 4; k++) {
                float4 *dst = o4 + 128 * ws + 32 * k + lane;
                const float4 o = mode == TLC_MODE_OVERWRITE ? make_float4(0, 0, 0, 0) : *dst;
                __stcs(dst, dq4(w[k], scale, o, mode));
            }
        }
        head = 512 * nw;
    }
    for (uint64_t i = head + (uint64_t)blockIdx.x * kI8Threads + threadIdx.x; i < n; i += stride) {
        const int8_t c = codes[i];
        if (mode == TLC_MODE_OVERWRITE) out[i] = dq(c, scale);
        else if (c) out[i] = __fadd_rn(out[i], dq(c, scale));
    }
}

template <class K>
static int grid_for(K kernel, uint64_t work) {
    int blocks = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kernel, kI8Threads, 0);
    return (int)tmax<uint64_t>(1, tmin<uint64_t>((work + kI8Threads - 1) / kI8Threads,
                                                 (uint64_t)num_sms() * tmax(1, blocks)));
}

int launch_int8_compress(const float *t, uint64_t n, int8_t *codes, tlc_header *hdr, void *ws, cudaStream_t st) {
    uint64_t scratch = 0;
    const SegTable T = single_table(t, nullptr, nullptr, nullptr, hdr, n, scratch);
    const WsLayout L = ws_layout(T, 0);
    unsigned int *maxkey = reinterpret_cast<unsigned int *>(reinterpret_cast<char *>(ws) + L.maxkey);
    if (cudaMemsetAsync(ws, 0, L.memset_c, st) != cudaSuccess) return TLC_ERR_CUDA;
    launch_absmax(T, maxkey, false, st);
    {
        KernelScope ks(kKq8, st);
        static int grid = 0;
        if (!grid) grid = grid_for(tlc_int8_quant_kernel, ~0ull >> 8);
        const int vec = aligned16(t) && aligned16(codes);
        const int g = (int)tmin<uint64_t>((uint64_t)grid, tmax<uint64_t>(1, (n / 16 + kI8Threads - 1) / kI8Threads));
        tlc_int8_quant_kernel<<<g, kI8Threads, 0, st>>>(t, n, codes, hdr, maxkey, vec);
    }
    return cudaPeekAtLastError() == cudaSuccess ? TLC_OK : TLC_ERR_CUDA;
}

int launch_int8_decompress(const int8_t *codes, tlc_header *hdr, uint64_t n, float *out, int mode, cudaStream_t st) {
    KernelScope ks(kKd8, st);
    static int grid = 0;
    if (!grid) grid = grid_for(tlc_int8_dequant_kernel, ~0ull >> 8);
    const int vec = aligned16(codes) && aligned16(out);
    const int g = (int)tmin<uint64_t>((uint64_t)grid, tmax<uint64_t>(1, (n / 16 + kI8Threads - 1) / kI8Threads));
    tlc_int8_dequant_kernel<<<g, kI8Threads, 0, st>>>(codes, hdr, n, out, mode, vec);
    return cudaPeekAtLastError() == cudaSuccess ? TLC_OK : TLC_ERR_CUDA;
}

}  // namespace tlc
