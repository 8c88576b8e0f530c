// decompress.cu -- the 3LC decompressor on sm_100a (rows a5-a6).
//
//  K4 tlc_zre_scan_kernel: validates the header; with ZRE, scans the
//     expansion lengths len(b) = b >= 243 ? b-241 : 1 (inverse of P:545-546)
//     with a decoupled look-back and writes, for every output tile start
//     J0 = k*kOutTile, a seek entry (payload byte covering J0, offset inside
//     it).  The last tile checks that the expansion is exactly P bytes.
//  K5 tlc_expand_dequant_kernel: output-driven, one tile = kOutTile quartic
//     bytes = 5*kOutTile fp32 outputs, so every CTA does the same work whatever
//     the run structure.  Expands the covering payload bytes into shared
//     memory, decodes base 3 through a 243-entry digit table, and
//     writes M*q (Eq. 3) -- or adds it where q != 0 (R16) -- to the
//     five partitions with coalesced 128-bit stores.
#include "tlc_device.cuh"
#include "tlc_launch.h"

namespace tlc {

constexpr int kK4Threads = 256;
constexpr int kK4BytesPerThread = 8;
constexpr int kK4Tile = kK4Threads * kK4BytesPerThread;   // payload bytes per scan tile
constexpr int kK4Warps = kK4Threads / 32;

constexpr int kK5Threads = 256;
constexpr int kOutTile = 2048;                             // quartic bytes per output tile

constexpr unsigned long long kSumMask = (1ull << 62) - 1;

__device__ __forceinline__ void raise_format(tlc_header *hdr) {
    atomicCAS(&hdr->status, (unsigned int)TLC_OK, (unsigned int)TLC_ERR_FORMAT);
}

__device__ __forceinline__ uint32_t zre_len(uint32_t b) { return b >= kFirstRunCode ? b - 241u : 1u; }

// ============================================================== K4
__global__ void __launch_bounds__(kK4Threads)
tlc_zre_scan_kernel(const uint8_t *__restrict__ payload, tlc_header *hdr, uint64_t n, Ctrl *ctrl,
                    unsigned long long *states, unsigned long long *seek) {
    __shared__ unsigned int s_warp[kK4Warps];
    __shared__ unsigned long long s_tile_excl;
    __shared__ unsigned int s_tile;
    const uint64_t P = (n + 4) / 5;
    const unsigned int status = hdr->status;
    const uint64_t Z = hdr->payload_len;
    const bool zre = (hdr->flags & TLC_FLAG_ZRE) != 0;
    const bool valid = status == TLC_OK && hdr->n == n && Z <= P && Z >= 1 && (zre || Z == P);
    if (!valid) {
        if (blockIdx.x == 0 && threadIdx.x == 0 && status == TLC_OK) raise_format(hdr);
        return;
    }
    if (!zre) return;
    const uint64_t num_tiles = (Z + kK4Tile - 1) / kK4Tile;
    const uint64_t num_out_tiles = (P + kOutTile - 1) / kOutTile;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

    while (true) {
        if (threadIdx.x == 0) s_tile = atomicAdd(&ctrl->tile_counter, 1u);
        __syncthreads();
        const uint64_t tile = s_tile;
        if (tile >= num_tiles) break;
        const uint64_t z0 = tile * kK4Tile + (uint64_t)threadIdx.x * kK4BytesPerThread;
        uint8_t b[kK4BytesPerThread];
        uint32_t len[kK4BytesPerThread];
        uint32_t sum = 0;
#pragma unroll
        for (int m = 0; m < kK4BytesPerThread; m++) {
            b[m] = (z0 + m < Z) ? payload[z0 + m] : 0;
            len[m] = (z0 + m < Z) ? zre_len(b[m]) : 0u;
            sum += len[m];
        }
        // block exclusive scan of the per-thread sums
        uint32_t x = sum;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
            if (lane >= d) x += y;
        }
        if (lane == 31) s_warp[warp] = x;
        __syncthreads();
        if (warp == 0) {
            uint32_t agg = 0;
#pragma unroll
            for (int w = 0; w < kK4Warps; w++) agg += s_warp[w];
            unsigned long long excl = 0;
            if (tile == 0) {
                if (lane == 0) st_relaxed_u64(states, kStatusPrefix | agg);
            } else {
                if (lane == 0) st_relaxed_u64(states + tile, kStatusAgg | agg);
                int64_t pred = (int64_t)tile - 1;
                while (true) {
                    const int64_t idx = pred - lane;
                    unsigned long long w = idx >= 0 ? ld_relaxed_u64(states + idx) : kStatusPrefix;
                    const unsigned int st = (unsigned int)(w >> 62);
                    const unsigned int pref = __ballot_sync(0xffffffffu, st == 2u);
                    const unsigned int inval = __ballot_sync(0xffffffffu, st == 0u);
                    const int first = pref ? (__ffs(pref) - 1) : 31;
                    const unsigned int window = (first == 31) ? 0xffffffffu : ((2u << first) - 1u);
                    if (inval & window) { __nanosleep(32); continue; }
                    unsigned long long v = (lane <= first) ? (w & kSumMask) : 0ull;
#pragma unroll
                    for (int d = 16; d >= 1; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
                    excl += v;
                    if (pref) break;
                    pred -= 32;
                }
                if (lane == 0) st_relaxed_u64(states + tile, kStatusPrefix | (excl + agg));
            }
            if (lane == 0) {
                s_tile_excl = excl;
                if (tile == num_tiles - 1 && excl + agg != P) raise_format(hdr);
            }
            __syncwarp();
            if (lane == 0) {   // exclusive warp offsets
                uint32_t acc = 0;
                for (int w = 0; w < kK4Warps; w++) { uint32_t t = s_warp[w]; s_warp[w] = acc; acc += t; }
            }
        }
        __syncthreads();
        // seek entries: the byte whose expansion [pos, pos+len) contains J0 = k*kOutTile
        uint64_t pos = s_tile_excl + s_warp[warp] + (x - sum);
#pragma unroll
        for (int m = 0; m < kK4BytesPerThread; m++) {
            if (len[m]) {
                const uint64_t k = (pos + kOutTile - 1) / kOutTile;
                const uint64_t J0 = k * kOutTile;
                if (J0 < pos + len[m] && k < num_out_tiles)
                    seek[k] = ((z0 + m) << 4) | (J0 - pos);
                pos += len[m];
            }
        }
        __syncthreads();
    }
}

// ============================================================== K5
struct K5Smem {
    alignas(16) uint8_t E[kOutTile];     // expanded quartic bytes of the tile
    uint16_t lut[256];                   // base-3 digits d0..d4, 2 bits each (d0 highest)
    unsigned int warp_sum[kK5Threads / 32];
};

__device__ __forceinline__ float trit_value(float M, uint32_t d) {
    // Eq. 3: M * q with q = d - 1 in {-1, 0, 1}; the same single fp32 multiply
    // as T_out = M * T_quantized.
    const float qf = d == 0 ? -1.0f : (d == 2 ? 1.0f : 0.0f);
    return __fmul_rn(M, qf);
}

template <bool kVec, int kMode>
__global__ void __launch_bounds__(kK5Threads)
tlc_expand_dequant_kernel(const uint8_t *__restrict__ payload, tlc_header *hdr, uint64_t n,
                          float *__restrict__ out, const unsigned long long *__restrict__ seek) {
    __shared__ K5Smem sm;
    if (hdr->status != TLC_OK) return;
    const float M = hdr->M;
    const bool zre = (hdr->flags & TLC_FLAG_ZRE) != 0;
    const uint64_t Z = hdr->payload_len;
    const uint64_t P = (n + 4) / 5;
    const uint64_t num_tiles = (P + kOutTile - 1) / kOutTile;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

    // digit table: step 1 of decoding, "dividing a by a power of 3 and taking
    // the remainder", precomputed for the 243 byte values.
    for (int v = threadIdx.x; v < 256; v += kK5Threads) {
        uint32_t w = 0, r = v < 243 ? v : 121;
#pragma unroll
        for (int i = 0; i < 5; i++) { w |= (r % 3u) << (2 * i); r /= 3u; }
        sm.lut[v] = (uint16_t)w;   // bits 2i..2i+1 = digit of partition 4-i
    }
    bool bad = false;

    for (uint64_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const uint64_t J0 = tile * kOutTile;
        const int tl = (int)tmin<uint64_t>(kOutTile, P - J0);
        __syncthreads();   // previous tile's readers of sm.E are done (and lut is built)
        if (zre) {
            const unsigned long long sk = seek[tile];
            const uint64_t bi = sk >> 4;
            const uint32_t skip = (uint32_t)(sk & 15);
            // thread owns window bytes [8*tid, 8*tid+8) of payload[bi, bi + kK5Window)
            const uint64_t zb = bi + (uint64_t)threadIdx.x * 8;
            uint8_t b[8];
            uint32_t len[8], sum = 0;
#pragma unroll
            for (int m = 0; m < 8; m++) {
                b[m] = (zb + m < Z) ? payload[zb + m] : 0;
                len[m] = (zb + m < Z) ? zre_len(b[m]) : 0u;
                sum += len[m];
            }
            uint32_t x = sum;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
                if (lane >= d) x += y;
            }
            if (lane == 31) sm.warp_sum[warp] = x;
            __syncthreads();
            uint32_t wofs = 0;
            for (int w = 0; w < warp; w++) wofs += sm.warp_sum[w];
            // local position (relative to J0) of this thread's first byte
            int64_t p = (int64_t)wofs + (x - sum) - (int64_t)skip;
#pragma unroll
            for (int m = 0; m < 8; m++) {
                const int64_t lo = tmax<int64_t>(p, 0), hi = tmin<int64_t>(p + len[m], tl);
                const uint8_t v = b[m] >= kFirstRunCode ? kZeroGroup : b[m];
                for (int64_t q = lo; q < hi; q++) sm.E[q] = v;
                p += len[m];
            }
        } else {
            for (int jl = threadIdx.x; jl < tl; jl += kK5Threads) {
                uint8_t v = payload[J0 + jl];
                if (v > 242) { bad = true; v = kZeroGroup; }
                sm.E[jl] = v;
            }
        }
        __syncthreads();

        // ---- base-3 decode + dequantize, 4 consecutive quartic bytes per thread
        for (int jl = 4 * threadIdx.x; jl < tl; jl += 4 * kK5Threads) {
            const uint32_t w4 = *reinterpret_cast<const uint32_t *>(sm.E + jl);
            uint32_t dg[4];
#pragma unroll
            for (int c = 0; c < 4; c++) dg[c] = sm.lut[(w4 >> (8 * c)) & 0xff];
            const uint64_t j = J0 + jl;
#pragma unroll
            for (int i = 0; i < 5; i++) {
                const int sh = 2 * (4 - i);
                uint32_t d[4];
#pragma unroll
                for (int c = 0; c < 4; c++) d[c] = (dg[c] >> sh) & 3u;
                const uint64_t e = (uint64_t)i * P + j;
                const bool full = kVec && (jl + 3 < tl) && (e + 3 < n);
                if (kMode == TLC_MODE_OVERWRITE) {
                    if (full) {
                        __stcs(reinterpret_cast<float4 *>(out + e),
                               make_float4(trit_value(M, d[0]), trit_value(M, d[1]),
                                           trit_value(M, d[2]), trit_value(M, d[3])));
                    } else {
#pragma unroll
                        for (int c = 0; c < 4; c++)
                            if (jl + c < tl && e + c < n) out[e + c] = trit_value(M, d[c]);
                    }
                } else {
                    const bool any = (d[0] != 1) | (d[1] != 1) | (d[2] != 1) | (d[3] != 1);
                    if (!any) continue;                       // skip-zero: sector untouched (R16)
                    if (full) {
                        float4 o = *reinterpret_cast<float4 *>(out + e);
                        if (d[0] != 1) o.x = __fadd_rn(o.x, trit_value(M, d[0]));
                        if (d[1] != 1) o.y = __fadd_rn(o.y, trit_value(M, d[1]));
                        if (d[2] != 1) o.z = __fadd_rn(o.z, trit_value(M, d[2]));
                        if (d[3] != 1) o.w = __fadd_rn(o.w, trit_value(M, d[3]));
                        *reinterpret_cast<float4 *>(out + e) = o;
                    } else {
#pragma unroll
                        for (int c = 0; c < 4; c++)
                            if (jl + c < tl && e + c < n && d[c] != 1)
                                out[e + c] = __fadd_rn(out[e + c], trit_value(M, d[c]));
                    }
                }
            }
        }
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) raise_format(hdr);
}

// ============================================================== host launchers
static int g_k5_blocks = 0;

int launch_decompress(const uint8_t *payload, tlc_header *hdr, uint64_t n, float *out, int mode,
                      void *ws, cudaStream_t st) {
    const uint64_t P = (n + 4) / 5;
    const uint64_t scan_tiles = (P + kK4Tile - 1) / kK4Tile;
    const uint64_t out_tiles = (P + kOutTile - 1) / kOutTile;
    Ctrl *ctrl = reinterpret_cast<Ctrl *>(ws);
    unsigned long long *states = reinterpret_cast<unsigned long long *>((char *)ws + sizeof(Ctrl));
    unsigned long long *seek = reinterpret_cast<unsigned long long *>(
        (char *)ws + sizeof(Ctrl) + align256(scan_tiles * sizeof(unsigned long long)));
    if (cudaMemsetAsync(ws, 0, sizeof(Ctrl) + scan_tiles * sizeof(unsigned long long), st) != cudaSuccess)
        return TLC_ERR_CUDA;
    const int sms = num_sms();
    if (!g_k5_blocks)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_k5_blocks, tlc_expand_dequant_kernel<true, 0>, kK5Threads, 0);
    const int grid4 = (int)tmin<uint64_t>(scan_tiles, (uint64_t)sms * 8);
    {
        KernelScope ks(kK4, st);
        tlc_zre_scan_kernel<<<grid4, kK4Threads, 0, st>>>(payload, hdr, n, ctrl, states, seek);
    }
    const int grid5 = (int)tmin<uint64_t>(out_tiles, (uint64_t)sms * max(1, g_k5_blocks));
    const bool vec = (P % 4 == 0) && aligned16(out);
    KernelScope ks(kK5, st);
    if (mode == TLC_MODE_OVERWRITE) {
        if (vec) tlc_expand_dequant_kernel<true, 0><<<grid5, kK5Threads, 0, st>>>(payload, hdr, n, out, seek);
        else tlc_expand_dequant_kernel<false, 0><<<grid5, kK5Threads, 0, st>>>(payload, hdr, n, out, seek);
    } else {
        if (vec) tlc_expand_dequant_kernel<true, 1><<<grid5, kK5Threads, 0, st>>>(payload, hdr, n, out, seek);
        else tlc_expand_dequant_kernel<false, 1><<<grid5, kK5Threads, 0, st>>>(payload, hdr, n, out, seek);
    }
    return cudaPeekAtLastError() == cudaSuccess ? TLC_OK : TLC_ERR_CUDA;
}

size_t decompress_workspace_bytes(uint64_t n) {
    const uint64_t P = (n + 4) / 5;
    const uint64_t scan_tiles = (P + kK4Tile - 1) / kK4Tile;
    const uint64_t out_tiles = (P + kOutTile - 1) / kOutTile;
    return sizeof(Ctrl) + align256(scan_tiles * sizeof(unsigned long long)) +
           align256(out_tiles * sizeof(unsigned long long));
}

}  // namespace tlc
