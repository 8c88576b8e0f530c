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


constexpr int kK5Threads = 256;
constexpr int kOutTile = 4096;                             // quartic bytes per output tile


// ============================================================== K4
// Same chunked single-pass scan as K3 (compress.cu), over the sum monoid of
// expansion lengths: phase 1 sums each chunk, phase 2 adds the preceding
// chunks' sums, phase 3 re-scans the chunk (L2-resident) and writes the seek
// entry of every output tile start that falls inside one of its bytes.
constexpr int kK4Threads = kScanThreads;
constexpr int kK4Seg = 16;
constexpr int kK4Row = kK4Threads * kK4Seg;

__device__ __forceinline__ int load_pay16(const uint8_t *__restrict__ p, uint64_t pos, uint64_t hi,
                                          uint32_t (&len)[kK4Seg]) {
    const int n = pos < hi ? (int)tmin<uint64_t>(kK4Seg, hi - pos) : 0;
    uint8_t b[kK4Seg];
    if (n == kK4Seg && (reinterpret_cast<uintptr_t>(p + pos) & 15u) == 0) {
        const uint4 w = __ldg(reinterpret_cast<const uint4 *>(p + pos));
        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int k = 0; k < kK4Seg; k++) b[k] = (ws[k >> 2] >> (8 * (k & 3))) & 0xff;
    } else {
#pragma unroll
        for (int k = 0; k < kK4Seg; k++) b[k] = k < n ? p[pos + k] : 0;
    }
#pragma unroll
    for (int k = 0; k < kK4Seg; k++) len[k] = k < n ? zre_len(b[k]) : 0u;
    return n;
}

__global__ void __launch_bounds__(kK4Threads)
tlc_zre_scan_kernel(const uint8_t *__restrict__ payload, tlc_header *hdr, uint64_t n, Ctrl *ctrl,
                    unsigned long long *states, unsigned long long *seek) {
    __shared__ unsigned long long s_warp[kScanWarps];
    __shared__ unsigned int s_id;
    const uint64_t P = (n + 4) / 5;
    const unsigned int status = hdr->status;
    const uint64_t Z = hdr->payload_len;
    const bool zre = (hdr->flags & TLC_FLAG_ZRE) != 0;
    const bool valid = header_valid(hdr, n);
    if (!valid) {
        if (blockIdx.x == 0 && threadIdx.x == 0 && status == TLC_OK) raise_format(hdr);
        return;
    }
    if (!zre) return;
    // chunk size from the device-side payload length: at most gridDim.x chunks
    const uint64_t chunk = tmax<uint64_t>(kK4Row, ((Z + gridDim.x - 1) / gridDim.x + kK4Seg - 1) / kK4Seg * kK4Seg);
    const uint64_t nchunks = (Z + chunk - 1) / chunk;
    const uint64_t num_out_tiles = (P + kOutTile - 1) / kOutTile;
    if (threadIdx.x == 0) s_id = atomicAdd(&ctrl->tile_counter, 1u);
    __syncthreads();
    const uint64_t b = s_id;
    if (b >= nchunks) return;
    const uint64_t lo = b * chunk, hi = tmin<uint64_t>(Z, lo + chunk);
    uint32_t len[kK4Seg];

    // ---- phase 1: expansion length of the chunk
    uint64_t agg = 0;
    for (uint64_t row = lo; row < hi; row += kK4Row) {
        load_pay16(payload, row + (uint64_t)kK4Seg * threadIdx.x, hi, len);
        uint32_t sum = 0;
#pragma unroll
        for (int k = 0; k < kK4Seg; k++) sum += len[k];
        agg += block_reduce_sum(sum, s_warp);
    }
    if (threadIdx.x == 0) st_relaxed_u64(states + b, kReady | agg);

    // ---- phase 2: quartic position of the chunk's first byte
    uint64_t part = 0;
    const uint64_t per = (b + kK4Threads - 1) / kK4Threads;
    const uint64_t i0 = per * threadIdx.x, i1 = tmin<uint64_t>(b, i0 + per);
    for (uint64_t i = i0; i < i1; i++) part += wait_ready(states + i) & ~kReady;
    uint64_t run = block_reduce_sum(part, s_warp);
    if (b == nchunks - 1 && threadIdx.x == 0 && run + agg != P) raise_format(hdr);

    // ---- phase 3: seek entries (payload byte covering J0 = k*kOutTile, offset inside it)
    for (uint64_t row = lo; row < hi; row += kK4Row) {
        const uint64_t pos0 = row + (uint64_t)kK4Seg * threadIdx.x;
        load_pay16(payload, pos0, hi, len);
        uint32_t sum = 0;
#pragma unroll
        for (int k = 0; k < kK4Seg; k++) sum += len[k];
        uint64_t row_total;
        uint64_t q = run + block_excl_scan_sum(sum, s_warp, row_total);
#pragma unroll
        for (int k = 0; k < kK4Seg; k++) {
            if (len[k]) {
                const uint64_t kt = (q + kOutTile - 1) / kOutTile;
                const uint64_t J0 = kt * kOutTile;
                if (J0 < q + len[k] && kt < num_out_tiles) seek[kt] = ((pos0 + k) << 4) | (J0 - q);
                q += len[k];
            }
        }
        run += row_total;
    }
}

// ============================================================== K5
constexpr int kK5BytesPerThread = kOutTile / kK5Threads;   // 16 quartic bytes per thread per tile
constexpr int kK5Words = kK5BytesPerThread / 4;

struct K5Smem {
    alignas(16) uint8_t E[kOutTile];     // expanded quartic bytes of the tile
    uint32_t V[5][256];                  // Eq. 3 output bits of partition i for byte value b
    uint16_t lut[256];                   // per byte: bit i = (digit_i != 1), bit 8+i = (digit_i == 0)
    unsigned int warp_sum[kK5Threads / 32];
};

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
    const bool pal = (reinterpret_cast<uintptr_t>(payload) & 3u) == 0;   // word loads allowed

    // Decoding step 1, "dividing a by a power of 3 and taking the remainder"
    // (P:514-515), tabulated for the 243 byte values, and Eq. 3,
    // T_out = M * q, tabulated per partition: V[i][b] = M * (digit_i(b) - 1).
    for (int v = threadIdx.x; v < 256; v += kK5Threads) {
        uint32_t w = 0, r = v < 243 ? v : 121;
#pragma unroll
        for (int i = 4; i >= 0; i--) {
            const uint32_t d = r % 3u;
            r /= 3u;
            w |= (uint32_t)(d != 1) << i;
            w |= (uint32_t)(d == 0) << (8 + i);
            sm.V[i][v] = __float_as_uint(__fmul_rn(M, (float)((int)d - 1)));
        }
        sm.lut[v] = (uint16_t)w;
    }
    bool bad = false;

    for (uint64_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const uint64_t J0 = tile * kOutTile;
        const int tl = (int)tmin<uint64_t>(kOutTile, P - J0);
        // valid positions of partition i in this tile: e = i*P + J0 + jl < n
        int lim[5];
        float *ob[5];
#pragma unroll
        for (int i = 0; i < 5; i++) {
            const uint64_t e0 = (uint64_t)i * P + J0;
            lim[i] = e0 >= n ? 0 : (int)tmin<uint64_t>(tl, n - e0);
            ob[i] = out + e0;
        }
        __syncthreads();   // previous tile's readers of sm.E are done (and the tables are built)
        if (zre) {
            // pre-fill with 121: zero-run codes expand to 121s and need no further writes
            *reinterpret_cast<uint4 *>(sm.E + kK5BytesPerThread * threadIdx.x) =
                make_uint4(0x79797979u, 0x79797979u, 0x79797979u, 0x79797979u);
            const unsigned long long sk = seek[tile];
            const uint64_t bi = sk >> 4;                      // payload byte covering J0
            const int skip = (int)(sk & 15);                  // J0 - (first position of that byte)
            const uint64_t be = tile + 1 < num_tiles ? (seek[tile + 1] >> 4) : Z - 1;   // last byte needed
            const int wl = (int)(be - bi) + 1;                // <= kOutTile + 1
            // thread owns window bytes [16*tid, 16*tid+16) relative to w0 = bi rounded down
            // to 4; the last thread also owns the next 4 bytes, so the <= kOutTile bytes
            // from bi on are always covered
            const uint64_t w0 = bi & ~3ull;
            const int sh = (int)(bi - w0);
            constexpr int NW = kK5Words + 1;
            const int nwords = threadIdx.x == kK5Threads - 1 ? NW : kK5Words;
            uint32_t wd[NW];
#pragma unroll
            for (int h = 0; h < NW; h++) {
                wd[h] = 0;
                if (h >= nwords) continue;
                const int r = kK5BytesPerThread * threadIdx.x + 4 * h - sh;   // window offset of the word
                if (pal && r >= 0 && r + 3 < wl) {
                    wd[h] = __ldg(reinterpret_cast<const uint32_t *>(payload + w0) + kK5Words * threadIdx.x + h);
                } else {
                    uint32_t x = 0;
#pragma unroll
                    for (int c = 0; c < 4; c++)
                        if (r + c >= 0 && r + c < wl) x |= (uint32_t)payload[bi + r + c] << (8 * c);
                    wd[h] = x;
                }
            }
            uint32_t len[4 * NW], sum = 0;
#pragma unroll
            for (int m = 0; m < 4 * NW; m++) {
                const int r = kK5BytesPerThread * threadIdx.x + m - sh;
                const uint32_t b = (wd[m >> 2] >> (8 * (m & 3))) & 0xffu;
                len[m] = (m < 4 * nwords && r >= 0 && r < wl) ? zre_len(b) : 0u;
                sum += len[m];
            }
            uint32_t x = sum;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
                if (lane >= d) x += y;
            }
            if (lane == 31) sm.warp_sum[warp] = x;
            __syncthreads();
            uint32_t wofs = 0;
#pragma unroll
            for (int w = 0; w < kK5Threads / 32; w++) wofs += (w < warp) ? sm.warp_sum[w] : 0u;
            int p = (int)(wofs + x - sum) - skip;   // tile position of this thread's first byte
#pragma unroll
            for (int m = 0; m < 4 * NW; m++) {
                const uint32_t b = (wd[m >> 2] >> (8 * (m & 3))) & 0xffu;
                if (len[m] == 1 && p >= 0 && p < tl) sm.E[p] = (uint8_t)b;   // literal byte
                p += (int)len[m];
            }
        } else {
            for (int jl = threadIdx.x; jl < tl; jl += kK5Threads) {
                uint8_t v = payload[J0 + jl];
                if (v > 242) { bad = true; v = kZeroGroup; }
                sm.E[jl] = v;
            }
        }
        __syncthreads();

        // ---- base-3 decode + dequantize, 4 consecutive quartic bytes per step
#pragma unroll
        for (int k = 0; k < kK5BytesPerThread / 4; k++) {
            const int jl = 4 * threadIdx.x + 4 * kK5Threads * k;
            if (jl >= tl) break;
            const uint32_t w4 = *reinterpret_cast<const uint32_t *>(sm.E + jl);
            const uint32_t b0 = w4 & 0xffu, b1 = (w4 >> 8) & 0xffu, b2 = (w4 >> 16) & 0xffu, b3 = w4 >> 24;
            if (kMode == TLC_MODE_OVERWRITE) {
                const bool zero4 = w4 == 0x79797979u;   // four all-zero groups: 20 x +0
#pragma unroll
                for (int i = 0; i < 5; i++) {
                    float *o = ob[i] + jl;
                    uint4 v = make_uint4(0u, 0u, 0u, 0u);
                    if (!zero4) v = make_uint4(sm.V[i][b0], sm.V[i][b1], sm.V[i][b2], sm.V[i][b3]);
                    if (kVec && jl + 3 < lim[i]) {
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
                    if (kVec && jl + 3 < lim[i]) {
                        float4 v = *reinterpret_cast<float4 *>(o);
                        float *vv = reinterpret_cast<float *>(&v);
#pragma unroll
                        for (int c = 0; c < 4; c++)
                            if ((L[c] >> i) & 1u) vv[c] = __fadd_rn(vv[c], __uint_as_float(sm.V[i][bb[c]]));
                        *reinterpret_cast<float4 *>(o) = v;
                    } else {
#pragma unroll
                        for (int c = 0; c < 4; c++)
                            if (jl + c < lim[i] && ((L[c] >> i) & 1u))
                                o[c] = __fadd_rn(o[c], __uint_as_float(sm.V[i][bb[c]]));
                    }
                }
            }
        }
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) raise_format(hdr);
}

// ============================================================== host launchers
static int g_k5_blocks = 0;

static int g_k4_blocks = 0;
constexpr int kMaxScanChunks = kMaxSms * 16;

int launch_decompress(const uint8_t *payload, tlc_header *hdr, uint64_t n, float *out, int mode,
                      void *ws, cudaStream_t st) {
    const uint64_t P = (n + 4) / 5;
    const uint64_t out_tiles = (P + kOutTile - 1) / kOutTile;
    Ctrl *ctrl = reinterpret_cast<Ctrl *>(ws);
    unsigned long long *states = reinterpret_cast<unsigned long long *>((char *)ws + sizeof(Ctrl));
    unsigned long long *seek = reinterpret_cast<unsigned long long *>(
        (char *)ws + sizeof(Ctrl) + align256(kMaxScanChunks * sizeof(unsigned long long)));
    if (cudaMemsetAsync(ws, 0, sizeof(Ctrl) + kMaxScanChunks * sizeof(unsigned long long), st) != cudaSuccess)
        return TLC_ERR_CUDA;
    const int sms = num_sms();
    if (!g_k5_blocks)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_k5_blocks, tlc_expand_dequant_kernel<true, 0>, kK5Threads, 0);
    if (!g_k4_blocks)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_k4_blocks, tlc_zre_scan_kernel, kK4Threads, 0);
    {
        KernelScope ks(kK4, st);
        const uint64_t rows = (P + kK4Row - 1) / kK4Row;
        const int grid4 = (int)tmax<uint64_t>(1, tmin<uint64_t>(rows, (uint64_t)sms * tmin(16, tmax(1, g_k4_blocks))));
        tlc_zre_scan_kernel<<<grid4, kK4Threads, 0, st>>>(payload, hdr, n, ctrl, states, seek);
    }
    const int grid5 = (int)tmin<uint64_t>(out_tiles, (uint64_t)sms * tmax(1, g_k5_blocks));
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
    const uint64_t out_tiles = (P + kOutTile - 1) / kOutTile;
    return sizeof(Ctrl) + align256(kMaxScanChunks * sizeof(unsigned long long)) +
           align256(out_tiles * sizeof(unsigned long long));
}

}  // namespace tlc
