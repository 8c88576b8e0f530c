// batched.cu -- one launch for a whole list of small tensors (SURVEY 8(a),
// "small-tensor regime"; BASELINE configs[1], the ResNet-110 gradient set).
//
//  K6 tlc_compress_batched_kernel: one CTA per tensor.  Pass 1 reduces
//     max|err + t| (Eq. 1) in the CTA; pass 2 re-reads t/err (L2-resident at
//     these sizes), quantizes (Eq. 2), writes err (steps a,b) and folds the
//     quartic bytes into shared memory; the CTA then zero-run
//     encodes its bytes with the warp-row scan of tlc_device.cuh
//     (no cross-CTA dependency) and writes payload and header.
//  K7 tlc_decompress_batched_kernel: one CTA per tensor.  Expands the payload
//     into shared memory (121 prefill, literal scatter at scanned positions),
//     checks the expansion is exactly P bytes before writing anything, then
//     decodes base 3 and writes M*q (or adds it where q != 0).
//
// Tensors up to kBatchMaxN elements (P <= 32 KiB of shared memory) take this
// path; the host wrapper sends larger ones through K1-K5.
#include "tlc_device.cuh"
#include "tlc_launch.h"

namespace tlc {

constexpr int kBThreads = kScanThreads;
constexpr int kBMaxP = 32768;

// Load shared-memory bytes [pos, min(pos+32, hi)) as 8 words, padding with 121.
__device__ __forceinline__ int load_smem_seg(const uint8_t *sb, uint32_t pos, uint32_t hi, uint32_t (&w)[8]) {
    const int len = pos < hi ? (int)min(32u, hi - pos) : 0;
    if (len == 32) {
        const uint4 a = *reinterpret_cast<const uint4 *>(sb + pos);
        const uint4 c = *reinterpret_cast<const uint4 *>(sb + pos + 16);
        w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w; w[4] = c.x; w[5] = c.y; w[6] = c.z; w[7] = c.w;
    } else {
#pragma unroll
        for (int k = 0; k < 8; k++) {
            uint32_t x = 0;
#pragma unroll
            for (int c = 0; c < 4; c++) {
                const int mm = 4 * k + c;
                x |= (uint32_t)(mm < len ? sb[pos + mm] : kZeroGroup) << (8 * c);
            }
            w[k] = x;
        }
    }
    return len;
}

// ============================================================== K6
__global__ void __launch_bounds__(kBThreads)
tlc_compress_batched_kernel(const tlc_tensor_desc *__restrict__ descs, float s, int use_zre) {
    extern __shared__ __align__(16) uint8_t smem_b[];   // kBMaxP quartic bytes
    __shared__ unsigned int s_red[kScanWarps];
    __shared__ unsigned long long s_wagg[kScanWarps];
    const tlc_tensor_desc d = descs[blockIdx.x];
    const float *__restrict__ t = d.t;
    float *__restrict__ err = d.err;
    const uint64_t n = d.n;
    if (n == 0 || n > kBatchMaxN) {                              // per-tensor argument error
        if (threadIdx.x == 0) { d.hdr->status = TLC_ERR_ARG; d.hdr->payload_len = 0; d.hdr->n = n; }
        return;
    }
    const uint32_t P = (uint32_t)((n + 4) / 5);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

    // ---- pass 1: max |u|, u = err + t (step 1, Eq. 1); NaN/Inf flagged by the key
    unsigned int m = 0;
#pragma unroll 4
    for (uint64_t i = threadIdx.x; i < n; i += kBThreads)
        m = max(m, __float_as_uint(__fadd_rn(__ldg(err + i), __ldg(t + i))) & 0x7fffffffu);
    m = __reduce_max_sync(0xffffffffu, m);
    if (lane == 0) s_red[warp] = m;
    __syncthreads();
    unsigned int key = 0;
#pragma unroll
    for (int w = 0; w < kScanWarps; w++) key = max(key, s_red[w]);
    unsigned int status = TLC_OK;
    float M = 0.0f;
    if (key >= 0x7f800000u) {
        status = TLC_ERR_NONFINITE;                              // R6
    } else {
        M = __fmul_rn(__uint_as_float(key), s);                  // Eq. 1
        if (isinf(M)) { status = TLC_ERR_RANGE; M = 0.0f; }
    }
    if (status != TLC_OK) {                                      // err untouched
        if (threadIdx.x == 0) {
            d.hdr->M = 0.0f; d.hdr->flags = use_zre ? TLC_FLAG_ZRE : 0u; d.hdr->n = n;
            d.hdr->payload_len = 0; d.hdr->status = status; d.hdr->reserved = 0;
        }
        return;
    }
    const Quant Q(M);

    // ---- pass 2: quantize, residual, quartic bytes into shared memory
    uint8_t *B = use_zre ? smem_b : d.payload;
    for (uint32_t j = threadIdx.x; j < P; j += kBThreads) {
        uint32_t b = 0;
#pragma unroll
        for (int i = 0; i < 5; i++) {
            const uint64_t e = (uint64_t)i * P + j;
            const bool ok = e < n;
            const float u = ok ? __fadd_rn(err[e], t[e]) : 0.0f;
            const int q = Q.q(u);
            if (ok) err[e] = Q.residual(u, q);
            b = b * 3u + (ok ? (uint32_t)(q + 1) : 0u);
        }
        B[j] = (uint8_t)b;
    }
    if (!use_zre) {
        if (threadIdx.x == 0) {
            d.hdr->M = M; d.hdr->flags = 0u; d.hdr->n = n;
            d.hdr->payload_len = P; d.hdr->status = TLC_OK; d.hdr->reserved = 0;
        }
        return;
    }
    __syncthreads();

    // ---- zero-run encoding of the tensor's bytes: one sub-range per warp
    const uint32_t sub = ((P + kScanWarps - 1) / kScanWarps + 31u) / 32u * 32u;
    const uint32_t wlo = min(P, (uint32_t)warp * sub), whi = min(P, wlo + sub);
    uint32_t w[8];
    RunSum wagg = run_identity();
    for (uint32_t row = wlo; row < whi; row += 1024u) {
        const int len = load_smem_seg(smem_b, row + 32u * lane, whi, w);
        const uint32_t mask = literal_mask(w);
        wagg = compose(wagg, warp_row_summary(mask, len, mask_summary(mask, len), min(1024u, whi - row)));
    }
    if (lane == 0) s_wagg[warp] = pack(wagg);
    __syncthreads();
    RunSum before = run_identity(), all = run_identity();
#pragma unroll
    for (int k = 0; k < kScanWarps; k++) {
        const RunSum x = unpack(s_wagg[k]);
        if (k < warp) before = compose(before, x);
        all = compose(all, x);
    }
    uint64_t off;
    uint32_t carry;
    run_eval(before, 0, off, carry);
    for (uint32_t row = wlo; row < whi; row += 1024u) {
        const uint32_t pos = row + 32u * lane;
        const int len = load_smem_seg(smem_b, pos, whi, w);
        const uint32_t mask = literal_mask(w);
        const WarpRow r = warp_row(mask, len, mask_summary(mask, len), carry, min(1024u, whi - row));
        uint32_t ex = r.count;
#pragma unroll
        for (int dd = 1; dd < 32; dd <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, ex, dd);
            if (lane >= dd) ex += y;
        }
        ex -= r.count;
        if (len > 0) {
            uint64_t o = off + ex;
            uint32_t c = r.carry_in;
            mask_emit(w, mask, len, c, d.payload, o);
            if (c > 0 && pos + (uint32_t)len == P) d.payload[o] = run_code(c);
        }
        off += r.row_count;
        carry = r.carry_out;
    }
    if (threadIdx.x == 0) {
        uint64_t total;
        uint32_t c;
        run_eval(all, 0, total, c);
        d.hdr->M = M; d.hdr->flags = TLC_FLAG_ZRE; d.hdr->n = n;
        d.hdr->payload_len = total + (c > 0); d.hdr->status = TLC_OK; d.hdr->reserved = 0;
    }
}

// ============================================================== K7
template <int kMode>
__global__ void __launch_bounds__(kBThreads)
tlc_decompress_batched_kernel(const tlc_tensor_desc *__restrict__ descs) {
    extern __shared__ __align__(16) uint8_t smem_e[];   // kBMaxP expanded quartic bytes
    __shared__ uint32_t s_V[5][256];
    __shared__ unsigned long long s_warp[kScanWarps];
    const tlc_tensor_desc d = descs[blockIdx.x];
    tlc_header *hdr = d.hdr;
    const uint64_t n = d.n;
    if (n == 0 || n > kBatchMaxN || !header_valid(hdr, n)) {
        if (threadIdx.x == 0 && hdr->status == TLC_OK) raise_format(hdr);
        return;
    }
    const uint32_t P = (uint32_t)((n + 4) / 5);
    const uint32_t Z = (uint32_t)hdr->payload_len;
    const bool zre = (hdr->flags & TLC_FLAG_ZRE) != 0;
    const float M = hdr->M;
    const uint8_t *__restrict__ pay = d.payload;

    // Eq. 3 per partition and byte value: V[i][b] = M * (digit_i(b) - 1)
    for (int v = threadIdx.x; v < 256; v += kBThreads) {
        uint32_t r = v < 243 ? v : 121;
#pragma unroll
        for (int i = 4; i >= 0; i--) {
            s_V[i][v] = __float_as_uint(__fmul_rn(M, (float)((int)(r % 3u) - 1)));
            r /= 3u;
        }
    }
    bool bad = false;
    if (zre) {
        for (uint32_t j = 4 * threadIdx.x; j < P; j += 4 * kBThreads)
            *reinterpret_cast<uint32_t *>(smem_e + j) = 0x79797979u;   // 121 prefill
        __syncthreads();
        // scan the payload in rows of kBThreads x 16 bytes; literal bytes land at their positions
        uint64_t base = 0;
        for (uint32_t row = 0; row < Z; row += kBThreads * 16u) {
            const uint32_t z0 = row + 16u * threadIdx.x;
            uint8_t b[16];
            uint32_t len[16], sum = 0;
#pragma unroll
            for (int k = 0; k < 16; k++) {
                b[k] = z0 + k < Z ? pay[z0 + k] : 0;
                len[k] = z0 + k < Z ? zre_len(b[k]) : 0u;
                sum += len[k];
            }
            uint64_t tot;
            uint64_t p = base + block_excl_scan_sum(sum, s_warp, tot);
#pragma unroll
            for (int k = 0; k < 16; k++) {
                if (len[k] == 1 && p < P) smem_e[p] = b[k];
                p += len[k];
            }
            base += tot;
        }
        bad = base != P;                                       // S:235 (uniform)
    } else {
        for (uint32_t j = threadIdx.x; j < P; j += kBThreads) {
            uint8_t v = pay[j];
            if (v > 242) { bad = true; v = kZeroGroup; }
            smem_e[j] = v;
        }
    }
    if (__syncthreads_or(bad)) {                               // nothing written to out
        if (threadIdx.x == 0) raise_format(hdr);
        return;
    }
    float *__restrict__ out = d.out;
    for (uint32_t j = threadIdx.x; j < P; j += kBThreads) {
        const uint32_t bv = smem_e[j];
#pragma unroll
        for (int i = 0; i < 5; i++) {
            const uint64_t e = (uint64_t)i * P + j;
            if (e >= n) continue;
            const uint32_t v = s_V[i][bv];
            if (kMode == TLC_MODE_OVERWRITE) {
                out[e] = __uint_as_float(v);
            } else {
                // digit != 1  <=>  q != 0 (R16)
                uint32_t r = bv;
                for (int k = 4; k > i; k--) r /= 3u;
                if (r % 3u != 1u) out[e] = __fadd_rn(out[e], __uint_as_float(v));
            }
        }
    }
}

// ============================================================== host launchers
int launch_compress_batched(int count, const tlc_tensor_desc *d_descs, float s, int use_zre, cudaStream_t st) {
    if (count <= 0) return TLC_OK;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(tlc_compress_batched_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kBMaxP);
        attr = true;
    }
    KernelScope ks(kK6, st);
    tlc_compress_batched_kernel<<<count, kBThreads, use_zre ? kBMaxP : 0, st>>>(d_descs, s, use_zre);
    return cudaPeekAtLastError() == cudaSuccess ? TLC_OK : TLC_ERR_CUDA;
}

int launch_decompress_batched(int count, const tlc_tensor_desc *d_descs, int mode, cudaStream_t st) {
    if (count <= 0) return TLC_OK;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(tlc_decompress_batched_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBMaxP);
        cudaFuncSetAttribute(tlc_decompress_batched_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBMaxP);
        attr = true;
    }
    KernelScope ks(kK7, st);
    if (mode == TLC_MODE_OVERWRITE) tlc_decompress_batched_kernel<0><<<count, kBThreads, kBMaxP, st>>>(d_descs);
    else tlc_decompress_batched_kernel<1><<<count, kBThreads, kBMaxP, st>>>(d_descs);
    return cudaPeekAtLastError() == cudaSuccess ? TLC_OK : TLC_ERR_CUDA;
}

}  // namespace tlc
