// api.cu -- the extern "C" boundary declared in include/tlc.h.
//
// Argument marshalling and synchronous validation only; every step of the
// method runs in the kernels of compress.cu / decompress.cu.
#include <cmath>
#include <cstring>

#include "tlc_launch.h"

using namespace tlc;

extern "C" {

int tlc_version(void) { return 200; }

#ifndef TLC_BUILD_ID
#define TLC_BUILD_ID "unknown"
#endif
// the marker lets build.py read the id from the file without loading the library
static const char kBuildIdTagged[] = "TLC_BUILD_ID:" TLC_BUILD_ID;
const char *tlc_build_id(void) { return kBuildIdTagged + 13; }

// [a, a+na) and [b, b+nb) share a byte
static bool overlap(const void *a, uint64_t na, const void *b, uint64_t nb) {
    const uintptr_t x = reinterpret_cast<uintptr_t>(a), y = reinterpret_cast<uintptr_t>(b);
    return x < y + nb && y < x + na;
}

const char *tlc_status_string(int status) {
    switch (status) {
        case TLC_OK: return "TLC_OK";
        case TLC_ERR_ARG: return "TLC_ERR_ARG";
        case TLC_ERR_NONFINITE: return "TLC_ERR_NONFINITE";
        case TLC_ERR_RANGE: return "TLC_ERR_RANGE";
        case TLC_ERR_FORMAT: return "TLC_ERR_FORMAT";
        case TLC_ERR_CAPACITY: return "TLC_ERR_CAPACITY";
        case TLC_ERR_CUDA: return "TLC_ERR_CUDA";
        case TLC_ERR_NCCL: return "TLC_ERR_NCCL";
        default: return "TLC_ERR_UNKNOWN";
    }
}

uint64_t tlc_quartic_bytes(uint64_t n) { return n / 5 + (n % 5 != 0); }

uint64_t tlc_max_payload_bytes(uint64_t n) { return tlc_quartic_bytes(n); }

size_t tlc_compress_workspace_bytes(uint64_t n) { return compress_workspace_bytes(n); }

size_t tlc_decompress_workspace_bytes(uint64_t n) { return decompress_workspace_bytes(n); }

int tlc_compress(const float *t, float *err, uint64_t n, float s, int use_zre, uint8_t *payload,
                 uint64_t payload_cap, tlc_header *hdr, void *ws, size_t ws_bytes, void *stream) {
    if (!t || !err || !payload || !hdr || !ws || n == 0) return TLC_ERR_ARG;
    if (!(s >= 1.0f && s < 2.0f)) return TLC_ERR_ARG;
    if (n >= (1ull << 42)) return TLC_ERR_ARG;                         // 44-bit run counters
    // t, err, payload and hdr must not share bytes (err is rewritten while t is read; the
    // payload and header are written by other CTAs than the ones reading t and err)
    if (overlap(t, 4 * n, err, 4 * n) || overlap(payload, payload_cap, t, 4 * n) ||
        overlap(payload, payload_cap, err, 4 * n) || overlap(hdr, sizeof(tlc_header), t, 4 * n) ||
        overlap(hdr, sizeof(tlc_header), err, 4 * n) || overlap(hdr, sizeof(tlc_header), payload, payload_cap))
        return TLC_ERR_ARG;
    if (payload_cap < tlc_max_payload_bytes(n)) return TLC_ERR_CAPACITY;
    if (ws_bytes < compress_workspace_bytes(n)) return TLC_ERR_CAPACITY;
    if ((reinterpret_cast<uintptr_t>(ws) & 255u) != 0) return TLC_ERR_ARG;
    if ((reinterpret_cast<uintptr_t>(hdr) & 7u) != 0) return TLC_ERR_ARG;
    return launch_compress(t, err, n, s, use_zre ? 1 : 0, payload, hdr, ws,
                           reinterpret_cast<cudaStream_t>(stream));
}

int tlc_decompress(const uint8_t *payload, tlc_header *hdr, uint64_t n, float *out, int mode,
                   void *ws, size_t ws_bytes, void *stream) {
    if (!payload || !hdr || !out || !ws || n == 0) return TLC_ERR_ARG;
    if (mode != TLC_MODE_OVERWRITE && mode != TLC_MODE_ACCUMULATE) return TLC_ERR_ARG;
    if (n >= (1ull << 42)) return TLC_ERR_ARG;
    if (ws_bytes < decompress_workspace_bytes(n)) return TLC_ERR_CAPACITY;
    if ((reinterpret_cast<uintptr_t>(ws) & 255u) != 0) return TLC_ERR_ARG;
    if ((reinterpret_cast<uintptr_t>(hdr) & 7u) != 0) return TLC_ERR_ARG;
    return launch_decompress(payload, hdr, n, out, mode, ws, reinterpret_cast<cudaStream_t>(stream));
}

int tlc_stoch_compress(const float *t, uint64_t n, uint64_t seed, uint64_t step, int use_zre, uint8_t *payload,
                       uint64_t payload_cap, tlc_header *hdr, void *ws, size_t ws_bytes, void *stream) {
    if (!t || !payload || !hdr || !ws || n == 0) return TLC_ERR_ARG;
    if (n >= (1ull << 42)) return TLC_ERR_ARG;
    if (overlap(payload, payload_cap, t, 4 * n) || overlap(hdr, sizeof(tlc_header), t, 4 * n) ||
        overlap(hdr, sizeof(tlc_header), payload, payload_cap))
        return TLC_ERR_ARG;
    if (payload_cap < tlc_max_payload_bytes(n)) return TLC_ERR_CAPACITY;
    if (ws_bytes < compress_workspace_bytes(n)) return TLC_ERR_CAPACITY;
    if ((reinterpret_cast<uintptr_t>(ws) & 255u) != 0) return TLC_ERR_ARG;
    if ((reinterpret_cast<uintptr_t>(hdr) & 7u) != 0) return TLC_ERR_ARG;
    uint64_t scratch = 0;
    const SegTable T = single_table(t, nullptr, nullptr, payload, hdr, n, scratch);
    return launch_stoch_compress_table(T, seed, step, use_zre ? 1 : 0, ws, reinterpret_cast<cudaStream_t>(stream));
}

size_t tlc_int8_workspace_bytes(uint64_t n) {
    uint64_t scratch = 0;
    const SegTable T = single_table(nullptr, nullptr, nullptr, nullptr, nullptr, n ? n : 1, scratch);
    return ws_layout(T, 0).memset_c;
}

int tlc_int8_compress(const float *t, uint64_t n, int8_t *codes, tlc_header *hdr, void *ws, size_t ws_bytes,
                      void *stream) {
    if (!t || !codes || !hdr || !ws || n == 0) return TLC_ERR_ARG;
    if (n >= (1ull << 42)) return TLC_ERR_ARG;
    if (overlap(codes, n, t, 4 * n) || overlap(hdr, sizeof(tlc_header), t, 4 * n) ||
        overlap(hdr, sizeof(tlc_header), codes, n))
        return TLC_ERR_ARG;
    if (ws_bytes < tlc_int8_workspace_bytes(n)) return TLC_ERR_CAPACITY;
    if ((reinterpret_cast<uintptr_t>(ws) & 255u) != 0) return TLC_ERR_ARG;
    if ((reinterpret_cast<uintptr_t>(hdr) & 7u) != 0) return TLC_ERR_ARG;
    return launch_int8_compress(t, n, codes, hdr, ws, reinterpret_cast<cudaStream_t>(stream));
}

int tlc_int8_decompress(const int8_t *codes, tlc_header *hdr, uint64_t n, float *out, int mode, void *stream) {
    if (!codes || !hdr || !out || n == 0) return TLC_ERR_ARG;
    if (mode != TLC_MODE_OVERWRITE && mode != TLC_MODE_ACCUMULATE) return TLC_ERR_ARG;
    if ((reinterpret_cast<uintptr_t>(hdr) & 7u) != 0) return TLC_ERR_ARG;
    return launch_int8_decompress(codes, hdr, n, out, mode, reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"

// ---------------------------------------------------------------------------- 3LC1 blobs
// Host-side container of one compressed tensor, SPEC S:272-279 (the "blob" module):
// "3LC1", version 1, codec id, flags, rank, rank x u64 dims, f32 m, u64 payload_len,
// payload -- all little-endian.  Artifact plumbing for file-based parity dumps; the
// kernels never touch it.
namespace {
constexpr uint8_t kBlobMagic[4] = {'3', 'L', 'C', '1'};
constexpr uint64_t kBlobFixed = 4 + 1 + 1 + 1 + 1 + 4 + 8;     // without dims and payload
template <class V> void put_le(uint8_t *p, V v) {
    for (size_t i = 0; i < sizeof(V); i++) p[i] = (uint8_t)((uint64_t)v >> (8 * i));
}
uint64_t get_u64(const uint8_t *p) {
    uint64_t v = 0;
    for (int i = 7; i >= 0; i--) v = (v << 8) | p[i];
    return v;
}
}  // namespace

extern "C" {

uint64_t tlc_blob_size(int rank, uint64_t payload_len) {
    return (rank < 0 || rank > 255) ? 0 : kBlobFixed + 8ull * (uint64_t)rank + payload_len;
}

int tlc_blob_write(const tlc_header *hdr, int rank, const uint64_t *dims, const uint8_t *payload, uint8_t *out,
                   uint64_t out_cap, uint64_t *written) {
    if (!hdr || rank < 0 || rank > 255 || (rank && !dims) || !out || (hdr->payload_len && !payload))
        return TLC_ERR_ARG;
    if (hdr->status != TLC_OK) return TLC_ERR_ARG;                 // only a successful compression
    uint64_t prod = 1;
    for (int i = 0; i < rank; i++) prod *= dims[i];
    if (prod != hdr->n) return TLC_ERR_ARG;
    const uint64_t need = tlc_blob_size(rank, hdr->payload_len);
    if (out_cap < need) return TLC_ERR_CAPACITY;
    uint8_t *p = out;
    std::memcpy(p, kBlobMagic, 4);
    p[4] = 1;                                                      // version
    p[5] = (hdr->flags & TLC_FLAG_INT8) ? 2 : 0;                   // codec: 0 = 3LC pipeline, 2 = 8-bit int
    p[6] = (uint8_t)(hdr->flags & TLC_FLAG_ZRE);
    p[7] = (uint8_t)rank;
    p += 8;
    for (int i = 0; i < rank; i++, p += 8) put_le<uint64_t>(p, dims[i]);
    uint32_t mb;
    std::memcpy(&mb, &hdr->M, 4);
    put_le<uint32_t>(p, mb);
    put_le<uint64_t>(p + 4, hdr->payload_len);
    p += 12;
    if (hdr->payload_len) std::memcpy(p, payload, hdr->payload_len);
    if (written) *written = need;
    return TLC_OK;
}

int tlc_blob_read(const uint8_t *blob, uint64_t len, tlc_header *hdr, int *rank, uint64_t *dims, int dims_cap,
                  uint64_t *payload_offset) {
    if (!blob || !hdr || !rank) return TLC_ERR_ARG;
    if (len < kBlobFixed || std::memcmp(blob, kBlobMagic, 4) != 0 || blob[4] != 1) return TLC_ERR_FORMAT;
    const uint8_t codec = blob[5], flags = blob[6], r = blob[7];
    if ((codec != 0 && codec != 2) || (flags & ~1u) || (codec == 2 && flags)) return TLC_ERR_FORMAT;
    if (len < kBlobFixed + 8ull * r) return TLC_ERR_FORMAT;
    if (r > dims_cap || (r && !dims)) return TLC_ERR_CAPACITY;
    const uint8_t *p = blob + 8;
    uint64_t n = 1;
    for (int i = 0; i < r; i++, p += 8) {
        dims[i] = get_u64(p);
        n *= dims[i];
    }
    uint32_t mb = 0;
    for (int i = 3; i >= 0; i--) mb = (mb << 8) | p[i];
    const uint64_t plen = get_u64(p + 4);
    p += 12;
    if (plen != len - (uint64_t)(p - blob)) return TLC_ERR_FORMAT;  // payload_len = byte length of payload
    if (n == 0) return TLC_ERR_FORMAT;
    if (codec == 0 && (plen > tlc_quartic_bytes(n) || (!flags && plen != tlc_quartic_bytes(n)))) return TLC_ERR_FORMAT;
    if (codec == 2 && plen != n) return TLC_ERR_FORMAT;
    std::memset(hdr, 0, sizeof(*hdr));
    std::memcpy(&hdr->M, &mb, 4);
    hdr->flags = codec == 2 ? TLC_FLAG_INT8 : flags;
    hdr->n = n;
    hdr->payload_len = plen;
    *rank = r;
    if (payload_offset) *payload_offset = (uint64_t)(p - blob);
    return TLC_OK;
}

}  // extern "C"
