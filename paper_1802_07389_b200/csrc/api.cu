// api.cu -- the extern "C" boundary declared in include/tlc.h.
//
// Argument marshalling and synchronous validation only; every step of the
// method runs in the kernels of compress.cu / decompress.cu.
#include <cmath>

#include "tlc_launch.h"

using namespace tlc;

extern "C" {

int tlc_version(void) { return 100; }

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
    if ((const void *)t == (const void *)err) return TLC_ERR_ARG;
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
