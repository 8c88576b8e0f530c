// tlc_launch.h -- host-side helpers shared by the kernel launchers.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/tlc.h"

namespace tlc {

constexpr int kMaxSms = 256;          // workspace sizing bound (B200 has 148)
constexpr int kK1BlocksPerSm = 2;     // K1 grid = SMs x 2 x 512 threads (2 waves of 1 CTA/SM)

template <class T> __host__ __device__ inline T tmin(T a, T b) { return a < b ? a : b; }
template <class T> __host__ __device__ inline T tmax(T a, T b) { return a < b ? b : a; }

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
inline bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
inline bool aligned4(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 3u) == 0; }

inline int num_sms() {
    static int sms[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!sms[dev]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        sms[dev] = v > 0 ? (v > kMaxSms ? kMaxSms : v) : 1;
    }
    return sms[dev];
}

// Kernel ids for launch counting / profiling (prof.cu).
enum KernelId { kK1 = 0, kK2 = 1, kK3 = 2, kK4 = 3, kK5 = 4, kK6 = 5, kK7 = 6, kK8 = 7, kNumKernelIds = 8 };

// RAII bracket around one kernel launch: counts it and, when profiling is on,
// records CUDA events before and after it on `st`.
class KernelScope {
  public:
    KernelScope(int id, cudaStream_t st);
    ~KernelScope();
  private:
    int id_;
    cudaStream_t st_;
    void *a_;
};

int launch_compress(const float *t, float *err, uint64_t n, float s, int use_zre, uint8_t *payload,
                    tlc_header *hdr, void *ws, cudaStream_t st);
size_t compress_workspace_bytes(uint64_t n);

constexpr uint64_t kBatchMaxN = 5 * 32768;   // P <= 32 KiB of shared memory per CTA
int launch_compress_batched(int count, const tlc_tensor_desc *d_descs, float s, int use_zre, cudaStream_t st);
int launch_decompress_batched(int count, const tlc_tensor_desc *d_descs, int mode, cudaStream_t st);

int launch_decompress(const uint8_t *payload, tlc_header *hdr, uint64_t n, float *out, int mode,
                      void *ws, cudaStream_t st);
size_t decompress_workspace_bytes(uint64_t n);

}  // namespace tlc
