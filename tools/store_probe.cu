// Development probe: HBM write bandwidth of 128-bit vs 256-bit streaming stores, flat and
// in K5's pattern (five partitions of P floats written side by side by each CTA tile).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o store_probe tools/store_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int V, bool kCs>
__global__ void __launch_bounds__(256) flat(float *o, size_t n, float a) {
    const size_t nv = n / (4 * V);
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nv; i += (size_t)gridDim.x * blockDim.x) {
        float *p = o + i * 4 * V;
        if (V == 2) {
            if (kCs) asm volatile("st.global.cs.v8.f32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p), "f"(a) : "memory");
            else asm volatile("st.global.v8.f32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p), "f"(a) : "memory");
        } else {
            if (kCs) __stcs(reinterpret_cast<float4 *>(p), make_float4(a, a, a, a));
            else *reinterpret_cast<float4 *>(p) = make_float4(a, a, a, a);
        }
    }
}
// K5 pattern: tile of T positions; partition i at o + i*P; thread t writes 4V floats per step
template <int V>
__global__ void __launch_bounds__(256) parts(float *o, size_t P, int T, float a) {
    const size_t ntiles = P / T;
    for (size_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
        for (int i = 0; i < 5; i++)
            for (int jl = 4 * V * threadIdx.x; jl < T; jl += 4 * V * blockDim.x) {
                float *p = o + i * P + tile * T + jl;
                if (V == 2) asm volatile("st.global.cs.v8.f32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p), "f"(a) : "memory");
                else __stcs(reinterpret_cast<float4 *>(p), make_float4(a, a, a, a));
            }
}
template <typename F>
float timeit(F f) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int w = 0; w < 3; w++) f();
    cudaEventRecord(a);
    for (int r = 0; r < 20; r++) f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    return ms / 20;
}
int main() {
    const size_t n = 1ull << 28, P = n / 5 / 4096 * 4096;
    float *o; cudaMalloc(&o, n * 4 + 64);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int cpsm : {2, 4, 8}) {
        const int g = sms * cpsm;
        printf("CTAs/SM %d: flat v4 %.0f  v4.cs %.0f  v8 %.0f  v8.cs %.0f GB/s\n", cpsm,
               n * 4 / 1e6 / timeit([&] { flat<1, false><<<g, 256>>>(o, n, 1.f); }),
               n * 4 / 1e6 / timeit([&] { flat<1, true><<<g, 256>>>(o, n, 1.f); }),
               n * 4 / 1e6 / timeit([&] { flat<2, false><<<g, 256>>>(o, n, 1.f); }),
               n * 4 / 1e6 / timeit([&] { flat<2, true><<<g, 256>>>(o, n, 1.f); }));
        for (int T : {2048, 4096, 8192})
            printf("   parts T=%d: v4.cs %.0f  v8.cs %.0f GB/s\n", T,
                   5 * P * 4 / 1e6 / timeit([&] { parts<1><<<g, 256>>>(o, P, T, 1.f); }),
                   5 * P * 4 / 1e6 / timeit([&] { parts<2><<<g, 256>>>(o, P, T, 1.f); }));
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
