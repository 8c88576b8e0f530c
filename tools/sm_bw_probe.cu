// Probe: what one SM (one 512-thread CTA) can load from and store to HBM, as a function
// of the bytes it moves; grids of 1..148 such CTAs on distinct SMs.  Per-launch device time
// in CUDA graphs of 20 dependent launches, minus an empty launch of the same grid.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sm_bw_probe tools/sm_bw_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

// mode 0: float4 loads (8 in flight per thread); 1: float4 stores (.cs); 2: scalar stores
// (.cs); 3: float4 stores (default policy); 4: load+store float4 (copy)
__global__ void __launch_bounds__(512, 1) k(float *buf, size_t per_cta, int mode, float *sink) {
    float4 *b4 = reinterpret_cast<float4 *>(buf + (size_t)blockIdx.x * per_cta / 4);
    float *b = buf + (size_t)blockIdx.x * per_cta / 4;
    const size_t n4 = per_cta / 16;
    float acc = 0.f;
    if (mode == 0) {
        for (size_t g0 = threadIdx.x; g0 < n4; g0 += 8 * 512) {
            float4 v[8];
#pragma unroll
            for (int u = 0; u < 8; u++) v[u] = g0 + u * 512 < n4 ? __ldcs(b4 + g0 + u * 512) : make_float4(0, 0, 0, 0);
#pragma unroll
            for (int u = 0; u < 8; u++) acc += v[u].x + v[u].y + v[u].z + v[u].w;
        }
    } else if (mode == 1) {
        for (size_t g = threadIdx.x; g < n4; g += 512) __stcs(b4 + g, make_float4(1, 2, 3, 4));
    } else if (mode == 2) {
        for (size_t g = threadIdx.x; g < 4 * n4; g += 512) __stcs(b + g, 1.f);
    } else if (mode == 3) {
        for (size_t g = threadIdx.x; g < n4; g += 512) b4[g] = make_float4(1, 2, 3, 4);
    } else if (mode == 4) {
        float4 *o4 = reinterpret_cast<float4 *>(sink) + (size_t)blockIdx.x * n4;
        for (size_t g0 = threadIdx.x; g0 < n4; g0 += 8 * 512) {
            float4 v[8];
#pragma unroll
            for (int u = 0; u < 8; u++) v[u] = g0 + u * 512 < n4 ? __ldcs(b4 + g0 + u * 512) : make_float4(0, 0, 0, 0);
#pragma unroll
            for (int u = 0; u < 8; u++) if (g0 + u * 512 < n4) __stcs(o4 + g0 + u * 512, v[u]);
        }
    }
    if (acc == 12345.f && mode == 0) sink[0] = acc;
}

static float timed(int grid, size_t per_cta, int mode, float *buf, float *sink, cudaStream_t s) {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; i < 20; i++) k<<<grid, 512, 0, s>>>(buf, per_cta, mode, sink);
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    for (int i = 0; i < 3; i++) cudaGraphLaunch(ge, s);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
    for (int i = 0; i < 10; i++) cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    return ms * 1e3f / 200;
}

int main() {
    float *buf, *sink;
    cudaMalloc(&buf, 1ull << 30);
    cudaMalloc(&sink, 1ull << 30);
    cudaStream_t s;
    cudaStreamCreate(&s);
    const char *names[] = {"load v4", "store v4 cs", "store f32 cs", "store v4", "copy v4"};
    for (int grid : {1, 16, 148}) {
        const float e = timed(grid, 0, 0, buf, sink, s);
        printf("grid %d: empty launch %.2f us\n", grid, e);
        for (size_t kb : {16, 64, 256, 1024})
            for (int mode = 0; mode < 5; mode++) {
                const float t = timed(grid, kb << 10, mode, buf, sink, s) - e;
                printf("grid %3d %5zu KB/CTA %-13s %7.2f us  %7.1f GB/s per SM\n", grid, kb, names[mode], t,
                       (kb << 10) / (t * 1e3));
            }
    }
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) printf("error %s\n", cudaGetErrorString(err));
    return 0;
}
