// Probe: fixed cost of a cluster launch and of barrier.cluster on B200, in CUDA graphs of
// 20 back-to-back dependent launches (us per launch).  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_plain(int *p, int nb) {
    for (int i = 0; i < nb; i++) __syncthreads();
    if (threadIdx.x == 0 && p) p[blockIdx.x] += 1;
}
__global__ void k_cluster(int *p, int nb) {
    for (int i = 0; i < nb; i++)
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (threadIdx.x == 0 && p) p[blockIdx.x] += 1;
}

static float run(bool cluster, int grid, int threads, int nb, size_t smem, int *p) {
    cudaStream_t s;
    cudaStreamCreate(&s);
    auto launch = [&]() {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(threads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute a[1];
        a[0].id = cudaLaunchAttributeClusterDimension;
        a[0].val.clusterDim.x = 2; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
        cfg.attrs = a;
        cfg.numAttrs = cluster ? 1 : 0;
        cudaLaunchKernelEx(&cfg, cluster ? k_cluster : k_plain, p, nb);
    };
    for (int i = 0; i < 3; i++) launch();
    cudaStreamSynchronize(s);
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; i < 20; i++) launch();
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
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
    return ms * 1e3f / 200;
}

int main() {
    int *p;
    cudaMalloc(&p, 1 << 20);
    cudaFuncSetAttribute(k_plain, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
    cudaFuncSetAttribute(k_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
    for (int grid : {2, 220, 296})
        for (size_t smem : {(size_t)0, (size_t)90000})
            for (int nb : {0, 2, 20})
                printf("grid %d smem %zu syncs %d: plain %.2f us  cluster2 %.2f us\n", grid, smem, nb,
                       run(false, grid, 512, nb, smem, p), run(true, grid, 512, nb, smem, p));
    return 0;
}
