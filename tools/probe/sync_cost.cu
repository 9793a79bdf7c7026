// Measures the cost of grid-wide (cooperative) and cluster barriers on B200.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void grid_sync_kernel(int iters, int* out) {
    cg::grid_group g = cg::this_grid();
    for (int i = 0; i < iters; ++i) g.sync();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = iters;
}

__global__ void __cluster_dims__(16, 1, 1) cluster_sync_kernel(int iters, int* out) {
    cg::cluster_group cl = cg::this_cluster();
    for (int i = 0; i < iters; ++i) cl.sync();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = iters;
}

__global__ void __cluster_dims__(8, 1, 1) cluster8_sync_kernel(int iters, int* out) {
    cg::cluster_group cl = cg::this_cluster();
    for (int i = 0; i < iters; ++i) cl.sync();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = iters;
}

int main() {
    int* out;
    cudaMalloc(&out, 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int blocks : {16, 64, 148, 296}) {
        const int iters = 2000;
        void* args[] = {(void*)&iters, (void*)&out};
        cudaLaunchCooperativeKernel((void*)grid_sync_kernel, blocks, 256, args, 0, 0);
        cudaDeviceSynchronize();
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void*)grid_sync_kernel, blocks, 256, args, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("grid.sync blocks=%d: %.3f us per sync (%s)\n", blocks, ms * 1e3 / iters,
               cudaGetErrorString(cudaGetLastError()));
    }
    cudaFuncSetAttribute(cluster_sync_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int blocks : {16, 144}) {
        const int iters = 20000;
        cluster_sync_kernel<<<blocks, 256>>>(iters, out);
        cudaDeviceSynchronize();
        cudaEventRecord(a);
        cluster_sync_kernel<<<blocks, 256>>>(iters, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("cluster16.sync blocks=%d: %.3f us per sync (%s)\n", blocks, ms * 1e3 / iters,
               cudaGetErrorString(cudaGetLastError()));
        cluster8_sync_kernel<<<blocks, 256>>>(iters, out);
        cudaDeviceSynchronize();
        cudaEventRecord(a);
        cluster8_sync_kernel<<<blocks, 256>>>(iters, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("cluster8.sync blocks=%d: %.3f us per sync (%s)\n", blocks, ms * 1e3 / iters,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
