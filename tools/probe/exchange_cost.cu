// Cost of one cross-CTA all-reduce step of the QR panel kernel (32 doubles
// per CTA, every CTA needs every CTA's 32 partials), G CTAs x 512 threads:
//   A: cooperative-groups grid.sync between the partial stores and the loads
//   B: per-lane release/acquire flags (no grid barrier): lane l of warp 0
//      stores its partial then st.release a step-tagged flag; gathering lanes
//      spin with ld.acquire on the flags of the CTAs they read.
//   C: 16-CTA cluster, distributed shared memory + cluster.sync (reference)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe/exchange_cost tools/probe/exchange_cost.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

constexpr int kWarps = 16, kLW = 16;

__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__global__ void __launch_bounds__(kWarps * 32, 1) grid_kernel(int steps, double* part, double* out) {
    __shared__ double xs[kLW * 32];
    cg::grid_group gg = cg::this_grid();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, G = gridDim.x, rank = blockIdx.x;
    double acc = 0.0;
    for (int s = 0; s < steps; ++s) {
        const int buf = s & 1;
        double* pb = part + static_cast<long>(buf) * G * 32;
        if (warp == 0) pb[rank * 32 + lane] = acc + rank + lane;
        gg.sync();
        if (warp < kLW) {
            double t = 0.0;
            for (int c = warp; c < G; c += kLW) t += __ldcg(pb + c * 32 + lane);
            xs[warp * 32 + lane] = t;
        }
        __syncthreads();
        if (warp == 0) {
            double t = 0.0;
            for (int w = 0; w < kLW; ++w) t += xs[w * 32 + lane];
            acc = t * 1e-9;
        }
        __syncthreads();
    }
    if (warp == 0) out[rank * 32 + lane] = acc;
}

__global__ void __launch_bounds__(kWarps * 32, 1) flag_kernel(int steps, double* part, unsigned* flags, double* out) {
    __shared__ double xs[kLW * 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, G = gridDim.x, rank = blockIdx.x;
    double acc = 0.0;
    for (int s = 0; s < steps; ++s) {
        const int buf = s & 1;
        double* pb = part + static_cast<long>(buf) * G * 32;
        const unsigned tag = static_cast<unsigned>(s + 1);
        if (warp == 0) {
            pb[rank * 32 + lane] = acc + rank + lane;
            st_release(flags + rank * 32 + lane, tag);
        }
        if (warp < kLW) {
            double t = 0.0;
            for (int c = warp; c < G; c += kLW) {
                while (ld_acquire(flags + c * 32 + lane) < tag) {
                }
                t += __ldcg(pb + c * 32 + lane);
            }
            xs[warp * 32 + lane] = t;
        }
        __syncthreads();
        if (warp == 0) {
            double t = 0.0;
            for (int w = 0; w < kLW; ++w) t += xs[w * 32 + lane];
            acc = t * 1e-9;
        }
        __syncthreads();
    }
    if (warp == 0) out[rank * 32 + lane] = acc;
}

__global__ void __launch_bounds__(kWarps * 32, 1) cluster_kernel(int steps, double* out) {
    __shared__ double part_s[2 * 32];
    __shared__ double xs[8 * 32];
    cg::cluster_group cl = cg::this_cluster();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int G = static_cast<int>(cl.num_blocks()), rank = static_cast<int>(cl.block_rank());
    double acc = 0.0;
    for (int s = 0; s < steps; ++s) {
        const int buf = s & 1;
        if (warp == 0) part_s[buf * 32 + lane] = acc + rank + lane;
        cl.sync();
        if (warp < 8) {
            double t = 0.0;
            for (int c = warp; c < G; c += 8) t += cl.map_shared_rank(part_s, c)[buf * 32 + lane];
            xs[warp * 32 + lane] = t;
        }
        __syncthreads();
        if (warp == 0) {
            double t = 0.0;
            for (int w = 0; w < 8; ++w) t += xs[w * 32 + lane];
            acc = t * 1e-9;
        }
        __syncthreads();
    }
    cl.sync();
    if (warp == 0) out[blockIdx.x * 32 + lane] = acc;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *part, *out;
    unsigned* flags;
    cudaMalloc(&part, 2 * 160 * 32 * 8);
    cudaMalloc(&out, 160 * 32 * 8);
    cudaMalloc(&flags, 160 * 32 * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int steps = 2000;
    for (int G : {16, 64, 128, sms}) {
        float ms;
        void* args[] = {(void*)&steps, (void*)&part, (void*)&out};
        cudaLaunchCooperativeKernel((void*)grid_kernel, G, kWarps * 32, args, 0, 0);
        cudaEventRecord(e0);
        cudaLaunchCooperativeKernel((void*)grid_kernel, G, kWarps * 32, args, 0, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        std::printf("G=%3d grid.sync      : %.3f us/step  (%s)\n", G, ms * 1e3 / steps,
                    cudaGetErrorString(cudaGetLastError()));
        // flags: co-resident via cooperative launch as well
        cudaMemset(flags, 0, 160 * 32 * 4);
        void* fargs[] = {(void*)&steps, (void*)&part, (void*)&flags, (void*)&out};
        cudaLaunchCooperativeKernel((void*)flag_kernel, G, kWarps * 32, fargs, 0, 0);
        cudaMemset(flags, 0, 160 * 32 * 4);
        cudaEventRecord(e0);
        cudaLaunchCooperativeKernel((void*)flag_kernel, G, kWarps * 32, fargs, 0, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        std::printf("G=%3d release/acquire: %.3f us/step  (%s)\n", G, ms * 1e3 / steps,
                    cudaGetErrorString(cudaGetLastError()));
    }
    {
        cudaFuncSetAttribute(cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(16);
        cfg.blockDim = dim3(kWarps * 32);
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 16;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        float ms;
        cudaLaunchKernelEx(&cfg, cluster_kernel, steps, out);
        cudaEventRecord(e0);
        cudaLaunchKernelEx(&cfg, cluster_kernel, steps, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        std::printf("G= 16 cluster DSMEM  : %.3f us/step  (%s)\n", ms * 1e3 / steps,
                    cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
