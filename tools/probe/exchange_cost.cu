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

__device__ __forceinline__ void ll_store(unsigned long long* dst, double v, unsigned tag) {
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
    const unsigned long long hi = static_cast<unsigned long long>(tag) << 32;
    asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};\n" ::"l"(dst), "l"(hi | (b & 0xffffffffull)),
                 "l"(hi | (b >> 32)) : "memory");
}
__device__ __forceinline__ bool ll_load(const unsigned long long* src, unsigned tag, double& v) {
    unsigned long long w0, w1;
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];\n" : "=l"(w0), "=l"(w1) : "l"(src) : "memory");
    if (static_cast<unsigned>(w0 >> 32) != tag || static_cast<unsigned>(w1 >> 32) != tag) return false;
    v = __longlong_as_double(static_cast<long long>((w1 << 32) | (w0 & 0xffffffffull)));
    return true;
}

// LL: every lane polls its column's tagged words of <= 10 CTAs (all in flight); SLEEP ns backoff
template <int SLEEP>
__global__ void __launch_bounds__(kWarps * 32, 1) ll_kernel(int steps, unsigned long long* slots, unsigned base, double* out) {
    __shared__ double xs[kLW * 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, G = gridDim.x, rank = blockIdx.x;
    double acc = 0.0;
    for (int s = 0; s < steps; ++s) {
        const int buf = s & 1;
        const unsigned tag = base + s;
        unsigned long long* sb = slots + buf * 160 * 32 * 2;
        if (warp == 0) ll_store(sb + (rank * 32 + lane) * 2, acc + rank + lane, tag);
        if (warp < kLW) {
            constexpr int kL = 10;
            double v[kL];
            unsigned pend = 0;
#pragma unroll
            for (int u = 0; u < kL; ++u) { v[u] = 0.0; if (warp + kLW * u < G) pend |= 1u << u; }
            while (pend) {
#pragma unroll
                for (int u = 0; u < kL; ++u) {
                    double t;
                    if ((pend >> u) & 1u)
                        if (ll_load(sb + ((warp + kLW * u) * 32 + lane) * 2, tag, t)) { v[u] = t; pend &= ~(1u << u); }
                }
                if (SLEEP && pend) __nanosleep(SLEEP);
            }
            double t = 0.0;
#pragma unroll
            for (int u = 0; u < kL; ++u) t += v[u];
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

// one flag per source CTA: warp 0 stores 32 partials, syncwarp, lane 0 st.release flag;
// readers: lanes of warps 0..4 poll one source flag each (ld.acquire), barrier, then plain loads
__global__ void __launch_bounds__(kWarps * 32, 1) ctaflag_kernel(int steps, double* part, unsigned* flags, unsigned base,
                                                                  double* out) {
    __shared__ double xs[kLW * 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, G = gridDim.x, rank = blockIdx.x;
    double acc = 0.0;
    for (int s = 0; s < steps; ++s) {
        const int buf = s & 1;
        const unsigned tag = base + s;
        double* pb = part + static_cast<long>(buf) * 160 * 32;
        if (warp == 0) {
            pb[rank * 32 + lane] = acc + rank + lane;
            __syncwarp();
            if (lane == 0) st_release(flags + rank * 32, tag);
        }
        const int t = threadIdx.x;
        if (t < G)
            while (ld_acquire(flags + t * 32) != tag) {
            }
        __syncthreads();
        if (warp < kLW) {
            double a = 0.0;
            for (int c = warp; c < G; c += kLW) a += __ldcg(pb + c * 32 + lane);
            xs[warp * 32 + lane] = a;
        }
        __syncthreads();
        if (warp == 0) {
            double a = 0.0;
            for (int w = 0; w < kLW; ++w) a += xs[w * 32 + lane];
            acc = a * 1e-9;
        }
        __syncthreads();
    }
    if (warp == 0) out[rank * 32 + lane] = acc;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *part, *out;
    unsigned* flags;
    cudaMalloc(&part, 2 * 160 * 32 * 8);
    cudaMalloc(&out, 160 * 32 * 8);
    cudaMalloc(&flags, 160 * 32 * 4);
    unsigned long long* slots;
    cudaMalloc(&slots, 2 * 160 * 32 * 2 * 8);
    cudaMemset(slots, 0, 2 * 160 * 32 * 2 * 8);
    unsigned* flags2;
    cudaMalloc(&flags2, 160 * 32 * 4);
    cudaMemset(flags2, 0, 160 * 32 * 4);
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
        auto run_ll = [&](auto kern, const char* name) {
            static unsigned base = 1;
            unsigned b0 = base;
            base += steps + 1;
            void* la[] = {(void*)&steps, (void*)&slots, (void*)&b0, (void*)&out};
            cudaLaunchCooperativeKernel((void*)kern, G, kWarps * 32, la, 0, 0);
            b0 = base;
            base += steps + 1;
            cudaEventRecord(e0);
            cudaLaunchCooperativeKernel((void*)kern, G, kWarps * 32, la, 0, 0);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float t;
            cudaEventElapsedTime(&t, e0, e1);
            std::printf("G=%3d %-16s: %.3f us/step  (%s)\n", G, name, t * 1e3 / steps, cudaGetErrorString(cudaGetLastError()));
        };
        run_ll(ll_kernel<0>, "LL poll");
        run_ll(ll_kernel<64>, "LL poll sleep64");
        run_ll(ll_kernel<256>, "LL poll sleep256");
        {
            static unsigned fb = 1;
            unsigned b0 = fb;
            fb += steps + 1;
            void* ca[] = {(void*)&steps, (void*)&part, (void*)&flags2, (void*)&b0, (void*)&out};
            cudaLaunchCooperativeKernel((void*)ctaflag_kernel, G, kWarps * 32, ca, 0, 0);
            b0 = fb;
            fb += steps + 1;
            cudaEventRecord(e0);
            cudaLaunchCooperativeKernel((void*)ctaflag_kernel, G, kWarps * 32, ca, 0, 0);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float t;
            cudaEventElapsedTime(&t, e0, e1);
            std::printf("G=%3d %-16s: %.3f us/step  (%s)\n", G, "CTA flag", t * 1e3 / steps, cudaGetErrorString(cudaGetLastError()));
        }
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
