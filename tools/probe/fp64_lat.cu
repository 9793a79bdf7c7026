// Latency/throughput of fp64 div, sqrt, rsqrt-based paths, shuffles and smem
// round trips on one warp (dependent chains), B200 probe.
#include <cstdio>
__global__ void lat(double* out, double x0, int iters, long long* cyc) {
    double x = x0 + threadIdx.x * 1e-9;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) x = 1.0 / (x + 1.0);          // div chain
    long long t1 = clock64();
    for (int i = 0; i < iters; ++i) x = sqrt(x + 2.0);             // sqrt chain
    long long t2 = clock64();
    for (int i = 0; i < iters; ++i) x = fma(x, 0.999, 1e-3);       // dfma chain
    long long t3 = clock64();
    for (int i = 0; i < iters; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) + 1e-3;  // shfl chain
    long long t4 = clock64();
    __shared__ double sm[64];
    for (int i = 0; i < iters; ++i) { sm[threadIdx.x & 31] = x; __syncwarp(); x = sm[(threadIdx.x + 1) & 31] * 0.5 + 1.0; __syncwarp(); }
    long long t5 = clock64();
    for (int i = 0; i < iters; ++i) { sm[threadIdx.x & 63] = x; __syncthreads(); x = sm[(threadIdx.x + 1) & 63] * 0.5 + 1.0; __syncthreads(); }
    long long t6 = clock64();
    for (int i = 0; i < iters; ++i) x = __drcp_rn(x + 1.0);        // rcp chain
    long long t7 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5; cyc[6] = t7 - t6; }
}
int main() {
    double* out; long long* cyc; cudaMalloc(&out, 8 * 1024); cudaMallocManaged(&cyc, 8 * 8);
    const int iters = 1000;
    for (int threads : {32, 256, 1024}) {
        lat<<<1, threads>>>(out, 0.5, iters, cyc);
        cudaDeviceSynchronize();
        printf("threads %4d cycles/op: div %.1f sqrt %.1f dfma %.1f shfl64 %.1f smem+syncwarp %.1f smem+syncthreads %.1f rcp %.1f\n", threads,
               cyc[0] / (double)iters, cyc[1] / (double)iters, cyc[2] / (double)iters, cyc[3] / (double)iters,
               cyc[4] / (double)iters, cyc[5] / (double)iters, cyc[6] / (double)iters);
    }
}
