// Phase timing of the batched small sCQR3 (qr_chol.cu K4e; clock64 per phase on
// thread 0 of every CTA, summed): nvcc -DTTR_SQ_TRACE, includes the kernel
// source; links the other objects of the library build:
//   nvcc -DTTR_SQ_TRACE ... sq_trace.cu $(build/*.o except qr_chol.o) -lcudart
// run on the GPU box: sq_trace m n batch
#include "../../paper_2511_03598_b200/csrc/qr_chol.cu"
#include <cstdio>
#include <random>
#include <vector>
using namespace ttr;
template <int NT>
void go(int m, int n, int batch) {
    std::mt19937_64 g(1);
    std::normal_distribution<double> nd;
    std::vector<double> a((size_t)m * n * batch);
    for (auto& x : a) x = nd(g);
    double *dA, *dQ; int* flags;
    cudaMalloc(&dA, sizeof(double) * a.size()); cudaMalloc(&dQ, sizeof(double) * a.size()); cudaMalloc(&flags, 4 * batch);
    cudaMemcpy(dA, a.data(), sizeof(double) * a.size(), cudaMemcpyHostToDevice);
    const std::size_t smem = sq_smem<NT>(m, n);
    cudaFuncSetAttribute(cholqr_small_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int tiles = (m + 7) / 8;
    const int warps = getenv("TTR_SQ_WARPS") ? atoi(getenv("TTR_SQ_WARPS")) : std::max(kSqGramWarps, std::min(8, (tiles + 3) / 4));
    const double coeff = 11.0 * ((double)m * n + (double)n * (n + 1)) * (DBL_EPSILON / 2);
    for (int rep = 0; rep < 3; ++rep) {
        unsigned long long z[8] = {0};
        cudaMemcpyToSymbol(g_sq_trace, z, sizeof(z));
        cudaMemset(flags, 0, 4 * batch);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        cholqr_small_kernel<NT><<<batch, 32 * warps, smem>>>(m, n, dA, m, (i64)m * n, dQ, m, (i64)m * n, coeff, flags);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long t[8]; cudaMemcpyFromSymbol(t, g_sq_trace, sizeof(t));
        printf("m=%d n=%d batch=%d warps=%d smem=%zu: %.1f us %s | cycles/CTA: load %llu gram %llu reduce %llu chol %llu trsm %llu store %llu\n",
               m, n, batch, warps, smem, ms * 1e3, cudaGetErrorString(cudaGetLastError()), t[0] / batch, t[1] / batch,
               t[2] / batch, t[3] / batch, t[4] / batch, t[5] / batch);
    }
}
int main(int argc, char** argv) {
    int m = argc > 1 ? atoi(argv[1]) : 320, n = argc > 2 ? atoi(argv[2]) : 20, b = argc > 3 ? atoi(argv[3]) : 2048;
    switch ((n + 7) / 8) { case 1: go<1>(m, n, b); break; case 2: go<2>(m, n, b); break; case 3: go<3>(m, n, b); break; default: go<4>(m, n, b); }
}
