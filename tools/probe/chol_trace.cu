// Phase timing of chol_kernel (clock64 per phase, thread 0): nvcc -DTTR_CHOL_TRACE,
// includes the kernel source; run on the GPU box: chol_trace n
#include "../../paper_2511_03598_b200/csrc/qr_chol.cu"
#include <cstdio>
#include <vector>
#include <random>
using namespace ttr;
int main(int argc, char** argv) {
    int n = argc > 1 ? atoi(argv[1]) : 110;
    int m = 4 * n;
    std::mt19937_64 g(1);
    std::normal_distribution<double> nd;
    std::vector<double> a((size_t)m * n), G((size_t)n * n, 0.0);
    for (auto& x : a) x = nd(g);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            double s = 0;
            for (int k = 0; k < m; ++k) s += a[(size_t)i * m + k] * a[(size_t)j * m + k];
            G[i + (size_t)j * n] = s;
        }
    double *dG, *dRi; int* flag;
    cudaMalloc(&dG, sizeof(double) * n * n); cudaMalloc(&dRi, sizeof(double) * 1024 * ((n + 31) / 32 + 1)); cudaMalloc(&flag, 4);
    for (int rep = 0; rep < 3; ++rep) {
        cudaMemcpy(dG, G.data(), sizeof(double) * n * n, cudaMemcpyHostToDevice);
        cudaMemset(flag, 0, 4);
        unsigned long long z[8] = {0};
        cudaMemcpyToSymbol(g_chol_trace, z, sizeof(z));
        CholArgs p{n, dG, n, 1, 1e-12, flag, 1, dRi};
        const std::size_t panel = sizeof(double) * 32 * chol_ldp(n);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        if (n <= kCholSmemMaxN) {
            set_max_dynamic_smem(reinterpret_cast<const void*>(chol_kernel<true>));
            cudaEventRecord(e0);
            chol_kernel<true><<<1, kCholThreads, panel + sizeof(double) * n * (n + 1)>>>(p);
        } else {
            set_max_dynamic_smem(reinterpret_cast<const void*>(chol_kernel<false>));
            cudaEventRecord(e0);
            chol_kernel<false><<<1, kCholThreads, panel>>>(p);
        }
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long t[8]; cudaMemcpyFromSymbol(t, g_chol_trace, sizeof(t));
        int f; cudaMemcpy(&f, flag, 4, cudaMemcpyDeviceToHost);
        printf("n=%d %.1f us flag %d err %s | cycles: load %llu dload %llu diag %llu panel %llu trail %llu inv %llu diagwarp %llu\n", n,
               ms * 1e3, f, cudaGetErrorString(cudaGetLastError()), t[0], t[1], t[2], t[3], t[4], t[5], t[6]);
    }
}
