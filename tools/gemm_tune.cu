// Tile-configuration sweep for the fp64 DMMA GEMM (measurement tool).
// Includes the library's kernel source and times instantiations on the
// shapes of config 5b. Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude -o tools/gemm_tune tools/gemm_tune.cu
#include <cstdio>
#include <vector>

#include "../paper_2511_03598_b200/csrc/gemm_dmma.cu"

namespace ttr {
double* Ctx::scratch(std::size_t bytes) {
    if (bytes > work_bytes) {
        if (work) cudaFree(work);
        cudaMalloc(reinterpret_cast<void**>(&work), bytes);
        work_bytes = bytes;
    }
    return work;
}
void cuda_fail(cudaError_t e, const char* expr, const char* file, int line) {
    std::printf("CUDA error %s at %s:%d (%s)\n", cudaGetErrorString(e), file, line, expr);
    std::exit(1);
}
const char* errc_name(Errc) { return "err"; }
void scale(Ctx&, double*, std::size_t, double) {}
}  // namespace ttr

using namespace ttr;

template <int BM, int BN, int BK, int WM, int WN, int ST, bool AT, int KM>
float run_cfg(Ctx& c, GemmArgs a, int splits, int reps) {
    const int total_kt = (a.K + BK - 1) / BK;
    a.ktiles_per_split = (total_kt + splits - 1) / splits;
    splits = (total_kt + a.ktiles_per_split - 1) / a.ktiles_per_split;
    if (splits > 1) a.work = c.scratch(static_cast<std::size_t>(splits) * a.M * a.N * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int w = 0; w < 2; ++w) launch<BM, BN, BK, WM, WN, ST, AT, KM, 2, 2>(c, a, splits);
    cudaEventRecord(e0, c.stream);
    for (int r = 0; r < reps; ++r) {
        launch<BM, BN, BK, WM, WN, ST, AT, KM, 2, 2>(c, a, splits);
        if (splits > 1) {
            const i64 total = static_cast<i64>(a.M) * a.N;
            splitk_reduce<<<std::min<i64>((total + 255) / 256, 592), 256, 0, c.stream>>>(a.work, splits, a.M, a.N, 1.0,
                                                                                       0.0, a.C, a.ldc, nullptr, 0);
        }
    }
    cudaEventRecord(e1, c.stream);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) std::printf("  error %s\n", cudaGetErrorString(err));
    return ms / reps;
}

template <int BM, int BN, bool AT, int KM, int ST = 4>
float run_tma(Ctx& c, GemmArgs a, int splits, int reps) {
    const int total_kt = (a.K + 15) / 16;
    a.ktiles_per_split = (total_kt + splits - 1) / splits;
    splits = (total_kt + a.ktiles_per_split - 1) / a.ktiles_per_split;
    if (splits > 1) a.work = c.scratch(static_cast<std::size_t>(splits) * a.M * a.N * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int w = 0; w < 2; ++w) launch_tma<BM, BN, AT, KM, ST>(c, a, splits);
    cudaEventRecord(e0, c.stream);
    for (int r = 0; r < reps; ++r) {
        launch_tma<BM, BN, AT, KM, ST>(c, a, splits);
        if (splits > 1) {
            const i64 total = static_cast<i64>(a.M) * a.N;
            splitk_reduce_wide<<<(total + 31) / 32, 256, 0, c.stream>>>(a.work, splits, a.M, a.N, 1.0, 0.0, a.C, a.ldc,
                                                                       nullptr, 0);
        }
    }
    cudaEventRecord(e1, c.stream);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) std::printf("  error %s\n", cudaGetErrorString(err));
    return ms / reps;
}

int main() {
    Ctx c;
    c.stream = 0;
    cudaDeviceGetAttribute(&c.sm_count, cudaDevAttrMultiProcessorCount, 0);
    // buffers big enough for all shapes
    const size_t big = 1000ull * 128000;  // 1 G doubles? no: 128M doubles = 1 GB
    double *A, *B, *Cm, *Wt;
    cudaMalloc(&A, big * 8);
    cudaMalloc(&B, 128ull * 1024 * 1024 * 8);
    cudaMalloc(&Cm, 64ull * 1024 * 1024 * 8);
    cudaMalloc(&Wt, 4ull * 1024 * 1024 * 8);
    cudaMemset(A, 0, big * 8);
    cudaMemset(B, 0, 128ull * 1024 * 1024 * 8);
    cudaMemset(Wt, 0, 4ull * 1024 * 1024 * 8);

    struct Shape { const char* name; int M, N, K; bool at; int km; int splits; };
    std::vector<Shape> shapes = {
        {"sketch 1000x320x128000 (KRP) s74", 1000, 320, 128000, false, 1, 74},
        {"sketch 1000x320x128000 (KRP) s37", 1000, 320, 128000, false, 1, 37},
        {"sketch 1000x320x128000 (KRP) s19", 1000, 320, 128000, false, 1, 19},
        {"plain 1000x320x128000 s37", 1000, 320, 128000, false, 0, 37},
        {"S=V*W 40960x320x1000", 40960, 320, 1000, false, 0, 1},
        {"M=Q^T V 320x1000x40960", 320, 1000, 40960, true, 0, 8},
        {"next=M*H 320x128000x1000", 320, 128000, 1000, false, 0, 1},
    };
    for (auto& s : shapes) {
        GemmArgs a{};
        a.M = s.M; a.N = s.N; a.K = s.K;
        a.A = A; a.lda = s.at ? s.K : s.M;
        a.B = B; a.ldb = s.km == 1 ? 128 : s.K;
        a.Wt = Wt; a.ldw = s.N; a.nmode = 128;
        a.C = Cm; a.ldc = s.M; a.alpha = 1.0; a.beta = 0.0;
        const double gf = 2.0 * s.M * s.N * s.K / 1e9;
        std::printf("%s (%.1f GF)\n", s.name, gf);
#define RUN(BM, BN, BK, WM, WN, ST)                                                                      \
        {                                                                                                \
            float ms;                                                                                    \
            if (s.km == 1) ms = run_cfg<BM, BN, BK, WM, WN, ST, false, 1>(c, a, s.splits, 5);            \
            else if (s.at) ms = run_cfg<BM, BN, BK, WM, WN, ST, true, 0>(c, a, s.splits, 5);             \
            else ms = run_cfg<BM, BN, BK, WM, WN, ST, false, 0>(c, a, s.splits, 5);                      \
            std::printf("  %3dx%-3d bk%-2d w%dx%d st%d : %8.3f ms %6.2f TF/s\n", BM, BN, BK, WM, WN, ST, ms, \
                        gf / ms);                                                                        \
        }
        {
            float ms;
            if (s.km == 1) ms = run_tma<128, 64, false, 1>(c, a, s.splits, 5);
            else if (s.at) ms = run_tma<128, 64, true, 0>(c, a, s.splits, 5);
            else ms = run_tma<128, 64, false, 0>(c, a, s.splits, 5);
            std::printf("  TMA 128x64        : %8.3f ms %6.2f TF/s\n", ms, gf / ms);
            if (s.km == 1) ms = run_tma<128, 64, false, 1, 6>(c, a, s.splits, 5);
            else if (s.at) ms = run_tma<128, 64, true, 0, 6>(c, a, s.splits, 5);
            else ms = run_tma<128, 64, false, 0, 6>(c, a, s.splits, 5);
            std::printf("  TMA 128x64 st6    : %8.3f ms %6.2f TF/s\n", ms, gf / ms);
            if (s.km == 0) {
                ms = s.at ? run_tma<64, 64, true, 0>(c, a, s.splits, 5) : run_tma<64, 64, false, 0>(c, a, s.splits, 5);
                std::printf("  TMA 64x64         : %8.3f ms %6.2f TF/s\n", ms, gf / ms);
            }
        }
        RUN(128, 64, 16, 32, 32, 4)
        RUN(64, 64, 16, 32, 32, 4)
        RUN(64, 64, 16, 32, 32, 3)
    }
    // ---- blocked-QR shapes (memory-bound): trailing update and V^T A ----
    {
        GemmArgs a{};
        a.M = 40960; a.N = 288; a.K = 32;
        a.A = A; a.lda = 40960; a.B = B; a.ldb = 32; a.C = Cm; a.ldc = 40960; a.alpha = -1.0; a.beta = 1.0;
        const double gb = (2.0 * 40960 * 288 + 40960 * 32) * 8 / 1e9;
        std::printf("update A -= V W2 40960x288x32 beta=1 (%.0f MB min traffic)\n", gb * 1e3);
        auto pr = [&](const char* nm, float ms) { std::printf("  %-22s: %8.4f ms %7.0f GB/s\n", nm, ms, gb / ms * 1e3); };
        pr("TMA 128x64 st4", run_tma<128, 64, false, 0, 4>(c, a, 1, 10));
        pr("TMA 128x64 st2", run_tma<128, 64, false, 0, 2>(c, a, 1, 10));
        pr("TMA 64x64 st2", run_tma<64, 64, false, 0, 2>(c, a, 1, 10));
        pr("TMA 64x64 st4", run_tma<64, 64, false, 0, 4>(c, a, 1, 10));
        pr("cp.async 128x64", run_cfg<128, 64, 16, 32, 32, 4, false, 0>(c, a, 1, 10));
    }
    {
        GemmArgs a{};
        a.M = 32; a.N = 288; a.K = 40960;
        a.A = A; a.lda = 40960; a.B = B; a.ldb = 40960; a.C = Cm; a.ldc = 32; a.alpha = 1.0; a.beta = 0.0;
        const double gb = (40960.0 * 288 + 40960 * 32) * 8 / 1e9;
        std::printf("V^T A 32x288x40960 (%.0f MB min traffic)\n", gb * 1e3);
        auto pr = [&](const char* nm, float ms) { std::printf("  %-22s: %8.4f ms %7.0f GB/s\n", nm, ms, gb / ms * 1e3); };
        for (int sp : {142, 74, 37}) {
            char nm[64];
            std::snprintf(nm, sizeof nm, "cp.async 32x128 s%d", sp);
            pr(nm, run_cfg<32, 128, 16, 32, 32, 4, true, 0>(c, a, sp, 10));
            std::snprintf(nm, sizeof nm, "TMA 32x128 s%d", sp);
            pr(nm, run_tma<32, 128, true, 0, 4>(c, a, sp, 10));
            std::snprintf(nm, sizeof nm, "TMA 32x64 s%d", sp);
            pr(nm, run_tma<32, 64, true, 0, 4>(c, a, sp, 10));
        }
    }
    return 0;
}
