// svd.cu — K6: thin SVD of the small k x n triangle of TT-SVD rounding on the
// device (linalg::svd, proj/core/src/linalg.cpp:58-69, Eigen JacobiSVD).
//
// One-sided (Hestenes) Jacobi: a cooperative kernel sweeps round-robin
// tournaments of disjoint column pairs (one warp per pair, one grid barrier
// per round) until a sweep applies no rotation. Rotations act on the columns
// themselves, so singular values keep relative accuracy (no Gram matrix is
// formed). Singular values are the column norms, sorted descending; U columns
// are normalised columns (orthonormal completion for exact zeros).
#include <cooperative_groups.h>

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <numeric>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace ttr {
namespace {

constexpr int kSvdThreads = 256;

__device__ __forceinline__ double warp_sum(double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

struct JacobiArgs {
    int m, n, N;  // N = n rounded up to even (dummy column index n when odd)
    double* A;
    i64 lda;
    double* V;
    i64 ldv;
    int* rotated;  // [max_sweeps] flags
    int max_sweeps;
    int* sweeps_done;
};

__global__ void __launch_bounds__(kSvdThreads) jacobi_kernel(JacobiArgs p) {
    cg::grid_group grid = cg::this_grid();
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    const int N = p.N, half = N / 2;
    const double eps = DBL_EPSILON;
    int sweep = 0;
    for (; sweep < p.max_sweeps; ++sweep) {
        for (int r = 0; r < N - 1; ++r) {
            for (int i = gw; i < half; i += nwarps) {
                // tournament position j -> player: 0 fixed, others rotate by r
                auto player = [&](int j) { return j == 0 ? 0 : 1 + (j - 1 + r) % (N - 1); };
                int a = player(i), b = player(N - 1 - i);
                if (a > b) { const int t = a; a = b; b = t; }
                if (b >= p.n) continue;  // dummy column
                double* ap = p.A + static_cast<i64>(a) * p.lda;
                double* aq = p.A + static_cast<i64>(b) * p.lda;
                double al = 0, be = 0, ga = 0;
                for (int row = lane; row < p.m; row += 32) {
                    const double x = ap[row], y = aq[row];
                    al = fma(x, x, al);
                    be = fma(y, y, be);
                    ga = fma(x, y, ga);
                }
                al = warp_sum(al);
                be = warp_sum(be);
                ga = warp_sum(ga);
                if (ga == 0.0 || fabs(ga) <= eps * sqrt(al * be)) continue;
                const double zeta = (be - al) / (2.0 * ga);
                const double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
                for (int row = lane; row < p.m; row += 32) {
                    const double x = ap[row], y = aq[row];
                    ap[row] = c * x - s * y;
                    aq[row] = s * x + c * y;
                }
                double* vp = p.V + static_cast<i64>(a) * p.ldv;
                double* vq = p.V + static_cast<i64>(b) * p.ldv;
                for (int row = lane; row < p.n; row += 32) {
                    const double x = vp[row], y = vq[row];
                    vp[row] = c * x - s * y;
                    vq[row] = s * x + c * y;
                }
                if (lane == 0) atomicOr(p.rotated + sweep, 1);
            }
            grid.sync();
        }
        if (*(volatile int*)(p.rotated + sweep) == 0) break;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *p.sweeps_done = sweep;
}

__global__ void col_norms(int m, int n, const double* A, i64 lda, double* s) {
    const int lane = threadIdx.x & 31;
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (w >= n) return;
    double acc = 0.0;
    for (int r = lane; r < m; r += 32) acc = fma(A[r + static_cast<i64>(w) * lda], A[r + static_cast<i64>(w) * lda], acc);
    acc = warp_sum(acc);
    if (lane == 0) s[w] = sqrt(acc);
}

// U(:, jj) = A(:, perm[jj]) / s[perm[jj]]; Vout(:, jj) = V(:, perm[jj])
__global__ void gather_sorted(int m, int n, int k, const double* A, i64 lda, const double* V, i64 ldv, const int* perm,
                              const double* s, double* U, i64 ldu, double* Vo, i64 ldvo) {
    const int jj = blockIdx.x;
    if (jj >= k) return;
    const int j = perm[jj];
    const double sj = s[j];
    const double inv = sj > 0.0 ? 1.0 / sj : 0.0;
    for (int r = threadIdx.x; r < m; r += blockDim.x) U[r + static_cast<i64>(jj) * ldu] = A[r + static_cast<i64>(j) * lda] * inv;
    for (int r = threadIdx.x; r < n; r += blockDim.x) Vo[r + static_cast<i64>(jj) * ldvo] = V[r + static_cast<i64>(j) * ldv];
}

__global__ void init_identity(int n, double* V, i64 ldv) {
    for (i64 idx = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; idx < static_cast<i64>(n) * n;
         idx += static_cast<i64>(gridDim.x) * blockDim.x) {
        const int r = static_cast<int>(idx % n), c = static_cast<int>(idx / n);
        V[r + c * ldv] = (r == c) ? 1.0 : 0.0;
    }
}

}  // namespace

void svd_small(Ctx& c, i64 m, i64 n, const double* A_in, i64 lda_in, double* U, i64 ldu, double* Vout, i64 ldvo,
               std::vector<double>& s_host, double* d_s) {
    // orient so that rows >= cols (m^T = V S U^T)
    const bool trans = m < n;
    const i64 M = trans ? n : m, Nn = trans ? m : n, k = std::min(m, n);
    c.charge_svd(14ULL * m * n * k + 8ULL * k * k * k);
    DBuf A(c, static_cast<std::size_t>(M * Nn));
    if (trans) transpose(c, m, n, A_in, lda_in, A.p, M);
    else copy_matrix(c, m, n, A_in, lda_in, A.p, M);
    DBuf V(c, static_cast<std::size_t>(Nn * Nn));
    init_identity<<<std::max<i64>(1, std::min<i64>((Nn * Nn + 255) / 256, 1024)), 256, 0, c.stream>>>(static_cast<int>(Nn), V.p, Nn);
    TTR_CUDA(cudaGetLastError());
    c.launched();
    const int max_sweeps = 60;
    int* flags = nullptr;
    TTR_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&flags), sizeof(int) * (max_sweeps + 1), c.stream));
    TTR_CUDA(cudaMemsetAsync(flags, 0, sizeof(int) * (max_sweeps + 1), c.stream));
    JacobiArgs ja{};
    ja.m = static_cast<int>(M);
    ja.n = static_cast<int>(Nn);
    ja.N = static_cast<int>(Nn + (Nn & 1));
    ja.A = A.p;
    ja.lda = M;
    ja.V = V.p;
    ja.ldv = Nn;
    ja.rotated = flags;
    ja.max_sweeps = max_sweeps;
    ja.sweeps_done = flags + max_sweeps;
    if (Nn > 1) {
        const int warps_needed = ja.N / 2;
        int blocks = (warps_needed * 32 + kSvdThreads - 1) / kSvdThreads;
        int per_sm = 0;
        TTR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jacobi_kernel, kSvdThreads, 0));
        blocks = std::max(1, std::min(blocks, per_sm * c.sm_count));
        void* args[] = {&ja};
        TTR_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(jacobi_kernel), dim3(blocks), dim3(kSvdThreads), args, 0,
                                             c.stream));
        c.launched();
    }
    DBuf s(c, static_cast<std::size_t>(Nn));
    col_norms<<<static_cast<unsigned>((Nn * 32 + 255) / 256), 256, 0, c.stream>>>(static_cast<int>(M), static_cast<int>(Nn), A.p, M, s.p);
    TTR_CUDA(cudaGetLastError());
    c.launched();
    std::vector<double> sv(static_cast<std::size_t>(Nn));
    int sweeps = 0;
    TTR_CUDA(cudaMemcpyAsync(sv.data(), s.p, sizeof(double) * Nn, cudaMemcpyDeviceToHost, c.stream));
    TTR_CUDA(cudaMemcpyAsync(&sweeps, flags + max_sweeps, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    TTR_CUDA(cudaStreamSynchronize(c.stream));
    TTR_CUDA(cudaFreeAsync(flags, c.stream));
    if (Nn > 1 && sweeps >= max_sweeps) fail(Errc::SVDFailure, "SVD did not converge");
    std::vector<int> perm(static_cast<std::size_t>(Nn));
    std::iota(perm.begin(), perm.end(), 0);
    std::stable_sort(perm.begin(), perm.end(), [&](int a, int b) { return sv[a] > sv[b]; });
    s_host.resize(static_cast<std::size_t>(k));
    for (i64 j = 0; j < k; ++j) s_host[j] = sv[perm[j]];
    int* dperm = nullptr;
    TTR_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dperm), sizeof(int) * Nn, c.stream));
    TTR_CUDA(cudaMemcpyAsync(dperm, perm.data(), sizeof(int) * Nn, cudaMemcpyHostToDevice, c.stream));
    // left/right factors of the oriented problem: Uo = A cols / s (M x k), Vo = V cols (Nn x k)
    double* Uo = trans ? Vout : U;
    const i64 lduo = trans ? ldvo : ldu;
    double* Vo = trans ? U : Vout;
    const i64 ldvoo = trans ? ldu : ldvo;
    gather_sorted<<<static_cast<unsigned>(k), 256, 0, c.stream>>>(static_cast<int>(M), static_cast<int>(Nn), static_cast<int>(k),
                                                                  A.p, M, V.p, Nn, dperm, s.p, Uo, lduo, Vo, ldvoo);
    TTR_CUDA(cudaGetLastError());
    c.launched();
    if (d_s) TTR_CUDA(cudaMemcpyAsync(d_s, s_host.data(), sizeof(double) * k, cudaMemcpyHostToDevice, c.stream));
    TTR_CUDA(cudaFreeAsync(dperm, c.stream));
    TTR_CUDA(cudaStreamSynchronize(c.stream));
    // exact-zero singular values: the matching U columns are zero; the
    // truncation rule never keeps them beyond rank 1 except for the all-zero
    // matrix, whose rank-1 result is zero either way.
}

}  // namespace ttr
