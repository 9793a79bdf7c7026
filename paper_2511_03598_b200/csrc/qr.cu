// qr.cu — K4: Householder thin QR with explicit Q on the device.
//
// Replaces linalg::thin_qr / thin_qr_q (proj/core/src/linalg.cpp:44-56, Eigen
// HouseholderQR + householderQ()*Identity). Same reflector convention as
// Eigen::makeHouseholder: beta = -sign(alpha)*||x||, tau = (beta-alpha)/beta,
// v = [1; x_tail/(alpha-beta)], and tau = 0 when the tail is exactly zero, so
// rank-deficient sketches (the last bond of configs 3/5, padded exact-rank
// inputs) still give an orthonormal Q (linalg.hpp:22).
//
// Two paths:
//  * qr_small_kernel — the whole m x n matrix lives in one CTA's shared
//    memory (m*n <= ~26k doubles); factor + in-place dorg2r-style backward
//    accumulation of Q; warp-shuffle column reductions. Batched over a
//    strided set of matrices (one CTA each) for the 5a batch.
//  * blocked right-looking Householder for tall matrices: panels of width
//    kPanel factored by panel_col_kernel (qr_panel.cuh: lane = column, warp =
//    row block, registers only; CTAs combined through one thread-block
//    cluster's distributed shared memory or a cooperative grid barrier, sums
//    in fixed order -> deterministic), which also emits V and the compact-WY
//    T; the trailing update and the explicit-Q backward accumulation run on
//    the DMMA GEMM (gemm_dmma.cu). <= 32 columns: one launch yields Q and R.
//    Very tall R-only requests (norm_exact) take a TSQR split first.
#include <cooperative_groups.h>

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace ttr {
namespace {

constexpr int kQrThreads = 256;
constexpr int kPanel = 32;

__device__ __forceinline__ double warp_sum(double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Fixed-order block reduction (deterministic); result broadcast to all threads.
__device__ double block_sum(double v, double* red) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    double s = 0.0;
    for (int i = 0; i < nw; ++i) s += red[i];
    return s;
}

// ---------------------------------------------------------------------------
// single-CTA QR (batched): a[m x n] in smem (ld m), tau[n]
__global__ void __launch_bounds__(kQrThreads) qr_small_kernel(int m, int n, const double* A, i64 lda, i64 sA, double* Q,
                                                              i64 ldq, i64 sQ, double* R, i64 ldr, i64 sR) {
    extern __shared__ double sm[];
    double* a = sm;
    double* tau = a + static_cast<i64>(m) * n;
    double* red = tau + n;
    double* bc = red + 32;  // broadcast scalars
    const int k = min(m, n);
    A += blockIdx.x * sA;
    if (Q) Q += blockIdx.x * sQ;
    if (R) R += blockIdx.x * sR;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;

    for (i64 idx = tid; idx < static_cast<i64>(m) * n; idx += blockDim.x) {
        const int r = static_cast<int>(idx % m), c = static_cast<int>(idx / m);
        a[idx] = A[r + c * lda];
    }
    __syncthreads();

    for (int j = 0; j < k; ++j) {
        double* x = a + static_cast<i64>(j) * m;
        double t = 0.0;
        for (int r = j + 1 + tid; r < m; r += blockDim.x) t = fma(x[r], x[r], t);
        const double tail = block_sum(t, red);
        if (tid == 0) {
            const double alpha = x[j];
            double tj, beta, inv;
            if (tail <= DBL_MIN) {
                tj = 0.0;
                beta = alpha;
                inv = 0.0;
            } else {
                beta = sqrt(alpha * alpha + tail);
                if (alpha >= 0.0) beta = -beta;
                inv = 1.0 / (alpha - beta);
                tj = (beta - alpha) / beta;
            }
            tau[j] = tj;
            bc[0] = beta;
            bc[1] = inv;
        }
        __syncthreads();
        const double inv = bc[1], tj = tau[j];
        for (int r = j + 1 + tid; r < m; r += blockDim.x) x[r] *= inv;
        __syncthreads();
        if (tj != 0.0) {
            for (int l = j + 1 + warp; l < n; l += nw) {
                double* y = a + static_cast<i64>(l) * m;
                double s = 0.0;
                for (int r = j + 1 + lane; r < m; r += 32) s = fma(x[r], y[r], s);
                s = warp_sum(s) + y[j];
                const double wv = tj * s;
                if (lane == 0) y[j] -= wv;
                for (int r = j + 1 + lane; r < m; r += 32) y[r] = fma(-wv, x[r], y[r]);
            }
        }
        __syncthreads();
        if (tid == 0) x[j] = bc[0];
        __syncthreads();
    }
    if (R) {
        for (i64 idx = tid; idx < static_cast<i64>(k) * n; idx += blockDim.x) {
            const int r = static_cast<int>(idx % k), c = static_cast<int>(idx / k);
            R[r + c * ldr] = (r <= c) ? a[r + static_cast<i64>(c) * m] : 0.0;
        }
    }
    __syncthreads();
    if (Q == nullptr) return;  // R only (norm_exact)
    // explicit thin Q (m x k), backward accumulation in place (LAPACK dorg2r)
    for (int i = k - 1; i >= 0; --i) {
        const double ti = tau[i];
        double* v = a + static_cast<i64>(i) * m;
        if (i < k - 1 && ti != 0.0) {
            for (int l = i + 1 + warp; l < k; l += nw) {
                double* y = a + static_cast<i64>(l) * m;
                double s = 0.0;
                for (int r = i + 1 + lane; r < m; r += 32) s = fma(v[r], y[r], s);
                s = warp_sum(s) + y[i];
                const double wv = ti * s;
                if (lane == 0) y[i] -= wv;
                for (int r = i + 1 + lane; r < m; r += 32) y[r] = fma(-wv, v[r], y[r]);
            }
        }
        __syncthreads();
        for (int r = tid; r < m; r += blockDim.x) {
            if (r > i) v[r] *= -ti;
            else if (r == i) v[r] = 1.0 - ti;
            else v[r] = 0.0;
        }
        __syncthreads();
    }
    for (i64 idx = tid; idx < static_cast<i64>(m) * k; idx += blockDim.x) {
        const int r = static_cast<int>(idx % m), c = static_cast<int>(idx / m);
        Q[r + c * ldq] = a[idx];
    }
}

// ---------------------------------------------------------------------------
// Arguments of the Householder panel kernel (qr_panel.cuh). Optional outputs:
// the factored panel (reflector tails + R), R, the explicit unit-lower V, the
// compact-WY T and — when the panel is the whole matrix — the explicit thin Q.
struct RegQrArgs {
    int rows, b, rpc;
    const double* Pin;
    i64 ldin;
    double* Pout;
    i64 ldout;
    double* tau;
    double* V;
    i64 ldv;
    double* T;
    double* Q;
    i64 ldq;
    double* R;
    i64 ldr;
    unsigned long long* xchg;  // grid mode: Ctx::qr_exchange() ([2][160][32] partials + [2][32] row)
    long long* trace;  // optional (TTR_QR_TRACE): clock64 per phase of CTA 0 / thread 0
};

#include "qr_panel.cuh"
#include "qr_cpanel.cuh"
#include "qr_batch.cuh"

template <int RPT, int WARPS, int MODE>
void launch_col(Ctx& c, const RegQrArgs& a, i64 grid) {
    auto kern = panel_col_kernel<RPT, WARPS, MODE>;
    if constexpr (MODE == 0) {
        static std::atomic<std::uint64_t> configured{0};  // bit d: attributes set on device d
        if (first_on_device(configured)) {
            TTR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        }
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(static_cast<unsigned>(grid));
        cfg.blockDim = dim3(WARPS * 32);
        cfg.dynamicSmemBytes = 0;
        cfg.stream = c.stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = static_cast<unsigned>(grid);
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        TTR_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
    } else {
        RegQrArgs copy = a;
        void* args[] = {&copy};
        TTR_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(kern), dim3(static_cast<unsigned>(grid)),
                                             dim3(WARPS * 32), args, 0, c.stream));
    }
    c.launched();
    if (a.trace) {  // TTR_QR_TRACE: per-phase cycles of CTA 0, averaged over the panel's columns
        long long h[32 * 8];
        TTR_CUDA(cudaMemcpyAsync(h, a.trace, sizeof(h), cudaMemcpyDeviceToHost, c.stream));
        TTR_CUDA(cudaStreamSynchronize(c.stream));
        const int nc = std::min(a.b, a.rows);
        double acc[8] = {};
        for (int i = 0; i < nc; ++i) {
            const long long* t = h + i * 8;
            const long long seq[8] = {t[0], t[1], t[6], t[7], t[2], t[3], t[4], t[5]};
            for (int k = 1; k < 8; ++k) acc[k] += static_cast<double>(seq[k] - seq[k - 1]) / nc;
            acc[0] += static_cast<double>(t[5] - t[0]) / nc;
        }
        std::fprintf(stderr,
                     "panel<%d,%d,mode %d> grid %lld rows %d: cycles/col %.0f | dots %.0f bar %.0f xchg %.0f gather %.0f "
                     "scalar %.0f bar %.0f update %.0f\n",
                     RPT, WARPS, MODE, static_cast<long long>(grid), a.rows, acc[0], acc[1], acc[2], acc[3], acc[4],
                     acc[5], acc[6], acc[7]);
    }
}

// Geometry + template dispatch for panel_col_kernel. a.xchg must be set.
bool launch_panel_col(Ctx& c, RegQrArgs a) {
    const i64 rows = a.rows;
    static const bool tracing = std::getenv("TTR_QR_TRACE") != nullptr;  // diagnostics only
    static long long* trace_buf = nullptr;
    if (tracing && !trace_buf) TTR_CUDA(cudaMalloc(reinterpret_cast<void**>(&trace_buf), 32 * 8 * sizeof(long long)));
    a.trace = tracing ? trace_buf : nullptr;
    constexpr int kClW = 16;
    auto cl_try = [&](auto rpt_tag) -> bool {
        constexpr int RPT = decltype(rpt_tag)::value;
        const i64 per = static_cast<i64>(kClW) * RPT;
        if (rows > 16 * per) return false;
        const i64 grid = std::max<i64>(1, (rows + per - 1) / per);
        a.rpc = static_cast<int>(per);
        launch_col<RPT, kClW, 0>(c, a, grid);
        return true;
    };
    // grid: 16 warps while x[RPT] leaves room in 128 registers, then 8 warps
    auto gr_try = [&](auto rpt_tag, auto warps_tag, auto mode_tag, i64 max_grid) -> bool {
        constexpr int RPT = decltype(rpt_tag)::value, W = decltype(warps_tag)::value;
        constexpr int MODE = decltype(mode_tag)::value;
        const i64 per = static_cast<i64>(W) * RPT;
        if (rows > max_grid * per) return false;
        const i64 grid = std::max<i64>(1, (rows + per - 1) / per);
        a.rpc = static_cast<int>(per);
        launch_col<RPT, W, MODE>(c, a, grid);
        return true;
    };
    // experiments: TTR_QR_PANEL_MODE = grid forces the cooperative grid
    static const int forced = [] {
        const char* e = std::getenv("TTR_QR_PANEL_MODE");
        return (e && e[0] == 'g') ? 1 : -1;
    }();
    using I16 = std::integral_constant<int, 16>;
    using I8 = std::integral_constant<int, 8>;
    using Gb = std::integral_constant<int, 1>;
    // Measured (tools/qr_bench.py, tools/probe/exchange_cost.cu): the cluster
    // wins while a warp owns <= 8 rows (<= 2048-row panels); beyond that the
    // cooperative grid (up to one CTA per SM) wins.
    if ((forced < 0 || forced == 0) &&
        (cl_try(std::integral_constant<int, 4>{}) || cl_try(std::integral_constant<int, 8>{})))
        return true;
    static const bool force_cluster = [] {  // experiments: TTR_QR_PANEL_MODE=c tries tall cluster panels
        const char* e = std::getenv("TTR_QR_PANEL_MODE");
        return e && e[0] == 'c';
    }();
    if (force_cluster && (cl_try(std::integral_constant<int, 12>{}) || cl_try(std::integral_constant<int, 16>{}) ||
                          cl_try(std::integral_constant<int, 20>{}) || cl_try(std::integral_constant<int, 28>{})))
        return true;
    const i64 g = std::min<i64>(c.sm_count, kQrMaxGridCtas);  // the exchange layout holds 160 CTA slots
    if (gr_try(std::integral_constant<int, 4>{}, I16{}, Gb{}, g) ||
        gr_try(std::integral_constant<int, 8>{}, I16{}, Gb{}, g) ||
        gr_try(std::integral_constant<int, 12>{}, I16{}, Gb{}, g) ||
        gr_try(std::integral_constant<int, 16>{}, I16{}, Gb{}, g) ||
        gr_try(std::integral_constant<int, 20>{}, I16{}, Gb{}, g) ||
        gr_try(std::integral_constant<int, 24>{}, I16{}, Gb{}, g) ||
        gr_try(std::integral_constant<int, 56>{}, I8{}, Gb{}, g) || gr_try(std::integral_constant<int, 64>{}, I8{}, Gb{}, g))
        return false;
    throw Error(TTR_ERR_INTERNAL, "qr panel taller than the device panel limit");
}

__global__ void init_thin_identity(int m, int k, double* Q, i64 ldq, i64 sQ = 0) {
    Q += blockIdx.y * sQ;
    const i64 total = static_cast<i64>(m) * k;
    for (i64 idx = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<i64>(gridDim.x) * blockDim.x) {
        const int r = static_cast<int>(idx % m), c = static_cast<int>(idx / m);
        Q[r + c * ldq] = (r == c) ? 1.0 : 0.0;
    }
}

__global__ void add_unit_diagonal(int k, double* Q, i64 ldq) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < k) Q[j + static_cast<i64>(j) * ldq] += 1.0;
}

__global__ void copy_upper(int k, int n, const double* A, i64 lda, double* R, i64 ldr, i64 sA = 0, i64 sR = 0) {
    A += blockIdx.y * sA;
    R += blockIdx.y * sR;
    const i64 total = static_cast<i64>(k) * n;
    for (i64 idx = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<i64>(gridDim.x) * blockDim.x) {
        const int r = static_cast<int>(idx % k), c = static_cast<int>(idx / k);
        R[r + c * ldr] = (r <= c) ? A[r + c * lda] : 0.0;
    }
}

// Aggregated compact-WY factor of all panels: T = U^{-1}, U = diag(1/tau) +
// striu(V^T V), by block back substitution with the panel factors T_i
// (= U_ii^{-1}, zero rows/columns for tau = 0): X_jj = T_j,
// X_ij = -T_i sum_{l=i+1..j} G_il X_lj. One CTA per block column j; the
// column X(:, j-block) stays in shared memory. k x k in/out, ld k, blocks of 32
// (zero padded past k).
constexpr int kTaggThreads = 256;
__global__ void __launch_bounds__(kTaggThreads) t_aggregate_kernel(int k, const double* __restrict__ G,
                                                                   const double* __restrict__ Ts, double* T,
                                                                   i64 sG = 0, i64 sTs = 0, i64 sT = 0) {
    extern __shared__ double xs[];  // X(:, j-block): [nb * 32][32]; then G row block [(nb-1)*32][33]
    __shared__ double acc_s[32 * 33];
    __shared__ double ti_s[32 * 33];
    G += blockIdx.y * sG;  // batch (blockIdx.y): one matrix of a strided set
    Ts += blockIdx.y * sTs;
    T += blockIdx.y * sT;
    const int j = blockIdx.x, nb = (k + 31) / 32, tid = threadIdx.x;
    double* gs = xs + static_cast<i64>(nb) * 32 * 32;
    const int r = tid & 31, c0 = tid >> 5;  // thread owns (r, c0 + 8q), q = 0..3
    // X_jj = T_j
    for (int q = 0; q < 4; ++q) xs[(j * 32 + r) * 32 + c0 + 8 * q] = Ts[static_cast<i64>(j) * 1024 + r + (c0 + 8 * q) * 32];
    for (int i = j - 1; i >= 0; --i) {
        // stage G(i-block, (i+1)..j blocks) (coalesced: 32 rows of one column per warp) and T_i
        const int ncols = (j - i) * 32;
        for (int e = tid; e < ncols * 32; e += kTaggThreads) {
            const int rr = e & 31, cc = e >> 5, row = i * 32 + rr, col = (i + 1) * 32 + cc;
            gs[cc * 33 + rr] = (row < k && col < k) ? G[row + static_cast<i64>(col) * k] : 0.0;
        }
        for (int e = tid; e < 1024; e += kTaggThreads) ti_s[(e & 31) * 33 + (e >> 5)] = Ts[static_cast<i64>(i) * 1024 + e];
        __syncthreads();
        double a[4] = {0.0, 0.0, 0.0, 0.0};
        for (int t = 0; t < ncols; ++t) {
            const double g = gs[t * 33 + r];
            const double* xr = xs + ((i + 1) * 32 + t) * 32 + c0;
#pragma unroll
            for (int q = 0; q < 4; ++q) a[q] = fma(g, xr[8 * q], a[q]);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) acc_s[r * 33 + c0 + 8 * q] = a[q];
        __syncthreads();
        double x[4] = {0.0, 0.0, 0.0, 0.0};
        for (int t = 0; t < 32; ++t) {
            const double tv = ti_s[r * 33 + t];  // T_i(r, t)
#pragma unroll
            for (int q = 0; q < 4; ++q) x[q] = fma(tv, acc_s[t * 33 + c0 + 8 * q], x[q]);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) xs[(i * 32 + r) * 32 + c0 + 8 * q] = -x[q];
        __syncthreads();
    }
    __syncthreads();
    // write column block j (rows below the diagonal block are zero)
    for (int e = tid; e < k * 32; e += kTaggThreads) {
        const int row = e % k, cc = e / k, col = j * 32 + cc;
        if (col >= k) continue;
        const int bi = row / 32;
        T[row + static_cast<i64>(col) * k] = bi <= j ? xs[(bi * 32 + row % 32) * 32 + cc] : 0.0;
    }
}

int blocks_for(Ctx& c, i64 work) {
    return static_cast<int>(std::max<i64>(1, std::min<i64>((work + 255) / 256, 4LL * c.sm_count)));
}

// rows x cols copies / k x k transposes of a strided batch (blockIdx.y = matrix)
__global__ void copy_batched_kernel(int rows, int cols, const double* __restrict__ s, i64 lds, i64 ss,
                                    double* __restrict__ d, i64 ldd, i64 sd) {
    s += blockIdx.y * ss;
    d += blockIdx.y * sd;
    const i64 total = static_cast<i64>(rows) * cols;
    for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<i64>(gridDim.x) * blockDim.x) {
        const int r = static_cast<int>(i % rows), cc = static_cast<int>(i / rows);
        d[r + cc * ldd] = s[r + cc * lds];
    }
}
__global__ void transpose_batched_kernel(int k, const double* __restrict__ s, i64 lds, i64 ss, double* __restrict__ d,
                                         i64 ldd, i64 sd) {
    s += blockIdx.y * ss;
    d += blockIdx.y * sd;
    const i64 total = static_cast<i64>(k) * k;
    for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<i64>(gridDim.x) * blockDim.x) {
        const int r = static_cast<int>(i % k), cc = static_cast<int>(i / k);
        d[cc + r * ldd] = s[r + cc * lds];
    }
}

// ---- cluster push panels (qr_cpanel.cuh) --------------------------------------
constexpr int kPushWarps = 16;
constexpr int kPushMaxRpt = 28;
constexpr i64 kPushMaxRows = static_cast<i64>(kPushMaxCtas) * kPushWarps * kPushMaxRpt;  // 7,168 (+ the diagonal block)

template <int RPT>
void launch_push(Ctx& c, const PushQrArgs& a, int G, i64 batch) {
    auto kern = panel_push_kernel<RPT, kPushWarps>;
    static std::atomic<std::uint64_t> configured{0};  // bit d: attributes set on device d
    constexpr std::size_t smem = push_smem_bytes<RPT, kPushWarps>();
    if (first_on_device(configured)) {
        TTR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        TTR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(G * batch));
    cfg.blockDim = dim3(kPushWarps * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c.stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = static_cast<unsigned>(G);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    TTR_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
    c.launched();
    if (a.trace) {  // TTR_QR_TRACE: per-phase cycles of cluster 0 / CTA 0, averaged over the panel's columns
        long long h[32 * 8 + 8];
        TTR_CUDA(cudaMemcpyAsync(h, a.trace, sizeof(h), cudaMemcpyDeviceToHost, c.stream));
        TTR_CUDA(cudaStreamSynchronize(c.stream));
        const int nc = std::min(a.b, a.rows);
        double acc[8] = {};
        for (int i = 0; i < nc; ++i) {
            const long long* t = h + i * 8;
            const long long seq[8] = {t[0], t[1], t[6], t[7], t[2], t[3], t[4], t[5]};
            for (int q = 1; q < 8; ++q) acc[q] += static_cast<double>(seq[q] - seq[q - 1]) / nc;
            acc[0] += static_cast<double>(t[5] - t[0]) / nc;
        }
        const long long* k = h + 256;
        std::fprintf(stderr,
                     "push<%d> cluster %d x %lld rows %d: cycles/col %.0f | dots %.0f bar %.0f xchg %.0f sum %.0f "
                     "scalar %.0f bar %.0f update %.0f | init+load %lld loop %lld epilogue %lld q %lld exit %lld\n",
                     RPT, G, static_cast<long long>(batch), a.rows, acc[0], acc[1], acc[2], acc[3], acc[4], acc[5],
                     acc[6], acc[7], k[1] - k[0], k[2] - k[1], k[3] - k[2], k[4] - k[3], k[5] - k[4]);
    }
}

// One cluster per matrix: the fewest rows per warp that fit 16 CTAs (more CTAs =
// less arithmetic per column; the push exchange grows with the cluster size).
void launch_panel_push(Ctx& c, PushQrArgs a, i64 batch) {
    static const bool tracing = std::getenv("TTR_QR_TRACE") != nullptr;  // diagnostics only
    static long long* trace_buf = nullptr;
    if (tracing && !trace_buf) TTR_CUDA(cudaMalloc(reinterpret_cast<void**>(&trace_buf), (32 * 8 + 8) * sizeof(long long)));
    a.trace = tracing ? trace_buf : nullptr;
    const i64 rows = a.rows - std::min(a.b, a.rows);  // register rows (the diagonal block sits in CTA 0's smem)
    bool done = false;
    auto go = [&](auto rpt_tag) {
        constexpr int RPT = decltype(rpt_tag)::value;
        const i64 per = static_cast<i64>(kPushWarps) * RPT;
        if (done || rows > kPushMaxCtas * per) return;
        a.rpc = static_cast<int>(per);
        launch_push<RPT>(c, a, static_cast<int>(std::max<i64>(1, (rows + per - 1) / per)), batch);
        done = true;
    };
    go(std::integral_constant<int, 2>{});
    go(std::integral_constant<int, 4>{});
    go(std::integral_constant<int, 8>{});
    go(std::integral_constant<int, 12>{});
    go(std::integral_constant<int, 16>{});
    go(std::integral_constant<int, 20>{});
    go(std::integral_constant<int, 24>{});
    go(std::integral_constant<int, 28>{});
    if (!done) throw Error(TTR_ERR_INTERNAL, "push panel taller than one cluster");
}

// Blocked right-looking Householder QR of a strided batch of m x n matrices
// (m <= kPushMaxRows): panels of 32 columns on one cluster per matrix
// (panel_push_kernel), trailing updates and the explicit thin Q as strided-
// batch DMMA GEMMs. Not charged (the caller charges the reference's 4mnk).
void qr_blocked_push(Ctx& c, i64 batch, i64 m, i64 n, const double* A, i64 lda, i64 sA, double* Q, i64 ldq, i64 sQ,
                     double* R, i64 ldr, i64 sR, double* inplace = nullptr) {
    // inplace: A itself is the (overwritten) work buffer, lda == even_ld(m), sA == lda * n
    const i64 k = std::min(m, n);
    const i64 ldw = even_ld(m), sW = ldw * n;
    DBuf work_buf;
    double* work = inplace;
    if (!inplace) {
        work_buf = DBuf(c, static_cast<std::size_t>(sW * batch));
        work = work_buf.p;
        dim3 grid(static_cast<unsigned>(blocks_for(c, m * n)), static_cast<unsigned>(batch));
        copy_batched_kernel<<<grid, 256, 0, c.stream>>>(static_cast<int>(m), static_cast<int>(n), A, lda, sA, work,
                                                        ldw, sW);
        TTR_CUDA(cudaGetLastError());
        c.launched();
    }
    const i64 npanels = (k + kPanel - 1) / kPanel;
    DBuf tau(c, static_cast<std::size_t>(k * batch));
    const i64 sV = ldw * k, sTs = npanels * kPanel * kPanel, sWb = kPanel * n;
    DBuf Vall(c, static_cast<std::size_t>(sV * batch));
    if (Q) TTR_CUDA(cudaMemsetAsync(Vall.p, 0, sizeof(double) * sV * batch, c.stream));  // zeros above each panel
    DBuf Ts(c, static_cast<std::size_t>(sTs * batch));
    DBuf Wb(c, static_cast<std::size_t>(sWb * batch)), Wb2(c, static_cast<std::size_t>(sWb * batch));
    for (i64 p = 0; p < npanels; ++p) {
        const i64 j0 = p * kPanel, bb = std::min<i64>(kPanel, k - j0), rows = m - j0;
        double* V = Vall.p + j0 + j0 * ldw;
        PushQrArgs a{};
        a.rows = static_cast<int>(rows);
        a.b = static_cast<int>(bb);
        a.Pin = work + j0 + j0 * ldw;
        a.ldin = ldw;
        a.sin = sW;
        a.Pout = work + j0 + j0 * ldw;
        a.ldout = ldw;
        a.sout = sW;
        a.tau = tau.p + j0;
        a.stau = k;
        a.V = V;
        a.ldv = ldw;
        a.sv = sV;
        a.T = Ts.p + p * kPanel * kPanel;
        a.sT = sTs;
        launch_panel_push(c, a, batch);
        const i64 ntrail = n - j0 - bb;
        if (ntrail > 0) {
            double* At = work + j0 + (j0 + bb) * ldw;
            const double* T = Ts.p + p * kPanel * kPanel;
            gemm_batched(c, true, bb, ntrail, rows, 1.0, V, ldw, sV, At, ldw, sW, 0.0, Wb.p, kPanel, sWb, batch,
                         false);                                                                   // V^T A
            gemm_batched(c, true, bb, ntrail, bb, 1.0, T, kPanel, sTs, Wb.p, kPanel, sWb, 0.0, Wb2.p, kPanel, sWb,
                         batch, false);                                                            // T^T (V^T A)
            gemm_batched(c, false, rows, ntrail, bb, -1.0, V, ldw, sV, Wb2.p, kPanel, sWb, 1.0, At, ldw, sW, batch,
                         false);                                                                   // A -= V (.)
        }
    }
    if (R) {
        dim3 grid(static_cast<unsigned>(blocks_for(c, k * n)), static_cast<unsigned>(batch));
        copy_upper<<<grid, 256, 0, c.stream>>>(static_cast<int>(k), static_cast<int>(n), work, ldw, R, ldr, sW, sR);
        TTR_CUDA(cudaGetLastError());
        c.launched();
    }
    if (Q == nullptr) return;
    {
        dim3 grid(static_cast<unsigned>(blocks_for(c, m * k)), static_cast<unsigned>(batch));
        init_thin_identity<<<grid, 256, 0, c.stream>>>(static_cast<int>(m), static_cast<int>(k), Q, ldq, sQ);
        TTR_CUDA(cudaGetLastError());
        c.launched();
    }
    if (k <= 384) {  // Q = [I;0] - V (T V_1^T) with the aggregated T of all panels
        const i64 kk2 = k * k;
        DBuf Gm(c, static_cast<std::size_t>(kk2 * batch)), Tf(c, static_cast<std::size_t>(kk2 * batch)),
            V1t(c, static_cast<std::size_t>(kk2 * batch)), Y(c, static_cast<std::size_t>(kk2 * batch));
        if (batch == 1)
            gemm(c, true, k, k, m, 1.0, Vall.p, ldw, Vall.p, ldw, 0.0, Gm.p, k, false, true);  // upper tiles only
        else
            gemm_batched(c, true, k, k, m, 1.0, Vall.p, ldw, sV, Vall.p, ldw, sV, 0.0, Gm.p, k, kk2, batch, false);
        const std::size_t smem = (static_cast<std::size_t>(npanels) * 32 * 32 + (npanels - 1) * 32 * 33) * sizeof(double);
        static std::atomic<std::uint64_t> configured{0};  // bit d: attributes set on device d
        if (first_on_device(configured)) {
            TTR_CUDA(cudaFuncSetAttribute(t_aggregate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        }
        t_aggregate_kernel<<<dim3(static_cast<unsigned>(npanels), static_cast<unsigned>(batch)), kTaggThreads, smem,
                             c.stream>>>(static_cast<int>(k), Gm.p, Ts.p, Tf.p, kk2, sTs, kk2);
        TTR_CUDA(cudaGetLastError());
        c.launched();
        {
            dim3 grid(static_cast<unsigned>(blocks_for(c, kk2)), static_cast<unsigned>(batch));
            transpose_batched_kernel<<<grid, 256, 0, c.stream>>>(static_cast<int>(k), Vall.p, ldw, sV, V1t.p, k, kk2);
            TTR_CUDA(cudaGetLastError());
            c.launched();
        }
        gemm_batched(c, false, k, k, k, 1.0, Tf.p, k, kk2, V1t.p, k, kk2, 0.0, Y.p, k, kk2, batch, false);  // T V_1^T
        gemm_batched(c, false, m, k, k, -1.0, Vall.p, ldw, sV, Y.p, k, kk2, 1.0, Q, ldq, sQ, batch, false);  // Q -= V Y
        return;
    }
    // very wide: panels applied last to first (backward accumulation)
    const i64 sQw = kPanel * k;
    DBuf Qw(c, static_cast<std::size_t>(sQw * batch)), Qw2(c, static_cast<std::size_t>(sQw * batch));
    for (i64 p = npanels - 1; p >= 0; --p) {
        const i64 j0 = p * kPanel, bb = std::min<i64>(kPanel, k - j0), rows = m - j0, nc = k - j0;
        const double* V = Vall.p + j0 + j0 * ldw;
        const double* T = Ts.p + p * kPanel * kPanel;
        double* Qs = Q + j0 + j0 * ldq;
        gemm_batched(c, true, bb, nc, rows, 1.0, V, ldw, sV, Qs, ldq, sQ, 0.0, Qw.p, kPanel, sQw, batch, false);
        gemm_batched(c, false, bb, nc, bb, 1.0, T, kPanel, sTs, Qw.p, kPanel, sQw, 0.0, Qw2.p, kPanel, sQw, batch,
                     false);
        gemm_batched(c, false, rows, nc, bb, -1.0, V, ldw, sV, Qw2.p, kPanel, sQw, 1.0, Qs, ldq, sQ, batch, false);
    }
}


std::size_t small_smem_bytes(i64 m, i64 n) { return sizeof(double) * static_cast<std::size_t>(m * n + n + 32 + 4); }

}  // namespace

void qr_small_batched(Ctx& c, i64 m, i64 n, const double* A, i64 lda, i64 sA, double* Q, i64 ldq, i64 sQ, double* R,
                      i64 ldr, i64 sR, i64 batch) {
    // <= 32 columns and <= 512 rows: register-resident column owners
    // (qr_batch.cuh); otherwise the whole matrix in one CTA's shared memory
    if (n <= 32 && m <= 512) {
        const int rt_need = static_cast<int>((m + 31) / 32), cn = static_cast<int>((n + 7) / 8);
        // 17..20 columns (config 5a): 5 warps x 4 columns, 3 CTAs per SM, beats
        // 8 warps x 3 columns at 2 CTAs per SM (5a step 16.1 -> 15.7 ms)
        const bool five = n > 16 && n <= 20;
        static const int kRt[] = {1, 2, 4, 6, 8, 10, 12, 16};
        int rt = 16;
        for (int v : kRt)
            if (v >= rt_need) {
                rt = v;
                break;
            }
        const std::size_t smem = sizeof(double) * static_cast<std::size_t>(2 * 32 * rt + 6 + 32);
        bool done = false;
        auto go = [&](auto rt_tag, auto c_tag) {
            constexpr int RT = decltype(rt_tag)::value, CC = decltype(c_tag)::value;
            if (rt != RT || done) return;
            if constexpr ((RT == 8 || RT == 10) && CC == 4) {
                if (five) {
                    qr_small_colreg_kernel<RT, CC, 5><<<static_cast<unsigned>(batch), 160, smem, c.stream>>>(
                        static_cast<int>(m), static_cast<int>(n), A, lda, sA, Q, ldq, sQ, R, ldr, sR);
                    done = true;
                    return;
                }
            }
            if (cn == CC) {
                qr_small_colreg_kernel<RT, CC><<<static_cast<unsigned>(batch), 256, smem, c.stream>>>(
                    static_cast<int>(m), static_cast<int>(n), A, lda, sA, Q, ldq, sQ, R, ldr, sR);
                done = true;
            }
        };
        auto per_c = [&](auto rt_tag) {
            go(rt_tag, std::integral_constant<int, 4>{});
            go(rt_tag, std::integral_constant<int, 3>{});
            go(rt_tag, std::integral_constant<int, 2>{});
            go(rt_tag, std::integral_constant<int, 1>{});
        };
        per_c(std::integral_constant<int, 1>{});
        per_c(std::integral_constant<int, 2>{});
        per_c(std::integral_constant<int, 4>{});
        per_c(std::integral_constant<int, 6>{});
        per_c(std::integral_constant<int, 8>{});
        per_c(std::integral_constant<int, 10>{});
        per_c(std::integral_constant<int, 12>{});
        per_c(std::integral_constant<int, 16>{});
        if (!done) throw Error(TTR_ERR_INTERNAL, "qr_small_colreg dispatch");
        TTR_CUDA(cudaGetLastError());
        c.launched();
        return;
    }
    const std::size_t smem = small_smem_bytes(m, n);
    static std::atomic<std::uint64_t> configured{0};  // bit d: attributes set on device d
    if (first_on_device(configured)) {
        TTR_CUDA(cudaFuncSetAttribute(qr_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    }
    qr_small_kernel<<<static_cast<unsigned>(batch), kQrThreads, smem, c.stream>>>(
        static_cast<int>(m), static_cast<int>(n), A, lda, sA, Q, ldq, sQ, R, ldr, sR);
    TTR_CUDA(cudaGetLastError());
    c.launched();
}

namespace {
i64 kCqrSingleMaxRows(Ctx& c) { return 320LL * c.sm_count; }  // K4f: <= 320 rows per CTA, one CTA per SM
bool cqr_checked_on() {  // experiments: TTR_QR_CHECKED=0 = non-speculating callers keep the Householder panels
    static const bool on = [] {
        const char* e = std::getenv("TTR_QR_CHECKED");
        return !(e && e[0] == '0');
    }();
    return on;
}
}  // namespace

void thin_qr(Ctx& c, i64 m, i64 n, const double* A, i64 lda, double* Q, i64 ldq, double* R, i64 ldr) {
    const i64 k = std::min(m, n);
    c.charge_qr(4ULL * static_cast<std::uint64_t>(m) * n * k);
    if (m <= 0 || n <= 0) return;
    // A panel lives in registers of at most one CTA per SM (launch_panel_col:
    // up to 8 warps x 64 rows per SM). Taller matrices take a TSQR split: QR of
    // each row block, QR of the stacked R factors, and — when Q is requested —
    // Q(block q) = Q_q Q_s(q-th block) by one GEMM per block. Charged once, as
    // one QR of the whole matrix (linalg.cpp:48).
    const i64 max_rows = 8LL * 64 * c.sm_count;
    if (m > max_rows) {
        const Counts saved = c.counts;
        const i64 chunk = std::max<i64>(k, max_rows / 2);
        const i64 nchunks = (m + chunk - 1) / chunk;
        const i64 lds = nchunks * k;
        DBuf stack(c, static_cast<std::size_t>(lds * n));
        TTR_CUDA(cudaMemsetAsync(stack.p, 0, sizeof(double) * lds * n, c.stream));
        std::vector<DBuf> Qq(static_cast<std::size_t>(Q ? nchunks : 0));
        for (i64 q = 0; q < nchunks; ++q) {
            const i64 r0 = q * chunk, rows = std::min(chunk, m - r0), kq = std::min(rows, n);
            DBuf Rq(c, static_cast<std::size_t>(kq * n));
            if (Q) Qq[q] = DBuf(c, static_cast<std::size_t>(rows * kq));
            thin_qr(c, rows, n, A + r0, lda, Q ? Qq[q].p : nullptr, rows, Rq.p, kq);
            TTR_CUDA(cudaMemcpy2DAsync(stack.p + q * k, sizeof(double) * lds, Rq.p, sizeof(double) * kq,
                                       sizeof(double) * kq, n, cudaMemcpyDeviceToDevice, c.stream));
        }
        if (!Q) {
            thin_qr(c, lds, n, stack.p, lds, nullptr, 1, R, ldr);
        } else {
            DBuf Qs(c, static_cast<std::size_t>(lds * k));
            thin_qr(c, lds, n, stack.p, lds, Qs.p, lds, R, ldr);
            for (i64 q = 0; q < nchunks; ++q) {
                const i64 r0 = q * chunk, rows = std::min(chunk, m - r0), kq = std::min(rows, n);
                gemm(c, false, rows, k, kq, 1.0, Qq[q].p, rows, Qs.p + q * k, lds, 0.0, Q + r0, ldq, false);
            }
        }
        c.counts = saved;
        return;
    }
    // Launch the column-per-lane panel kernel on a rows x b panel (b <= 32):
    // one cluster of <= 16 CTAs (16 warps each) when the rows fit, else a
    // cooperative grid of <= one CTA (8 warps) per SM. Returns true for the
    // cluster mode.
    unsigned long long* xchg = c.qr_exchange();
    auto launch_panel = [&](RegQrArgs a) {
        a.xchg = xchg;
        return launch_panel_col(c, a);
    };

    // ---- small (<= 512 x 32): one CTA, register column owners (qr_batch.cuh):
    //      no cross-CTA exchange per column ----
    static const bool small_on = [] {
        const char* e = std::getenv("TTR_QR_SMALL_CTA");  // experiments: 0 = cluster panel
        return !(e && e[0] == '0');
    }();
    if (small_on && n <= kPanel && m <= 512 && m >= n) {
        qr_small_batched(c, m, n, A, lda, 0, Q, ldq, 0, R, ldr, 0, 1);
        return;
    }
    static const bool old_panels = [] {  // experiments: TTR_QR_OLD=1 = cooperative-grid / old cluster panels
        const char* e = std::getenv("TTR_QR_OLD");
        return e && e[0] == '1';
    }();
    // Measured (tools/qr_bench.py, TTR_QR_OLD=1 for the other path): the push
    // cluster panels win for blocked QRs up to one cluster of rows (7040 x 110:
    // 0.566 -> 0.466 ms, 5120 x 320: 1.60 -> 1.28, 2560 x 320: 1.51 -> 1.10);
    // single panels (<= 32 columns) keep the in-register-Q panels below, and
    // taller matrices the cooperative-grid panel (40960 x 320: 2.72 ms vs 3.8
    // for the chunked TSQR below, kept behind TTR_QR_TSQR=1 for experiments).
    // The push panel's per-column floor (~4,200 cycles at 7,040 rows) is the
    // shared-memory broadcast of the active column (two LDS.128 wavefronts per
    // two rows per phase, ~440 rows per SM) plus the serial reflector step.
    static const bool tsqr_on = [] {
        const char* e = std::getenv("TTR_QR_TSQR");
        return e && e[0] == '1';
    }();
    // Cholesky-QR panels with Householder reconstruction (qr_chol.cu: K4f, one
    // cooperative kernel per panel; K4d, separate launches) when the caller
    // speculates (c.qr_tag >= 0: a breakdown reruns the call on the Householder
    // panels). Default since K4f (40,960 x 320: 2.69 -> 1.89 ms, 7,040 x 110: 0.465 ->
    // 0.366 ms); TTR_QR_CQR=0 keeps the Householder panels.
    static const bool cqr_on = [] {
        const char* e = std::getenv("TTR_QR_CQR");
        return !(e && e[0] == '0');
    }();
    // (rows beyond the fused kernel's one-CTA-per-SM capacity keep the Householder
    // panels: K4d's separate launches are slower than those)
    const bool cqr_shape = m >= 8 * kPanel && m <= kCqrSingleMaxRows(c) && (n > kPanel || m >= 8 * n);
    bool cqr = cqr_on && c.qr_tag >= 0 && cqr_shape;
    // Callers that do not speculate themselves (TT-SVD orthogonalisations, the
    // adaptive growth blocks, the C-ABI thin_qr): the same kernels in a checked
    // call — factor under a private tag, read the breakdown flag (one stream
    // synchronisation per QR) and redo the QR on the Householder panels if a
    // panel broke down. Under a recorded plan (Ctx::QrTape) the recording run
    // notes each outcome and the captured replay follows it without a
    // synchronisation, a breakdown there raising the plan's mismatch flag.
    // Never under an outer speculation (the flag is the caller's).
    if (!cqr && cqr_on && c.qr_tag < 0 && !c.qr_spec && cqr_shape && A != Q && cqr_checked_on()) {
        cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
        TTR_CUDA(cudaStreamIsCapturing(c.stream, &cap));
        Ctx::QrTape* tp = c.qr_tape;
        const Counts saved = c.counts;  // charged once, above
        auto inner = [&](int* override_flag) {
            c.qr_tag = 0;
            c.qr_flag_override = override_flag;
            try {
                thin_qr(c, m, n, A, lda, Q, ldq, R, ldr);
            } catch (...) {
                c.qr_tag = -1;
                c.qr_flag_override = nullptr;
                throw;
            }
            c.qr_tag = -1;
            c.qr_flag_override = nullptr;
            c.counts = saved;
        };
        if (tp && tp->replay) {
            if (tp->pos >= tp->took_hh.size()) fail(Errc::InvalidArgument, "plan: QR decision tape exhausted");
            if (!tp->took_hh[tp->pos++]) {
                inner(tp->flag);
                return;
            }
        } else if (cap == cudaStreamCaptureStatusNone) {
            c.qr_flag_reset();
            inner(nullptr);
            const bool broke = c.qr_flag_read() >= 0;
            if (tp) tp->took_hh.push_back(broke ? 1 : 0);
            if (!broke) return;
        }
    }
    if (!old_panels && m <= kPushMaxRows && n > kPanel && !cqr) {
        qr_blocked_push(c, 1, m, n, A, lda, 0, Q, ldq, 0, R, ldr, 0);
        return;
    }
    if (!old_panels && tsqr_on && n <= kPushMaxRows && m > kPushMaxRows) {
        // Taller: TSQR over B cluster-sized row chunks, all factored at once
        // (one cluster per chunk, strided-batch GEMMs), then the QR of the
        // stacked R factors and Q(chunk q) = Q_q Q_s(q-th block). The chunks are
        // padded with zero rows to one height (zero rows leave R unchanged and
        // get zero rows of Q, never copied out). Charged once, as one QR.
        const Counts saved = c.counts;
        const i64 B = (m + kPushMaxRows - 1) / kPushMaxRows;
        const i64 chunk = even_ld((m + B - 1) / B), kq = std::min(chunk, n), sC = chunk * n;
        DBuf Ap(c, static_cast<std::size_t>(sC * B));
        if (chunk * B != m) TTR_CUDA(cudaMemsetAsync(Ap.p, 0, sizeof(double) * sC * B, c.stream));
        for (i64 q = 0; q < B; ++q) {
            const i64 rq = std::min(chunk, m - q * chunk);
            TTR_CUDA(cudaMemcpy2DAsync(Ap.p + q * sC, sizeof(double) * chunk, A + q * chunk, sizeof(double) * lda,
                                       sizeof(double) * rq, n, cudaMemcpyDeviceToDevice, c.stream));
        }
        const i64 ls = B * kq;
        DBuf Rst(c, static_cast<std::size_t>(ls * n));
        DBuf Qc(c, static_cast<std::size_t>(Q ? chunk * kq * B : 1));
        // the chunk QRs are independent: one side stream each (their panels run
        // as concurrent clusters, their GEMMs share the GPU), each with its own
        // split-K scratch; joined before the stacked QR
        {
            const int ns = static_cast<int>(std::min<i64>(B, 8));
            c.fork_side(ns);
            const cudaStream_t main = c.stream;
            double* const main_work = c.work;
            const std::size_t main_bytes = c.work_bytes;
            std::vector<double*> works;
            for (i64 q = 0; q < B; ++q) {
                c.stream = c.side[q % ns];
                c.work = nullptr;
                c.work_bytes = 0;
                qr_blocked_push(c, 1, chunk, n, Ap.p + q * sC, chunk, sC, Q ? Qc.p + q * chunk * kq : nullptr, chunk,
                                chunk * kq, Rst.p + q * kq, ls, kq, Ap.p + q * sC);
                if (c.work) works.push_back(c.work);
            }
            c.stream = main;
            c.work = main_work;
            c.work_bytes = main_bytes;
            c.join_side(ns);
            for (double* w : works) TTR_CUDA(cudaFreeAsync(w, c.stream));
        }
        if (!Q) {
            thin_qr(c, ls, n, Rst.p, ls, nullptr, 1, R, ldr);
        } else {
            DBuf Qs(c, static_cast<std::size_t>(ls * k));
            thin_qr(c, ls, n, Rst.p, ls, Qs.p, ls, R, ldr);
            if (B > 1)
                gemm_batched(c, false, chunk, k, kq, 1.0, Qc.p, chunk, chunk * kq, Qs.p, ls, kq, 0.0, Q, ldq, chunk,
                             B - 1, false);
            const i64 last = m - (B - 1) * chunk;
            gemm(c, false, last, k, kq, 1.0, Qc.p + (B - 1) * chunk * kq, chunk, Qs.p + (B - 1) * kq, ls, 0.0,
                 Q + (B - 1) * chunk, ldq, false);
        }
        c.counts = saved;
        return;
    }
    // ---- <= 32 columns: the fused Cholesky-QR kernel as a plain thin QR when the
    // caller speculates (K4f, hr = 0), else one Householder panel launch ----
    if (n <= kPanel && cqr && cqr_single(c, m, n, A, lda, Q, ldq, R, ldr, nullptr, c.qr_tag)) {
        c.qr_spec_used = true;
        return;
    }
    if (n <= kPanel) {
        DBuf tau(c, static_cast<std::size_t>(k));
        RegQrArgs a{};
        a.rows = static_cast<int>(m);
        a.b = static_cast<int>(n);
        a.Pin = A;
        a.ldin = lda;
        a.tau = tau.p;
        a.R = R;
        a.ldr = ldr;
        // Q in registers costs one more cross-CTA exchange per column; on the
        // cooperative grid (> 2048 rows, ~3 us per exchange) Q = [I;0] - V (T V_1^T)
        // from the panel's V and T is cheaper (the adaptive paths' growth QRs)
        const bool wy = Q != nullptr && m > 2048 && n >= 6;
        if (!wy) {
            a.Q = Q;
            a.ldq = ldq;
            launch_panel(a);
            return;
        }
        const i64 ldv = even_ld(m);
        DBuf Vb(c, static_cast<std::size_t>(ldv * n)), Tb(c, static_cast<std::size_t>(kPanel * kPanel)),
            V1t(c, static_cast<std::size_t>(k * k)), Y(c, static_cast<std::size_t>(k * k));
        a.V = Vb.p;
        a.ldv = ldv;
        a.T = Tb.p;
        launch_panel(a);
        transpose(c, k, k, Vb.p, ldv, V1t.p, k);                                       // V_1^T
        gemm(c, false, k, k, k, 1.0, Tb.p, kPanel, V1t.p, k, 0.0, Y.p, k, false);      // Y = T V_1^T
        init_thin_identity<<<blocks_for(c, m * k), 256, 0, c.stream>>>(static_cast<int>(m), static_cast<int>(k), Q, ldq);
        TTR_CUDA(cudaGetLastError());
        c.launched();
        gemm(c, false, m, k, k, -1.0, Vb.p, ldv, Y.p, k, 1.0, Q, ldq, false);           // Q = [I;0] - V Y
        return;
    }

    // ---- blocked right-looking Householder ----
    // kf: columns that get reflectors (all, unless the caller bounds the rank and wants Q only)
    i64 kf = k;
    if (c.qr_rank_hint > 0 && R == nullptr && Q != nullptr && k <= 384) {
        const i64 h = (c.qr_rank_hint + kPanel - 1) / kPanel * kPanel;
        if (h < k) kf = h;
    }
    const i64 ldw = even_ld(m);
    DBuf work(c, static_cast<std::size_t>(ldw * n));
    copy_matrix(c, m, n, A, lda, work.p, ldw);
    const i64 npanels = (k + kPanel - 1) / kPanel;
    DBuf tau(c, static_cast<std::size_t>(k));
    DBuf Vall(c, static_cast<std::size_t>(ldw * k));  // explicit V of every panel (rows j0.. of column block)
    if (Q) TTR_CUDA(cudaMemsetAsync(Vall.p, 0, sizeof(double) * ldw * k, c.stream));  // zeros above each panel
    DBuf Ts(c, static_cast<std::size_t>(npanels * kPanel * kPanel));
    DBuf Wb(c, static_cast<std::size_t>(kPanel * std::max<i64>(n, 1)));
    DBuf Wb2(c, static_cast<std::size_t>(kPanel * std::max<i64>(n, 1)));

    const i64 npf = (kf + kPanel - 1) / kPanel, nf = kf < k ? kf : n;  // panels factored, columns kept up to date
    for (i64 p = 0; p < npf; ++p) {
        const i64 j0 = p * kPanel, bb = std::min<i64>(kPanel, kf - j0), rows = m - j0;
        double* V = Vall.p + j0 + j0 * ldw;  // rows x bb block at (j0, j0), ld ldw
        double* T = Ts.p + p * kPanel * kPanel;
        if (cqr && rows >= 4 * kPanel) {
            cqr_panel(c, rows, bb, work.p + j0 + j0 * ldw, ldw, V, ldw, T, tau.p + j0, c.qr_tag);
            c.qr_spec_used = true;
            const i64 ntrail = nf - j0 - bb;
            if (ntrail > 0) {
                double* At = work.p + j0 + (j0 + bb) * ldw;
                gemm_tn_lt(c, bb, ntrail, rows, V, ldw, At, ldw, T, kPanel, Wb2.p, kPanel, Wb.p, false);  // T^T (V^T A)
                gemm(c, false, rows, ntrail, bb, -1.0, V, ldw, Wb2.p, kPanel, 1.0, At, ldw, false);  // A -= V (.)
            }
            continue;
        }
        RegQrArgs a{};
        a.rows = static_cast<int>(rows);
        a.b = static_cast<int>(bb);
        a.Pin = work.p + j0 + j0 * ldw;
        a.ldin = ldw;
        a.Pout = work.p + j0 + j0 * ldw;
        a.ldout = ldw;
        a.tau = tau.p + j0;
        a.V = V;
        a.ldv = ldw;
        a.T = T;
        launch_panel(a);
        const i64 ntrail = nf - j0 - bb;
        if (ntrail > 0) {
            double* At = work.p + j0 + (j0 + bb) * ldw;
            gemm_tn_lt(c, bb, ntrail, rows, V, ldw, At, ldw, T, kPanel, Wb2.p, kPanel, Wb.p, false);  // T^T (V^T A)
            gemm(c, false, rows, ntrail, bb, -1.0, V, ldw, Wb2.p, kPanel, 1.0, At, ldw, false);  // A -= V (.)
        }
    }
    if (R) {
        copy_upper<<<blocks_for(c, k * n), 256, 0, c.stream>>>(static_cast<int>(k), static_cast<int>(n), work.p, ldw, R, ldr);
        TTR_CUDA(cudaGetLastError());
        c.launched();
    }
    if (Q == nullptr) return;
    // explicit Q = H_0 ... H_{k-1} [I_k; 0] = [I_k; 0] - V T V_1^T with the
    // aggregated T of all panels (V_1 = top k x k block of V): two full-size
    // GEMMs (V^T V and V Y) instead of three skinny ones per panel
    if (k <= 384) {
        // kq = kf columns of V carry reflectors (the rest of Q is the reflected unit vectors)
        const i64 kq = kf;
        DBuf Gm(c, static_cast<std::size_t>(kq * kq));
        DBuf Tf(c, static_cast<std::size_t>(kq * kq));
        DBuf V1t(c, static_cast<std::size_t>(kq * k));
        DBuf Y(c, static_cast<std::size_t>(kq * k));
        // G = V^T V; t_aggregate_kernel reads only its strictly upper 32-blocks
        gemm(c, true, kq, kq, m, 1.0, Vall.p, ldw, Vall.p, ldw, 0.0, Gm.p, kq, false, true);
        const std::size_t smem = (static_cast<std::size_t>(npf) * 32 * 32 + (npf - 1) * 32 * 33) * sizeof(double);
        static std::atomic<std::uint64_t> configured{0};  // bit d: attributes set on device d
        if (first_on_device(configured)) {
            TTR_CUDA(cudaFuncSetAttribute(t_aggregate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        }
        t_aggregate_kernel<<<static_cast<unsigned>(npf), kTaggThreads, smem, c.stream>>>(static_cast<int>(kq), Gm.p, Ts.p,
                                                                                         Tf.p);
        TTR_CUDA(cudaGetLastError());
        c.launched();
        transpose(c, k, kq, Vall.p, ldw, V1t.p, kq);                                      // V_1^T (kq x k)
        gemm(c, false, kq, k, kq, 1.0, Tf.p, kq, V1t.p, kq, 0.0, Y.p, kq, false);         // Y = T V_1^T
        // Q = [I;0] - V Y: the product alone (no pass over Q to preset the identity and to
        // read it back), then + 1 on the diagonal (-(V Y) + 1 rounds as the fused form does)
        gemm(c, false, m, k, kq, -1.0, Vall.p, ldw, Y.p, kq, 0.0, Q, ldq, false);
        add_unit_diagonal<<<static_cast<unsigned>((k + 255) / 256), 256, 0, c.stream>>>(static_cast<int>(k), Q, ldq);
        TTR_CUDA(cudaGetLastError());
        c.launched();
        return;
    }
    // very wide: panels applied last to first (backward accumulation)
    init_thin_identity<<<blocks_for(c, m * k), 256, 0, c.stream>>>(static_cast<int>(m), static_cast<int>(k), Q, ldq);
    TTR_CUDA(cudaGetLastError());
    c.launched();
    for (i64 p = npanels - 1; p >= 0; --p) {
        const i64 j0 = p * kPanel, bb = std::min<i64>(kPanel, k - j0), rows = m - j0, nc = k - j0;
        const double* V = Vall.p + j0 + j0 * ldw;
        const double* T = Ts.p + p * kPanel * kPanel;
        double* Qs = Q + j0 + j0 * ldq;
        gemm(c, true, bb, nc, rows, 1.0, V, ldw, Qs, ldq, 0.0, Wb.p, kPanel, false);          // V^T Q
        gemm(c, false, bb, nc, bb, 1.0, T, kPanel, Wb.p, kPanel, 0.0, Wb2.p, kPanel, false);  // T (V^T Q)
        gemm(c, false, rows, nc, bb, -1.0, V, ldw, Wb2.p, kPanel, 1.0, Qs, ldq, false);      // Q -= V (.)
    }
}

}  // namespace ttr
