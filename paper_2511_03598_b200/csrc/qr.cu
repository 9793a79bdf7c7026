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
//    strided set of matrices (one CTA each), which covers the 5a batch and
//    every mode of the small configs.
//  * blocked right-looking Householder for tall matrices: panels of width
//    kPanel factored by ONE cooperative kernel (each CTA keeps its row block
//    of the panel in shared memory, one grid-wide barrier per column, partial
//    dot products reduced in fixed CTA order -> deterministic), then the
//    compact-WY trailing update and the explicit-Q backward accumulation run
//    on the DMMA GEMM (gemm_dmma.cu).
#include <cooperative_groups.h>

#include <algorithm>
#include <cfloat>
#include <cmath>

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
// cooperative panel factorization of P (rows x b, ld), b <= kPanel
struct PanelArgs {
    int rows, b, rpc;  // rows per CTA
    double* P;
    i64 ld;
    double* tau;
    double* partials;  // [2][grid][kPanel]
    double* diag;      // [2][kPanel]
};

// Layout: the CTA's row block lives in shared memory column-major with an
// odd leading dimension (conflict-free 64-bit accesses); lane l of every
// warp owns column l for the partial dot products, warps split the rows.
__global__ void __launch_bounds__(kQrThreads) panel_kernel(PanelArgs p) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ double sm[];
    const int rpc = p.rpc, b = p.b, ldx = rpc | 1;
    double* x = sm;                                  // [b][ldx]
    double* wred = x + static_cast<i64>(ldx) * b;    // [8][32] warp partials
    double* red = wred + 8 * 32;                     // kPanel sums
    double* sc = red + kPanel;                       // scalars
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    const int r0 = blockIdx.x * rpc, r1 = min(p.rows, r0 + rpc), nr = max(0, r1 - r0);
    const int G = gridDim.x;
    const int rpw = (nr + nw - 1) / nw;  // rows per warp

    for (int idx = tid; idx < nr * b; idx += blockDim.x) {
        const int rr = idx % nr, l = idx / nr;
        x[rr + l * ldx] = p.P[(r0 + rr) + l * p.ld];
    }
    __syncthreads();

    const int kk = min(b, p.rows);
    for (int i = 0; i < kk; ++i) {
        const int buf = i & 1;
        double* part = p.partials + static_cast<i64>(buf) * G * kPanel;
        double* dg = p.diag + buf * kPanel;
        // (a) partial dot products x(:,i) . x(:,l) over my rows strictly below row i
        {
            const int lo = max(0, i + 1 - r0);
            const int ra = max(lo, warp * rpw), rb = min(nr, (warp + 1) * rpw);
            double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;  // 4 chains for ILP
            if (lane >= i && lane < b) {
                const double* xi = x + i * ldx;
                const double* xl = x + lane * ldx;
                int rr = ra;
                for (; rr + 3 < rb; rr += 4) {
                    s0 = fma(xi[rr], xl[rr], s0);
                    s1 = fma(xi[rr + 1], xl[rr + 1], s1);
                    s2 = fma(xi[rr + 2], xl[rr + 2], s2);
                    s3 = fma(xi[rr + 3], xl[rr + 3], s3);
                }
                for (; rr < rb; ++rr) s0 = fma(xi[rr], xl[rr], s0);
            }
            wred[warp * 32 + lane] = (s0 + s1) + (s2 + s3);
        }
        __syncthreads();
        if (tid < 32) {
            double s = 0.0;
            for (int w = 0; w < nw; ++w) s += wred[w * 32 + tid];
            part[blockIdx.x * kPanel + tid] = s;
            if (i >= r0 && i < r1 && tid >= i && tid < b) dg[tid] = x[(i - r0) + tid * ldx];
        }
        grid.sync();
        // (d) reduce partials in fixed order: 8 CTA groups x 32 columns, then groups in order
        {
            // all loads issued before any add: one L2 round trip (G <= 8 * kMaxLoads)
            constexpr int kMaxLoads = 20;
            const int grp = tid >> 5;
            double v[kMaxLoads];
#pragma unroll
            for (int q = 0; q < kMaxLoads; ++q) {
                const int c = grp + 8 * q;
                v[q] = (c < G) ? __ldcg(part + c * kPanel + lane) : 0.0;
            }
            double s = 0.0;
#pragma unroll
            for (int q = 0; q < kMaxLoads; ++q) s += v[q];
            wred[grp * 32 + lane] = s;
        }
        __syncthreads();
        if (tid < 32) {
            double s = 0.0;
            for (int g = 0; g < 8; ++g) s += wred[g * 32 + tid];
            red[tid] = s;
            sc[40 + tid] = __ldcg(dg + tid);
        }
        __syncthreads();
        const double alpha = sc[40 + i], tail = red[i];
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
        // w_l = tau * (A(i,l) + s_l/(alpha-beta)) for l > i
        if (tid < kPanel) {
            const int l = tid;
            sc[1 + l] = (l > i && l < b) ? tj * (sc[40 + l] + red[l] * inv) : 0.0;
        }
        __syncthreads();
        for (int idx = tid; idx < nr; idx += blockDim.x) {
            const int gr = r0 + idx;
            if (gr > i) {
                const double v = x[idx + i * ldx] * inv;
                x[idx + i * ldx] = v;
                for (int l = i + 1; l < b; ++l) x[idx + l * ldx] = fma(-sc[1 + l], v, x[idx + l * ldx]);
            } else if (gr == i) {
                x[idx + i * ldx] = beta;
                for (int l = i + 1; l < b; ++l) x[idx + l * ldx] -= sc[1 + l];
            }
        }
        if (blockIdx.x == 0 && tid == 0) p.tau[i] = tj;
        __syncthreads();
    }
    for (int idx = tid; idx < nr * b; idx += blockDim.x) {
        const int rr = idx % nr, l = idx / nr;
        p.P[(r0 + rr) + l * p.ld] = x[rr + l * ldx];
    }
}

// V (rows x b): unit lower trapezoid from the factored panel P.
__global__ void extract_v(int rows, int b, const double* P, i64 ldp, double* V, i64 ldv) {
    const i64 total = static_cast<i64>(rows) * b;
    for (i64 idx = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<i64>(gridDim.x) * blockDim.x) {
        const int r = static_cast<int>(idx % rows), c = static_cast<int>(idx / rows);
        V[r + c * ldv] = r > c ? P[r + c * ldp] : (r == c ? 1.0 : 0.0);
    }
}

// T (b x b upper) of the compact WY form H_0..H_{b-1} = I - V T V^T, from
// G = V^T V: T(i,i) = tau_i, T(0:i,i) = -tau_i T(0:i,0:i) G(0:i,i).
__global__ void build_t(int b, const double* G, i64 ldg, const double* tau, double* T, i64 ldt) {
    __shared__ double t[kPanel * kPanel];
    __shared__ double g[kPanel * kPanel];
    __shared__ double ts[kPanel];
    __shared__ double z[kPanel];
    const int tid = threadIdx.x;
    for (int idx = tid; idx < kPanel * kPanel; idx += blockDim.x) {
        t[idx] = 0.0;
        const int r = idx % kPanel, cc = idx / kPanel;
        g[idx] = (r < b && cc < b) ? G[r + cc * ldg] : 0.0;
    }
    if (tid < kPanel) ts[tid] = tid < b ? tau[tid] : 0.0;
    __syncthreads();
    for (int i = 0; i < b; ++i) {
        const double ti = ts[i];
        if (tid < i) {
            double s = 0.0;
            for (int q = tid; q < i; ++q) s = fma(t[tid + q * kPanel], g[q + i * kPanel], s);
            z[tid] = -ti * s;
        }
        __syncthreads();
        if (tid < i) t[tid + i * kPanel] = z[tid];
        if (tid == 0) t[i + i * kPanel] = ti;
        __syncthreads();
    }
    for (int idx = tid; idx < b * b; idx += blockDim.x) {
        const int r = idx % b, c = idx / b;
        T[r + c * ldt] = t[r + c * kPanel];
    }
}

__global__ void init_thin_identity(int m, int k, double* Q, i64 ldq) {
    const i64 total = static_cast<i64>(m) * k;
    for (i64 idx = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<i64>(gridDim.x) * blockDim.x) {
        const int r = static_cast<int>(idx % m), c = static_cast<int>(idx / m);
        Q[r + c * ldq] = (r == c) ? 1.0 : 0.0;
    }
}

__global__ void copy_upper(int k, int n, const double* A, i64 lda, double* R, i64 ldr) {
    const i64 total = static_cast<i64>(k) * n;
    for (i64 idx = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<i64>(gridDim.x) * blockDim.x) {
        const int r = static_cast<int>(idx % k), c = static_cast<int>(idx / k);
        R[r + c * ldr] = (r <= c) ? A[r + c * lda] : 0.0;
    }
}

int blocks_for(Ctx& c, i64 work) {
    return static_cast<int>(std::max<i64>(1, std::min<i64>((work + 255) / 256, 4LL * c.sm_count)));
}

constexpr i64 kSmallMaxElems = 26000;  // ~203 KB of shared memory

std::size_t small_smem_bytes(i64 m, i64 n) { return sizeof(double) * static_cast<std::size_t>(m * n + n + 32 + 4); }

}  // namespace

void qr_small_batched(Ctx& c, i64 m, i64 n, const double* A, i64 lda, i64 sA, double* Q, i64 ldq, i64 sQ, double* R,
                      i64 ldr, i64 sR, i64 batch) {
    const std::size_t smem = small_smem_bytes(m, n);
    static bool configured = false;
    if (!configured) {
        TTR_CUDA(cudaFuncSetAttribute(qr_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        configured = true;
    }
    qr_small_kernel<<<static_cast<unsigned>(batch), kQrThreads, smem, c.stream>>>(
        static_cast<int>(m), static_cast<int>(n), A, lda, sA, Q, ldq, sQ, R, ldr, sR);
    TTR_CUDA(cudaGetLastError());
    c.launched();
}

void thin_qr(Ctx& c, i64 m, i64 n, const double* A, i64 lda, double* Q, i64 ldq, double* R, i64 ldr) {
    const i64 k = std::min(m, n);
    c.charge_qr(4ULL * static_cast<std::uint64_t>(m) * n * k);
    if (m <= 0 || n <= 0) return;
    if (m * n <= kSmallMaxElems) {
        qr_small_batched(c, m, n, A, lda, 0, Q, ldq, 0, R, ldr, 0, 1);
        return;
    }
    // ---- blocked Householder ----
    const i64 ldw = even_ld(m);
    DBuf work(c, static_cast<std::size_t>(ldw * n));
    copy_matrix(c, m, n, A, lda, work.p, ldw);
    const i64 npanels = (k + kPanel - 1) / kPanel;
    DBuf tau(c, static_cast<std::size_t>(k));
    DBuf Vall(c, static_cast<std::size_t>(ldw * k));  // explicit V of every panel (rows j0.. of column block)
    DBuf Ts(c, static_cast<std::size_t>(npanels * kPanel * kPanel));
    DBuf G(c, kPanel * kPanel);
    DBuf Wb(c, static_cast<std::size_t>(kPanel * std::max<i64>(n, 1)));
    DBuf Wb2(c, static_cast<std::size_t>(kPanel * std::max<i64>(n, 1)));

    // cooperative panel launch geometry
    int max_blocks_per_sm = 0;
    static bool configured = false;
    if (!configured) {
        TTR_CUDA(cudaFuncSetAttribute(panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        configured = true;
    }
    DBuf partials(c, static_cast<std::size_t>(2 * 4 * c.sm_count * kPanel));
    DBuf diag(c, 2 * kPanel);

    for (i64 p = 0; p < npanels; ++p) {
        const i64 j0 = p * kPanel, bb = std::min<i64>(kPanel, k - j0), rows = m - j0;
        // one CTA per SM at most (grid barrier cost grows with the CTA count),
        // at least 64 rows per CTA; the row block must fit in shared memory
        auto smem_for = [&](i64 rpc_) {
            return sizeof(double) * static_cast<std::size_t>((rpc_ | 1) * bb + 8 * 32 + kPanel + 80);
        };
        i64 grid = std::max<i64>(1, std::min<i64>((rows + 63) / 64, c.sm_count));
        i64 rpc = (rows + grid - 1) / grid;
        std::size_t smem = smem_for(rpc);
        TTR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&max_blocks_per_sm, panel_kernel, kQrThreads, smem));
        const i64 max_grid = static_cast<i64>(max_blocks_per_sm) * c.sm_count;
        if (smem > 220 * 1024 || grid > max_grid) throw Error(TTR_ERR_INTERNAL, "qr panel does not fit the GPU");
        grid = (rows + rpc - 1) / rpc;
        if (grid > 4LL * c.sm_count) throw Error(TTR_ERR_INTERNAL, "qr panel grid too large");
        PanelArgs pa{};
        pa.rows = static_cast<int>(rows);
        pa.b = static_cast<int>(bb);
        pa.rpc = static_cast<int>(rpc);
        pa.P = work.p + j0 + j0 * ldw;
        pa.ld = ldw;
        pa.tau = tau.p + j0;
        pa.partials = partials.p;
        pa.diag = diag.p;
        void* args[] = {&pa};
        TTR_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(panel_kernel), dim3(static_cast<unsigned>(grid)),
                                             dim3(kQrThreads), args, smem, c.stream));
        c.launched();
        double* V = Vall.p + j0 + j0 * ldw;  // rows x bb block at (j0, j0), ld ldw
        extract_v<<<blocks_for(c, rows * bb), 256, 0, c.stream>>>(static_cast<int>(rows), static_cast<int>(bb),
                                                                   work.p + j0 + j0 * ldw, ldw, V, ldw);
        TTR_CUDA(cudaGetLastError());
        c.launched();
        double* T = Ts.p + p * kPanel * kPanel;
        gemm(c, true, bb, bb, rows, 1.0, V, ldw, V, ldw, 0.0, G.p, kPanel, false);
        build_t<<<1, 64, 0, c.stream>>>(static_cast<int>(bb), G.p, kPanel, tau.p + j0, T, kPanel);
        TTR_CUDA(cudaGetLastError());
        c.launched();
        const i64 ntrail = n - j0 - bb;
        if (ntrail > 0) {
            double* At = work.p + j0 + (j0 + bb) * ldw;
            gemm(c, true, bb, ntrail, rows, 1.0, V, ldw, At, ldw, 0.0, Wb.p, kPanel, false);    // V^T A
            gemm(c, true, bb, ntrail, bb, 1.0, T, kPanel, Wb.p, kPanel, 0.0, Wb2.p, kPanel, false);  // T^T (V^T A)
            gemm(c, false, rows, ntrail, bb, -1.0, V, ldw, Wb2.p, kPanel, 1.0, At, ldw, false);  // A -= V (.)
        }
    }
    if (R) {
        copy_upper<<<blocks_for(c, k * n), 256, 0, c.stream>>>(static_cast<int>(k), static_cast<int>(n), work.p, ldw, R, ldr);
        TTR_CUDA(cudaGetLastError());
        c.launched();
    }
    if (Q == nullptr) return;
    // explicit Q = H_0 ... H_{k-1} [I_k; 0], panels applied last to first
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
