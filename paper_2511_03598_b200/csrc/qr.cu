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
// Register-resident Householder panel (b <= 32 columns). Every thread keeps
// R rows x 32 columns of the panel in registers, so a column step touches no
// shared memory except the reductions: per-column dot products are formed in
// registers, reduced across the warp with a 31-shuffle transpose-reduce
// (lane l ends up holding column l), across warps through an 8x32 shared
// tile, and across CTAs either through distributed shared memory inside ONE
// thread-block cluster (CL = true: <= 16 CTAs, cluster barriers ~0.24 us) or
// through global memory and a grid barrier (CL = false: cooperative launch,
// up to one CTA per SM, ~1.2 us). Every reduction runs in a fixed order, so
// the factorization is deterministic. Optional outputs: the factored panel
// (reflector tails + R), R, the explicit unit-lower V, the compact-WY T
// (cluster mode) and — when the panel is the whole matrix — the explicit thin
// Q (in-register dorg2r backward accumulation).
constexpr int kRegThreads = 256;

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
    double* partials;  // grid mode: [2][gridDim][32]
    double* diag;      // grid mode: [2][32]
};

// lane l returns the warp sum of a[l] (a is destroyed); 31 shuffles.
__device__ __forceinline__ double transpose_reduce32(double (&a)[32]) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
        const bool up = (lane & s) != 0;
#pragma unroll
        for (int k = 0; k < s; ++k) {
            const double send = up ? a[k] : a[k + s];
            const double keep = up ? a[k + s] : a[k];
            a[k] = keep + __shfl_xor_sync(0xffffffffu, send, s);
        }
    }
    return a[0];
}

// register-array element i for a runtime i (keeps the array in registers)
__device__ __forceinline__ double reg_pick(const double (&row)[32], int i) {
    double v = 0.0;
#pragma unroll
    for (int l = 0; l < 32; ++l) v = (l == i) ? row[l] : v;
    return v;
}
__device__ __forceinline__ void reg_set(double (&row)[32], int i, double v) {
#pragma unroll
    for (int l = 0; l < 32; ++l) row[l] = (l == i) ? v : row[l];
}

// this CTA's sums of x(r,i) * x(r,l) over its rows r with global index > i
// (column l in lane l of threads 0..31); wsum is an 8x32 scratch tile.
template <int R>
__device__ __forceinline__ double reg_col_dots(const double (&x)[R][32], const int i, int r0, int nr, double* wsum) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double a[32];
#pragma unroll
    for (int l = 0; l < 32; ++l) a[l] = 0.0;
#pragma unroll
    for (int j = 0; j < R; ++j) {
        const int rr = tid + j * kRegThreads;
        const double xi = (rr < nr && r0 + rr > i) ? reg_pick(x[j], i) : 0.0;
#pragma unroll
        for (int l = 0; l < 32; ++l) a[l] = fma(xi, x[j][l], a[l]);
    }
    wsum[warp * 32 + lane] = transpose_reduce32(a);
    __syncthreads();
    double s = 0.0;
    if (tid < 32) {
#pragma unroll
        for (int w = 0; w < 8; ++w) s += wsum[w * 32 + tid];
    }
    __syncthreads();
    return s;
}

// the thread holding local row orr copies its 32 values to dst
template <int R>
__device__ __forceinline__ void reg_publish_row(const double (&x)[R][32], int orr, int nr, double* dst) {
    if (orr < 0 || orr >= nr || threadIdx.x != (orr % kRegThreads)) return;
    const int jo = orr / kRegThreads;
#pragma unroll
    for (int j = 0; j < R; ++j)
        if (j == jo)
#pragma unroll
            for (int l = 0; l < 32; ++l) dst[l] = x[j][l];
}

template <int R, bool CL>
__global__ void __launch_bounds__(kRegThreads, 1) panel_reg_kernel(RegQrArgs p) {
    __shared__ double wsum[8 * 32];
    __shared__ double part_s[2 * 32];
    __shared__ double dg_s[2 * 32];
    __shared__ double red[32], wv[32], ts[32], dgv[32], sc[4], gcol[32];
    __shared__ double tb[32 * 32];  // compact-WY T, built column by column
    for (int e = threadIdx.x; e < 32 * 32; e += blockDim.x) tb[e] = 0.0;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int rank, G;
    if constexpr (CL) {
        cg::cluster_group cl = cg::this_cluster();
        rank = static_cast<int>(cl.block_rank());
        G = static_cast<int>(cl.num_blocks());
    } else {
        rank = blockIdx.x;
        G = gridDim.x;
    }
    const int b = p.b, rpc = p.rpc;
    const int r0 = rank * rpc, nr = max(0, min(p.rows, r0 + rpc) - r0);
    const int kk = min(b, p.rows);
    int xc = 0;  // exchange counter: double-buffer parity

    double x[R][32];
#pragma unroll
    for (int j = 0; j < R; ++j) {
        const int rr = tid + j * kRegThreads;
#pragma unroll
        for (int l = 0; l < 32; ++l)
            x[j][l] = (rr < nr && l < b) ? p.Pin[(r0 + rr) + static_cast<i64>(l) * p.ldin] : 0.0;
    }

    // Cross-CTA: red[l] = sum over CTAs of `mine` (column tid, valid in tid < 32)
    // in fixed CTA order; dgv[l] = row `orow` of the panel (from its owner).
    // (the owner of row `orow` has already published it with reg_publish_row
    // into row_slot(): dg_s[buf] in cluster mode, p.diag[buf] in grid mode)
    auto row_slot = [&]() { return CL ? dg_s + (xc & 1) * 32 : p.diag + (xc & 1) * 32; };
    auto exchange = [&](double mine, int orow) {
        const int buf = xc & 1;
        ++xc;
        if constexpr (CL) {
            cg::cluster_group cl = cg::this_cluster();
            if (tid < 32) part_s[buf * 32 + tid] = mine;
            cl.sync();
            const int g = tid >> 5;
            const double a0 = (g < G) ? cl.map_shared_rank(part_s, g)[buf * 32 + lane] : 0.0;
            const double a1 = (g + 8 < G) ? cl.map_shared_rank(part_s, g + 8)[buf * 32 + lane] : 0.0;
            wsum[g * 32 + lane] = a0 + a1;
            if (g == 0) dgv[lane] = cl.map_shared_rank(dg_s, orow / rpc)[buf * 32 + lane];
        } else {
            cg::grid_group gg = cg::this_grid();
            double* part = p.partials + static_cast<i64>(buf) * G * 32;
            if (tid < 32) part[rank * 32 + tid] = mine;
            gg.sync();
            constexpr int kMaxLoads = 20;  // G <= 160
            const int g = tid >> 5;
            double v[kMaxLoads];
#pragma unroll
            for (int q = 0; q < kMaxLoads; ++q) {
                const int c = g + 8 * q;
                v[q] = (c < G) ? __ldcg(part + c * 32 + lane) : 0.0;
            }
            double s = 0.0;
#pragma unroll
            for (int q = 0; q < kMaxLoads; ++q) s += v[q];
            wsum[g * 32 + lane] = s;
            if (g == 0) dgv[lane] = __ldcg(p.diag + buf * 32 + lane);
        }
        __syncthreads();
        if (tid < 32) {
            double s = 0.0;
#pragma unroll
            for (int w = 0; w < 8; ++w) s += wsum[w * 32 + tid];
            red[tid] = s;
        }
        __syncthreads();
    };

    // ---- factorization (runtime column loop; registers are indexed only by
    // compile-time l, the active column is selected with predicates) ----
    for (int i = 0; i < kk; ++i) {
        {
            const double mine = reg_col_dots<R>(x, i, r0, nr, wsum);
            reg_publish_row<R>(x, i - r0, nr, row_slot());
            exchange(mine, i);
            if (tid == 0) {
                const double alpha = dgv[i], tail = red[i];
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
                ts[i] = tj;
                sc[0] = beta;
                sc[1] = inv;
            }
            __syncthreads();
            if (tid < 32) {
                // update weights (l > i) and, for l < i, the Gram entries
                // v_l^T v_i = v_l(i) + inv * sum_{r>i} v_l(r) x_i(r), which the
                // same reduction produced: column i of the compact-WY T follows
                // (T(0:i,i) = -tau_i T(0:i,0:i) G(0:i,i)) with no extra pass.
                wv[tid] = (tid > i && tid < b) ? ts[i] * (dgv[tid] + red[tid] * sc[1]) : 0.0;
                if (tid < i) gcol[tid] = dgv[tid] + sc[1] * red[tid];
            }
            __syncthreads();
            if (p.T && tid <= i) {
                double s = 0.0;
                for (int q = tid; q < i; ++q) s = fma(tb[tid + q * 32], gcol[q], s);
                tb[tid + i * 32] = (tid == i) ? ts[i] : -ts[i] * s;
            }
            const double beta = sc[0], inv = sc[1];
            double vj[R];
#pragma unroll
            for (int j = 0; j < R; ++j) {
                const int rr = tid + j * kRegThreads, gr = r0 + rr;
                const double xi = reg_pick(x[j], i);
                vj[j] = (rr < nr && gr > i) ? xi * inv : 0.0;
                if (rr < nr && gr >= i) reg_set(x[j], i, gr > i ? vj[j] : beta);
            }
#pragma unroll
            for (int l = 0; l < 32; ++l) {
                if (l > i) {
                    const double wl = wv[l];
#pragma unroll
                    for (int j = 0; j < R; ++j) {
                        const int rr = tid + j * kRegThreads, gr = r0 + rr;
                        if (rr < nr) x[j][l] = (gr == i) ? x[j][l] - wl : fma(-wl, vj[j], x[j][l]);
                    }
                }
            }
        }
    }
    if (tid < 32) {
        if (tid >= kk) ts[tid] = 0.0;
        if (rank == 0 && tid < kk) p.tau[tid] = ts[tid];
    }
    __syncthreads();

    // ---- factored panel / R / V ----
#pragma unroll
    for (int j = 0; j < R; ++j) {
        const int rr = tid + j * kRegThreads, gr = r0 + rr;
        if (rr < nr) {
#pragma unroll
            for (int l = 0; l < 32; ++l) {
                if (l < b) {
                    if (p.Pout) p.Pout[gr + static_cast<i64>(l) * p.ldout] = x[j][l];
                    if (p.R && gr < kk) p.R[gr + static_cast<i64>(l) * p.ldr] = (gr <= l) ? x[j][l] : 0.0;
                    if (p.V) p.V[gr + static_cast<i64>(l) * p.ldv] = gr > l ? x[j][l] : (gr == l ? 1.0 : 0.0);
                }
            }
        }
    }

    // ---- compact-WY T (identical in every CTA; rank 0 writes it) ----
    if (p.T && rank == 0)
        for (int e = tid; e < 32 * 32; e += kRegThreads) p.T[e] = tb[e];

    // ---- explicit thin Q of the whole (single-panel) matrix ----
    if (p.Q) {
        for (int i = kk - 1; i >= 0; --i) {
            {
                const double ti = ts[i];
                if (i < kk - 1 && ti != 0.0) {
                    const double mine = reg_col_dots<R>(x, i, r0, nr, wsum);
                    reg_publish_row<R>(x, i - r0, nr, row_slot());
                    exchange(mine, i);
                    if (tid < 32) wv[tid] = (tid > i && tid < kk) ? ti * (dgv[tid] + red[tid]) : 0.0;
                    __syncthreads();
                    double vi[R];
#pragma unroll
                    for (int j = 0; j < R; ++j) vi[j] = reg_pick(x[j], i);
#pragma unroll
                    for (int l = 0; l < 32; ++l) {
                        if (l > i) {
                            const double wl = wv[l];
#pragma unroll
                            for (int j = 0; j < R; ++j) {
                                const int rr = tid + j * kRegThreads, gr = r0 + rr;
                                if (rr < nr && gr >= i) x[j][l] = (gr == i) ? x[j][l] - wl : fma(-wl, vi[j], x[j][l]);
                            }
                        }
                    }
                }
#pragma unroll
                for (int j = 0; j < R; ++j) {
                    const int gr = r0 + tid + j * kRegThreads;
                    const double xi = reg_pick(x[j], i);
                    reg_set(x[j], i, gr > i ? -ti * xi : (gr == i ? 1.0 - ti : 0.0));
                }
            }
        }
#pragma unroll
        for (int j = 0; j < R; ++j) {
            const int rr = tid + j * kRegThreads;
            if (rr < nr)
#pragma unroll
                for (int l = 0; l < 32; ++l)
                    if (l < kk) p.Q[(r0 + rr) + static_cast<i64>(l) * p.ldq] = x[j][l];
        }
    }
    if constexpr (CL) cg::this_cluster().sync();  // peers may still read this CTA's shared memory
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
    (void)kSmallMaxElems;  // the single-CTA smem kernel serves the batched API only
    // Panels hold at most 2 rows x 32 columns per thread in registers (one CTA
    // per SM): taller R-only factorizations (norm_exact of very tall cores)
    // go through a TSQR split — R of each row block, then R of the stacked Rs.
    const i64 max_rows = 2LL * kRegThreads * c.sm_count;
    if (m > max_rows) {
        if (Q != nullptr) throw Error(TTR_ERR_INTERNAL, "thin_qr with Q: matrix taller than the device panel limit");
        const i64 chunk = std::max<i64>(k, max_rows / 2);
        const i64 nchunks = (m + chunk - 1) / chunk;
        DBuf stack(c, static_cast<std::size_t>(nchunks * k * n));
        const i64 lds = nchunks * k;
        for (i64 q = 0; q < nchunks; ++q) {
            const i64 r0 = q * chunk, rows = std::min(chunk, m - r0), kq = std::min(rows, n);
            DBuf Rq(c, static_cast<std::size_t>(kq * n));
            thin_qr(c, rows, n, A + r0, lda, nullptr, 1, Rq.p, kq);
            if (kq < k)
                TTR_CUDA(cudaMemset2DAsync(stack.p + q * k, sizeof(double) * lds, 0, sizeof(double) * k, n, c.stream));
            TTR_CUDA(cudaMemcpy2DAsync(stack.p + q * k, sizeof(double) * lds, Rq.p, sizeof(double) * kq,
                                       sizeof(double) * kq, n, cudaMemcpyDeviceToDevice, c.stream));
        }
        thin_qr(c, lds, n, stack.p, lds, nullptr, 1, R, ldr);
        return;
    }
    static bool configured = false;
    if (!configured) {
        TTR_CUDA(cudaFuncSetAttribute(panel_reg_kernel<1, true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        TTR_CUDA(cudaFuncSetAttribute(panel_reg_kernel<2, true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        configured = true;
    }
    // Launch the register-resident panel kernel on a rows x b panel (b <= 32):
    // one cluster of <= 16 CTAs when rows <= 16 * 512, else a cooperative grid
    // of <= one CTA per SM. Returns true if the cluster mode was used.
    DBuf partials(c, static_cast<std::size_t>(2 * 160 * 32));
    DBuf diag(c, 2 * 32);
    auto launch_panel = [&](RegQrArgs a) {
        const i64 rows = a.rows;
        const bool cl = rows <= 16 * 2 * kRegThreads;
        i64 grid;
        if (cl) {
            grid = std::max<i64>(1, std::min<i64>(16, (rows + kRegThreads - 1) / kRegThreads));
        } else {
            grid = std::min<i64>(c.sm_count, (rows + 2 * kRegThreads - 1) / (2 * kRegThreads) * 2);
            grid = std::max<i64>(grid, (rows + 2 * kRegThreads - 1) / (2 * kRegThreads));
            grid = std::min<i64>(grid, c.sm_count);
        }
        const i64 rpc = (rows + grid - 1) / grid;
        if (rpc > 2 * kRegThreads) throw Error(TTR_ERR_INTERNAL, "qr panel too tall for the device");
        grid = (rows + rpc - 1) / rpc;
        a.rpc = static_cast<int>(rpc);
        a.partials = partials.p;
        a.diag = diag.p;
        const bool two = rpc > kRegThreads;
        if (cl) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(static_cast<unsigned>(grid));
            cfg.blockDim = dim3(kRegThreads);
            cfg.dynamicSmemBytes = 0;
            cfg.stream = c.stream;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = static_cast<unsigned>(grid);
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            if (two) TTR_CUDA(cudaLaunchKernelEx(&cfg, panel_reg_kernel<2, true>, a));
            else TTR_CUDA(cudaLaunchKernelEx(&cfg, panel_reg_kernel<1, true>, a));
        } else {
            void* args[] = {&a};
            void* fn = two ? reinterpret_cast<void*>(panel_reg_kernel<2, false>)
                           : reinterpret_cast<void*>(panel_reg_kernel<1, false>);
            TTR_CUDA(cudaLaunchCooperativeKernel(fn, dim3(static_cast<unsigned>(grid)), dim3(kRegThreads), args, 0,
                                                 c.stream));
        }
        c.launched();
        return cl;
    };

    // ---- <= 32 columns: factorization and explicit Q in one launch ----
    if (n <= kPanel) {
        DBuf tau(c, static_cast<std::size_t>(k));
        RegQrArgs a{};
        a.rows = static_cast<int>(m);
        a.b = static_cast<int>(n);
        a.Pin = A;
        a.ldin = lda;
        a.tau = tau.p;
        a.Q = Q;
        a.ldq = ldq;
        a.R = R;
        a.ldr = ldr;
        launch_panel(a);
        return;
    }

    // ---- blocked right-looking Householder ----
    const i64 ldw = even_ld(m);
    DBuf work(c, static_cast<std::size_t>(ldw * n));
    copy_matrix(c, m, n, A, lda, work.p, ldw);
    const i64 npanels = (k + kPanel - 1) / kPanel;
    DBuf tau(c, static_cast<std::size_t>(k));
    DBuf Vall(c, static_cast<std::size_t>(ldw * k));  // explicit V of every panel (rows j0.. of column block)
    DBuf Ts(c, static_cast<std::size_t>(npanels * kPanel * kPanel));
    DBuf Wb(c, static_cast<std::size_t>(kPanel * std::max<i64>(n, 1)));
    DBuf Wb2(c, static_cast<std::size_t>(kPanel * std::max<i64>(n, 1)));

    for (i64 p = 0; p < npanels; ++p) {
        const i64 j0 = p * kPanel, bb = std::min<i64>(kPanel, k - j0), rows = m - j0;
        double* V = Vall.p + j0 + j0 * ldw;  // rows x bb block at (j0, j0), ld ldw
        double* T = Ts.p + p * kPanel * kPanel;
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
