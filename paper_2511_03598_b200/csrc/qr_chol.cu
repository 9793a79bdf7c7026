// qr_chol.cu — Cholesky-QR kernels:
//   K4c  whole-matrix shifted Cholesky QR of a tall-skinny sketch (opt-in, below),
//   K4d  Cholesky-QR panels with Householder reconstruction as separate launches,
//   K4e  batched CholeskyQR2 / sCQR3 of small matrices (the batched sweep, config 5a),
//   K4f  the K4d panel as ONE cooperative kernel — the default panel factorisation
//        of the blocked Householder QR and the thin QR of <= 32-column blocks.
//
// K4c: shifted Cholesky QR (sCQR) for the tall-skinny sketches of the Rand-Orth
// sweep and the TT-SVD orthogonalisations.
//
// linalg::thin_qr_q (proj/core/src/linalg.cpp:44-56) is called by the sweep
// only for an orthonormal basis of range(S) (round_rand.cpp:33-37); the
// Householder path (qr.cu) is latency-bound: every column of every panel waits
// on one cross-CTA exchange (~2.5-4.5 us per column at 7,040-40,960 rows).
// Shifted CholeskyQR (Fukaya, Kannan, Nakatsukasa, Yamamoto, Yanagisawa, SIAM
// J. Sci. Comput. 2020) needs no per-column exchange: four passes of
//   G = A^T A            (DMMA GEMM, upper tiles, split-K — gemm_dmma.cu)
//   R = chol(G [+ s I])  (chol_kernel: one CTA, blocked right-looking)
//   Q = A R^{-1}         (trsm_kernel: row tiles, DMMA + substitution)
// the first two with the shift s = 11 (m n + n (n+1)) u ||A||_F^2 (each pass
// lowers the condition number by ~sqrt(s)/||A||), the last two (CholeskyQR2) on
// the previous Q without. For kappa(A) up to ~u^{-1} the result is backward
// stable with an orthonormal Q (the same guarantees as Householder); Q spans
// the same space as the Householder Q up to column signs, so the rounded
// tensor — a product of projections Q Q^T — is the same.
//
// Breakdown: a non-positive or non-finite pivot in any of the three Cholesky
// factorisations, or ||G_4 - I||_F > 1/2 (the earlier passes did not deliver a
// well-conditioned Q_3), sets the context's QR flag. Callers speculate: they
// run the whole rounding with sCQR, read the flag once, and redo the call on
// the Householder path if it is set (tt_round.cu), so exactly rank-deficient
// sketches still get the reference's behaviour.
#include <cfloat>
#include <cmath>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace ttr {
namespace {

constexpr int kCholThreads = 256;
constexpr int kCholSmemMaxN = 144;  // whole matrix in shared memory up to this order

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(double* dst, const double* src, int bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src), "r"(bytes));
}
__device__ __forceinline__ void cp_async8(double* dst, const double* src, int bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(dst)), "l"(src), "r"(bytes));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// row panel: n - j0 columns + 32 appended identity columns (-> inv(R_JJ)) + 4 pad
__host__ __device__ constexpr int chol_ldp(int n) { return ((n + 3) / 4) * 4 + 36; }
__host__ __device__ constexpr int trsm_ld(int n) { return ((n + 31) / 32) * 32 + 4; }  // % 16 == 4

struct CholArgs {
    int n;
    double* G;  // n x n (ld ldg): upper triangle in, R (upper, zeros below) out
    int ldg;
    int mode;  // bit 0: add shift_coeff * trace(G) to the diagonal; bit 1: require ||G - I||_F <= 1/2
    double shift_coeff;
    int* flag;  // atomicMin(flag, tag) on breakdown
    int tag;
    double* Rinv;  // [ceil(n/32)][32 x 32] column-major inverses of the diagonal blocks of R
};

// Blocked (32) right-looking Cholesky G = R^T R in one CTA. Per block row J
// the 32 x (n - j0) row panel is copied to shared memory and eliminated in
// place with deferred scaling (step k: G(i, c) -= G(k, i) G(k, c) / g_kk for
// the panel rows i > k; one barrier per step, every thread owning columns),
// which factors the diagonal block and solves the panel rows together; the
// rows are then scaled by 1/sqrt(g_kk) into R and the trailing upper triangle
// is updated with 4 x 4 register tiles. Finally the inverses of the 32 x 32
// diagonal blocks of R are formed (one warp per block, one row per step) for
// the blocked TRSM. All loops stay rolled: this kernel is latency-bound on one
// SM, and straight-line code would run from instruction-cache misses.
// SM: the matrix lives in shared memory (n <= kCholSmemMaxN); otherwise it is
// updated in place in global memory (L2-resident).
#ifdef TTR_CHOL_TRACE
__device__ unsigned long long g_chol_trace[8];
#define CHOL_T(i) do { __syncthreads(); if (threadIdx.x == 0) { long long t = clock64(); atomicAdd(&g_chol_trace[i], static_cast<unsigned long long>(t - t_last)); t_last = t; } } while (0)
#else
#define CHOL_T(i) do { } while (0)
#endif
template <bool SM>
__global__ void __launch_bounds__(kCholThreads) chol_kernel(CholArgs p) {
#ifdef TTR_CHOL_TRACE
    long long t_last = clock64();
#endif
    extern __shared__ __align__(16) double smem[];
    __shared__ double pv[32], rsq[32], rinv[32];  // pivots of the current block, sqrt, 1 / sqrt
    __shared__ double prcp[32];                   // 1 / pivot
    __shared__ double red[kCholThreads / 32];
    __shared__ int bad;
    const int n = p.n, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int ldp = chol_ldp(n);
    double* RP = smem;  // row panel [32][ldp]: RP[i * ldp + c'] = G(j0 + i, j0 + c')
    double* A;
    i64 lda;
    if constexpr (SM) {
        A = smem + 32 * ldp;
        lda = n + 1;
        for (int cc = warp; cc < n; cc += kCholThreads / 32)
            for (int r = lane; r <= cc; r += 32) cp_async8(A + r + cc * lda, p.G + r + static_cast<i64>(cc) * p.ldg, 8);
        cp_commit();
        cp_wait<0>();
    } else {
        A = p.G;
        lda = p.ldg;
    }
    if (tid == 0) bad = 0;
    __syncthreads();
    CHOL_T(0);
    double shift = 0.0;
    if (p.mode & 3) {
        double acc = 0.0;
        if (p.mode & 1) {
            for (int i = tid; i < n; i += kCholThreads) acc += A[i + i * lda];
        } else {
            for (int cc = warp; cc < n; cc += kCholThreads / 32)
                for (int r = lane; r <= cc; r += 32) {
                    const double v = A[r + cc * lda] - (r == cc ? 1.0 : 0.0);
                    acc += (r == cc ? 1.0 : 2.0) * v * v;
                }
        }
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) red[warp] = acc;
        __syncthreads();
        double total = 0.0;
        for (int w = 0; w < kCholThreads / 32; ++w) total += red[w];
        if (p.mode & 1)
            shift = p.shift_coeff * total;
        else if (tid == 0 && !(total <= 0.25))
            bad = 1;
    }
    for (int j0 = 0; j0 < n; j0 += 32) {
        const int b = min(32, n - j0), nt = n - j0;  // panel columns c' in [0, nt), then 32 identity columns
        for (int cc = tid; cc < nt; cc += kCholThreads)
            for (int i = 0; i < 32; ++i) {
                const bool in = i < b && i <= cc;
                if constexpr (SM)
                    RP[i * ldp + cc] = in ? A[(j0 + i) + (j0 + cc) * lda] : 0.0;
                else  // global -> shared without a register round trip (latency-bound otherwise)
                    cp_async8(RP + i * ldp + cc, A + (in ? (j0 + i) + (j0 + cc) * lda : 0), in ? 8 : 0);
            }
        cp_commit();
        for (int e = tid; e < 32 * 32; e += kCholThreads) {
            const int i = e & 31, a = e >> 5;
            RP[i * ldp + nt + a] = (i == a && a < b) ? 1.0 : 0.0;
        }
        cp_wait<0>();
        __syncthreads();
        if (tid < b && shift != 0.0) RP[tid * ldp + tid] += shift;
        __syncthreads();
        CHOL_T(1);
        // elimination with deferred scaling: row_i -= (G(k, i) / g_kk) row_k, i > k,
        // over the whole row panel (diagonal block, panel columns, identity
        // columns) at once: thread (row group rg, column lane cl) owns rows
        // rg + 4q and columns cl + 64p; one barrier per step. Regular columns
        // only need their upper part (i <= c), the identity columns all rows.
        const int ncol = nt + 32;
        {
            const int rg = tid >> 6, cl = tid & 63;
            for (int k = 0; k < b; ++k) {
                double piv = RP[k * ldp + k];
                if (!(piv > 0.0) || !isfinite(piv)) {
                    if (tid == 0) bad = 1;
                    piv = 1.0;  // keep the factor finite; the result is discarded
                }
                if (tid == 0) pv[k] = piv;
                const double invp = 1.0 / piv;
                const double* rk = RP + k * ldp;
                double ri[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) ri[q] = rk[rg + 4 * q] * invp;  // multipliers G(k, i) / g_kk
                for (int c0 = k + 1; c0 < ncol; c0 += 64) {
                    const int cc = c0 + cl;
                    if (cc >= ncol) continue;
                    const double rc = rk[cc];
                    const int iend = cc < nt ? min(cc, b - 1) : b - 1;
                    double v[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q) v[q] = RP[(rg + 4 * q) * ldp + cc];
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const int i = rg + 4 * q;
                        if (i > k && i <= iend) RP[i * ldp + cc] = fma(-ri[q], rc, v[q]);
                    }
                }
                __syncthreads();
            }
        }
        CHOL_T(2);
        // R rows: R(j0 + k, c) = G(k, c) / sqrt(g_kk) (c > k), R(k, k) = sqrt(g_kk); the
        // identity columns become inv(R_JJ)^T
        if (tid < 32) {
            const double r = tid < b ? sqrt(pv[tid]) : 1.0;
            rsq[tid] = r;
            rinv[tid] = 1.0 / r;
        }
        __syncthreads();
        {
            const int rg = tid >> 6, cl = tid & 63;
            for (int cc = cl; cc < ncol; cc += 64) {
                const int kend = cc < nt ? min(cc, b - 1) : b - 1;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int k = rg + 4 * q;
                    if (k <= kend) {
                        const double v = (k == cc) ? rsq[k] : RP[k * ldp + cc] * rinv[k];
                        RP[k * ldp + cc] = v;
                        if (cc < nt) A[(j0 + k) + (j0 + cc) * lda] = v;
                    }
                }
            }
        }
        __syncthreads();
        // inv(R_JJ) (column-major 32 x 32) = transpose of the identity columns
        for (int e = tid; e < 32 * 32; e += kCholThreads) {
            const int i = e & 31, c = e >> 5;
            p.Rinv[static_cast<i64>(j0 / 32) * 1024 + i + 32 * c] = (i < b && c < b) ? RP[c * ldp + nt + i] : 0.0;
        }
        __syncthreads();  // the identity columns are read above before the padding below overwrites them
        // zero the panel's padding columns past the trailing block so the 4-wide tiles read zeros
        for (int e = tid; e < 32 * 8; e += kCholThreads) {
            const int r = e >> 3, cc = nt + (e & 7);
            RP[r * ldp + cc] = 0.0;
        }
        __syncthreads();
        CHOL_T(3);
        // trailing update of the upper triangle: G(i, j) -= sum_r P(r, i) P(r, j)
        // over the panel columns past the diagonal block, 4 (i) x 8 (j) register
        // tiles with i <= j somewhere in the tile; lanes of a warp share the
        // j-tile (broadcast loads), so the update is FMA-bound; the next tile's
        // old values load while this tile computes
        const int c1 = j0 + b, nr = n - c1;
        const double* Pb = RP + b;
        const int nj = (nr + 7) / 8, ntiles = nj * (nj + 1);  // j-tile tj holds i-tiles 0 .. 2 tj + 1
        auto tile_of = [&](int t, int& ti, int& tj) {
            tj = static_cast<int>((sqrt(4.0 * t + 1.0) - 1.0) * 0.5);
            while (tj * (tj + 1) > t) --tj;
            while ((tj + 1) * (tj + 2) <= t) ++tj;
            ti = t - tj * (tj + 1);
        };
        double oldv[4][8];
        auto load_old = [&](int ti, int tj) {
#pragma unroll
            for (int v = 0; v < 8; ++v)
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int i = 4 * ti + u, j = 8 * tj + v;
                    oldv[u][v] = (i <= j && j < nr) ? A[(c1 + i) + (c1 + j) * lda] : 0.0;
                }
        };
        int ti = 0, tj = 0;
        if (tid < ntiles) {
            tile_of(tid, ti, tj);
            load_old(ti, tj);
        }
        for (int t = tid; t < ntiles; t += kCholThreads) {
            double acc[4][8];
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 8; ++v) acc[u][v] = oldv[u][v];
            const int cti = ti, ctj = tj;
            if (t + kCholThreads < ntiles) {
                tile_of(t + kCholThreads, ti, tj);
                load_old(ti, tj);
            }
#pragma unroll 2
            for (int r = 0; r < b; ++r) {
                const double* pr = Pb + r * ldp;
                const double2 i01 = *reinterpret_cast<const double2*>(pr + 4 * cti);
                const double2 i23 = *reinterpret_cast<const double2*>(pr + 4 * cti + 2);
                const double2 j01 = *reinterpret_cast<const double2*>(pr + 8 * ctj);
                const double2 j23 = *reinterpret_cast<const double2*>(pr + 8 * ctj + 2);
                const double2 j45 = *reinterpret_cast<const double2*>(pr + 8 * ctj + 4);
                const double2 j67 = *reinterpret_cast<const double2*>(pr + 8 * ctj + 6);
                const double pi[4] = {i01.x, i01.y, i23.x, i23.y};
                const double pj[8] = {j01.x, j01.y, j23.x, j23.y, j45.x, j45.y, j67.x, j67.y};
#pragma unroll
                for (int u = 0; u < 4; ++u)
#pragma unroll
                    for (int v = 0; v < 8; ++v) acc[u][v] = fma(-pi[u], pj[v], acc[u][v]);
            }
#pragma unroll
            for (int v = 0; v < 8; ++v)
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int i = 4 * cti + u, j = 8 * ctj + v;
                    if (i <= j && j < nr) A[(c1 + i) + (c1 + j) * lda] = acc[u][v];
                }
        }
        __syncthreads();
        CHOL_T(4);
    }
    CHOL_T(5);
    // R out (upper) with zeros below the diagonal
    for (int cc = warp; cc < n; cc += kCholThreads / 32)
        for (int r = lane; r < n; r += 32) {
            double* g = p.G + r + static_cast<i64>(cc) * p.ldg;
            if (r > cc)
                *g = 0.0;
            else if constexpr (SM)
                *g = A[r + cc * lda];
        }
    if (tid == 0 && bad) atomicMin(p.flag, p.tag);
}

// Q = A R^{-1} for R upper triangular (n x n), one CTA per BM-row tile (BM/16
// warps, 16 rows each). The tile lives column-major in shared memory; per
// 32-column block J each warp forms acc = A(:, J) - Q(:, <J) R(<J, J) on DMMA,
// with R(<J, J) streamed through shared memory in 32 x 32 chunks (cp.async,
// double buffered), then Q(:, J) = acc * inv(R_JJ) with the 32 x 32 inverse of
// the diagonal block written by chol_kernel (blocked TRSM with inverted
// diagonal blocks). With the two shifted passes every factor here has
// kappa(R) <= ~||A|| / sqrt(s) ~ 1e4, so the inverted blocks cost at most that
// factor in the rowwise residual. A and Q may alias (in place).
constexpr int kRcLd = 36;  // chunk [32 cols][32 k + 4]: conflict-free B fragments

template <int BM>
__global__ void __launch_bounds__(BM * 2) trsm_kernel(int m, int n, const double* A, i64 lda, const double* R,
                                                     int ldr, const double* Rinv, double* Q, i64 ldq) {
    constexpr int kThreads = BM * 2, kLdm = BM + 4;  // kLdm % 16 == 4: conflict-free A fragments
    extern __shared__ __align__(16) double smem[];
    const int npad = ((n + 31) / 32) * 32;
    double* Qs = smem;                    // [npad][kLdm] column-major tile
    double* Rc = smem + npad * kLdm;      // [2][32][kRcLd] chunks of R(<J, J)
    double* Ui = Rc + 2 * 32 * kRcLd;     // [32][kRcLd] inv(R_JJ)
    const i64 row0 = static_cast<i64>(blockIdx.x) * BM;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool vec = ((lda & 1) == 0) && ((reinterpret_cast<std::uintptr_t>(A) & 15) == 0);
    for (int e = tid; e < npad * (BM / 2); e += kThreads) {
        const int cc = e / (BM / 2), r2 = (e % (BM / 2)) * 2;
        const i64 gr = row0 + r2;
        double* dst = Qs + cc * kLdm + r2;
        const int rows = (cc < n && gr < m) ? static_cast<int>(m - gr < 2 ? m - gr : 2) : 0;
        const double* src = A + (rows ? gr + cc * lda : 0);
        if (vec) {
            cp_async16(dst, src, rows * 8);
        } else {
            cp_async8(dst, src, rows >= 1 ? 8 : 0);
            cp_async8(dst + 1, src + (rows >= 2 ? 1 : 0), rows >= 2 ? 8 : 0);
        }
    }
    cp_commit();
    const bool rvec = (ldr & 1) == 0;
    auto load_block = [&](double* dst, const double* base, i64 ld, int k0, int c0, bool v16) {
        // base(k0:k0+32, c0:c0+32) -> dst[col][k] (zero fill past n)
        for (int e = tid; e < 32 * 16; e += kThreads) {
            const int col = e >> 4, kk = (e & 15) * 2;
            const int gc = c0 + col, gk = k0 + kk;
            const int cnt = gc < n ? max(0, min(2, n - gk)) : 0;
            const double* src = base + (cnt ? static_cast<i64>(gc) * ld + gk : 0);
            double* d = dst + col * kRcLd + kk;
            if (v16) {
                cp_async16(d, src, cnt * 8);
            } else {
                cp_async8(d, src, cnt >= 1 ? 8 : 0);
                cp_async8(d + 1, src + (cnt >= 2 ? 1 : 0), cnt >= 2 ? 8 : 0);
            }
        }
    };
    const int fr = lane >> 2, fc = lane & 3, wr = warp * 16;
    for (int c0 = 0; c0 < n; c0 += 32) {
        const int nch = c0 / 32;
        __syncthreads();  // the previous block's reads of Ui / Rc are done
        {
            // inv(R_JJ): stored 32 x 32 column-major per block (ld 32, c0 local)
            const double* ub = Rinv + static_cast<i64>(c0 / 32) * 1024;
            for (int e = tid; e < 32 * 16; e += kThreads) {
                const int col = e >> 4, kk = (e & 15) * 2;
                cp_async16(Ui + col * kRcLd + kk, ub + col * 32 + kk, 16);
            }
        }
        if (nch > 0) load_block(Rc, R, ldr, 0, c0, rvec);
        cp_commit();
        double acc[2][4][2];
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
            for (int t = 0; t < 4; ++t)
#pragma unroll
                for (int h = 0; h < 2; ++h) acc[mi][t][h] = 0.0;
        for (int ch = 0; ch < nch; ++ch) {
            if (ch + 1 < nch) load_block(Rc + ((ch + 1) & 1) * 32 * kRcLd, R, ldr, (ch + 1) * 32, c0, rvec);
            cp_commit();
            cp_wait<1>();
            __syncthreads();
            const double* rc = Rc + (ch & 1) * 32 * kRcLd;
            const double* qa = Qs + (ch * 32) * kLdm + wr + fr;
#pragma unroll
            for (int k = 0; k < 32; k += 4) {
                const double a0 = qa[(k + fc) * kLdm], a1 = qa[(k + fc) * kLdm + 8];
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const double bv = rc[(t * 8 + fr) * kRcLd + k + fc];
                    dmma(acc[0][t][0], acc[0][t][1], a0, bv);
                    dmma(acc[1][t][0], acc[1][t][1], a1, bv);
                }
            }
            __syncthreads();  // buffer (ch & 1) is refilled two chunks later
        }
        cp_wait<0>();
        __syncthreads();
        // acc_J = A(:, J) - Q(:, <J) R(<J, J) into the tile (own rows only)
        double* qj = Qs + c0 * kLdm + wr + fr;
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
            for (int t = 0; t < 4; ++t)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    double* d = qj + (t * 8 + 2 * fc + h) * kLdm + mi * 8;
                    *d = *d - acc[mi][t][h];
                }
        __syncwarp();
        // Q(:, J) = acc_J inv(R_JJ)
        double x[2][4][2];
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
            for (int t = 0; t < 4; ++t) x[mi][t][0] = x[mi][t][1] = 0.0;
#pragma unroll
        for (int k = 0; k < 32; k += 4) {
            const double a0 = qj[(k + fc) * kLdm], a1 = qj[(k + fc) * kLdm + 8];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const double bv = Ui[(t * 8 + fr) * kRcLd + k + fc];
                dmma(x[0][t][0], x[0][t][1], a0, bv);
                dmma(x[1][t][0], x[1][t][1], a1, bv);
            }
        }
        __syncwarp();
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
            for (int t = 0; t < 4; ++t)
#pragma unroll
                for (int h = 0; h < 2; ++h) qj[(t * 8 + 2 * fc + h) * kLdm + mi * 8] = x[mi][t][h];
        __syncwarp();
    }
    __syncthreads();
    for (int e = tid; e < n * BM; e += kThreads) {
        const int cc = e / BM, r = e % BM;
        const i64 gr = row0 + r;
        if (gr < m) Q[gr + cc * ldq] = Qs[cc * kLdm + r];
    }
}

template <int BM>
std::size_t trsm_smem(i64 n) {
    const std::size_t npad = static_cast<std::size_t>((n + 31) / 32) * 32;
    return sizeof(double) * (npad * (BM + 4) + 3 * 32 * kRcLd);
}

// opt in to the largest dynamic shared memory the kernel's static usage leaves
void set_max_dynamic_smem(const void* fn) {
    cudaFuncAttributes fa{};
    TTR_CUDA(cudaFuncGetAttributes(&fa, fn));
    int dev = 0, optin = 0;
    TTR_CUDA(cudaGetDevice(&dev));
    TTR_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    TTR_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  optin - static_cast<int>(fa.sharedSizeBytes)));
}

void launch_chol(Ctx& c, i64 n, double* G, i64 ldg, int mode, double coeff, double* Rinv, int tag) {
    CholArgs a{static_cast<int>(n), G, static_cast<int>(ldg), mode, coeff, c.qr_flag_dev(), static_cast<int>(tag), Rinv};
    const std::size_t panel = sizeof(double) * 32 * chol_ldp(static_cast<int>(n));
    static std::atomic<std::uint64_t> configured{0};
    if (first_on_device(configured)) {
        set_max_dynamic_smem(reinterpret_cast<const void*>(chol_kernel<true>));
        set_max_dynamic_smem(reinterpret_cast<const void*>(chol_kernel<false>));
    }
    if (n <= kCholSmemMaxN) {
        const std::size_t smem = panel + sizeof(double) * static_cast<std::size_t>(n * (n + 1));
        chol_kernel<true><<<1, kCholThreads, smem, c.stream>>>(a);
    } else {
        chol_kernel<false><<<1, kCholThreads, panel, c.stream>>>(a);
    }
    TTR_CUDA(cudaGetLastError());
    c.launched();
}

void launch_trsm(Ctx& c, i64 m, i64 n, const double* A, i64 lda, const double* R, i64 ldr, const double* Rinv,
                 double* Q, i64 ldq) {
    static std::atomic<std::uint64_t> configured{0};
    if (first_on_device(configured)) {
        set_max_dynamic_smem(reinterpret_cast<const void*>(trsm_kernel<64>));
        set_max_dynamic_smem(reinterpret_cast<const void*>(trsm_kernel<32>));
    }
    if (trsm_smem<64>(n) <= 220 * 1024) {
        const unsigned grid = static_cast<unsigned>((m + 63) / 64);
        trsm_kernel<64><<<grid, 128, trsm_smem<64>(n), c.stream>>>(static_cast<int>(m), static_cast<int>(n), A, lda, R,
                                                                  static_cast<int>(ldr), Rinv, Q, ldq);
    } else {
        const unsigned grid = static_cast<unsigned>((m + 31) / 32);
        trsm_kernel<32><<<grid, 64, trsm_smem<32>(n), c.stream>>>(static_cast<int>(m), static_cast<int>(n), A, lda, R,
                                                                 static_cast<int>(ldr), Rinv, Q, ldq);
    }
    TTR_CUDA(cudaGetLastError());
    c.launched();
}

// ---------------------------------------------------------------------------
// K4d: Cholesky-QR panels with Householder reconstruction (the blocked
// Householder QR's panel factorisation without a cross-CTA exchange per
// column). A rows x b panel (b <= 32) is orthogonalised by shifted CholeskyQR3
// (every pass: partial Grams per CTA -> one CTA reduces them in a fixed order,
// factors the 32 x 32 Gram and inverts the factor -> Q = P R^{-1} row by row),
// then the Householder vectors are rebuilt from Q (Ballard, Demmel, Grigori,
// Jacquelin, Nguyen, Solomonik 2014): the LU without pivoting of Q_1 - S with
// s_k = -sign of the running pivot gives Y_1 = L, U, and Y_2 = Q_2 U^{-1},
// T = -U S Y_1^{-T}, R = S R_chol — exactly the (V, T, R) of the panel the
// blocked QR's trailing updates and explicit-Q formation consume (H = I - V T V^T
// with H [R; 0] = P).

constexpr int kCqrThreads = 256;

__global__ void __launch_bounds__(kCqrThreads) cqr_gram_partial(int rows, int b, const double* P, i64 ldp, int rpc,
                                                               double* part) {
    __shared__ double tile[32][33];
    const int tid = threadIdx.x;
    const int r0 = blockIdx.x * rpc, r1 = min(rows, r0 + rpc);
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int c0 = r0; c0 < r1; c0 += 32) {
        __syncthreads();
        for (int e = tid; e < 1024; e += kCqrThreads) {
            const int rr = e & 31, col = e >> 5, r = c0 + rr;
            tile[rr][col] = (r < r1 && col < b) ? P[r + static_cast<i64>(col) * ldp] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int e = tid + kCqrThreads * q, i = e & 31, j = e >> 5;
            double a = acc[q];
#pragma unroll 8
            for (int rr = 0; rr < 32; ++rr) a = fma(tile[rr][i], tile[rr][j], a);
            acc[q] = a;
        }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) part[static_cast<i64>(blockIdx.x) * 1024 + tid + kCqrThreads * q] = acc[q];
}

// One CTA of 1024 threads, thread = matrix entry (i, j): G = sum of the
// partial Grams (fixed order, 8 interleaved partial sums); mode 1 adds the
// shift coeff * trace(G), mode 2 requires ||G - I||_F <= 1/2; R = chol(G) by
// 32 deferred-scaling elimination steps (one barrier each), Rinv by
// Gauss-Jordan on [R | I] (32 steps), Rtot = R Rtot (first: Rtot = R).
// Breakdown -> atomicMin(flag, tag).
constexpr int kCholSmall = 1024;
__global__ void __launch_bounds__(kCholSmall) cqr_chol32(int nparts, const double* part, int b, int mode, double coeff,
                                                        double* Rinv, double* Rtot, int first, int* flag, int tag) {
    __shared__ double G[32][33], X[32][33], Rt[32][33];
    __shared__ double red[32], pv[32];
    __shared__ int bad;
    const int e = threadIdx.x, i = e & 31, j = e >> 5, lane = e & 31, warp = e >> 5;
    if (e == 0) bad = 0;
    {
        double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        int g = 0;
        for (; g + 8 <= nparts; g += 8) {
            double v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = part[static_cast<i64>(g + q) * 1024 + e];
#pragma unroll
            for (int q = 0; q < 8; ++q) acc[q] += v[q];
        }
        for (int q = 0; g < nparts; ++g, ++q) acc[q] += part[static_cast<i64>(g) * 1024 + e];
        const double sacc = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
        G[i][j] = (i < b && j < b) ? sacc : (i == j ? 1.0 : 0.0);
        if (!first) Rt[i][j] = Rtot[e];
    }
    __syncthreads();
    if (mode != 0) {
        double v = 0.0;
        if (i < b && j < b) {
            if (mode == 1) v = (i == j) ? G[i][i] : 0.0;
            else {
                const double d = G[i][j] - (i == j ? 1.0 : 0.0);
                v = d * d;
            }
        }
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) red[warp] = v;
        __syncthreads();
        double tot = 0.0;
        for (int w = 0; w < 32; ++w) tot += red[w];
        if (mode == 1 && i == j && i < b) G[i][i] += coeff * tot;
        if (mode == 2 && e == 0 && !(tot <= 0.25)) bad = 1;
        __syncthreads();
    }
    // Cholesky with deferred scaling: step k, G(i, j) -= G(k, i) G(k, j) / g_kk for k < i <= j
    for (int k = 0; k < 32; ++k) {
        double piv = G[k][k];
        if (!(piv > 0.0) || !isfinite(piv)) {
            if (e == 0) bad = 1;
            piv = 1.0;
        }
        if (e == 0) pv[k] = piv;
        const double upd = (i > k && j >= i) ? G[k][i] * G[k][j] / piv : 0.0;
        __syncthreads();
        if (i > k && j >= i) G[i][j] -= upd;
        __syncthreads();
    }
    // R(i, j) = G(i, j) / sqrt(g_ii) (j > i), R(i, i) = sqrt(g_ii)
    {
        const double r = sqrt(pv[i]);
        const double v = (j > i) ? G[i][j] / r : (j == i ? r : 0.0);
        __syncthreads();
        G[i][j] = v;
        X[i][j] = (i == j) ? 1.0 : 0.0;
        __syncthreads();
    }
    // Gauss-Jordan on the upper triangle, last column first: X <- R^{-1}
    for (int k = 31; k >= 0; --k) {
        const double rkk = G[k][k];
        const double xk = X[k][j] / rkk;  // row k scaled (read before the barrier)
        const double rik = G[i][k];
        __syncthreads();
        if (i == k) X[k][j] = xk;
        else if (i < k) X[i][j] = fma(-rik, xk, X[i][j]);
        __syncthreads();
    }
    Rinv[e] = i <= j ? X[i][j] : 0.0;
    double v;
    if (first) {
        v = i <= j ? G[i][j] : 0.0;
    } else {  // Rtot <- R Rtot (both upper)
        v = 0.0;
        for (int q = i; q <= j; ++q) v = fma(G[i][q], Rt[q][j], v);
        if (i > j) v = 0.0;
    }
    Rtot[e] = v;
    if (e == 0 && bad) atomicMin(flag, tag);
}

// Q = P M for M upper triangular 32 x 32 (column-major), one row per thread
// (P and Q may alias: a thread reads its whole row before writing it).
__global__ void __launch_bounds__(kCqrThreads) cqr_apply(int rows, int b, const double* P, i64 ldp, const double* M,
                                                        double* Q, i64 ldq) {
    __shared__ double Ms[32][33];
    for (int e = threadIdx.x; e < 1024; e += kCqrThreads) Ms[e & 31][e >> 5] = M[e];
    __syncthreads();
    for (int r = blockIdx.x * kCqrThreads + threadIdx.x; r < rows; r += gridDim.x * kCqrThreads) {
        double x[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) x[k] = k < b ? P[r + static_cast<i64>(k) * ldp] : 0.0;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            double sacc = 0.0;
#pragma unroll
            for (int k = 0; k <= j; ++k) sacc = fma(x[k], Ms[k][j], sacc);
            if (j < b) Q[r + static_cast<i64>(j) * ldq] = sacc;
        }
    }
}

// Householder reconstruction (one CTA of 1024 threads, thread = entry (i, j)):
// from Q_1 (top b x b of Q) and the Cholesky-QR factor Rtot -> T (ld 32,
// upper), the top block of V (unit lower), R = S Rtot into the panel's top
// block (ld ldr), Uinv = U^{-1}, tau = diag(T).
__global__ void __launch_bounds__(kCholSmall) cqr_hr(int b, const double* Q, i64 ldq, const double* Rtot, double* T,
                                                    double* V, i64 ldv, double* Rout, i64 ldr, double* Uinv, double* tau) {
    __shared__ double A[32][33], Li[32][33], Ui[32][33];
    __shared__ double s[32];
    const int e = threadIdx.x, i = e & 31, j = e >> 5;
    A[i][j] = (i < b && j < b) ? Q[i + static_cast<i64>(j) * ldq] : (i == j ? 1.0 : 0.0);
    Li[i][j] = (i == j) ? 1.0 : 0.0;
    Ui[i][j] = (i == j) ? 1.0 : 0.0;
    __syncthreads();
    // LU without pivoting of Q_1 - S, s_k = -sign(running pivot): step k (one barrier pair)
    for (int k = 0; k < 32; ++k) {
        const double akk = A[k][k];
        const double sk = k < b ? (akk >= 0.0 ? -1.0 : 1.0) : 0.0;
        const double ukk = akk - sk;  // |ukk| >= 1 for k < b
        const double lik = (i > k) ? A[i][k] / ukk : 0.0;
        const double akj = A[k][j];
        __syncthreads();
        if (e == 0) s[k] = sk;
        if (i == k && j == k) A[k][k] = ukk;
        if (i > k && j == k) A[i][k] = lik;
        if (i > k && j > k) A[i][j] = fma(-lik, akj, A[i][j]);
        __syncthreads();
    }
    // Li = L^{-1} (unit lower; forward Gauss-Jordan), Ui = U^{-1} (upper; backward)
    for (int k = 0; k < 32; ++k) {
        const double lik = (i > k) ? A[i][k] : 0.0;
        const double xk = Li[k][j];
        __syncthreads();
        if (i > k) Li[i][j] = fma(-lik, xk, Li[i][j]);
        __syncthreads();
    }
    for (int k = 31; k >= 0; --k) {
        const double ukk = A[k][k];
        const double xk = Ui[k][j] / ukk;
        const double uik = A[i][k];
        __syncthreads();
        if (i == k) Ui[k][j] = xk;
        else if (i < k) Ui[i][j] = fma(-uik, xk, Ui[i][j]);
        __syncthreads();
    }
    // T = -U S L^{-T}: T(i, j) = -sum_{i <= k <= j} U(i, k) s_k Li(j, k)
    double t = 0.0;
    if (i <= j) {
        for (int k = i; k <= j; ++k) t = fma(A[i][k] * s[k], Li[j][k], t);
        t = -t;
    }
    T[i + 32 * j] = (i < b && j < b) ? t : 0.0;  // the whole block: zero past b (the T aggregation reads all of it)
    if (i < b && j < b) {
        if (i == j) tau[j] = t;
        V[i + static_cast<i64>(j) * ldv] = i > j ? A[i][j] : (i == j ? 1.0 : 0.0);
        if (i <= j) Rout[i + static_cast<i64>(j) * ldr] = s[i] * Rtot[i + 32 * j];
    }
    Uinv[e] = i <= j ? Ui[i][j] : 0.0;
}

// ---------------------------------------------------------------------------
// K4e: batched CholeskyQR2 / shifted CholeskyQR3 of small tall matrices (config
// 5a: 4096 x 5 QRs of 256/320 x 20 per call), one CTA per matrix, the matrix
// column-major in shared memory (ld = 4 mod 16: the DMMA fragment loads below are
// conflict-free) and updated in place. Per pass:
//   G = S^T S      fp64 DMMA m8n8k4, the upper tile pairs of the NT x NT tile
//                  grid (8-column tiles, padded columns read as zero), k split
//                  over kSqGramWarps warps, partials summed in a fixed order
//                  (deterministic);
//   R, R^{-1}      one warp, lane c holding column c of [G | I] (the G part in
//                  registers, the I part in registers for NT <= 3, else in G's
//                  storage): Gaussian elimination with symmetric multipliers (row
//                  k of the trailing upper part, broadcast through shared
//                  memory); the scaled rows give R and R^{-T};
//   S <- S R^{-1}  fp64 DMMA, warp per 8-row tile, R^{-1} fragments in registers.
// Passes: CholeskyQR2 (plain, plain with the ||G - I||_F <= 1/2 check: Q_1 well
// conditioned, so the second pass is accurate to O(u)); if that breaks down (a
// non-positive or non-finite pivot, or the check), the CTA reloads A and runs
// the shifted CholeskyQR3 (s = 11 (m n + n (n+1)) u tr(G), then plain, then plain
// with the check). A breakdown there sets flags[b] (never cleared; the batched
// caller redoes that tensor on the Householder path).
constexpr int kSqGramWarps = 4;
#ifndef SQ_MINB
#define SQ_MINB 2  // CTAs per SM the register budget is sized for (3 spills the NT = 3 Cholesky)
#endif

__device__ __forceinline__ void sq_dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

__host__ __device__ constexpr int sq_ld(int m) { return ((m + 7) / 8 * 8 + 11) / 16 * 16 + 4; }

template <int NT>
__host__ __device__ constexpr int sq_pairs() {
    return NT * (NT + 1) / 2;
}

template <int NT>
std::size_t sq_smem(int m, int n) {
    const int np = 8 * NT;
    return sizeof(double) * (static_cast<std::size_t>(n) * sq_ld(m) + kSqGramWarps * sq_pairs<NT>() * 64 +
                             static_cast<std::size_t>(np) * (np + 2));
}

#ifdef TTR_SQ_TRACE
__device__ unsigned long long g_sq_trace[8];
#define SQ_T(i) do { if (threadIdx.x == 0) { long long t_ = clock64(); atomicAdd(&g_sq_trace[i], static_cast<unsigned long long>(t_ - t_last)); t_last = t_; } } while (0)
#else
#define SQ_T(i) do { } while (0)
#endif

template <int NT>
__global__ void __launch_bounds__(256, SQ_MINB) cholqr_small_kernel(int m, int n, const double* A, i64 lda, i64 sA, double* Q,
                                                          i64 ldq, i64 sQ, double coeff, int* flags) {
#ifdef TTR_SQ_TRACE
    long long t_last = clock64();
#endif
    constexpr int NP = 8 * NT, NPAIR = sq_pairs<NT>();
    extern __shared__ __align__(16) double sq[];
    const int ld = sq_ld(m), m8 = (m + 7) / 8 * 8;
    double* S = sq;                                   // [n][ld]
    double* part = S + static_cast<i64>(n) * ld;      // [kSqGramWarps][NPAIR][64]
    double* G = part + kSqGramWarps * NPAIR * 64;     // [NP][NP + 1]: G, then R^{-T}
    __shared__ int bad;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    const int lr = lane & 3, lc = lane >> 2;
    A += blockIdx.x * sA;
    Q += blockIdx.x * sQ;
    // S <- A: 16-byte cp.async chunks when the columns allow (all in flight at
    // once), else plain loads; rows m..m8-1 zero
    auto load_s = [&] {
        if ((m & 1) == 0 && (lda & 1) == 0 && (reinterpret_cast<std::uintptr_t>(A) & 15) == 0) {
            const int hm = m >> 1;
            for (int e = tid; e < n * hm; e += blockDim.x) {
                const int c = e / hm, r = 2 * (e - c * hm);
                const unsigned dst = smem_u32(S + c * ld + r);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(A + r + static_cast<i64>(c) * lda));
            }
            asm volatile("cp.async.commit_group;\n" ::);
        } else {
            for (int e = tid; e < n * m; e += blockDim.x) {
                const int c = e / m, r = e - c * m;
                S[c * ld + r] = A[r + static_cast<i64>(c) * lda];
            }
        }
        for (int e = tid; e < n * (m8 - m); e += blockDim.x) {
            const int c = e / (m8 - m), r = m + e - c * (m8 - m);
            S[c * ld + r] = 0.0;
        }
        if (tid == 0) bad = 0;
        asm volatile("cp.async.wait_all;\n" ::);
        __syncthreads();
    };
    load_s();
    SQ_T(0);
    // CholeskyQR2 (plain, plain with the check) first; if it breaks down, the
    // shifted CholeskyQR3 (shifted, plain, plain with the check) from A again
    bool fallback = false;
    for (int stage = 0; stage < (fallback ? 3 : 2);) {
        const int kind = fallback ? stage : stage + 1;  // 0 shifted, 1 plain, 2 plain + check
        // ---- Gram partials: warp w takes k-steps w, w + kSqGramWarps, ... ----
        if (warp < kSqGramWarps) {
            double acc[NPAIR][2];
#pragma unroll
            for (int p = 0; p < NPAIR; ++p) acc[p][0] = acc[p][1] = 0.0;
            for (int k0 = 4 * warp; k0 < m8; k0 += 4 * kSqGramWarps) {
                double v[NT];
#pragma unroll
                for (int t = 0; t < NT; ++t) {
                    const int col = 8 * t + lc;
                    v[t] = (col < n) ? S[col * ld + k0 + lr] : 0.0;
                }
                int p = 0;
#pragma unroll
                for (int i = 0; i < NT; ++i)
#pragma unroll
                    for (int j = i; j < NT; ++j, ++p) sq_dmma(acc[p][0], acc[p][1], v[i], v[j]);
            }
#pragma unroll
            for (int p = 0; p < NPAIR; ++p) {
                part[(warp * NPAIR + p) * 64 + 2 * lane] = acc[p][0];
                part[(warp * NPAIR + p) * 64 + 2 * lane + 1] = acc[p][1];
            }
        }
        __syncthreads();
        SQ_T(1);
        // ---- fixed-order sum of the partials into G (tile pair p = (i, j), i <= j) ----
        for (int e = tid; e < NPAIR * 64; e += blockDim.x) {
            const int p = e >> 6, q = e & 63;
            double g = 0.0;
#pragma unroll
            for (int w = 0; w < kSqGramWarps; ++w) g += part[(w * NPAIR + p) * 64 + q];
            int i = 0, pp = p;
            while (pp >= NT - i) {
                pp -= NT - i;
                ++i;
            }
            const int j = i + pp;
            const int ql = q >> 1;  // C fragment: row ql >> 2, columns 2 (ql & 3) + (q & 1)
            G[(8 * i + (ql >> 2)) * (NP + 1) + 8 * j + 2 * (ql & 3) + (q & 1)] = g;
        }
        __syncthreads();
        SQ_T(2);
        // ---- R and R^{-1} by one warp: lane c holds column c of the upper part
        // of G and column c of the identity (registers for NT <= 3, else the
        // identity part in G's own storage); padded steps k >= n are skipped ----
        if (warp == 0) {
            constexpr bool kXReg = NT <= 3;
            double L[NP], XR[kXReg ? NP : 1];
            double* xs = G + lane;  // X[k][lane] = xs[k * (NP + 1)] (kXReg: at the end)
            double* rowk = G + NP * (NP + 1);  // [NP], 16-byte aligned
#pragma unroll
            for (int k = 0; k < NP; ++k) {
                const bool real = lane < n;
                L[k] = real ? (k <= lane ? G[k * (NP + 1) + lane] : 0.0) : (k == lane ? 1.0 : 0.0);
            }
            auto xget = [&](int k) -> double {
                if constexpr (kXReg) return XR[k];
                else return (lane < NP) ? xs[k * (NP + 1)] : 0.0;
            };
            auto xset = [&](int k, double v) {
                if constexpr (kXReg) XR[k] = v;
                else if (lane < NP) xs[k * (NP + 1)] = v;
            };
#pragma unroll
            for (int k = 0; k < NP; ++k) xset(k, (k == lane) ? 1.0 : 0.0);
            if (kind != 1) {
                double acc = 0.0;
                if (lane < n) {
#pragma unroll
                    for (int k = 0; k < NP; ++k)
                        if (k <= lane) {
                            if (kind == 0) {
                                acc += (k == lane) ? L[k] : 0.0;
                            } else {
                                const double dd = L[k] - (k == lane ? 1.0 : 0.0);
                                acc = fma(k == lane ? 1.0 : 2.0, dd * dd, acc);
                            }
                        }
                }
                for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
                if (kind == 0) {
                    const double shift = coeff * acc;
#pragma unroll
                    for (int k = 0; k < NP; ++k)
                        if (k == lane && lane < n) L[k] += shift;
                } else if (!(acc <= 0.25) && lane == 0) {
                    bad = 1;
                }
            }
            bool broke = false;
#pragma unroll
            for (int k = 0; k < NP; ++k) {
                if (k < n) {
                    // row k of the trailing part, broadcast through shared memory
                    __syncwarp();
                    if (lane < NP) rowk[lane] = L[k];
                    __syncwarp();
                    double piv = rowk[k];
                    if (!(piv > 0.0) || !isfinite(piv)) {
                        broke = true;
                        piv = 1.0;
                    }
                    const double is = rsqrt(piv), rp = is * is;
                    const double fl = L[k] * rp;
                    const double xk = xget(k);
                    const double fx = xk * rp;
#pragma unroll
                    for (int i2 = (k + 1) & ~1; i2 < NP; i2 += 2) {
                        const double2 v = *reinterpret_cast<const double2*>(rowk + i2);
                        if (i2 > k) {
                            L[i2] = fma(-v.x, fl, L[i2]);
                            xset(i2, fma(-v.x, fx, xget(i2)));
                        }
                        L[i2 + 1] = fma(-v.y, fl, L[i2 + 1]);
                        xset(i2 + 1, fma(-v.y, fx, xget(i2 + 1)));
                    }
                    L[k] *= is;
                    xset(k, xk * is);
                }
            }
            if (broke && lane == 0) bad = 1;
            if constexpr (kXReg) {
                if (lane < NP) {
#pragma unroll
                    for (int k = 0; k < NP; ++k) xs[k * (NP + 1)] = XR[k];
                }
            }
            // now X = R^{-T}: R^{-1}[kk][jj] = G[jj * (NP + 1) + kk]
        }
        __syncthreads();
        SQ_T(3);
        if (!fallback && bad) {
            fallback = true;
            stage = 0;
            __syncthreads();
            load_s();
            continue;
        }
        // ---- S <- S R^{-1}: warp per 8-row tile, R^{-1} fragments in registers ----
        {
            double bf[NT][2 * NT];  // bf[j][ks]: k = 4 ks + lr, column 8 j + lc (ks < 2 (j + 1))
#pragma unroll
            for (int j = 0; j < NT; ++j)
#pragma unroll
                for (int ks = 0; ks < 2 * NT; ++ks)
                    bf[j][ks] = (ks < 2 * (j + 1)) ? G[(8 * j + lc) * (NP + 1) + 4 * ks + lr] : 0.0;
            for (int rt = warp; rt < m8 / 8; rt += nwarps) {
                const int r0 = 8 * rt;
                double af[2 * NT];
#pragma unroll
                for (int ks = 0; ks < 2 * NT; ++ks) {
                    const int col = 4 * ks + lr;
                    af[ks] = (col < n) ? S[col * ld + r0 + lc] : 0.0;
                }
                double cc[NT][2];
#pragma unroll
                for (int j = 0; j < NT; ++j) {
                    cc[j][0] = cc[j][1] = 0.0;
#pragma unroll
                    for (int ks = 0; ks < 2 * (j + 1); ++ks) sq_dmma(cc[j][0], cc[j][1], af[ks], bf[j][ks]);
                }
                __syncwarp();
#pragma unroll
                for (int j = 0; j < NT; ++j)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int col = 8 * j + 2 * lr + e;
                        if (col < n) S[col * ld + r0 + lc] = cc[j][e];
                    }
            }
        }
        __syncthreads();
        SQ_T(4);
        ++stage;
    }
    if ((m & 1) == 0 && (ldq & 1) == 0 && (reinterpret_cast<std::uintptr_t>(Q) & 15) == 0) {
        const int hm = m >> 1;
        for (int e = tid; e < n * hm; e += blockDim.x) {
            const int c = e / hm, r = 2 * (e - c * hm);
            *reinterpret_cast<double2*>(Q + r + static_cast<i64>(c) * ldq) = *reinterpret_cast<const double2*>(S + c * ld + r);
        }
    } else {
        for (int e = tid; e < n * m; e += blockDim.x) {
            const int c = e / m, r = e - c * m;
            Q[r + static_cast<i64>(c) * ldq] = S[c * ld + r];
        }
    }
    SQ_T(5);
    if (tid == 0 && bad) flags[blockIdx.x] = 1;  // sticky across the modes of one call
}

// ---------------------------------------------------------------------------
// K4f: the K4d panel (Cholesky-QR + Householder reconstruction) as ONE
// cooperative kernel, so a 32-column panel costs 4-6 grid barriers instead of
// one cross-CTA exchange per column (qr_panel.cuh: ~4.5 us per column at
// 40,960 rows) or K4d's eleven dependent launches. CTA `rank` keeps its rpc
// rows of the panel column-major in shared memory (the K4e layout, ld = 4 mod
// 16) plus a shadow copy of the panel's top b x b block, which takes every
// S <- S R^{-1} with the own rows: all CTAs then hold the same Q_1 bit for bit
// and run the Householder reconstruction redundantly (no broadcast barrier).
// Per pass:
//   partial Gram of the own rows   fp64 DMMA, upper 8 x 8 tile pairs, k split
//                                  over kFpGramWarps warps, fixed-order sums;
//   grid sum                       partials to global, grid barrier, CTA `rank`
//                                  sums a slice of the 640 entries over all
//                                  CTAs (one warp per entry, fixed order), grid
//                                  barrier, every CTA reads the 640 sums: all
//                                  CTAs see the same G and take the same branches;
//   R, R^{-T}                      warp 0 (the K4e elimination), redundantly;
//   S <- S R^{-1}                  fp64 DMMA, warp per 8-row tile.
// A pass factors G as it is unless a pivot fell below 1e-6 of its diagonal entry
// (or was not positive), in which case the same G is refactored with the sCQR
// shift s = coeff tr(G) (each shifted pass lowers the condition number by about
// sqrt(s)/||A||: one for kappa ~ 1e8, two for the 1e8-1e12 of a panel that
// straddles the numerical rank of the sketch). Every pass after the first tests
// ||G - I||_F <= 1/2 first: when it holds the pass is the last one (its input was
// well conditioned, so its output is orthonormal to O(u)); a seventh pass, a
// non-positive pivot under the shift or a non-finite entry is a breakdown (flag
// <- tag, nothing written; the caller reruns the QR on the Householder panels).
// A well conditioned panel takes two passes (4 grid barriers), an ill
// conditioned one three or four.
// Then (Ballard et al. 2014, as cqr_hr above): LU without pivoting of Q_1 - S,
// V_2 = Q_2 U^{-1} by the same DMMA apply, CTA 0 writes V_1 = L, T = -U S L^{-T},
// tau = diag(T) and R = S R_p ... R_1 into the panel's top block.
constexpr int kFpThreads = 512, kFpWarps = kFpThreads / 32, kFpGramWarps = 8, kFpFacWarps = 8, kFpPairs = 10, kFpEntries = kFpPairs * 64,
              kFpMaxRpc = 320, kFpMaxPasses = 6, kFpDirectG = 32;
constexpr double kFpAnalyticDev2 = 1e-18;  // ||G - I||_F^2 below which a pass takes the first-order factor

struct FusedPanelArgs {
    int rows, b, rpc;  // rpc: rows per CTA, a multiple of 8, <= kFpMaxRpc
    double* P;         // rows x b panel (R is written into its top block)
    i64 ldp;
    double* V;
    i64 ldv;
    double* T;
    double* tau;
    double* gpart;  // [gridDim.x][640] partial Grams (upper tile pairs, C-fragment order)
    double* gsum;   // [640] their sum
    double coeff;   // shift coefficient: s = coeff * trace(G)
    int* flag;
    int tag;
    long long* trace;  // [64] phase time stamps of CTA 0 (diagnostics) or null
    // hr = 0: a plain thin QR of the panel instead of the blocked QR's (V, T, R):
    // Q = P R^{-1} to V (ldv) when V is set, R = R_p ... R_1 (positive diagonal) to
    // Rout (ldr) when set; P is not written and no reconstruction runs
    int hr;
    double* Rout;
    i64 ldr;
};

__host__ __device__ constexpr int fp_ld(int rpc) { return sq_ld(rpc + 32); }
__host__ __device__ constexpr std::size_t fp_smem_doubles(int rpc) {
    return static_cast<std::size_t>(32) * fp_ld(rpc) + kFpGramWarps * kFpEntries + 4 * (32 * 33 + 2) + 5 * 32;
}

__global__ void __launch_bounds__(kFpThreads, 1) cqr_panel_fused(FusedPanelArgs p) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(16) double fsm[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int lr = lane & 3, lc = lane >> 2;
    const int rank = blockIdx.x, G = gridDim.x;
    const int b = p.b, rpc = p.rpc;
    const int r0 = rank * rpc, nr = max(0, min(p.rows, r0 + rpc) - r0);
    const int mt = rpc + 32, ld = fp_ld(rpc);
    constexpr int LM = 33, MS = 32 * 33 + 1;  // small-matrix row stride (odd: conflict-free columns), slot size (even)
    double* S = fsm;                                // [32][ld]: own rows 0..rpc-1, shadow top block rpc..rpc+31
    double* part = S + 32 * ld;                     // [kFpGramWarps][640]; the HR scratch afterwards
    double* Gm = part + kFpGramWarps * kFpEntries;  // [32][33] the summed Gram (upper)
    double* RX = Gm + MS + 1;    // [32][33] row k: R(k, c) for c >= k, X(k, c) = R^{-T}(k, c) for c < k
    double* RTa = RX + MS + 1;   // [32][33] R_p ... R_1 (CTA 0), ping
    double* RTb = RTa + MS + 1;  // pong
    double* rowk = RTb + MS + 1;  // [2][32] the pivot row, double buffered
    double* d0s = rowk + 64;      // [32] (spare)
    double* xdg = d0s + 32;       // [32] X(k, k) (then U^{-1}(k, k))
    double* sg = xdg + 32;        // [32] HR signs
    __shared__ int s_bad, s_final;
    int stamp = 0;
    auto mark = [&] {
        if (p.trace && rank == 0 && tid == 0 && stamp < 64) p.trace[stamp] = clock64();
        ++stamp;
    };
    mark();
    // ---- load: own rows, zero padding, shadow top block (all loads in flight) ----
    {
        constexpr int kLd = (32 * (kFpMaxRpc + 32) + kFpThreads - 1) / kFpThreads;  // 22 elements per thread
        double v[kLd];
#pragma unroll
        for (int u = 0; u < kLd; ++u) {
            const int e = tid + u * kFpThreads, c = e / mt, r = e - c * mt;
            v[u] = 0.0;
            if (c < b) {
                if (r < nr) v[u] = p.P[(r0 + r) + static_cast<i64>(c) * p.ldp];
                else if (r >= rpc && r - rpc < b) v[u] = p.P[(r - rpc) + static_cast<i64>(c) * p.ldp];
            }
        }
#pragma unroll
        for (int u = 0; u < kLd; ++u) {
            const int e = tid + u * kFpThreads, c = e / mt, r = e - c * mt;
            if (c < 32) S[c * ld + r] = v[u];
        }
    }
    if (tid == 0) {
        s_bad = 0;
        s_final = 0;
    }
    __syncthreads();
    mark();

    // S <- S M on `ntiles` 8-row tiles, M upper triangular in the RX/xdg layout:
    // M(k, c) = RX[c][k] for k < c, xdg[c] for k = c
    auto apply = [&](int ntiles, int nwarps) {
        double bf[4][8];
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                const int c = 8 * j + lc, k = 4 * ks + lr;
                bf[j][ks] = (ks < 2 * (j + 1)) ? (k < c ? RX[c * LM + k] : (k == c ? xdg[c] : 0.0)) : 0.0;
            }
        for (int rt = warp; rt < ntiles; rt += nwarps) {
            const int rr = 8 * rt;
            double af[8];
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) af[ks] = S[(4 * ks + lr) * ld + rr + lc];
            double cc[4][2];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                cc[j][0] = cc[j][1] = 0.0;
#pragma unroll
                for (int ks = 0; ks < 2 * (j + 1); ++ks) sq_dmma(cc[j][0], cc[j][1], af[ks], bf[j][ks]);
            }
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int col = 8 * j + 2 * lr + e;
                    if (col < b) S[col * ld + rr + lc] = cc[j][e];
                }
        }
    };

    double* RT = RTa;  // current R_p ... R_1 (CTA 0)
    bool done = false;
    for (int pass = 0; !done; ++pass) {
        // ---- partial Gram of the own rows ----
        if (warp < kFpGramWarps) {
            double acc[kFpPairs][2];
#pragma unroll
            for (int q = 0; q < kFpPairs; ++q) acc[q][0] = acc[q][1] = 0.0;
            for (int k0 = 4 * warp; k0 < rpc; k0 += 4 * kFpGramWarps) {
                double v[4];
#pragma unroll
                for (int t = 0; t < 4; ++t) v[t] = S[(8 * t + lc) * ld + k0 + lr];
                int q = 0;
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = i; j < 4; ++j, ++q) sq_dmma(acc[q][0], acc[q][1], v[i], v[j]);
            }
#pragma unroll
            for (int q = 0; q < kFpPairs; ++q)
                *reinterpret_cast<double2*>(part + (warp * kFpPairs + q) * 64 + 2 * lane) = make_double2(acc[q][0], acc[q][1]);
        }
        __syncthreads();
        // few CTAs (kFpDirectG): every CTA sums all partials itself after ONE barrier (the
        // partials double-buffered by pass parity: the next pass's writes cannot overtake
        // a late reader), else the two-stage sum below
        const bool direct = G <= kFpDirectG;
        double* gp = p.gpart + (direct && (pass & 1) ? static_cast<i64>(G) * kFpEntries : 0);
        for (int e = tid; e < kFpEntries; e += kFpThreads) {
            double g = 0.0;
#pragma unroll
            for (int w = 0; w < kFpGramWarps; ++w) g += part[w * kFpEntries + e];
            gp[static_cast<i64>(rank) * kFpEntries + e] = g;
        }
        mark();
        grid.sync();
        mark();
        if (direct) {
            for (int e = tid; e < kFpEntries; e += kFpThreads) {
                double a = 0.0;
                for (int g0 = 0; g0 < G; g0 += 8) {  // eight loads in flight, summed in rank order
                    double v[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        v[u] = (g0 + u < G) ? __ldcg(gp + static_cast<i64>(g0 + u) * kFpEntries + e) : 0.0;
#pragma unroll
                    for (int u = 0; u < 8; ++u) a += v[u];
                }
                const int q = e >> 6, f = e & 63;
                int i = 0, qq = q;
                while (qq >= 4 - i) {
                    qq -= 4 - i;
                    ++i;
                }
                const int j = i + qq, fl = f >> 1;
                Gm[(8 * i + (fl >> 2)) * LM + 8 * j + 2 * (fl & 3) + (f & 1)] = a;
            }
            mark();
            mark();
        } else {
        // ---- slice of the grid sum: one warp per entry, fixed order ----
        {
            const int eper = (kFpEntries + G - 1) / G, e0 = rank * eper;
            for (int ee = warp; ee < eper; ee += kFpWarps) {
                const int e = e0 + ee;
                if (e < kFpEntries) {
                    double a = 0.0;
                    for (int g = lane; g < G; g += 32) a += __ldcg(p.gpart + static_cast<i64>(g) * kFpEntries + e);
                    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
                    if (lane == 0) p.gsum[e] = a;
                }
            }
        }
        mark();
        grid.sync();
        mark();
        for (int e = tid; e < kFpEntries; e += kFpThreads) {
            const int q = e >> 6, f = e & 63;
            int i = 0, qq = q;
            while (qq >= 4 - i) {
                qq -= 4 - i;
                ++i;
            }
            const int j = i + qq, fl = f >> 1;  // C fragment: row fl >> 2, columns 2 (fl & 3) + (f & 1)
            Gm[(8 * i + (fl >> 2)) * LM + 8 * j + 2 * (fl & 3) + (f & 1)] = __ldcg(p.gsum + e);
        }
        }  // two-stage sum
        __syncthreads();
        // ---- R and R^{-T} by warps 0..7 (kFpFacWarps), four rows each, lane = column c.
        // One array holds both triangles: entry (i, c) is G(i, c) for i <= c and, as the
        // elimination reaches it, X(i, c) for i > c (the identity carried along; X(c, c)
        // = 1 implicit). Step k: the owner of row k publishes it, one named barrier, then
        // every row i > k takes W(i, c) -= G(k, i) f with ONE per-column factor: columns
        // c > k are in their G part (f = G(k, c)/piv, rows i <= c), columns c <= k in their
        // X part (f = X(k, c)/piv, every row). The scaled row k is R(k, c) for c >= k and
        // X(k, c) = R^{-T}(k, c) for c < k. Every warp derives the same pivots and flags. ----
        if (warp < kFpFacWarps) {
            double W[4];
            bool broke = false, ill = false, fin = false;
            double dev2 = 1.0;
            const bool real = lane < b;
            for (int attempt = 0; attempt < 2; ++attempt) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int i = 4 * warp + q;
                    W[q] = real ? (i <= lane ? Gm[i * LM + lane] : 0.0) : (i == lane ? 1.0 : 0.0);
                }
                const double dg = real ? Gm[lane * LM + lane] : 1.0;
                double shift = 0.0;
                if (attempt == 1) {  // sCQR shift
                    double tr = real ? dg : 0.0;
                    for (int o = 16; o > 0; o >>= 1) tr += __shfl_xor_sync(0xffffffffu, tr, o);
                    shift = p.coeff * tr;
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if (4 * warp + q == lane && real) W[q] += shift;
                }
                if (pass > 0) {  // ||G - I||_F^2 over the real columns (upper part counted twice)
                    double acc = 0.0;
                    if (real) {
                        for (int i = 0; i <= lane; ++i) {
                            const double dd = Gm[i * LM + lane] - (i == lane ? 1.0 : 0.0);
                            acc = fma(i == lane ? 1.0 : 2.0, dd * dd, acc);
                        }
                    }
                    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
                    fin = acc <= 0.25;  // false for NaN
                    dev2 = acc;
                }
                broke = false;
                ill = false;
                if (pass > 0 && dev2 <= kFpAnalyticDev2) {
                    // G = I + E with ||E||_F <= 1e-9: R = I + striu(E) + diag(E)/2 and R^{-1} = I -
                    // striu(E) - diag(E)/2 up to O(||E||^2) <= 1e-18 -- no elimination sweep
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int i = 4 * warp + q;
                        if (i < b) {
                            double v;
                            if (!real) v = 0.0;
                            else if (i < lane) v = Gm[i * LM + lane];                       // R(i, c) = E(i, c)
                            else if (i == lane) v = 1.0 + 0.5 * (Gm[i * LM + i] - 1.0);     // R(i, i)
                            else v = -Gm[lane * LM + i];                                    // X(i, c) = -E(c, i)
                            RX[i * LM + lane] = v;
                            if (i == lane) xdg[i] = 1.0 - 0.5 * (Gm[i * LM + i] - 1.0);
                        }
                    }
                    break;
                }
                // one elimination step; Q = k & 3 is a compile-time constant so that the
                // owner's row W[Q] is a register (a run-time select puts W in local memory)
                auto chol_step = [&](int k, auto qc) {
                    constexpr int Q = decltype(qc)::value;
                    double* rb = rowk + 32 * (k & 1);
                    const bool owner = warp == (k >> 2);
                    if (owner) rb[lane] = W[Q];
                    asm volatile("bar.sync 1, %0;" ::"n"(kFpFacWarps * 32) : "memory");
                    double piv = rb[k];
                    if (!(piv > 0.0) || !isfinite(piv)) {
                        broke = true;
                        piv = 1.0;
                    }
                    // original diagonal of column k: Gm (+ shift on the second attempt)
                    if (!(piv > 1e-6 * (Gm[k * LM + k] + shift))) ill = true;
                    const double is = rsqrt(piv), rp = is * is;
                    const double f = ((lane == k) ? 1.0 : rb[lane]) * rp;
                    const bool xpart = lane <= k;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int i2 = 4 * warp + q;
                        const double v = rb[i2];
                        const double upd = fma(-v, f, W[q]);
                        W[q] = (i2 > k && (xpart || i2 <= lane)) ? upd : W[q];
                    }
                    if (owner) {
                        W[Q] *= is;
                        RX[k * LM + lane] = W[Q];
                        if (lane == k) xdg[k] = is;
                    }
                };
#pragma unroll 1
                for (int k0 = 0; k0 < b; k0 += 4) {
                    chol_step(k0, std::integral_constant<int, 0>{});
                    if (k0 + 1 < b) chol_step(k0 + 1, std::integral_constant<int, 1>{});
                    if (k0 + 2 < b) chol_step(k0 + 2, std::integral_constant<int, 2>{});
                    if (k0 + 3 < b) chol_step(k0 + 3, std::integral_constant<int, 3>{});
                }
                if (!(attempt == 0 && (broke || ill))) break;
                asm volatile("bar.sync 1, %0;" ::"n"(kFpFacWarps * 32) : "memory");  // rowk reused by the second attempt
            }
            for (int i = b + warp; i < 32; i += kFpFacWarps) {  // padded rows: identity
                RX[i * LM + lane] = (i == lane) ? 1.0 : 0.0;
                if (lane == i) xdg[i] = 1.0;
            }
            if (tid == 0) {
                if (broke || (pass > 0 && !fin && pass + 1 >= kFpMaxPasses)) s_bad = 1;
                s_final = fin ? 1 : 0;
            }
        }
        __syncthreads();
        mark();
        if (s_bad) {  // the same decision in every CTA (identical G)
            if (rank == 0 && tid == 0) {
                atomicMin(p.flag, p.tag);
                if (p.trace) p.trace[63] = -(pass + 1);  // diagnostics: the pass that broke down
            }
            return;
        }
        done = s_final != 0;
        if (rank == 0) {  // RT <- R RT (first pass: RT = R), two entries per thread
            double* RTn = (RT == RTa) ? RTb : RTa;
            for (int e = tid; e < 1024; e += kFpThreads) {
                const int i = e >> 5, c = e & 31;
                double a = 0.0;
                if (i <= c) {
                    if (pass == 0) a = RX[i * LM + c];
                    else
                        for (int q = i; q <= c; ++q) a = fma(RX[i * LM + q], RT[q * LM + c], a);
                }
                RTn[i * LM + c] = a;
            }
            RT = RTn;
        }
        apply(mt / 8, kFpWarps);
        __syncthreads();
        mark();
    }

    if (!p.hr) {  // plain thin QR: Q from the own rows, R from CTA 0
        if (p.V) {
            for (int c = warp; c < b; c += kFpWarps) {
                double* dst = p.V + static_cast<i64>(c) * p.ldv;
                for (int r = lane; r < nr; r += 32) dst[r0 + r] = S[c * ld + r];
            }
        }
        if (rank == 0 && p.Rout) {
            for (int e = tid; e < 1024; e += kFpThreads) {
                const int i = e & 31, jj = e >> 5;
                if (i < b && jj < b) p.Rout[i + static_cast<i64>(jj) * p.ldr] = (i <= jj) ? RT[i * LM + jj] : 0.0;
            }
        }
        return;
    }

    // ---- Householder reconstruction from Q_1 (the shadow block), redundantly in every
    // CTA: ONE Gauss-Jordan sweep over A = Q_1 - S by warps 0..7 (four rows each, lane =
    // column), one named barrier per step. Step k: the owner publishes row k, every warp
    // the column-k entries of its rows; s_k = -sign(a_kk), u_kk = a_kk - s_k; every row
    // i != k takes A(i, c) -= m_i A(k, c) for c > k with m_i = A(i, k) / u_kk and keeps m_i
    // in place of A(i, k). Rows below k thus build L and U (LU without pivoting, the
    // pivot row saved to LUm as it is used), rows above k reduce U to its diagonal:
    // their multipliers are U^{-1}(i, k) = -m_i / u_ii. ----
    double* LUm = part;           // [32][33] L \ U
    double* ZS = LUm + MS + 1;    // [32][33] L^{-1} (CTA 0)
    double* colk = ZS + MS + 1;   // [2][32] column k of the sweep
    double* zrow = colk + 64;     // [2][32] row k of L^{-1} so far (CTA 0)
    if (warp < kFpFacWarps) {
        double W[4], Z[4];  // Z: rows of L^{-1} (CTA 0 only: the identity under the same row operations)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int i = 4 * warp + q;
            W[q] = (i < b && lane < b) ? S[lane * ld + rpc + i] : (i == lane ? 1.0 : 0.0);
            Z[q] = (i == lane) ? 1.0 : 0.0;
        }
        auto gj_step = [&](int k, auto qc) {  // Q = k & 3 at compile time (see chol_step)
            constexpr int Q = decltype(qc)::value;
            double* rb = rowk + 32 * (k & 1);
            double* cb = colk + 32 * (k & 1);
            double* zb = zrow + 32 * (k & 1);
            const bool owner = warp == (k >> 2);
            if (owner) {
                rb[lane] = W[Q];
                if (rank == 0) zb[lane] = Z[Q];
            }
            if (lane == k) {
#pragma unroll
                for (int q = 0; q < 4; ++q) cb[4 * warp + q] = W[q];
            }
            asm volatile("bar.sync 1, %0;" ::"n"(kFpFacWarps * 32) : "memory");
            const double akk = rb[k];
            const double sk = k < b ? (akk >= 0.0 ? -1.0 : 1.0) : 0.0;
            const double ukk = akk - sk;  // |ukk| >= 1 for k < b
            const double inv = 1.0 / ukk;
            const double rkc = rb[lane];
            const double zkc = rank == 0 ? zb[lane] : 0.0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int i = 4 * warp + q;
                const double m = cb[i] * inv;
                const double upd = fma(-m, rkc, W[q]);
                const double wq = (lane > k) ? upd : ((lane == k) ? m : W[q]);
                const double zu = fma(-m, zkc, Z[q]);
                if (!(owner && q == Q)) {
                    W[q] = wq;
                    if (rank == 0 && i > k) Z[q] = zu;
                }
            }
            if (owner) {
                if (lane == k) {
                    W[Q] = ukk;
                    sg[k] = sk;
                }
                if (lane >= k) LUm[k * LM + lane] = W[Q];  // U(k, c), c >= k
            }
        };
#pragma unroll 1
        for (int k0 = 0; k0 < 32; k0 += 4) {
            gj_step(k0, std::integral_constant<int, 0>{});
            gj_step(k0 + 1, std::integral_constant<int, 1>{});
            gj_step(k0 + 2, std::integral_constant<int, 2>{});
            gj_step(k0 + 3, std::integral_constant<int, 3>{});
        }
        // L below the diagonal; U^{-1} into the apply layout (RX/xdg; R no longer needed)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int i = 4 * warp + q;
            const double rd = 1.0 / __shfl_sync(0xffffffffu, W[q], i);
            if (lane < i) LUm[i * LM + lane] = W[q];
            else if (lane == i) xdg[i] = rd;
            else RX[lane * LM + i] = -W[q] * rd;
            if (rank == 0) ZS[i * LM + lane] = Z[q];
        }
    }
    __syncthreads();
    mark();
    apply(rpc / 8, kFpWarps);  // V_2 = Q_2 U^{-1} on the own rows
    __syncthreads();
    // ---- V: own rows (global rows < b: the unit lower L of the LU) ----
    for (int c = warp; c < b; c += kFpWarps) {
        double* dst = p.V + static_cast<i64>(c) * p.ldv;
        for (int r = lane; r < nr; r += 32) {
            const int g = r0 + r;
            double v;
            if (g >= b) v = S[c * ld + r];
            else v = g > c ? LUm[g * LM + c] : (g == c ? 1.0 : 0.0);
            dst[g] = v;
        }
    }
    if (rank == 0) {
        // T = -U S L^{-T}: T(i, j) = -sum_{i <= k <= j} U(i, k) s_k Z(j, k); R = S RT
        for (int e = tid; e < 1024; e += kFpThreads) {
            const int i = e & 31, jj = e >> 5;
            double t = 0.0;
            if (i <= jj) {
                for (int k = i; k <= jj; ++k) t = fma(LUm[i * LM + k] * sg[k], ZS[jj * LM + k], t);
                t = -t;
            }
            // the whole 32 x 32 block (zero past b: the T aggregation reads all of it)
            p.T[i + 32 * jj] = (i < b && jj < b) ? t : 0.0;
            if (i < b && jj < b) {
                if (i == jj) p.tau[jj] = t;
                if (i <= jj) p.P[i + static_cast<i64>(jj) * p.ldp] = sg[i] * RT[i * LM + jj];
            }
        }
    }
    mark();
}

}  // namespace

// Passes: two shifted (each lowers kappa by ~sqrt(11 (mn + n^2) u), enough for
// the ~1e10-1e12 condition numbers of the sweep's sketches), then two plain
// (CholeskyQR2), the last one checking that its Gram matrix is close to I.
constexpr int kCholQrPasses = 4, kCholQrShifted = 2;

bool cholqr_fits(i64 m, i64 n) { return n >= 1 && n <= kCholQrMaxN && m >= n; }

int* Ctx::qr_flag_dev() {
    if (!qr_flag) {
        TTR_CUDA(cudaMalloc(reinterpret_cast<void**>(&qr_flag), sizeof(int)));
        TTR_CUDA(cudaMemsetAsync(qr_flag, 0x7f, sizeof(int), stream));
    }
    return qr_flag;
}

void Ctx::qr_flag_reset() { TTR_CUDA(cudaMemsetAsync(qr_flag_dev(), 0x7f, sizeof(int), stream)); }

int Ctx::qr_flag_read() {
    int* hf = reinterpret_cast<int*>(host_scalars + 8);
    TTR_CUDA(cudaMemcpyAsync(hf, qr_flag_dev(), sizeof(int), cudaMemcpyDeviceToHost, stream));
    TTR_CUDA(cudaStreamSynchronize(stream));
    return *hf == kQrNoBreakdown ? -1 : *hf;
}

void thin_qr_cholesky(Ctx& c, i64 m, i64 n, const double* A, i64 lda, double* Q, i64 ldq, double* R, i64 ldr,
                      int tag) {
    if (!cholqr_fits(m, n)) fail(Errc::InvalidArgument, "sCQR: shape outside the Cholesky-QR path");
    c.charge_qr(4ULL * static_cast<std::uint64_t>(m) * n * n);  // the reference's Householder charge
    const double u = DBL_EPSILON / 2;
    const double coeff = 11.0 * (static_cast<double>(m) * n + static_cast<double>(n) * (n + 1)) * u;
    const std::size_t nn = static_cast<std::size_t>(n * n), ni = static_cast<std::size_t>((n + 31) / 32) * 1024;
    DBuf Gs(c, nn * (R ? kCholQrPasses : 1)), Ri(c, ni);
    const double* src = A;
    i64 lds = lda;
    for (int it = 0; it < kCholQrPasses; ++it) {
        double* G = Gs.p + (R ? it * nn : 0);
        gemm(c, true, n, n, m, 1.0, src, lds, src, lds, 0.0, G, n, false, true);  // upper tiles of src^T src
        const int mode = it < kCholQrShifted ? 1 : (it == kCholQrPasses - 1 ? 2 : 0);
        launch_chol(c, n, G, n, mode, coeff, Ri.p, tag);
        launch_trsm(c, m, n, src, lds, G, n, Ri.p, Q, ldq);
        src = Q;
        lds = ldq;
    }
    if (R) {  // R = R_p ... R_2 R_1
        DBuf T(c, nn), T2(c, nn);
        double* acc = Gs.p + (kCholQrPasses - 1) * nn;
        for (int it = kCholQrPasses - 2; it >= 0; --it) {
            double* dst = it == 0 ? R : (acc == T.p ? T2.p : T.p);
            const i64 ldd = it == 0 ? ldr : n;
            gemm(c, false, n, n, n, 1.0, acc, n, Gs.p + it * nn, n, 0.0, dst, ldd, false);
            acc = dst;
        }
    }
}


// K4d host: factor the rows x b panel P (ld ldp, b <= 32, rows >= 2b) into the
// blocked QR's (R in P's top block, V, T, tau); breakdown -> the context's QR
// flag with `tag` (the caller speculates, see with_qr_speculation).
// K4f host: the fused cooperative panel when the rows fit one CTA per SM
// (<= kFpMaxRpc rows each); false = not taken (the caller uses K4d's launches).
bool cqr_panel_fused_launch(Ctx& c, i64 rows, i64 b, double* P, i64 ldp, double* V, i64 ldv, double* T, double* tau,
                            int tag, int hr = 1, double* Rout = nullptr, i64 ldr = 1, int* flag = nullptr) {
    i64 rpc = ((rows + c.sm_count - 1) / c.sm_count + 7) / 8 * 8;
    rpc = std::max<i64>(rpc, 64);
    if (rpc > kFpMaxRpc) return false;
    const i64 G = (rows + rpc - 1) / rpc;
    static std::atomic<std::uint64_t> configured{0};  // bit d: attributes set on device d
    if (first_on_device(configured)) set_max_dynamic_smem(reinterpret_cast<const void*>(cqr_panel_fused));
    static const bool trace_on = std::getenv("TTR_QR_TRACE") != nullptr;  // diagnostics (eager calls only)
    const double u = DBL_EPSILON / 2;
    DBuf xb(c, static_cast<std::size_t>((2 * G + 1) * kFpEntries)), tr(c, trace_on ? 64 : 1);  // partials (x 2: kFpDirectG) + sum
    FusedPanelArgs a{};
    a.rows = static_cast<int>(rows);
    a.b = static_cast<int>(b);
    a.rpc = static_cast<int>(rpc);
    a.P = P;
    a.ldp = ldp;
    a.V = V;
    a.ldv = ldv;
    a.T = T;
    a.tau = tau;
    a.gpart = xb.p;
    a.gsum = xb.p + 2 * G * kFpEntries;
    a.coeff = 11.0 * (static_cast<double>(rows) * b + static_cast<double>(b) * (b + 1)) * u;
    a.flag = flag ? flag : (c.qr_flag_override ? c.qr_flag_override : c.qr_flag_dev());
    a.tag = c.qr_flag_override && !flag ? -1 : tag;
    a.hr = hr;
    a.Rout = Rout;
    a.ldr = ldr;
    a.trace = trace_on ? reinterpret_cast<long long*>(tr.p) : nullptr;
    if (trace_on) TTR_CUDA(cudaMemsetAsync(tr.p, 0, 64 * sizeof(double), c.stream));
    void* args[] = {&a};
    TTR_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(cqr_panel_fused), dim3(static_cast<unsigned>(G)),
                                         dim3(kFpThreads), args, sizeof(double) * fp_smem_doubles(static_cast<int>(rpc)),
                                         c.stream));
    c.launched();
    if (trace_on) {
        long long h[64];
        TTR_CUDA(cudaMemcpyAsync(h, tr.p, sizeof(h), cudaMemcpyDeviceToHost, c.stream));
        TTR_CUDA(cudaStreamSynchronize(c.stream));
        std::fprintf(stderr, "cqr_panel_fused rows %lld b %lld rpc %lld grid %lld: cycles", static_cast<long long>(rows),
                     static_cast<long long>(b), static_cast<long long>(rpc), static_cast<long long>(G));
        for (int i = 1; i < 63 && h[i]; ++i) std::fprintf(stderr, " %lld", h[i] - h[i - 1]);
        if (h[63] < 0) std::fprintf(stderr, " BREAKDOWN in pass %lld", -h[63] - 1);
        std::fprintf(stderr, "\n");
    }
    return true;
}

// K4f as a thin QR of an m x n matrix with n <= 32 (the adaptive growth blocks): Q
// (may be null) and R (may be null, n x n upper with a positive diagonal). A is
// only read. Breakdown -> atomicMin(*flag, tag) (flag null: the context's QR
// flag). false = shape outside the kernel (the caller keeps its Householder QR).
bool cqr_single(Ctx& c, i64 m, i64 n, const double* A, i64 lda, double* Q, i64 ldq, double* R, i64 ldr, int* flag,
                int tag) {
    if (n < 1 || n > 32 || m < 8 * n || m < 256) return false;
    return cqr_panel_fused_launch(c, m, n, const_cast<double*>(A), lda, Q, ldq, nullptr, nullptr, tag, 0, R, ldr, flag);
}

void cqr_panel(Ctx& c, i64 rows, i64 b, double* P, i64 ldp, double* V, i64 ldv, double* T, double* tau, int tag) {
    if (b < 1 || b > 32 || rows < 2 * b) fail(Errc::InvalidArgument, "cqr_panel: shape outside the panel path");
    static const bool fused_on = [] {  // experiments: TTR_QR_CQR_FUSED=0 = K4d's separate launches
        const char* e = std::getenv("TTR_QR_CQR_FUSED");
        return !(e && e[0] == '0');
    }();
    if (fused_on && cqr_panel_fused_launch(c, rows, b, P, ldp, V, ldv, T, tau, tag)) return;
    const i64 G = std::max<i64>(1, std::min<i64>(c.sm_count, (rows + 255) / 256));
    const i64 rpc = ((rows + G - 1) / G + 31) / 32 * 32;
    const double u = DBL_EPSILON / 2;
    const double coeff = 11.0 * (static_cast<double>(rows) * b + static_cast<double>(b) * (b + 1)) * u;
    DBuf part(c, static_cast<std::size_t>(G * 1024)), Qp(c, static_cast<std::size_t>(rows * 32)),
        mats(c, static_cast<std::size_t>(3 * 1024));
    double* Rinv = mats.p;
    double* Rtot = mats.p + 1024;
    double* Uinv = mats.p + 2048;
    const unsigned agrid = static_cast<unsigned>(std::min<i64>(4 * c.sm_count, (rows + kCqrThreads - 1) / kCqrThreads));
    int* flag = c.qr_flag_override ? c.qr_flag_override : c.qr_flag_dev();
    if (c.qr_flag_override) tag = -1;
    for (int pass = 0; pass < 3; ++pass) {
        const double* src = pass == 0 ? P : Qp.p;
        const i64 lds = pass == 0 ? ldp : rows;
        cqr_gram_partial<<<static_cast<unsigned>(G), kCqrThreads, 0, c.stream>>>(static_cast<int>(rows), static_cast<int>(b),
                                                                             src, lds, static_cast<int>(rpc), part.p);
        cqr_chol32<<<1, kCholSmall, 0, c.stream>>>(static_cast<int>(G), part.p, static_cast<int>(b),
                                                     pass == 0 ? 1 : (pass == 2 ? 2 : 0), coeff, Rinv, Rtot,
                                                     pass == 0 ? 1 : 0, flag, tag);
        cqr_apply<<<agrid, kCqrThreads, 0, c.stream>>>(static_cast<int>(rows), static_cast<int>(b), src, lds, Rinv, Qp.p,
                                                        rows);
        c.launched(3);
    }
    cqr_hr<<<1, kCholSmall, 0, c.stream>>>(static_cast<int>(b), Qp.p, rows, Rtot, T, V, ldv, P, ldp, Uinv, tau);
    cqr_apply<<<agrid, kCqrThreads, 0, c.stream>>>(static_cast<int>(rows - b), static_cast<int>(b), Qp.p + b, rows, Uinv,
                                                    V + b, ldv);
    TTR_CUDA(cudaGetLastError());
    c.launched(2);
}


bool cholqr_small_fits(i64 m, i64 n) {
    return n >= 1 && n <= 32 && m >= n && m <= 2048 && sq_smem<4>(static_cast<int>(m), static_cast<int>(n)) <= 200 * 1024;
}

template <int NT>
static void cholqr_small_launch(Ctx& c, int m, int n, const double* A, i64 lda, i64 sA, double* Q, i64 ldq, i64 sQ,
                                i64 batch, double coeff, int* flags) {
    const std::size_t smem = sq_smem<NT>(m, n);
    static std::atomic<std::uint64_t> configured{0};
    if (first_on_device(configured)) set_max_dynamic_smem(reinterpret_cast<const void*>(cholqr_small_kernel<NT>));
    static const int warps_env = [] {
        const char* e = std::getenv("TTR_SQ_WARPS");
        return e ? std::atoi(e) : 0;
    }();
    // 4 warps: more CTAs per SM hide the one-warp Cholesky (measured 154 vs 165 us
    // per 2048 320 x 20 matrices with 8)
    const int warps = warps_env > 0 ? std::max(kSqGramWarps, std::min(8, warps_env)) : kSqGramWarps;
    cholqr_small_kernel<NT><<<static_cast<unsigned>(batch), 32 * warps, smem, c.stream>>>(m, n, A, lda, sA, Q, ldq, sQ,
                                                                                        coeff, flags);
}

// K4e host: batched CholeskyQR2 / sCQR3 of `batch` m x n matrices (strided); flags[b] = 1 on breakdown.
void cholqr_small_batched(Ctx& c, i64 m, i64 n, const double* A, i64 lda, i64 sA, double* Q, i64 ldq, i64 sQ, i64 batch,
                          int* flags) {
    if (!cholqr_small_fits(m, n)) fail(Errc::InvalidArgument, "cholqr_small: shape outside the path");
    if (batch <= 0) return;
    const double u = DBL_EPSILON / 2;
    const double coeff = 11.0 * (static_cast<double>(m) * n + static_cast<double>(n) * (n + 1)) * u;
    const int mi = static_cast<int>(m), ni = static_cast<int>(n);
    switch ((ni + 7) / 8) {
        case 1: cholqr_small_launch<1>(c, mi, ni, A, lda, sA, Q, ldq, sQ, batch, coeff, flags); break;
        case 2: cholqr_small_launch<2>(c, mi, ni, A, lda, sA, Q, ldq, sQ, batch, coeff, flags); break;
        case 3: cholqr_small_launch<3>(c, mi, ni, A, lda, sA, Q, ldq, sQ, batch, coeff, flags); break;
        default: cholqr_small_launch<4>(c, mi, ni, A, lda, sA, Q, ldq, sQ, batch, coeff, flags); break;
    }
    TTR_CUDA(cudaGetLastError());
    c.launched();
}

}  // namespace ttr
