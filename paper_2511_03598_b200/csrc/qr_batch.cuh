// qr_batch.cuh — batched Householder QR of many small matrices (included by
// qr.cu): one CTA per matrix of m <= 512 rows and n <= 32 columns (the 5a
// batch: 4096 matrices of 320 x 20; linalg.cpp:44-56 per matrix).
//
// Measured on the 5a shape (ncu, one 4096-matrix launch): the shared-memory
// kernel in qr.cu (qr_small_kernel) 837 us and a column-owner variant with the
// matrix in shared memory 842 us — both bound by shared-memory bandwidth (two
// loads + a store per fma); lane-per-column registers (panel_col_kernel layout)
// 1.45-1.88 ms (64-bit shuffles / one CTA per SM); this kernel 668 us.
#pragma once

#include <cfloat>

__device__ __forceinline__ double colreg_warp_sum(double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// owner warp: stage its register column cj of x (rows lane + 32t) into cb
// and return sum_{r>j} of its squares (warp sum). The column is picked by
// selects, not x[cj] — a runtime index would put x in local memory.
template <int RT, int C>
__device__ __forceinline__ double colreg_stage(const double (&x)[C][RT], int cj, double* cb, int j, int lane) {
    double s = 0.0;
#pragma unroll
    for (int t = 0; t < RT; ++t) {
        double v = x[0][t];
#pragma unroll
        for (int c = 1; c < C; ++c) v = (cj == c) ? x[c][t] : v;
        const int r = lane + 32 * t;
        cb[r] = v;
        if (r > j) s = fma(v, v, s);
    }
    return colreg_warp_sum(s);
}

// Register-resident column owners (dispatched for m <= 32*RT, n <= NW*C): warp w
// owns columns l = w + NW*c (c < C) and lane holds rows lane + 32t (t < RT) of
// them in registers, so the only shared-memory traffic per step is the active
// column (staged once by its owner, double-buffered) — the smem-resident
// kernels above are bound by shared-memory bandwidth (5 accesses per 2 fma).
// Step j: the owner stages x_j and derives the reflector; ONE barrier; every
// warp loads the staged column once (masked to rows > j), dots its columns
// with it (warp sums) and updates them. n <= 32, so rows <= j all sit in the
// first chunk (lane <= j) and only the staged copy of that chunk is masked.
// One CTA's QR of one m x n matrix (the body of qr_small_colreg_kernel, also
// called from the fused batched sweep kernel, lr_batch.cuh): A is read with
// plain loads (it may have been written earlier in the same kernel); Q (m x k)
// and R (optional) are written; on return x holds Q in registers (column
// warp + NW c, rows lane + 32 t). sm: 2*32*RT + 38 doubles of shared memory.
template <int RT, int C, int NW>
__device__ __forceinline__ void colreg_qr_cta(int m, int n, const double* A, i64 lda, double* Q, i64 ldq, double* R,
                                              i64 ldr, double* sm, double (&x)[C][RT]) {
    double* colb = sm;                 // [2][32*RT] active column
    double* tl = colb + 2 * 32 * RT;   // [2][3] beta, inv, tau of the active reflector
    double* taus = tl + 6;             // [32]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int k = min(m, n);

#pragma unroll
    for (int c = 0; c < C; ++c) {
        const int l = warp + NW * c;
#pragma unroll
        for (int t = 0; t < RT; ++t) {
            const int r = lane + 32 * t;
            x[c][t] = (l < n && r < m) ? A[r + static_cast<i64>(l) * lda] : 0.0;
        }
    }
    double my_inv[C];
#pragma unroll
    for (int c = 0; c < C; ++c) my_inv[c] = 0.0;

    // the staged column, rows > j only (zero elsewhere). j < k <= 32, so every
    // row <= j sits in chunk t = 0 (lane <= j): only that chunk is masked.
    double cv[RT];
    auto load_masked = [&](const double* cb, int j) {
        cv[0] = (lane > j) ? cb[lane] : 0.0;
#pragma unroll
        for (int t = 1; t < RT; ++t) cv[t] = cb[lane + 32 * t];
    };

    // ---- factorization ----
    for (int j = 0; j < k; ++j) {
        const int buf = j & 1;
        if (warp == j % NW) {  // the owner stages x_j and derives the reflector (one warp: sqrt/div)
            double* cb = colb + buf * 32 * RT;
            const double tail = colreg_stage<RT, C>(x, j / NW, cb, j, lane);
            __syncwarp();
            const double alpha = cb[j];
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
            if (lane == 0) {
                tl[3 * buf] = beta;
                tl[3 * buf + 1] = inv;
                tl[3 * buf + 2] = tj;
                taus[j] = tj;
            }
        }
        __syncthreads();
        load_masked(colb + buf * 32 * RT, j);
        const double beta = tl[3 * buf], inv = tl[3 * buf + 1], tj = tl[3 * buf + 2];
#pragma unroll
        for (int c = 0; c < C; ++c) {
            const int l = warp + NW * c;
            const bool act = l > j && l < n, own = l == j;
            double s0 = 0.0, s1 = 0.0;
#pragma unroll
            for (int t = 0; t < RT; ++t) {
                if (t & 1) s1 = fma(cv[t], x[c][t], s1);
                else s0 = fma(cv[t], x[c][t], s0);
            }
            const double d = colreg_warp_sum(s0 + s1);
            const double row = __shfl_sync(0xffffffffu, x[c][0], j);
            const double wl = act ? tj * fma(inv, d, row) : 0.0;
            const double ca = -wl * inv;
            my_inv[c] = own ? inv : my_inv[c];
#pragma unroll
            for (int t = 0; t < RT; ++t) x[c][t] = fma(ca, cv[t], x[c][t]);  // rows <= j: cv = 0
            if (lane == j) x[c][0] = own ? beta : x[c][0] - wl;
        }
    }
    // scale the reflector tails v_l(r) = inv_l x_l(r), r > l
#pragma unroll
    for (int c = 0; c < C; ++c) {
        const int l = warp + NW * c;
#pragma unroll
        for (int t = 0; t < RT; ++t)
            if (lane + 32 * t > l && l < k) x[c][t] *= my_inv[c];
    }
    if (R) {
#pragma unroll
        for (int c = 0; c < C; ++c) {
            const int l = warp + NW * c;
#pragma unroll
            for (int t = 0; t < RT; ++t) {
                const int r = lane + 32 * t;
                if (r < k && l < n) R[r + static_cast<i64>(l) * ldr] = (r <= l) ? x[c][t] : 0.0;
            }
        }
    }
    if (Q == nullptr) return;
    __syncthreads();  // taus visible; the last factorization step's readers are done

    // ---- explicit thin Q (backward accumulation) ----
    for (int i = k - 1; i >= 0; --i) {
        const int buf = i & 1;
        const double ti = taus[i];
        if (warp == i % NW) colreg_stage<RT, C>(x, i / NW, colb + buf * 32 * RT, i, lane);
        __syncthreads();
        load_masked(colb + buf * 32 * RT, i);  // v_i below row i
#pragma unroll
        for (int c = 0; c < C; ++c) {
            const int l = warp + NW * c;
            const bool act = l > i && l < k && ti != 0.0, own = l == i;
            double s0 = 0.0, s1 = 0.0;
#pragma unroll
            for (int t = 0; t < RT; ++t) {
                if (t & 1) s1 = fma(cv[t], x[c][t], s1);
                else s0 = fma(cv[t], x[c][t], s0);
            }
            const double d = colreg_warp_sum(s0 + s1);
            const double row = __shfl_sync(0xffffffffu, x[c][0], i);
            const double wl = act ? ti * (d + row) : 0.0;
            // others: x_l -= w_l v_i; the owner: column i becomes e_i - tau_i v_i,
            // i.e. -tau_i v_i = -tau_i x below row i (cv holds exactly that tail)
            const double ca = own ? -ti : -wl;
#pragma unroll
            for (int t = 0; t < RT; ++t) {
                const double base = own ? 0.0 : x[c][t];
                x[c][t] = fma(ca, cv[t], base);
            }
            if (lane == i) x[c][0] = own ? 1.0 - ti : x[c][0] - wl;
        }
    }
#pragma unroll
    for (int c = 0; c < C; ++c) {
        const int l = warp + NW * c;
#pragma unroll
        for (int t = 0; t < RT; ++t) {
            const int r = lane + 32 * t;
            if (l < k && r < m) Q[r + static_cast<i64>(l) * ldq] = x[c][t];
        }
    }
}

template <int RT, int C, int NW = 8>
__global__ void __launch_bounds__(NW * 32, 16 / NW) qr_small_colreg_kernel(int m, int n, const double* __restrict__ A, i64 lda,
                                                                 i64 sA, double* Q, i64 ldq, i64 sQ, double* R,
                                                                 i64 ldr, i64 sR) {
    extern __shared__ double sm[];
    double x[C][RT];
    colreg_qr_cta<RT, C, NW>(m, n, A + blockIdx.x * sA, lda, Q ? Q + blockIdx.x * sQ : nullptr, ldq,
                             R ? R + blockIdx.x * sR : nullptr, ldr, sm, x);
}
