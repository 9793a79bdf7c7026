// lr_batch.cuh — fused left-to-right step of the batched Rand-Orth sweep
// (included by tt_batch.cu; config 5a: 4096 tensors, l = 20, ranks 64, n = 16).
//
// Per tensor, step k of rand_orth_sweep (round_rand.cpp:26-44) forms the next
// working unfolding H(Y_{k+1}) = M H(X_{k+1}) and step k+1 immediately sketches
// it, S_{k+1} = V(Y_{k+1}) W_{k+2}. Done as two strided-batch GEMMs, Y goes to
// HBM and comes straight back (the batch is far larger than L2), and the second
// tiny GEMM (320 x 20 x 64 per tensor) is one more launch. Here ONE CTA per
// tensor streams the core slice by slice: for every mode index j, X(:, j, :)
// (cols x rr) lands in shared memory by cp.async (double buffered) and
// Y_j = M X_j runs on the DMMA pipe; Y_j is written out (still needed for
// M_{k+1} = Q^T V(Y_{k+1})) and the S rows (a, j) = Y_j W are formed from
// shared memory one slice later, in the same loop as Y_{j+1} = M X_{j+1}, so
// the two dependent DMMA chains overlap (one CTA barrier per slice). Sums are
// in a fixed order (deterministic).
#pragma once

namespace lrb {

__device__ __forceinline__ unsigned su32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void cp16(double* dst, const double* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(su32(dst)), "l"(src));
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }
__device__ __forceinline__ void mma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// 68-double rows: 64-bit fragment loads (row = lane >> 2, k = lane & 3) of a
// half-warp hit 16 distinct 8-byte slots (68 = 4 mod 16); rows are 16-byte
// aligned for cp.async
constexpr int kLd = 68;
constexpr int kWarps = 8, kThreads = 32 * kWarps;

struct LrArgs {
    int l, cols, n, rr, l2;
    const double* M;  // l x cols, ld l
    i64 sM;
    const double* X;  // cols x n x rr core
    i64 sX;
    const double* W;  // rr x l2 (first l2 columns), ld ldw
    i64 ldw, sW;
    double* Y;        // l x (n rr), ld l
    i64 sY;
    double* S;        // (l n) x l2, ld l n
    i64 sS;
    // fused QR epilogue (lr_fused_kernel<.., RT > 0>): Q = qr(S) -> Q (the output
    // core, (l n) x l2, ld l n) and M_next = Q^T V(Y) (l2 x rr, ld l2)
    double* Q;
    i64 sQ;
    double* Mn;
    i64 sMn;
};

// Y slices are kept transposed, [g][a] with ld kLdY: the output stores read
// consecutive a (conflict free) and the S products' A fragments (a = lane >> 2,
// g = lane & 3) hit 16 distinct slots per half-warp (28 = 12, 36 = 4 mod 16)
template <int LT>
struct LrSmem {  // M, two X slices, two Y slices (2 CTAs per SM for LT <= 3)
    static constexpr int kLdY = LT <= 3 ? 28 : 36;
    static constexpr int kDoubles = 8 * LT * kLd + 2 * 64 * kLd + 2 * 64 * kLdY;
    static constexpr std::size_t kBytes = static_cast<std::size_t>(kDoubles) * sizeof(double);
};

// S output tiles t = c * LT + i (i < LT, c < LT2) are dealt round-robin to the
// warps (t = warp + 8q); each warp keeps the W fragments of its tiles in registers
template <int LT, int LT2>
struct STiles {
    static constexpr int kTiles = LT * LT2;
    static constexpr int kPerWarp = (kTiles + kWarps - 1) / kWarps;
};

// l <= 8 LT, l2 <= 8 LT2, cols <= 64 (even), rr <= 64; RT > 0: l n <= 32 RT and
// the QR + M_next epilogue (the per-tensor QR of step k+1 and M = Q^T V)
template <int LT, int LT2, int RT = 0>
__global__ void __launch_bounds__(kThreads, 2) lr_fused_kernel(const LrArgs p) {
    extern __shared__ __align__(16) double sm[];
    double* Ms = sm;                    // [8 LT][kLd]: M(a, b)
    double* Xs = Ms + 8 * LT * kLd;     // [2][64][kLd]: X(b, j, g) at [g][b]
    double* Ys = Xs + 2 * 64 * kLd;     // [2][64][kLdY]: Y(a, j, g) at [g][a]
    constexpr int kLdY = LrSmem<LT>::kLdY;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, fr = lane >> 2, fc = lane & 3;
    const i64 t = blockIdx.x;
    const int l = p.l, cols = p.cols, n = p.n, rr = p.rr, l2 = p.l2, rows = l * n;
    const double* M = p.M + t * p.sM;
    const double* X = p.X + t * p.sX;
    const double* W = p.W + t * p.sW;
    double* Y = p.Y + t * p.sY;
    double* S = p.S + t * p.sS;

    // zero padding (rows g >= rr and columns b >= cols of the X slices are never
    // overwritten, so Y_j's padded columns and the padded k of every product are 0)
    constexpr int kTot = LrSmem<LT>::kDoubles;
    for (int e = tid; e < kTot; e += kThreads) sm[e] = 0.0;
    __syncthreads();
    for (int e = tid; e < l * cols; e += kThreads) Ms[(e % l) * kLd + e / l] = M[e];
    const int halves = cols >> 1;  // 16-byte chunks per g-row
    const i64 gstride = static_cast<i64>(cols) * n;  // X(:, j, g) -> X(:, j, g + 1)
    auto issue = [&](int j) {      // always commits a group (empty past the last slice)
        if (j < n && lane < halves) {  // warp: rows g = warp + 8q; lane: 16-byte chunk (cols <= 64)
            double* dst = Xs + (j & 1) * 64 * kLd + warp * kLd + 2 * lane;
            const double* src = X + static_cast<i64>(cols) * j + warp * gstride + 2 * lane;
            for (int g = warp; g < rr; g += kWarps, dst += kWarps * kLd, src += kWarps * gstride) cp16(dst, src);
        }
        commit();
    };
    issue(0);

    // this warp's S tiles and their W fragments B(k = g, n = c): g = 4 kk + fc, c = 8 (t / LT) + fr
    constexpr int NT = STiles<LT, LT2>::kTiles, PW = STiles<LT, LT2>::kPerWarp;
    double wf[PW][16];
#pragma unroll
    for (int q = 0; q < PW; ++q) {
        const int tt = warp + kWarps * q, cc = 8 * (tt / LT) + fr;
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) {
            const int g = 4 * kk + fc;
            wf[q][kk] = (tt < NT && g < rr && cc < l2) ? __ldg(W + g + static_cast<i64>(cc) * p.ldw) : 0.0;
        }
    }
    const int kSteps = (cols + 3) >> 2;

    for (int j = 0; j <= n; ++j) {
        wait<0>();
        __syncthreads();  // X_j and Y_{j-1} visible; readers of the buffers rewritten below are done
        issue(j + 1);     // overlaps this slice's products
        const bool g1 = j < n, g2 = j > 0;
        const double* xs = Xs + (j & 1) * 64 * kLd + (8 * warp + fr) * kLd;
        const double* yp = Ys + ((j - 1) & 1) * 64 * kLdY;
        double a1[LT][2], a2[PW][2];
#pragma unroll
        for (int i = 0; i < LT; ++i) a1[i][0] = a1[i][1] = 0.0;
#pragma unroll
        for (int q = 0; q < PW; ++q) a2[q][0] = a2[q][1] = 0.0;
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) {  // full unroll: wf stays in registers
            const int b = 4 * kk + fc;
            if (g1 && kk < kSteps) {  // Y_j = M X_j: warp w owns columns g = 8w .. 8w + 7
                const double bf = xs[b];
#pragma unroll
                for (int i = 0; i < LT; ++i) mma(a1[i][0], a1[i][1], Ms[(8 * i + fr) * kLd + b], bf);
            }
            if (g2) {  // S rows (a, j - 1) = Y_{j-1} W
#pragma unroll
                for (int q = 0; q < PW; ++q) {
                    const int tt = warp + kWarps * q;
                    if (tt < NT) mma(a2[q][0], a2[q][1], yp[b * kLdY + 8 * (tt % LT) + fr], wf[q][kk]);
                }
            }
        }
        if (g2) {
            const int jj = j - 1;
#pragma unroll
            for (int q = 0; q < PW; ++q) {
                const int tt = warp + kWarps * q, a = 8 * (tt % LT) + fr, cc = 8 * (tt / LT) + 2 * fc;
                if (tt < NT && a < l) {
                    if (cc < l2) S[a + l * jj + static_cast<i64>(rows) * cc] = a2[q][0];
                    if (cc + 1 < l2) S[a + l * jj + static_cast<i64>(rows) * (cc + 1)] = a2[q][1];
                }
            }
            // Y_{j-1} out: Y(a, j-1, g) at a + l (j-1 + n g) (runs of l doubles)
            if (lane < l) {  // l <= 32
                double* yo = Y + lane + static_cast<i64>(l) * (jj + static_cast<i64>(n) * warp);
                for (int g = warp; g < rr; g += kWarps, yo += static_cast<i64>(l) * n * kWarps) *yo = yp[g * kLdY + lane];
            }
        }
        if (g1) {
            double* yc = Ys + (j & 1) * 64 * kLdY + (8 * warp + 2 * fc) * kLdY + fr;
#pragma unroll
            for (int i = 0; i < LT; ++i) {
                yc[8 * i] = a1[i][0];
                yc[kLdY + 8 * i] = a1[i][1];
            }
        }
    }
    if constexpr (RT > 0) {
        // ---- fused step k+1: Q = qr(S) (S just written by this CTA; plain loads),
        //      the output core, then M_next = Q^T V(Y) on the DMMA pipe ----
        __syncthreads();  // every S and Y store of this CTA is visible; Xs/Ys are free
        double* Q = p.Q + t * p.sQ;
        double qx[LT2][RT];
        colreg_qr_cta<RT, LT2, kWarps>(rows, l2, S, rows, Q, rows, nullptr, 1, Ys, qx);
        // Q^T staged row-major, [a][r] with ld kLdQ (% 16 == 4: conflict-free A fragments)
        constexpr int kLdQ = 32 * RT + 4;
        double* Qt = Xs;
        __syncthreads();  // the QR's shared-memory staging is done before Xs is reused
#pragma unroll
        for (int c = 0; c < LT2; ++c) {
            const int a = warp + kWarps * c;
#pragma unroll
            for (int tt = 0; tt < RT; ++tt) {
                const int r = lane + 32 * tt;
                if (a < 8 * LT2) Qt[a * kLdQ + r] = (a < l2 && r < rows) ? qx[c][tt] : 0.0;
            }
        }
        __syncthreads();
        // M_next (l2 x rr): warp w owns columns g = 8w .. 8w+7 (rr <= 64), all LT2 row tiles;
        // B fragments Y(r, g) from global (written above, L2-resident)
        double am[LT2][2];
#pragma unroll
        for (int i = 0; i < LT2; ++i) am[i][0] = am[i][1] = 0.0;
        const int g = 8 * warp + fr;
        const double* ycol = Y + static_cast<i64>(g < rr ? g : 0) * rows;
        for (int k4 = 0; k4 < 32 * RT; k4 += 4) {
            const int r = k4 + fc;
            const double bv = (g < rr && r < rows) ? ycol[r] : 0.0;
#pragma unroll
            for (int i = 0; i < LT2; ++i) mma(am[i][0], am[i][1], Qt[(8 * i + fr) * kLdQ + r], bv);
        }
        double* Mn = p.Mn + t * p.sMn;
#pragma unroll
        for (int i = 0; i < LT2; ++i) {
            const int a = 8 * i + fr;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int gg = 8 * warp + 2 * fc + h;
                if (a < l2 && gg < rr) Mn[a + static_cast<i64>(gg) * l2] = am[i][h];
            }
        }
    }

}

}  // namespace lrb
